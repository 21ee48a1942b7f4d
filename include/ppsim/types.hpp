// Drop-in path of the reference's ppsim/types.hpp (types.hpp:15-207): Kind, Policy, ClusterSpec, PolicyConfig, TaskEvent, Timeline, reports, Verdict.
// Every declaration lives in ppsim/ppsim.hpp (implemented in libamdp.so); this header keeps
// the reference's include paths so code written against it (P/README.md:96-116, the
// reference's own tests) compiles unmodified.
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <optional>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "ppsim/ppsim.hpp"
