// Drop-in path of the reference's ppsim/analysis.hpp (analysis.hpp:28-346): mismatch_report, window_mismatch, verify_steady_mismatch, verify_topology_invariance, memory_report, reduce_broadcast_cost.
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
