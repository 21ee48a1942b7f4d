// Drop-in path of the reference's ppsim/engine.hpp (engine.hpp:28-202): simulate, bubble_ratio (and simulate_with_order, which also returns the dispatch order).
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
