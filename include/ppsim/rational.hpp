// Drop-in path of the reference's ppsim/rational.hpp (rational.hpp:13-128): exact rational
// time `Rat`, implemented in ppsim/rat.hpp.
#pragma once

#include "ppsim/rat.hpp"
