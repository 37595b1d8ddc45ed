// Drop-in header name of the reference (proj/include/wavetune/wave_sim.hpp);
// the whole API is declared in wavetune.hpp.
#pragma once
#include "wavetune/wavetune.hpp"
