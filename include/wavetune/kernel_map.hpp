// Drop-in header name of the reference (proj/include/wavetune/kernel_map.hpp);
// the whole API is declared in wavetune.hpp.
#pragma once
#include "wavetune/wavetune.hpp"
