// Forwarding header: the whole C++ API is declared in synscale.hpp
// (calibration: the sweep, reference calibration.hpp:12-42).
#pragma once
#include "synscale/synscale.hpp"
