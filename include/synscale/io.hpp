// Forwarding header: the whole C++ API is declared in synscale.hpp.
#pragma once
#include "synscale/synscale.hpp"
