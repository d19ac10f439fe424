// shim_io.hpp — force-included (-include) into the reference unit tests: the
// declaration of the test-only network_to_json of shim_io.cpp.
#pragma once
#include <string>
#include "synscale/synscale.hpp"
namespace synscale {
std::string network_to_json(const NetworkSpec& spec);
}
