// Forwarding header: the reference's include path (proj/include/acs/tsp_instance.hpp)
// resolves to the B200 library's instance layer.
#pragma once
#include "instance.hpp"
