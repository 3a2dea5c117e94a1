// Forwarding header: the reference's include path (proj/include/acs/rng.hpp)
// resolves to the B200 library's host/device stream.
#pragma once
#include "rng_stream.hpp"
