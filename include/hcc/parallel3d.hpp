// Forwarding header: the B200 build of the hcc API lives in hcc_b200.hpp
// (one header for the whole drop-in surface; see its preamble).
#pragma once
#include "hcc/hcc_b200.hpp"
