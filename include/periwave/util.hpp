// Forwarding header: the whole drop-in API lives in periwave/periwave.hpp.
#pragma once
#include "periwave/periwave.hpp"
