// Reference header name (proj/core/include/cbp/fft.hpp) for drop-in includes.
#pragma once
#include "cbp/cbp.hpp"
