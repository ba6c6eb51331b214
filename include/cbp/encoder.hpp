// Reference header name (proj/core/include/cbp/encoder.hpp) for drop-in includes.
#pragma once
#include "cbp/cbp.hpp"
