// Reference header name (proj/core/include/cbp/decoder.hpp) for drop-in includes.
#pragma once
#include "cbp/cbp.hpp"
