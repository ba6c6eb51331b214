// Reference header name (proj/core/include/cbp/poly.hpp) for drop-in includes.
#pragma once
#include "cbp/cbp.hpp"
