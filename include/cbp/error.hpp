// Reference header name (proj/core/include/cbp/error.hpp) for drop-in includes.
#pragma once
#include "cbp/cbp.hpp"
