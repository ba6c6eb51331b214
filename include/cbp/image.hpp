// Reference header name (proj/core/include/cbp/image.hpp) for drop-in includes.
#pragma once
#include "cbp/cbp.hpp"
