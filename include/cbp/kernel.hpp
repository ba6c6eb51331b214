// Reference header name (proj/core/include/cbp/kernel.hpp) for drop-in includes.
#pragma once
#include "cbp/cbp.hpp"
