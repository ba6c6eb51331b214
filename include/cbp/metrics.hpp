// Reference header name (proj/core/include/cbp/metrics.hpp) for drop-in includes.
#pragma once
#include "cbp/cbp.hpp"
