// Reference header name (proj/core/include/cbp/synth.hpp) for drop-in includes.
#pragma once
#include "cbp/cbp.hpp"
