// Programs for the persistent stream engine (kernels_engine.cu); structs live in hm_internal.h.
#pragma once

#include "hm_internal.h"
