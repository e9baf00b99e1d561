// bf_plan_internal.h -- plan internals shared by bf_plan.cu and the streaming
// builder (bf_build.cpp).  Not part of the ABI.
#pragma once
#include <cstdint>

#include "../../include/bf.h"

// Device destination of blocks [begin, begin+count) of `stage`; marks them uploaded.
bf_status_t bfp_stage_dst(bf_plan_t p, int32_t stage, int64_t begin, int64_t count, void** dst);
int bfp_device(bf_plan_t p);
bf_status_t bfp_fail(bf_status_t s, const char* msg);
