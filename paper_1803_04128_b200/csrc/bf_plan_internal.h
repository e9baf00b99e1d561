// bf_plan_internal.h -- plan internals shared by bf_plan.cu and the streaming
// builder (bf_build.cpp).  Not part of the ABI.
#pragma once
#include <cstdint>

#include "../../include/bf.h"

// Device destination of blocks [begin, begin+count) of `stage` of shard `shard`; marks them uploaded.
bf_status_t bfp_stage_dst(bf_plan_t p, int shard, int32_t stage, int64_t begin, int64_t count, void** dst);
int bfp_device(bf_plan_t p);
int bfp_num_shards(bf_plan_t p);
int bfp_rank(bf_plan_t p);
bf_status_t bfp_fail(bf_status_t s, const char* msg);
// mode: BF_SHARD_NONE / BF_SHARD_NCCL / BF_SHARD_EMULATED
bf_status_t bfp_plan_alloc_sharded(const bf_desc_t* meta, int device, int64_t max_nrhs_chunk, int world, int rank,
                                   int mode, const void* nccl_id, bf_plan_t* out);
void bfp_plan_free(bf_plan_t p);
