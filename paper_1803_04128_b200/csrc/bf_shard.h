// bf_shard.h -- index arithmetic of the index-sharded butterfly, shared by the
// kernels (input remap of the first second-half launch) and the host (plan building, bf_shard_pairs).
//
// G = 2^g ranks, rank q.  Level-l pair (a, b), pair index p = a 2^(LN-l) + b  (include/bf.h).
//   levels l <= h  (first half):  owned by the xi-shard   q = b >> (LN - l - g);
//                                 local index  a 2^(LN-l-g) + (b mod 2^(LN-l-g))
//   levels l >= h  (second half): owned by the x-shard    q = a >> (l - g);
//                                 local index  (a mod 2^(l-g)) 2^(LN-l) + b   = p - q N/G
// With these local indices the first half on a rank is the butterfly of log2 size LN' = LN - g at the
// same levels, and the second half the butterfly of size LN' at levels l - g: the kernels run unchanged.
// Exchange at h (LN - h = h): the first-half local order is a-major, so the pairs a rank sends to rank d
// (a >> (h - g) = d) form the contiguous block d of G equal blocks; the receiver stores block q (from
// source q) as [q][a' < 2^(h-g)][b_l < 2^(h-g)], b = q 2^(h-g) + b_l.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#if defined(__CUDACC__)
#define BF_HD __host__ __device__ __forceinline__
#else
#define BF_HD inline
#endif

namespace bfs {

// Receive-buffer position of the second-half local level-h pair p = a' 2^h + b (rh = h, rhg = h - g).
BF_HD int64_t recv_index(int64_t p, int rh, int rhg)
{
    const int64_t a = p >> rh, b = p & ((int64_t(1) << rh) - 1);
    const int64_t q = b >> rhg, bl = b & ((int64_t(1) << rhg) - 1);
    return (q << (2 * rhg)) + (a << rhg) + bl;
}

// Global pair index of first-half local pair `loc` of rank q at level l.
BF_HD int64_t first_half_global(int64_t loc, int LN, int l, int g, int q)
{
    const int sb = LN - l - g;   // log2 local b-range
    const int64_t a = loc >> sb, bl = loc & ((int64_t(1) << sb) - 1);
    return (a << (LN - l)) + (int64_t(q) << sb) + bl;
}

// Global pair index of second-half local pair `loc` of rank q at level l.
BF_HD int64_t second_half_global(int64_t loc, int LN, int g, int q) { return (int64_t(q) << (LN - g)) + loc; }

// Fused exchange (peer stores): the launch that produces level h writes each output pair straight into
// its destination shard's receive array instead of its own send buffer.  Local first-half pair p goes to
// shard d = p >> lb (blocks of 2^lb pairs) at receive position src 2^lb + (p mod 2^lb) (the layout
// recv_index reads).  dst[d] are device pointers (same device for emulated shards, CUDA-IPC-mapped peer
// memory over NVLink for one shard per GPU).
constexpr int kMaxShards = 16;
struct PeerOut {
    float2* dst[kMaxShards];
    int lb;    // log2 pairs per destination block
    int src;   // this shard
    int on;    // 0: ordinary output array
};

#if defined(__CUDACC__)
__device__ __forceinline__ float2* pair_out(float2* out, const PeerOut& po, int64_t p, int R, int nv)
{
    if (!po.on) return out + p * R * int64_t(nv);
    const int64_t d = p >> po.lb, off = (p & ((int64_t(1) << po.lb) - 1)) + (int64_t(po.src) << po.lb);
    return po.dst[d] + off * R * int64_t(nv);
}
#endif

}  // namespace bfs
