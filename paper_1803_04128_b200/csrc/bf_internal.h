// bf_internal.h -- internal launcher interface between the plan (bf_plan.cu) and
// the sm_100a kernels (bf_kernels.cu).  Not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace bfk {

// Shape of one butterfly (notation of include/bf.h).
struct Dims {
    int LN, l0, h, D, R, n_amp;
    int64_t N;
};

// Kernel classes (indices of the per-kernel timing arrays, bf.h BF_NUM_KCLASS).
enum KClass { KC_S0 = 0, KC_XFER1 = 1, KC_SWITCH = 2, KC_XFER2 = 3, KC_SL = 4, KC_COUNT = 5 };

bool rank_supported(int R);

// S0 (eqn:1): out[p = a N/n0 + b][t][v] = sum_j V0[p](t, j) * b_k(x) F[x, c],  x = b n0 + j, v = c n_amp + k.
cudaError_t launch_s0(const Dims& d, const float2* F, int64_t ldf, const float2* ampb, const float2* V0,
                      float2* out, int nv, cudaStream_t s);

// Transfer level l (eqn:2 / eqn:3): out[p](t) = sum_{c,s} W[p](t, c r + s) in[(a>>1) 2^(LN-l+1) + 2b + c](s);
// with Sw != nullptr (only at l == h) the switch block Sw[p] is applied to the result.
// rh > 0: `in` is a receive buffer of the index-sharded exchange (input pair p at bfs::recv_index(p, rh, rhg)).
cudaError_t launch_xfer(const Dims& d, int l, const float2* in, float2* out, const float2* W, const float2* Sw,
                        int nv, cudaStream_t s, int rh = 0, int rhg = 0);

// Band of K (1 or 2) transfer levels l_first .. l_first+K-1 fused in shared memory; W[m] are the
// weights of level l_first+m; with m_sw in 1..K the switch Sw is applied after band level m_sw.
bool band_supported(int R, int nv);
cudaError_t launch_band(const Dims& d, int l_first, int K, const float2* in, float2* out, const float2* const* W,
                        const float2* Sw, int m_sw, int nv, cudaStream_t s, int rh = 0, int rhg = 0);

// Switch alone (used when no transfer level precedes it, h == l0).
cudaError_t launch_switch(const Dims& d, const float2* in, float2* out, const float2* Sw, int nv, cudaStream_t s);

// SL (eqn:bf3 + eqn:tg): G[x, c] = sum_k a_k(x) sum_{b<n0} sum_t U[a n0 + b](j, t) in[a n0 + b](t)[c n_amp + k],
// x = a n0 + j.
cudaError_t launch_sl(const Dims& d, const float2* in, const float2* U, const float2* ampa, float2* G, int64_t ldg,
                      int nv, cudaStream_t s);

}  // namespace bfk
