// bf_internal.h -- internal launcher interface between the plan (bf_plan.cu) and
// the sm_100a kernels (bf_kernels.cu).  Not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "bf_shard.h"

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

// Tensor-core leaf stages (bf_tc.cu).  They read the leaf weights in an expanded form built once at
// plan finalization: real-embedded, split hi/lo, in the shared-memory tile image of the MMA
// (leafx_floats(d) floats each for V0 and U).
bool leaf_tc_shape(const Dims& d);
int64_t leafx_floats(const Dims& d);
int64_t ux_floats(const Dims& d);
int64_t v0x_floats(const Dims& d);  // the S0 image: leafx_floats, or half of it for the 2x image   // the SL image: leafx_floats, or half of it for the 2x image (r in {8, 16})
cudaError_t expand_leaf_weights(const Dims& d, const float2* V0, const float2* U, float* V0x, float* Ux, cudaStream_t s);
// S0 on the tensor cores: same contract as launch_s0, weights from V0x.
bool s0_tc_supported(const Dims& d, int nv, int64_t ldf);
cudaError_t launch_s0_tc(const Dims& d, const float2* F, int64_t ldf, const float2* ampb, const float* V0x, float2* out,
                         int nv, cudaStream_t s,
                         bool multicast = true);

// SL on the tensor cores: same contract as launch_sl, weights from Ux.
bool sl_tc_supported(const Dims& d, int nv);
cudaError_t launch_sl_tc(const Dims& d, const float2* in, const float* Ux, const float2* ampa, float2* G, int64_t ldg,
                         int nv, cudaStream_t s,
                         bool multicast = true);

// Transfer level l (eqn:2 / eqn:3): out[p](t) = sum_{c,s} W[p](t, c r + s) in[(a>>1) 2^(LN-l+1) + 2b + c](s)
// (at l == h the switch is already folded into W).
// rh > 0: `in` is a receive buffer of the index-sharded exchange (input pair p at bfs::recv_index(p, rh, rhg)).
// po (fused exchange): the output pairs go to their destination shards' receive arrays (bf_shard.h).
cudaError_t launch_xfer(const Dims& d, int l, const float2* in, float2* out, const float2* W, int nv, cudaStream_t s,
                        int rh = 0, int rhg = 0, const bfs::PeerOut* po = nullptr);

// Band of K (1 or 2) transfer levels l_first .. l_first+K-1 fused in shared memory; W[m] are the
// weights of level l_first+m.
bool band_supported(int R, int nv);
cudaError_t launch_band(const Dims& d, int l_first, int K, const float2* in, float2* out, const float2* const* W, int nv,
                        cudaStream_t s, int rh = 0, int rhg = 0, const bfs::PeerOut* po = nullptr);

// Band of K (1 or 2) transfer levels for small vector batches (bf_small.cu: 8 <= nv < 128, nv % 8 == 0):
// persistent, bulk-copy-fed, one 4-pair job per warp; same contract as launch_band.
bool band_sv_supported(const Dims& d, int nv);
cudaError_t launch_band_sv(const Dims& d, int l_first, int K, const float2* in, float2* out, const float2* const* W,
                           int nv, cudaStream_t s, int rh = 0, int rhg = 0, const bfs::PeerOut* po = nullptr);

// S0 / SL for small vector batches (bf_small.cu): same contracts as launch_s0 / launch_sl.
bool s0_sv_supported(const Dims& d, int nv);
cudaError_t launch_s0_sv(const Dims& d, const float2* F, int64_t ldf, const float2* ampb, const float2* V0,
                         float2* out, int nv, cudaStream_t s);
bool sl_sv_supported(const Dims& d, int nv);
cudaError_t launch_sl_sv(const Dims& d, const float2* in, const float2* U, const float2* ampa, float2* G, int64_t ldg,
                         int nv, cudaStream_t s);

// Band of 2 transfer levels on the tensor cores (bf_tc.cu): same contract as launch_band with K = 2.
bool band_tc_supported(const Dims& d, int nv);
// which tensor-core band kernel runs (per plan: BF_OPT_BAND_COMPOSE)
struct BandVariant {
    bool compose = true;         // the composed two-level operator (band_cmp_kernel); else band_tc_kernel
};
// Cpre (optional): the band's operator precomposed at finalization (launch_compose_band) -- the kernel then
// only embeds and splits it instead of composing it on chip per group (small vector batches).
cudaError_t launch_band_tc(const Dims& d, int l_first, const float2* in, float2* out, const float2* const* W, int nv,
                           cudaStream_t s, int rh, int rhg, const bfs::PeerOut* po, const BandVariant& bv,
                           const float2* Cpre = nullptr);
// Plan finalization: the composed two-level operator of the band starting at l_first, 16 r^2 complex per group
// of 4 pairs (FP64 products, complex64 result).
cudaError_t launch_compose_band(const Dims& d, int l_first, const float2* W1, const float2* W2, float2* Cg,
                                cudaStream_t s);

// Band of 3 transfer levels on the tensor cores (bf_band3.cu, r in {6, 8}, nv >= 128): the band's precomposed
// 8 x 8 block operator per group of 8 pairs (launch_compose3 at finalization, band3_operator_elems complex).
bool band3_supported(const Dims& d, int nv);
int64_t band3_operator_elems(const Dims& d);
cudaError_t launch_band3(const Dims& d, int l_first, const float2* in, float2* out, const float2* Cpre, int nv,
                         cudaStream_t s);
cudaError_t launch_compose3(const Dims& d, int l_first, const float2* W1, const float2* W2, const float2* W3,
                            float2* Cg, cudaStream_t s);


// Plan finalization: W[p] <- Sw[p] W[p] for npairs blocks (W column-major R x cols, Sw R x R).
cudaError_t launch_fold_switch(const float2* Sw, float2* W, int64_t npairs, int R, int cols, cudaStream_t s);

// Adjoint plan: the factors of K* (same butterfly shape) from a finalized forward plan's factors (switch folded
// into the level-h factor): amplitudes conjugated and swapped, V0~ / U~ the conjugate transposes of U / V0 with
// the pair index transposed, transfer levels reversed and re-assembled (bf_kernels.cu).
cudaError_t launch_adjoint_factors(const Dims& d, const float2* amp_a, const float2* amp_b, const float2* v0,
                                   const float2* u, const float2* const* xfer, float2* adj_amp_a, float2* adj_amp_b,
                                   float2* adj_v0, float2* adj_u, float2* const* adj_xfer, cudaStream_t s);

// Structured interpolative factors (bf_struct.cu, NEXT-1): generic kernels (any nv, one level per launch).
// kind: 1 = first-half level (L1 r x 2r, psi [N][2r]), 2 = second-half level (L2 2 x r x r, chi [N][2r]).
// The Lagrange matrix of a stage travels BY VALUE in the kernel parameters (constant bank 0): with the loops over
// its rows and columns unrolled, every weight is a compile-time constant-bank operand of its FFMA -- no load
// instruction at all (a shared-memory copy cost one LDS per two FMAs and made the first version LDS-bound).
// The plan keeps a host copy of every level's matrix for this.
struct LagP {
    float v[1024];   // >= max(r n0, 2 r^2) floats (r <= 16, n0 <= 64)
};
cudaError_t launch_s0_st(const Dims& d, const float2* F, int64_t ldf, const float2* ampb, const LagP& L0,
                         const float2* om, float2* out, int nv, cudaStream_t s);
cudaError_t launch_xfer_st(const Dims& d, int l, int kind, const LagP& L, const float2* ph, const float2* in,
                           float2* out, int nv, cudaStream_t s);
cudaError_t launch_sl_st(const Dims& d, const float2* in, const float* Lsl, const float2* Om, const float2* ampa,
                         float2* G, int64_t ldg, int nv, cudaStream_t s);
// two transfer levels l, l+1 per launch on structured (kind 1 / 2) or dense (kind 0) levels; L carries level l's
// matrix at v[0] and level l+1's at v[512]; w1 / w2 the per-pair data (phases, or blocks for kind 0)
bool band_st_supported(const Dims& d, int nv);
bool band_st_kinds(int k1, int k2);   // level kinds (0 dense, 1 first, 2 second, 3 first + switch) the band fuses
cudaError_t launch_band_st(const Dims& d, int l, int k1, int k2, const LagP& L, const float2* w1, const float2* w2,
                           const float2* in, float2* out, int nv, cudaStream_t s);
// dense blocks of a structured stage (kind 0 S0, 1 first, 2 second, 3 first + switch, 4 SL; l = the level)
cudaError_t launch_expand_st(const Dims& d, int kind, int l, const float* L, const float2* ph, float2* out,
                             cudaStream_t s);

// Recompression (bf_recompress.cu, NEXT-3): the rank-rp factors of a dense rank-d.R (<= 12) factorization whose
// switch is folded into level h, by a balanced-truncation sweep in FP64.  Scratch: gout (D - l0 + 1) N r^2,
// q2 2 N r rp, gin2 2 N rp^2 complex doubles.
cudaError_t launch_recompress(const Dims& d, int rp, const float2* v0, const float2* const* xfer, const float2* u,
                              float2* out_v0, float2* const* out_x, float2* out_u, void* gout, void* q2, void* gin2,
                              cudaStream_t s);

// SL (eqn:bf3 + eqn:tg): G[x, c] = sum_k a_k(x) sum_{b<n0} sum_t U[a n0 + b](j, t) in[a n0 + b](t)[c n_amp + k],
// x = a n0 + j.
cudaError_t launch_sl(const Dims& d, const float2* in, const float2* U, const float2* ampa, float2* G, int64_t ldg,
                      int nv, cudaStream_t s);

}  // namespace bfk
