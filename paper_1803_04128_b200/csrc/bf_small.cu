// bf_small.cu -- transfer levels for SMALL vector batches (8 <= nv < 128, nv % 8 == 0): cfg2 (nv = 32),
// cfg5 (nv = 16) and cfg4 sharded over 8 GPUs (nv = 64).
//
// Transfer level l (eqn:2 P:748-752 for l <= h, eqn:3 P:780-785 for l > h; the switch P:755-766 is folded
// into the level-h blocks at plan finalization):
//     out[p](t) = sum_{c,s} W_l[p](t, c r + s) in[(a>>1) 2^(LN-l+1) + 2b + c](s),   p = a 2^(LN-l) + b.
// A JOB is 4 consecutive input pairs 4j .. 4j+3 of level l-1 (contiguous in the coefficient array):
//   K = 1: the two butterfly units 2j, 2j+1 of level l (4 output pairs);
//   K = 2: a band group closed under levels l, l+1 (SURVEY 8(a) "fusion geometry"): 4 output pairs at each
//          level, the level-l result kept in shared memory and only level l+1 written to HBM.
// With few vectors the weight stream dominates (cfg5: 6.7 GB of blocks vs 2 x 5.4 GB of coefficients per
// level), and every weight element is reused only nv times, so the kernel is built to keep both the FP32
// pipe and HBM busy:
//   * persistent CTAs (one per SM): a producer warp streams each job's input pairs and its 4 K weight blocks
//     into a ring of shared-memory slots with 1-D bulk copies (TMA engine), completion on mbarriers;
//   * C consumer warps, ONE JOB PER WARP: lane = (output pair slot os = lane / 8, vector lane vl = lane % 8);
//     a lane owns R rows x VPL consecutive vectors of its output pair (R x VPL complex accumulators, 4 FFMA
//     per complex MAC), so its indices are fixed for the whole job and computed once;
//   * weights are read as 16-byte shared-memory loads that the 8 lanes of an output pair share (broadcast);
//     the 4 blocks of a level sit at a stride = 32 (mod 128) bytes, so the 4 distinct addresses of one load
//     fall into disjoint bank groups (one wavefront);
//   * K = 2: level l is written back in place (unit u's outputs e = 0, 1 into its own input slots 2u, 2u+1),
//     level l+1 reads slots u, u+2 -- the slot algebra of band_kernel in bf_kernels.cu.
// nv > 8 VPL: the warp sweeps the vectors in passes of 8 VPL (weights re-read from shared memory).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "bf_internal.h"
#include "bf_shard.h"
#include "tc_sm100.cuh"

namespace bfk {

namespace {

constexpr int SV_MAX_CONSUMERS = 8;
constexpr int SV_SMEM_LIMIT = 227 * 1024;   // max dynamic shared memory per CTA
constexpr int SV_HDR = 1024;                // mbarriers

// Shared-memory image of one SUPER-JOB (J consecutive jobs: 4J input pairs, contiguous in HBM):
//   X                 [4J pairs][r][nv]           one bulk copy
//   level-1 run e     [2J blocks (u fastest)]     blocks (((2 a0 + e) << sh1) + 2 bq + u), J jobs' bq contiguous
//   level-2 run (u,e) [J blocks]                  blocks (((4 a0 + 2u + e) << shg) + bq)      (K = 2 only)
// Each run is ONE bulk copy (the TMA engine's per-request cost, ~170 clk, limited the one-copy-per-block
// version to 0.5 of HBM with loads alone).  A lane of output slot (u, e) reads block (2 jj + u) of level-1
// run e and block jj of level-2 run (u, e): the run bases are placed at 0 / 32 / 64 / 96 (mod 128) bytes so
// that the 4 distinct addresses of one weight load fall into disjoint bank groups (r = 10: a block is 64 mod
// 128 bytes, so u = 0 / 1 in a level-1 run are already 64 apart).
struct SvLayout {
    int xb;        // bytes of X
    int run[6];    // byte offsets of the runs: level-1 e = 0, 1; level-2 (u, e) = 2 + 2u + e
    int slot;      // bytes of the slot (multiple of 128)
};

__host__ __device__ constexpr int sv_blk(int R) { return 16 * R * R; }

__host__ __device__ inline SvLayout sv_layout(int R, int nv, int K, int J)
{
    SvLayout L{};
    L.xb = 4 * J * R * nv * 8;
    int pos = L.xb;
    const int nruns = K == 2 ? 6 : 2;
    for (int k = 0; k < nruns; k++) {
        const int target = (k < 2 ? k : k - 2) * 32;
        pos = (pos + 127) / 128 * 128 + target;
        L.run[k] = pos;
        pos += (k < 2 ? 2 * J : J) * sv_blk(R);
    }
    L.slot = (pos + 127) / 128 * 128;
    return L;
}

__device__ __forceinline__ void cmac(float2& acc, const float2 w, const float2 v)
{
    acc.x = fmaf(w.x, v.x, acc.x);
    acc.x = fmaf(-w.y, v.y, acc.x);
    acc.y = fmaf(w.x, v.y, acc.y);
    acc.y = fmaf(w.y, v.x, acc.y);
}

// The same complex MAC with packed FP32 pairs (sm_100a FFMA2: one instruction, two lanes of FMA):
//   acc += w.re (x.re, x.im);  acc += w.im (-x.im, x.re) = w.im (i x)
// w.re / w.im enter as scalar broadcasts (the .F32 operand mode), ix = i x is formed once per loaded x.  Per
// component the two FMAs and their order are those of cmac(): results are bitwise identical.
__device__ __forceinline__ unsigned long long pk2(float lo, float hi)
{
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void cmac2(unsigned long long& acc, const float wr, const float wi, const unsigned long long x,
                                      const unsigned long long ix)
{
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(pk2(wr, wr)), "l"(x));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(pk2(wi, wi)), "l"(ix));
}

template <int V>
__device__ __forceinline__ void ld_vec(float2 (&x)[V], const float2* p)
{
    if constexpr (V == 1) {
        x[0] = *p;
    } else {
#pragma unroll
        for (int i = 0; i < V / 2; i++) {
            const float4 q = reinterpret_cast<const float4*>(p)[i];
            x[2 * i] = make_float2(q.x, q.y);
            x[2 * i + 1] = make_float2(q.z, q.w);
        }
    }
}

template <int V>
__device__ __forceinline__ void st_vec(float2* p, const float2 (&x)[V])
{
    if constexpr (V == 1) {
        *p = x[0];
    } else {
#pragma unroll
        for (int i = 0; i < V / 2; i++)
            reinterpret_cast<float4*>(p)[i] = make_float4(x[2 * i].x, x[2 * i].y, x[2 * i + 1].x, x[2 * i + 1].y);
    }
}

struct SvArgs {
    const float2* W[2];   // weights of levels l_first, l_first + 1 (bf.h XFER layout, column-major r x 2r)
    bfs::PeerOut po;      // fused exchange: peer stores of the last level
    int rh, rhg;          // > 0: the input is a receive buffer of the index-sharded exchange
};

// global pair index of output (u, e) at band level m (1-based) of job j; shg = LN - l_first - 1
__device__ __forceinline__ int64_t sv_pair(int64_t j, int m, int u, int e, int LN, int l_first)
{
    const int shg = LN - l_first - 1;
    const int64_t a0 = j >> shg, bq = j & ((int64_t(1) << shg) - 1);
    if (m == 1) return (((a0 << 1) + e) << (LN - l_first)) + (bq << 1) + u;
    return (((a0 << 2) + 2 * u + e) << shg) + bq;
}

template <int R, int VPL, int K, int J>
// (9-12 warps put 3 on some SM sub-partition, whose 16K registers then cap a thread at 168 registers; the
// launch bounds let ptxas apply that cap)
__global__ void __launch_bounds__(32 * (SV_MAX_CONSUMERS + 1), 1)
    band_sv_kernel(const float2* __restrict__ in, float2* __restrict__ out, const SvArgs args, int LN, int l_first,
                   int nv, int64_t nsuper, int S, int C)
{
    extern __shared__ __align__(128) unsigned char sv_smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sv_smem);
    uint64_t* empty = full + S;
    unsigned char* slots = sv_smem + SV_HDR;
    const SvLayout L = sv_layout(R, nv, K, J);
    constexpr int BLK = sv_blk(R);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; s++) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], J);   // one arrival per job of the super-job
        }
        tc::mbar_fence_init();
    }
    __syncthreads();

    if (warp == 0) {
        // ---- producer: super-job q = blockIdx.x + i gridDim.x of this CTA -> slot i % S ----
        for (int64_t i = 0;; i++) {
            const int64_t q = blockIdx.x + i * gridDim.x;
            if (q >= nsuper) break;
            const int s = int(i % S);
            if (i >= S) tc::mbar_wait(&empty[s], uint32_t((i / S - 1) & 1));
#ifdef BF_SV_EXP_NOLOAD   // experiment: no copies (compute-only timing; results are garbage)
            if (lane == 0) tc::mbar_arrive(&full[s]);
            continue;
#endif
            unsigned char* slot = slots + size_t(s) * L.slot;
            if (lane == 0) tc::mbar_arrive_expect_tx(&full[s], uint32_t(L.xb + (K == 2 ? 8 : 4) * J * BLK));
            __syncwarp();
            const int64_t j0 = q * J;
            if (lane == 0) {
                if (!args.rh) {
                    tc::bulk_g2s(slot, in + 4 * j0 * R * int64_t(nv), uint32_t(L.xb), &full[s]);
                } else {   // receive buffer of the exchange: 4-pair groups are contiguous (h - g >= 2)
                    for (int jj = 0; jj < J; jj++)
                        tc::bulk_g2s(slot + jj * (L.xb / J),
                                     in + bfs::recv_index(4 * (j0 + jj), args.rh, args.rhg) * R * int64_t(nv),
                                     uint32_t(L.xb / J), &full[s]);
                }
            } else if (lane <= (K == 2 ? 6 : 2)) {
                const int k = lane - 1;
                const int m = k < 2 ? 1 : 2, u = k < 2 ? 0 : (k - 2) >> 1, e = k < 2 ? k : (k - 2) & 1;
                const int64_t p = sv_pair(j0, m, u, e, LN, l_first);
                tc::bulk_g2s(slot + L.run[k], args.W[m - 1] + p * 2 * R * R, uint32_t((m == 1 ? 2 * J : J) * BLK),
                             &full[s]);
            }
        }
        return;
    }

    // ---- consumers: warp w takes jobs i = w - 1, w - 1 + C, ... (C % J == 0: fixed position jj in the super-job)
    const int os = lane >> 3, vl = lane & 7, u = os >> 1, e = os & 1;
    const int passes = nv / (8 * VPL);
    for (int64_t i = warp - 1;; i += C) {
        const int64_t qi = i / J;
        const int jj = int(i % J);
        const int64_t q = blockIdx.x + qi * gridDim.x;
        if (q >= nsuper) break;
        const int64_t j = q * J + jj;
        const int s = int(qi % S);
        tc::mbar_wait(&full[s], uint32_t((qi / S) & 1));
        unsigned char* slot = slots + size_t(s) * L.slot;
        float2* X = reinterpret_cast<float2*>(slot) + jj * 4 * R * nv;
#ifdef BF_SV_EXP_NOCOMPUTE   // experiment: load-only timing
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&empty[s]);
        continue;
#endif
#pragma unroll 1
        for (int m = 1; m <= K; m++) {
            const int in0 = (m == 1) ? 2 * u : u, in1 = (m == 1) ? 2 * u + 1 : u + 2;
            const float2* Wb = reinterpret_cast<const float2*>(
                slot + (m == 1 ? L.run[e] + (2 * jj + u) * BLK : L.run[2 + 2 * u + e] + jj * BLK));
            float2* dst = (m < K) ? X + (2 * u + e) * R * nv
                                  : bfs::pair_out(out, args.po, sv_pair(j, m, u, e, LN, l_first), R, nv);
#pragma unroll 1
            for (int ps = 0; ps < passes; ps++) {
                const int vb = ps * 8 * VPL + vl * VPL;
                unsigned long long acc[R][VPL];
#pragma unroll
                for (int t = 0; t < R; t++)
#pragma unroll
                    for (int qq = 0; qq < VPL; qq++) acc[t][qq] = 0ull;
#pragma unroll
                for (int c = 0; c < 2; c++) {
                    const float2* xs = X + (c ? in1 : in0) * R * nv + vb;
                    const float2* wc = Wb + c * R * R;
#pragma unroll(K == 2 ? R : 2)   // K = 1: full unrolling let the compiler hoist every weight load (spills)
                    for (int sr = 0; sr < R; sr++) {
                        float2 x[VPL], w[R];
                        ld_vec<VPL>(x, xs + sr * nv);
                        ld_vec<R>(w, wc + sr * R);
                        unsigned long long xp[VPL], ixp[VPL];
#pragma unroll
                        for (int qq = 0; qq < VPL; qq++) {
                            xp[qq] = pk2(x[qq].x, x[qq].y);
                            ixp[qq] = pk2(-x[qq].y, x[qq].x);
                        }
#pragma unroll
                        for (int t = 0; t < R; t++)
#pragma unroll
                            for (int qq = 0; qq < VPL; qq++) cmac2(acc[t][qq], w[t].x, w[t].y, xp[qq], ixp[qq]);
                    }
                }
                if (m < K) __syncwarp();   // both outputs of unit u have read its input slots (this pass's columns)
#pragma unroll
                for (int t = 0; t < R; t++) {
                    float2 o[VPL];
#pragma unroll
                    for (int qq = 0; qq < VPL; qq++)
                        asm("mov.b64 {%0, %1}, %2;" : "=f"(o[qq].x), "=f"(o[qq].y) : "l"(acc[t][qq]));
                    st_vec<VPL>(dst + t * nv + vb, o);
                }
            }
            if (m < K) __syncwarp();   // level m in place before level m + 1 reads it
        }
        // generic-proxy writes to the slot (level l in place) -> ordered before the next bulk copy into it
        if (K > 1) tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&empty[s]);
    }
}

int env_int(const char* name)
{
    const char* e = getenv(name);
    return e ? atoi(e) : 0;
}

// vectors per lane: 2 (R x 2 register tile, passes of 16 vectors) unless nv is not a multiple of 16 (R x 4 tiles
// measured no faster at nv = 32 and spill at r >= 12 under the 168-register cap)
int sv_vpl(int nv) { return nv % 16 == 0 ? 2 : 1; }

// Super-job size J, ring depth S and consumer warps C for one CTA per SM.  J = 2 where 6+ slots fit (fewer,
// larger bulk copies), else J = 1.  C = min(8, J (S - 2)) rounded to a multiple of J: two slots of prefetch
// at least, and 2 consumer warps per SM sub-partition where they fit (an odd count leaves some sub-partitions
// with 2 warps and others with 1; jobs are dealt round robin and the in-order ring then runs at the pace of
// the shared ones).  BF_SV_CONSUMERS overrides C (tuning experiments).
bool sv_config(int R, int nv, int K, int& J, int& S, int& C)
{
    for (J = 2; J >= 1; J--) {
        S = (SV_SMEM_LIMIT - SV_HDR) / sv_layout(R, nv, K, J).slot;
        if (J == 1 || S >= 6) break;
    }
    if (S < 2) return false;
    C = J * (S - 2 > 0 ? S - 2 : 1);
    static const int c_env = env_int("BF_SV_CONSUMERS");
    if (c_env > 0) C = c_env;
    if (C > SV_MAX_CONSUMERS) C = SV_MAX_CONSUMERS;
    C = C / J * J;
    if (C < J) C = J;
    if (S > C / J + 4) S = C / J + 4;
    return true;
}

int num_sms()
{
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

template <int R, int VPL, int K, int J>
cudaError_t sv_go(const Dims& d, int l_first, const float2* in, float2* out, const float2* const* W, int nv, int S,
                  int C, cudaStream_t st, int rh, int rhg, const bfs::PeerOut* po)
{
    SvArgs a{};
    a.W[0] = W[0];
    a.W[1] = K > 1 ? W[1] : nullptr;
    if (po) a.po = *po;
    a.rh = rh;
    a.rhg = rhg;
    const size_t shm = SV_HDR + size_t(S) * sv_layout(R, nv, K, J).slot;
    auto kern = band_sv_kernel<R, VPL, K, J>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm));
    if (e != cudaSuccess) return e;
    const int64_t nsuper = d.N / (4 * J);
    const int64_t grid = nsuper < num_sms() ? nsuper : num_sms();
    kern<<<unsigned(grid), 32 * (C + 1), shm, st>>>(in, out, a, d.LN, l_first, nv, nsuper, S, C);
    return cudaGetLastError();
}

template <int R, int K>
cudaError_t sv_vpl_go(const Dims& d, int l_first, const float2* in, float2* out, const float2* const* W, int nv,
                      cudaStream_t st, int rh, int rhg, const bfs::PeerOut* po)
{
    int J = 1, S = 0, C = 0;
    if (!sv_config(R, nv, K, J, S, C)) return cudaErrorInvalidValue;
    // a super-job must stay inside one a0 block of the level (J | 2^shg) and, reading a receive buffer, inside
    // one source block (4 J | 2^rhg)
    const int shg = d.LN - l_first - 1;
    if (J == 2 && (shg < 1 || (rh && rhg < 3))) {
        J = 1;
        S = (SV_SMEM_LIMIT - SV_HDR) / sv_layout(R, nv, K, 1).slot;
        C = S - 2 > 0 ? (S - 2 > SV_MAX_CONSUMERS ? SV_MAX_CONSUMERS : S - 2) : 1;
    }
#define SV_J(VV)                                                                                  \
    return J == 2 ? sv_go<R, VV, K, 2>(d, l_first, in, out, W, nv, S, C, st, rh, rhg, po)        \
                  : sv_go<R, VV, K, 1>(d, l_first, in, out, W, nv, S, C, st, rh, rhg, po);
    switch (sv_vpl(nv)) {
    case 2: SV_J(2)
    default: SV_J(1)
    }
#undef SV_J
}

// =====================================================================================================
// Leaf stages for small vector batches (8 <= nv <= 64 / 32): the same structure as the band -- a producer warp
// bulk-copies the weight blocks into a ring, consumer warps hold fixed R x VPL (S0) or JPL x VPL (SL)
// register tiles and run packed FFMA2 complex MACs in the FP32 order of s0_kernel / sl_kernel (bitwise
// equal results).
// =====================================================================================================

// cmul of bf_kernels.cu (the amplitude pre-scale b_k(x) F[x, c], same rounding)
__device__ __forceinline__ float2 cmul_sv(const float2 a, const float2 b)
{
    return make_float2(fmaf(a.x, b.x, -(a.y * b.y)), fmaf(a.x, b.y, a.y * b.x));
}

__host__ __device__ constexpr int pad32(int bytes) { return bytes + ((32 - bytes % 128) % 128 + 128) % 128; }

// S0 (eqn:1 P:698-702, eqn:tg P:24-28): out[p = a N/n0 + b][t][v] = sum_j V0[p](t, j) y_b[j][v],
// y_b[j][v] = b_k(x) F[x, c], x = b n0 + j, v = c n_amp + k.
// A job is (leaf b, group g of 4 consecutive a): the 4 blocks V0[(4g + al) N/n0 + b] (4 bulk copies, bank-
// staggered), one job per consumer warp, lane = (al = lane / 8, vl = lane % 8) x R rows x VPL vectors.
// Warp 1 builds y_b (double-buffered by leaf) from F and b_k with ordinary loads.
template <int R, int VPL>
__global__ void __launch_bounds__(32 * (SV_MAX_CONSUMERS + 2), 1)
    s0_sv_kernel(const float2* __restrict__ F, int64_t ldf, const float2* __restrict__ ampb,
                 const float2* __restrict__ V0, float2* __restrict__ out, int LN, int l0, int n_amp, int nv, int S,
                 int C)
{
    extern __shared__ __align__(128) unsigned char sv_smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sv_smem);
    uint64_t* empty = full + S;
    uint64_t* yfull = empty + S;
    uint64_t* yempty = yfull + 2;
    const int n0 = 1 << l0, G = n0 / 4;
    const int64_t N = int64_t(1) << LN, nleaf = N >> l0;
    float2* Y = reinterpret_cast<float2*>(sv_smem + SV_HDR);   // [2][n0][nv]
    unsigned char* slots = sv_smem + SV_HDR + 2 * n0 * nv * 8;
    const int BLK = R * n0 * 8, WB = pad32(BLK), SB = (4 * WB + 127) / 128 * 128;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; s++) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int q = 0; q < 2; q++) {
            tc::mbar_init(&yfull[q], 1);
            tc::mbar_init(&yempty[q], G);
        }
        tc::mbar_fence_init();
    }
    __syncthreads();

    if (warp == 0) {   // ---- weight producer: job i = k G + g (k-th leaf of this CTA) -> slot i % S
        for (int64_t i = 0;; i++) {
            const int64_t k = i / G, b = blockIdx.x + k * gridDim.x;
            const int g = int(i % G);
            if (b >= nleaf) break;
            const int s = int(i % S);
            if (i >= S) tc::mbar_wait(&empty[s], uint32_t((i / S - 1) & 1));
            if (lane == 0) tc::mbar_arrive_expect_tx(&full[s], uint32_t(4 * BLK));
            __syncwarp();
            if (lane < 4)
                tc::bulk_g2s(slots + size_t(s) * SB + lane * WB, V0 + ((4 * g + lane) * nleaf + b) * int64_t(R) * n0,
                             uint32_t(BLK), &full[s]);
        }
        return;
    }
    if (warp == 1) {   // ---- y builder: y_b for the k-th leaf into buffer k % 2
        const int nrhs = nv / n_amp;
        for (int64_t k = 0;; k++) {
            const int64_t b = blockIdx.x + k * gridDim.x;
            if (b >= nleaf) break;
            const int yb = int(k & 1);
            if (k >= 2) tc::mbar_wait(&yempty[yb], uint32_t(((k >> 1) - 1) & 1));
            float2* Yb = Y + yb * n0 * nv;
            // 8 elements per lane per batch: all their loads are issued before the first product (one load, then
            // its stores, per element cost a memory round trip each -- 16 per leaf at cfg5: the y builder was
            // the S0 kernel's critical path)
            for (int e0 = 0; e0 < n0 * nrhs; e0 += 32 * 8) {
                float2 f[8], am[8][4];
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    const int e = e0 + q * 32 + lane;
                    f[q] = make_float2(0.f, 0.f);
                    if (e < n0 * nrhs) {
                        const int j = e % n0, c = e / n0;
                        const int64_t x = b * n0 + j;
                        f[q] = __ldg(F + x + c * ldf);
#pragma unroll
                        for (int kk = 0; kk < 4; kk++)
                            if (kk < n_amp) am[q][kk] = __ldg(ampb + kk * N + x);
                    }
                }
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    const int e = e0 + q * 32 + lane;
                    if (e >= n0 * nrhs) continue;
                    const int j = e % n0, c = e / n0;
#pragma unroll
                    for (int kk = 0; kk < 4; kk++)
                        if (kk < n_amp) Yb[j * nv + c * n_amp + kk] = cmul_sv(am[q][kk], f[q]);
                }
            }
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&yfull[yb]);
        }
        return;
    }
    // ---- consumers
    const int al = lane >> 3, vl = lane & 7;
    const int passes = nv / (8 * VPL);
    for (int64_t i = warp - 2;; i += C) {
        const int64_t k = i / G, b = blockIdx.x + k * gridDim.x;
        const int g = int(i % G);
        if (b >= nleaf) break;
        const int yb = int(k & 1), s = int(i % S);
        tc::mbar_wait(&yfull[yb], uint32_t((k >> 1) & 1));
        tc::mbar_wait(&full[s], uint32_t((i / S) & 1));
        const float2* Wb = reinterpret_cast<const float2*>(slots + size_t(s) * SB + al * WB);
        const float2* Yb = Y + yb * n0 * nv;
        const int64_t p = (4 * g + al) * nleaf + b;
#pragma unroll 1
        for (int ps = 0; ps < passes; ps++) {
            const int vb = ps * 8 * VPL + vl * VPL;
            unsigned long long acc[R][VPL];
#pragma unroll
            for (int t = 0; t < R; t++)
#pragma unroll
                for (int q = 0; q < VPL; q++) acc[t][q] = 0ull;
#pragma unroll 4
            for (int j = 0; j < n0; j++) {
                float2 x[VPL], w[R];
                ld_vec<VPL>(x, Yb + j * nv + vb);
                ld_vec<R>(w, Wb + j * R);
                unsigned long long xp[VPL], ixp[VPL];
#pragma unroll
                for (int q = 0; q < VPL; q++) {
                    xp[q] = pk2(x[q].x, x[q].y);
                    ixp[q] = pk2(-x[q].y, x[q].x);
                }
#pragma unroll
                for (int t = 0; t < R; t++)
#pragma unroll
                    for (int q = 0; q < VPL; q++) cmac2(acc[t][q], w[t].x, w[t].y, xp[q], ixp[q]);
            }
            float2* o = out + p * R * int64_t(nv) + vb;
#pragma unroll
            for (int t = 0; t < R; t++) {
                float2 ov[VPL];
#pragma unroll
                for (int q = 0; q < VPL; q++) asm("mov.b64 {%0, %1}, %2;" : "=f"(ov[q].x), "=f"(ov[q].y) : "l"(acc[t][q]));
                st_vec<VPL>(o + t * nv, ov);
            }
        }
        __syncwarp();
        if (lane == 0) {
            tc::mbar_arrive(&empty[s]);
            tc::mbar_arrive(&yempty[yb]);
        }
    }
}

// SL (eqn:bf3 P:791-797 + eqn:tg P:24-28): G[x, c] = sum_k a_k(x) sum_{b < n0} sum_t U[a n0 + b](j, t)
// delta[a n0 + b](t)[c n_amp + k], x = a n0 + j.  A consumer warp owns whole T_X leaves a (the reduction over
// b stays in registers); the producer streams each leaf's pairs in chunks of 4 (coefficients and U blocks,
// one bulk copy each) through a ring shared by the consumers in round-robin order.  Lane = (j group q < 4,
// v group vl < 8): rows j = 2 (4 m + q) + {0, 1} (m < n0 / 8: the 4 groups of one load are 4 consecutive
// 16-byte chunks -- conflict-free) x VPL = nv / 8 vectors (whole RHS columns: VPL % n_amp == 0).
constexpr int SL_SV_B = 4;   // pairs per chunk (2: twice the bulk copies, cfg5 SL 10.2 vs 9.4 ms)

template <int R, int VPL, int NA, int N0>
// (9-12 warps put 3 on some SM sub-partition, whose 16K registers then cap a thread at 168 registers; the
// launch bounds let ptxas apply that cap)
__global__ void __launch_bounds__(32 * (SV_MAX_CONSUMERS + 1), 1)
    sl_sv_kernel(const float2* __restrict__ in, const float2* __restrict__ U, const float2* __restrict__ ampa,
                 float2* __restrict__ G, int64_t ldg, int LN, int S, int C)
{
    constexpr int nv = 8 * VPL, JPL = N0 / 4, NCH = N0 / SL_SV_B;
    constexpr int DB = SL_SV_B * R * nv * 8, UB = SL_SV_B * N0 * R * 8, SB = (DB + UB + 127) / 128 * 128;
    extern __shared__ __align__(128) unsigned char sv_smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sv_smem);
    uint64_t* empty = full + S;
    unsigned char* slots = sv_smem + SV_HDR;
    const int64_t N = int64_t(1) << LN, nleaf = N / N0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // leaves of this CTA: a = blockIdx.x + m gridDim.x, m < Lc; round r has A_r = min(C, Lc - r C) consumers
    const int64_t Lc = (nleaf - blockIdx.x + gridDim.x - 1) / gridDim.x;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; s++) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        tc::mbar_fence_init();
    }
    __syncthreads();

    if (warp == 0) {   // ---- producer: round r, chunk n, consumer w' -> ring index i
        int64_t i = 0;
        for (int64_t r = 0; r * C < Lc; r++) {
            const int A = int(Lc - r * C < C ? Lc - r * C : C);
            for (int n = 0; n < NCH; n++)
                for (int wq = 0; wq < A; wq++, i++) {
                    const int64_t a = blockIdx.x + (r * C + wq) * gridDim.x;
                    const int s = int(i % S);
                    if (i >= S) tc::mbar_wait(&empty[s], uint32_t((i / S - 1) & 1));
                    if (lane == 0) {
                        const int64_t p0 = a * N0 + n * SL_SV_B;
                        tc::mbar_arrive_expect_tx(&full[s], uint32_t(DB + UB));
                        tc::bulk_g2s(slots + size_t(s) * SB, in + p0 * R * nv, uint32_t(DB), &full[s]);
                        tc::bulk_g2s(slots + size_t(s) * SB + DB, U + p0 * R * N0, uint32_t(UB), &full[s]);
                    }
                    __syncwarp();
                }
        }
        return;
    }
    const int wq = warp - 1, q = lane >> 3, vl = lane & 7;
    for (int64_t r = 0; r * C < Lc; r++) {
        const int A = int(Lc - r * C < C ? Lc - r * C : C);
        if (wq >= A) break;
        const int64_t a = blockIdx.x + (r * C + wq) * gridDim.x;
        unsigned long long acc[JPL][VPL];
#pragma unroll
        for (int jj = 0; jj < JPL; jj++)
#pragma unroll
            for (int v = 0; v < VPL; v++) acc[jj][v] = 0ull;
        for (int n = 0; n < NCH; n++) {
            const int64_t i = r * C * NCH + int64_t(n) * A + wq;
            const int s = int(i % S);
            tc::mbar_wait(&full[s], uint32_t((i / S) & 1));
            const float2* D = reinterpret_cast<const float2*>(slots + size_t(s) * SB);
            const float2* Ub = reinterpret_cast<const float2*>(slots + size_t(s) * SB + DB);
#pragma unroll
            for (int bb = 0; bb < SL_SV_B; bb++)
#pragma unroll 2
                for (int t = 0; t < R; t++) {
                    float2 x[VPL], w[JPL];
                    ld_vec<VPL>(x, D + (bb * R + t) * nv + vl * VPL);
                    const float2* uc = Ub + (bb * R + t) * N0 + 2 * q;   // column t of block bb (n0 rows)
#pragma unroll
                    for (int m = 0; m < JPL / 2; m++) {
                        const float4 u4 = *reinterpret_cast<const float4*>(uc + 8 * m);
                        w[2 * m] = make_float2(u4.x, u4.y);
                        w[2 * m + 1] = make_float2(u4.z, u4.w);
                    }
                    unsigned long long xp[VPL], ixp[VPL];
#pragma unroll
                    for (int v = 0; v < VPL; v++) {
                        xp[v] = pk2(x[v].x, x[v].y);
                        ixp[v] = pk2(-x[v].y, x[v].x);
                    }
#pragma unroll
                    for (int jj = 0; jj < JPL; jj++)
#pragma unroll
                        for (int v = 0; v < VPL; v++) cmac2(acc[jj][v], w[jj].x, w[jj].y, xp[v], ixp[v]);
                }
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&empty[s]);
        }
        // epilogue: g(x, c) = sum_k a_k(x) u_k(x) (cmac order of sl_kernel), c = (vl VPL) / NA + cc
#pragma unroll
        for (int jj = 0; jj < JPL; jj++) {
            const int j = 2 * (4 * (jj >> 1) + q) + (jj & 1);
            const int64_t x = a * N0 + j;
            float2 ak[NA];
#pragma unroll
            for (int k = 0; k < NA; k++) ak[k] = __ldg(ampa + k * N + x);
#pragma unroll
            for (int cc = 0; cc < VPL / NA; cc++) {
                float2 g = make_float2(0.f, 0.f);
#pragma unroll
                for (int k = 0; k < NA; k++) {
                    float2 u;
                    asm("mov.b64 {%0, %1}, %2;" : "=f"(u.x), "=f"(u.y) : "l"(acc[jj][cc * NA + k]));
                    cmac(g, ak[k], u);
                }
                G[x + int64_t(vl * VPL / NA + cc) * ldg] = g;
            }
        }
    }
}

template <int R, int VPL>
cudaError_t s0_sv_go(const Dims& d, const float2* F, int64_t ldf, const float2* ampb, const float2* V0, float2* out,
                     int nv, cudaStream_t st)
{
    const int n0 = 1 << d.l0;
    const int SB = (4 * pad32(R * n0 * 8) + 127) / 128 * 128;
    const int ybytes = 2 * n0 * nv * 8;
    int S = (SV_SMEM_LIMIT - SV_HDR - ybytes) / SB;
    if (S < 3) return cudaErrorInvalidValue;
    int C = S - 2 > SV_MAX_CONSUMERS ? SV_MAX_CONSUMERS : S - 2;
    if (S > C + 4) S = C + 4;
    const size_t shm = SV_HDR + ybytes + size_t(S) * SB;
    auto kern = s0_sv_kernel<R, VPL>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm));
    if (e != cudaSuccess) return e;
    const int64_t nleaf = d.N >> d.l0;
    const int64_t grid = nleaf < num_sms() ? nleaf : num_sms();
    kern<<<unsigned(grid), 32 * (C + 2), shm, st>>>(F, ldf, ampb, V0, out, d.LN, d.l0, d.n_amp, nv, S, C);
    e = cudaGetLastError();
    if (e != cudaSuccess && getenv("BF_DEBUG_LAUNCH")) {
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, kern);
        fprintf(stderr, "s0_sv<%d,%d>: threads %d shm %zu grid %lld S %d C %d | regs %d maxthreads %d static smem %zu local %zu\n",
                R, VPL, 32 * (C + 2), shm, (long long)grid, S, C, fa.numRegs, fa.maxThreadsPerBlock, fa.sharedSizeBytes,
                fa.localSizeBytes);
    }
    return e;
}

template <int R, int VPL, int NA, int N0>
cudaError_t sl_sv_go(const Dims& d, const float2* in, const float2* U, const float2* ampa, float2* G, int64_t ldg,
                     cudaStream_t st)
{
    constexpr int nv = 8 * VPL;
    constexpr int SB = (SL_SV_B * R * nv * 8 + SL_SV_B * N0 * R * 8 + 127) / 128 * 128;
    int S = (SV_SMEM_LIMIT - SV_HDR) / SB;
    int C = S - 2 > SV_MAX_CONSUMERS ? SV_MAX_CONSUMERS : S - 2;
    if (C < 1) return cudaErrorInvalidValue;
    if (S > 2 * C) S = 2 * C;
    const size_t shm = SV_HDR + size_t(S) * SB;
    auto kern = sl_sv_kernel<R, VPL, NA, N0>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm));
    if (e != cudaSuccess) return e;
    const int64_t nleaf = d.N / N0;
    const int64_t grid = nleaf < num_sms() ? nleaf : num_sms();
    kern<<<unsigned(grid), 32 * (C + 1), shm, st>>>(in, U, ampa, G, ldg, d.LN, S, C);
    return cudaGetLastError();
}

}  // namespace

bool band_sv_supported(const Dims& d, int nv)
{
    if (!(d.R == 6 || d.R == 8 || d.R == 10 || d.R == 12 || d.R == 14 || d.R == 16)) return false;
    if (nv < 8 || nv >= 128 || nv % 8) return false;
    if (d.N < 4) return false;
    int J, S, C;
    return sv_config(d.R, nv, 2, J, S, C);
}

cudaError_t launch_band_sv(const Dims& d, int l_first, int K, const float2* in, float2* out, const float2* const* W,
                           int nv, cudaStream_t s, int rh, int rhg, const bfs::PeerOut* po)
{
#define BF_SV_CASE(RR)                                                                                     \
    case RR:                                                                                               \
        return K == 2 ? sv_vpl_go<RR, 2>(d, l_first, in, out, W, nv, s, rh, rhg, po)                       \
                      : sv_vpl_go<RR, 1>(d, l_first, in, out, W, nv, s, rh, rhg, po);
    if (K != 1 && K != 2) return cudaErrorInvalidValue;
    switch (d.R) {
        BF_SV_CASE(6) BF_SV_CASE(8) BF_SV_CASE(10) BF_SV_CASE(12) BF_SV_CASE(14) BF_SV_CASE(16)
    default: return cudaErrorInvalidValue;
    }
#undef BF_SV_CASE
}


// S0 / SL for small vector batches: nv % 8 == 0, 8 <= nv <= 64 (S0) / 32 (SL), leaf 8..128 (S0) / 32, 64 (SL)
bool s0_sv_supported(const Dims& d, int nv)
{
    const int n0 = 1 << d.l0;
    if (!(d.R == 6 || d.R == 8 || d.R == 10 || d.R == 12 || d.R == 14 || d.R == 16)) return false;
    if (nv < 8 || nv > 64 || nv % 8 || n0 < 8) return false;
    const int SB = (4 * pad32(d.R * n0 * 8) + 127) / 128 * 128;
    return (SV_SMEM_LIMIT - SV_HDR - 2 * n0 * nv * 8) / SB >= 3;
}

cudaError_t launch_s0_sv(const Dims& d, const float2* F, int64_t ldf, const float2* ampb, const float2* V0,
                         float2* out, int nv, cudaStream_t s)
{
    const bool v2 = nv % 16 == 0;
#define S0SV_CASE(RR) \
    case RR: return v2 ? s0_sv_go<RR, 2>(d, F, ldf, ampb, V0, out, nv, s) : s0_sv_go<RR, 1>(d, F, ldf, ampb, V0, out, nv, s);
    switch (d.R) {
        S0SV_CASE(6) S0SV_CASE(8) S0SV_CASE(10) S0SV_CASE(12) S0SV_CASE(14) S0SV_CASE(16)
    default: return cudaErrorInvalidValue;
    }
#undef S0SV_CASE
}

bool sl_sv_supported(const Dims& d, int nv)
{
    const int n0 = 1 << d.l0;
    if (!(d.R == 6 || d.R == 8 || d.R == 10 || d.R == 12 || d.R == 14 || d.R == 16)) return false;
    if (!(nv == 8 || nv == 16 || nv == 32) || !(n0 == 32 || n0 == 64)) return false;
    if (nv == 32 && n0 == 64) return false;   // 16 x 4 accumulator tile: spills under the 168-register cap
    return (nv / 8) % d.n_amp == 0;
}

cudaError_t launch_sl_sv(const Dims& d, const float2* in, const float2* U, const float2* ampa, float2* G, int64_t ldg,
                         int nv, cudaStream_t s)
{
    const int n0 = 1 << d.l0;
#define SLSV_N0(RR, VV, NA)                                                                                \
    if constexpr (VV == 4) return sl_sv_go<RR, VV, NA, 32>(d, in, U, ampa, G, ldg, s);                     \
    else return n0 == 64 ? sl_sv_go<RR, VV, NA, 64>(d, in, U, ampa, G, ldg, s)                              \
                         : sl_sv_go<RR, VV, NA, 32>(d, in, U, ampa, G, ldg, s);
#define SLSV_V(RR)                                                              \
    if (nv == 8) {                                                              \
        SLSV_N0(RR, 1, 1)                                                       \
    } else if (nv == 16) {                                                      \
        if (d.n_amp == 2) { SLSV_N0(RR, 2, 2) } else { SLSV_N0(RR, 2, 1) }      \
    } else {                                                                    \
        if (d.n_amp == 4) { SLSV_N0(RR, 4, 4) }                                 \
        else if (d.n_amp == 2) { SLSV_N0(RR, 4, 2) } else { SLSV_N0(RR, 4, 1) } \
    }
    switch (d.R) {
    case 6: SLSV_V(6)
    case 8: SLSV_V(8)
    case 10: SLSV_V(10)
    case 12: SLSV_V(12)
    case 14: SLSV_V(14)
    case 16: SLSV_V(16)
    default: return cudaErrorInvalidValue;
    }
#undef SLSV_V
#undef SLSV_N0
}

}  // namespace bfk
