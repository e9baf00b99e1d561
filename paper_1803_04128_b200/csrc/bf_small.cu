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
#pragma unroll
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

// vectors per lane: 2 (R x 2 register tile, passes of 16 vectors) unless nv is not a multiple of 16
int sv_vpl(int nv)
{
    static const int v_env = env_int("BF_SV_VPL");   // tuning experiments
    if (v_env == 4 && nv % 32 == 0) return 4;
    if (v_env == 1) return 1;
    return nv % 16 == 0 ? 2 : 1;
}

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
    case 4: SV_J(4)
    case 2: SV_J(2)
    default: SV_J(1)
    }
#undef SV_J
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

}  // namespace bfk
