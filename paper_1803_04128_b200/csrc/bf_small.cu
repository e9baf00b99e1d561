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

#include "bf_internal.h"
#include "bf_shard.h"
#include "tc_sm100.cuh"

namespace bfk {

namespace {

constexpr int SV_MAX_CONSUMERS = 8;
constexpr int SV_SMEM_LIMIT = 220 * 1024;

// bytes of one weight block in shared memory: 2 r^2 complex, padded to 32 (mod 128)
__host__ __device__ constexpr int sv_wblk(int R)
{
    return 16 * R * R + ((32 - (16 * R * R) % 128) % 128 + 128) % 128;
}
__host__ __device__ constexpr int sv_xbytes(int R, int nv) { return 4 * R * nv * 8; }
__host__ __device__ constexpr int sv_slot(int R, int nv, int K) { return sv_xbytes(R, nv) + 4 * K * sv_wblk(R); }

__device__ __forceinline__ void cmac(float2& acc, const float2 w, const float2 v)
{
    acc.x = fmaf(w.x, v.x, acc.x);
    acc.x = fmaf(-w.y, v.y, acc.x);
    acc.y = fmaf(w.x, v.y, acc.y);
    acc.y = fmaf(w.y, v.x, acc.y);
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

template <int R, int VPL, int K>
__global__ void __launch_bounds__(32 * (SV_MAX_CONSUMERS + 1), 1)
    band_sv_kernel(const float2* __restrict__ in, float2* __restrict__ out, const SvArgs args, int LN, int l_first,
                   int nv, int64_t njobs, int S, int C)
{
    extern __shared__ __align__(128) unsigned char sv_smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sv_smem);
    uint64_t* empty = full + S;
    unsigned char* slots = sv_smem + 1024;
    const int WB = sv_wblk(R);
    const int XB = sv_xbytes(R, nv);
    const int SB = XB + 4 * K * WB;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; s++) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        tc::mbar_fence_init();
    }
    __syncthreads();

    if (warp == 0) {
        // ---- producer: job i of this CTA -> slot i % S ----
        for (int64_t i = 0;; i++) {
            const int64_t j = blockIdx.x + i * gridDim.x;
            if (j >= njobs) break;
            const int s = int(i % S);
            if (i >= S) tc::mbar_wait(&empty[s], uint32_t((i / S - 1) & 1));
            unsigned char* slot = slots + size_t(s) * SB;
            if (lane == 0) tc::mbar_arrive_expect_tx(&full[s], uint32_t(XB + 4 * K * 16 * R * R));
            __syncwarp();
            if (lane == 0) {
                const int64_t pin = args.rh ? bfs::recv_index(4 * j, args.rh, args.rhg) : 4 * j;
                tc::bulk_g2s(slot, in + pin * R * int64_t(nv), uint32_t(XB), &full[s]);
            } else if (lane <= 4 * K) {
                const int w = lane - 1, m = w / 4 + 1, os = w % 4;
                const int64_t p = sv_pair(j, m, os >> 1, os & 1, LN, l_first);
                tc::bulk_g2s(slot + XB + w * WB, args.W[m - 1] + p * 2 * R * R, uint32_t(16 * R * R), &full[s]);
            }
        }
        return;
    }

    // ---- consumers: warp w takes jobs i = w - 1, w - 1 + C, ... ----
    const int os = lane >> 3, vl = lane & 7, u = os >> 1, e = os & 1;
    const int passes = nv / (8 * VPL);
    for (int64_t i = warp - 1;; i += C) {
        const int64_t j = blockIdx.x + i * gridDim.x;
        if (j >= njobs) break;
        const int s = int(i % S);
        tc::mbar_wait(&full[s], uint32_t((i / S) & 1));
        float2* X = reinterpret_cast<float2*>(slots + size_t(s) * SB);
#pragma unroll 1
        for (int m = 1; m <= K; m++) {
            const int in0 = (m == 1) ? 2 * u : u, in1 = (m == 1) ? 2 * u + 1 : u + 2;
            const float2* Wb = reinterpret_cast<const float2*>(slots + size_t(s) * SB + XB + ((m - 1) * 4 + os) * WB);
            float2* dst;
            int64_t rs;   // row stride of the destination (complex)
            if (m < K) {
                dst = X + (2 * u + e) * R * nv;
                rs = nv;
            } else {
                dst = bfs::pair_out(out, args.po, sv_pair(j, m, u, e, LN, l_first), R, nv);
                rs = nv;
            }
#pragma unroll 1
            for (int ps = 0; ps < passes; ps++) {
                const int vb = ps * 8 * VPL + vl * VPL;
                float2 acc[R][VPL];
#pragma unroll
                for (int t = 0; t < R; t++)
#pragma unroll
                    for (int q = 0; q < VPL; q++) acc[t][q] = make_float2(0.f, 0.f);
#pragma unroll
                for (int c = 0; c < 2; c++) {
                    const float2* xs = X + (c ? in1 : in0) * R * nv + vb;
                    const float2* wc = Wb + c * R * R;
#pragma unroll 2
                    for (int sr = 0; sr < R; sr++) {
                        float2 x[VPL], w[R];
                        ld_vec<VPL>(x, xs + sr * nv);
                        ld_vec<R>(w, wc + sr * R);
#pragma unroll
                        for (int t = 0; t < R; t++)
#pragma unroll
                            for (int q = 0; q < VPL; q++) cmac(acc[t][q], w[t], x[q]);
                    }
                }
                if (m < K) __syncwarp();   // both outputs of unit u have read its input slots (this pass's columns)
#pragma unroll
                for (int t = 0; t < R; t++) st_vec<VPL>(dst + t * rs + vb, acc[t]);
            }
            if (m < K) __syncwarp();   // level m in place before level m + 1 reads it
        }
        // generic-proxy writes to the slot (level l in place) -> ordered before the next bulk copy into it
        if (K > 1) tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&empty[s]);
    }
}

int sv_vpl(int nv) { return (nv % 32 == 0) ? 4 : (nv % 16 == 0) ? 2 : 1; }

// ring depth and consumer warps for one CTA per SM
bool sv_config(int R, int nv, int K, int& S, int& C)
{
    const int sb = sv_slot(R, nv, K);
    S = (SV_SMEM_LIMIT - 1024) / sb;
    if (S < 2) return false;
    C = S - 2 > SV_MAX_CONSUMERS ? SV_MAX_CONSUMERS : S - 2;   // >= 2 slots of prefetch
    if (C < 1) {
        C = 1;
    }
    if (S > C + 4) S = C + 4;
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

template <int R, int VPL, int K>
cudaError_t sv_go(const Dims& d, int l_first, const float2* in, float2* out, const float2* const* W, int nv,
                  cudaStream_t st, int rh, int rhg, const bfs::PeerOut* po)
{
    int S = 0, C = 0;
    if (!sv_config(R, nv, K, S, C)) return cudaErrorInvalidValue;
    SvArgs a{};
    a.W[0] = W[0];
    a.W[1] = K > 1 ? W[1] : nullptr;
    if (po) a.po = *po;
    a.rh = rh;
    a.rhg = rhg;
    const size_t shm = 1024 + size_t(S) * sv_slot(R, nv, K);
    auto kern = band_sv_kernel<R, VPL, K>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm));
    if (e != cudaSuccess) return e;
    const int64_t njobs = d.N / 4;
    const int64_t grid = njobs < num_sms() ? njobs : num_sms();
    kern<<<unsigned(grid), 32 * (C + 1), shm, st>>>(in, out, a, d.LN, l_first, nv, njobs, S, C);
    return cudaGetLastError();
}

template <int R, int K>
cudaError_t sv_vpl_go(const Dims& d, int l_first, const float2* in, float2* out, const float2* const* W, int nv,
                      cudaStream_t st, int rh, int rhg, const bfs::PeerOut* po)
{
    switch (sv_vpl(nv)) {
    case 4: return sv_go<R, 4, K>(d, l_first, in, out, W, nv, st, rh, rhg, po);
    case 2: return sv_go<R, 2, K>(d, l_first, in, out, W, nv, st, rh, rhg, po);
    default: return sv_go<R, 1, K>(d, l_first, in, out, W, nv, st, rh, rhg, po);
    }
}

}  // namespace

bool band_sv_supported(const Dims& d, int nv)
{
    if (!(d.R == 6 || d.R == 8 || d.R == 10 || d.R == 12 || d.R == 14 || d.R == 16)) return false;
    if (nv < 8 || nv >= 128 || nv % 8) return false;
    if (d.N < 4) return false;
    int S, C;
    return sv_config(d.R, nv, 2, S, C);
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
