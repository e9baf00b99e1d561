// bf_kernels.cu -- sm_100a kernels of the IBF-MAT apply (arXiv:1803.04128).
//
// Every stage of eqn:BFM is a batch of small dense complex block
// products that share nothing but the coefficient arrays, so each is written
// as an FP32 register-blocked "outer product" loop: a thread owns TN
// consecutive vectors of one unit (leaf / butterfly / T_X leaf) and R (or JT)
// output rows; the block entries of one unit are warp-uniform loads (L1
// broadcast), the vector operands are coalesced 16-byte loads.  4 FFMA per
// complex MAC, FP32 accumulation (north_star).
//
// Coefficient layout (workspace): delta[pair][t][v], v < nv fastest,
// v = c * n_amp + k (RHS column c, amplitude term k).  See DESIGN.md section 4.
#include <cuda_runtime.h>
#include <cstdint>

#include "bf_internal.h"

namespace bfk {

__device__ __forceinline__ void cmac(float2& acc, const float2 w, const float2 v)
{
    acc.x = fmaf(w.x, v.x, acc.x);
    acc.x = fmaf(-w.y, v.y, acc.x);
    acc.y = fmaf(w.x, v.y, acc.y);
    acc.y = fmaf(w.y, v.x, acc.y);
}

__device__ __forceinline__ float2 cmul(const float2 a, const float2 b)
{
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// Load / store K consecutive complex values (16-byte vectors where possible).
template <int K>
__device__ __forceinline__ void ldc(float2 (&v)[K], const float2* p)
{
    if constexpr (K % 2 == 0) {
#pragma unroll
        for (int i = 0; i < K / 2; i++) {
            float4 q = reinterpret_cast<const float4*>(p)[i];
            v[2 * i] = make_float2(q.x, q.y);
            v[2 * i + 1] = make_float2(q.z, q.w);
        }
    } else {
#pragma unroll
        for (int i = 0; i < K; i++) v[i] = p[i];
    }
}

template <int K>
__device__ __forceinline__ void ldc_ro(float2 (&v)[K], const float2* __restrict__ p)
{
    if constexpr (K % 2 == 0) {
#pragma unroll
        for (int i = 0; i < K / 2; i++) {
            float4 q = __ldg(reinterpret_cast<const float4*>(p) + i);
            v[2 * i] = make_float2(q.x, q.y);
            v[2 * i + 1] = make_float2(q.z, q.w);
        }
    } else {
#pragma unroll
        for (int i = 0; i < K; i++) v[i] = __ldg(p + i);
    }
}

template <int K>
__device__ __forceinline__ void stc(float2* p, const float2 (&v)[K])
{
    if constexpr (K % 2 == 0) {
#pragma unroll
        for (int i = 0; i < K / 2; i++)
            reinterpret_cast<float4*>(p)[i] = make_float4(v[2 * i].x, v[2 * i].y, v[2 * i + 1].x, v[2 * i + 1].y);
    } else {
#pragma unroll
        for (int i = 0; i < K; i++) p[i] = v[i];
    }
}

// ---------------------------------------------------------------------------
// S0: amplitude pre-scale + leaf interpolation (eqn:1; eqn:tg P:24-28).
// CTA = 32 columns (lanes) x 8 warps.  A column is (leaf b, vector group vg).
// The scaled leaf inputs y[j][v] = b_k(x) F[x, c] are staged once in shared
// memory; warp w computes the pairs (a, b) for a = w, w+8, ...
// ---------------------------------------------------------------------------
template <int R, int TN>
__global__ void __launch_bounds__(256) s0_kernel(const float2* __restrict__ F, int64_t ldf,
                                                 const float2* __restrict__ ampb, const float2* __restrict__ V0,
                                                 float2* __restrict__ out, int LN, int l0, int n_amp, int nv)
{
    extern __shared__ float4 smem_s0[];
    float2* Ys = reinterpret_cast<float2*>(smem_s0);   // [n0][32 * TN]
    const int64_t N = int64_t(1) << LN;
    const int n0 = 1 << l0;
    const int64_t nleaf = N >> l0;
    const int cpu = nv / TN;   // columns per leaf
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int64_t col0 = int64_t(blockIdx.x) * 32;
    constexpr int W = 32 * TN;

    for (int e = threadIdx.x; e < n0 * W; e += blockDim.x) {
        const int j = e % n0, ci = e / n0, col = ci / TN, i = ci % TN;
        const int64_t gcol = col0 + col, b = gcol / cpu;
        float2 val = make_float2(0.f, 0.f);
        if (b < nleaf) {
            const int v = int(gcol % cpu) * TN + i, c = v / n_amp, k = v % n_amp;
            const int64_t x = b * n0 + j;
            val = cmul(__ldg(ampb + k * N + x), __ldg(F + x + c * ldf));
        }
        Ys[j * W + col * TN + i] = val;
    }
    __syncthreads();

    const int64_t gc = col0 + lane, b = gc / cpu;
    if (b >= nleaf) return;
    const int vg = int(gc % cpu);
    for (int a = warp; a < n0; a += nwarps) {
        const int64_t p = int64_t(a) * nleaf + b;
        const float2* Vb = V0 + p * n0 * R;   // column-major r x n0: column j at j*R
        float2 acc[R][TN];
#pragma unroll
        for (int t = 0; t < R; t++)
#pragma unroll
            for (int i = 0; i < TN; i++) acc[t][i] = make_float2(0.f, 0.f);
#pragma unroll 2
        for (int j = 0; j < n0; j++) {
            float2 y[TN], w[R];
            ldc<TN>(y, Ys + j * W + lane * TN);
            ldc_ro<R>(w, Vb + j * R);
#pragma unroll
            for (int t = 0; t < R; t++)
#pragma unroll
                for (int i = 0; i < TN; i++) cmac(acc[t][i], w[t], y[i]);
        }
        float2* o = out + p * R * nv + vg * TN;
#pragma unroll
        for (int t = 0; t < R; t++) stc<TN>(o + int64_t(t) * nv, acc[t]);
    }
}

// ---------------------------------------------------------------------------
// Transfer level (eqn:2 P:748-752 for l <= h, eqn:3 P:780-785 for l > h).
// A butterfly unit u = P 2^(LN-l) + b reads the two pairs 2u, 2u+1 of level
// l-1 (contiguous: [2 R][nv]) and writes the pairs (2P+e) 2^(LN-l) + b, e=0,1.
// One thread: both outputs (2 R rows) x TN vectors.  With SW, the switch block
// of each output pair is applied in registers before the store.
// ---------------------------------------------------------------------------
template <int R, int TN, bool SW>
__global__ void __launch_bounds__(128) xfer_kernel(const float2* __restrict__ in, float2* __restrict__ out,
                                                   const float2* __restrict__ Wl, const float2* __restrict__ Sw,
                                                   int LN, int l, int nv)
{
    const int64_t N = int64_t(1) << LN;
    const int cpu = nv / TN;
    const int64_t gc = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t u = gc / cpu;
    if (u >= N / 2) return;
    const int vg = int(gc % cpu);
    const int sh = LN - l;
    const int64_t P = u >> sh, b = u & ((int64_t(1) << sh) - 1);
    const int64_t p0 = (2 * P << sh) + b, p1 = p0 + (int64_t(1) << sh);
    const float2* x = in + 2 * u * R * nv + vg * TN;
    const float2* W0 = Wl + p0 * 2 * R * R;   // column-major r x 2r: column k at k*R
    const float2* W1 = Wl + p1 * 2 * R * R;

    float2 acc0[R][TN], acc1[R][TN];
#pragma unroll
    for (int t = 0; t < R; t++)
#pragma unroll
        for (int i = 0; i < TN; i++) acc0[t][i] = acc1[t][i] = make_float2(0.f, 0.f);

#pragma unroll 2
    for (int k = 0; k < 2 * R; k++) {
        float2 xv[TN], w[R];
        ldc_ro<TN>(xv, x + int64_t(k) * nv);
        ldc_ro<R>(w, W0 + k * R);
#pragma unroll
        for (int t = 0; t < R; t++)
#pragma unroll
            for (int i = 0; i < TN; i++) cmac(acc0[t][i], w[t], xv[i]);
        ldc_ro<R>(w, W1 + k * R);
#pragma unroll
        for (int t = 0; t < R; t++)
#pragma unroll
            for (int i = 0; i < TN; i++) cmac(acc1[t][i], w[t], xv[i]);
    }

#pragma unroll
    for (int e = 0; e < 2; e++) {
        float2 (&acc)[R][TN] = e ? acc1 : acc0;
        const int64_t p = e ? p1 : p0;
        float2* o = out + p * R * nv + vg * TN;
        if constexpr (SW) {
            const float2* S = Sw + p * R * R;   // column-major r x r: column s at s*R
            float2 res[R][TN];
#pragma unroll
            for (int t = 0; t < R; t++)
#pragma unroll
                for (int i = 0; i < TN; i++) res[t][i] = make_float2(0.f, 0.f);
#pragma unroll
            for (int s = 0; s < R; s++) {
                float2 w[R];
                ldc_ro<R>(w, S + s * R);
#pragma unroll
                for (int t = 0; t < R; t++)
#pragma unroll
                    for (int i = 0; i < TN; i++) cmac(res[t][i], w[t], acc[s][i]);
            }
#pragma unroll
            for (int t = 0; t < R; t++) stc<TN>(o + int64_t(t) * nv, res[t]);
        } else {
#pragma unroll
            for (int t = 0; t < R; t++) stc<TN>(o + int64_t(t) * nv, acc[t]);
        }
    }
}

// Switch alone: out[p] = Sw[p] in[p] (only when h == l0).
template <int R, int TN>
__global__ void __launch_bounds__(128) switch_kernel(const float2* __restrict__ in, float2* __restrict__ out,
                                                     const float2* __restrict__ Sw, int LN, int nv)
{
    const int64_t N = int64_t(1) << LN;
    const int cpu = nv / TN;
    const int64_t gc = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t p = gc / cpu;
    if (p >= N) return;
    const int vg = int(gc % cpu);
    const float2* x = in + p * R * nv + vg * TN;
    const float2* S = Sw + p * R * R;
    float2 res[R][TN];
#pragma unroll
    for (int t = 0; t < R; t++)
#pragma unroll
        for (int i = 0; i < TN; i++) res[t][i] = make_float2(0.f, 0.f);
#pragma unroll
    for (int s = 0; s < R; s++) {
        float2 xv[TN], w[R];
        ldc_ro<TN>(xv, x + int64_t(s) * nv);
        ldc_ro<R>(w, S + s * R);
#pragma unroll
        for (int t = 0; t < R; t++)
#pragma unroll
            for (int i = 0; i < TN; i++) cmac(res[t][i], w[t], xv[i]);
    }
    float2* o = out + p * R * nv + vg * TN;
#pragma unroll
    for (int t = 0; t < R; t++) stc<TN>(o + int64_t(t) * nv, res[t]);
}

// ---------------------------------------------------------------------------
// SL: leaf evaluation (eqn:bf3) + amplitude post-scale and sum over
// k (eqn:tg).  CTA = 32 columns (T_X leaf a, vector group) x n0/JT
// warps; warp w owns the JT output rows j in [w JT, w JT + JT).
// ---------------------------------------------------------------------------
template <int R, int TN, int JT, int NA>
__global__ void __launch_bounds__(256) sl_kernel(const float2* __restrict__ in, const float2* __restrict__ U,
                                                 const float2* __restrict__ ampa, float2* __restrict__ G, int64_t ldg,
                                                 int LN, int l0, int nv)
{
    static_assert(TN % NA == 0, "a thread owns whole RHS columns");
    const int64_t N = int64_t(1) << LN;
    const int n0 = 1 << l0;
    const int64_t nleaf = N >> l0;
    const int cpu = nv / TN;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t gc = int64_t(blockIdx.x) * 32 + lane, a = gc / cpu;
    if (a >= nleaf) return;
    const int vg = int(gc % cpu);
    const int j0 = warp * JT;

    float2 acc[JT][TN];
#pragma unroll
    for (int jj = 0; jj < JT; jj++)
#pragma unroll
        for (int i = 0; i < TN; i++) acc[jj][i] = make_float2(0.f, 0.f);

    for (int b = 0; b < n0; b++) {
        const int64_t p = a * n0 + b;
        const float2* x = in + p * R * nv + vg * TN;
        const float2* Ub = U + p * R * n0 + j0;   // column-major n0 x r: column t at t*n0
#pragma unroll 2
        for (int t = 0; t < R; t++) {
            float2 xv[TN], w[JT];
            ldc_ro<TN>(xv, x + int64_t(t) * nv);
            ldc_ro<JT>(w, Ub + t * n0);
#pragma unroll
            for (int jj = 0; jj < JT; jj++)
#pragma unroll
                for (int i = 0; i < TN; i++) cmac(acc[jj][i], w[jj], xv[i]);
        }
    }
    // epilogue: G[x, c] = sum_k a_k(x) u_k(x)
    const int c0 = vg * (TN / NA);
#pragma unroll
    for (int jj = 0; jj < JT; jj++) {
        const int64_t xrow = a * n0 + j0 + jj;
        float2 ak[NA];
#pragma unroll
        for (int k = 0; k < NA; k++) ak[k] = __ldg(ampa + k * N + xrow);
#pragma unroll
        for (int cc = 0; cc < TN / NA; cc++) {
            float2 g = make_float2(0.f, 0.f);
#pragma unroll
            for (int k = 0; k < NA; k++) cmac(g, ak[k], acc[jj][cc * NA + k]);
            G[xrow + int64_t(c0 + cc) * ldg] = g;
        }
    }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
bool rank_supported(int R) { return R == 6 || R == 8 || R == 10 || R == 12 || R == 14 || R == 16; }

static inline int pick_tn(int nv, int maxtn)
{
    if (maxtn >= 4 && nv % 4 == 0) return 4;
    if (maxtn >= 2 && nv % 2 == 0) return 2;
    return 1;
}

template <int R, int TN>
static cudaError_t s0_go(const Dims& d, const float2* F, int64_t ldf, const float2* ampb, const float2* V0, float2* out,
                         int nv, cudaStream_t s)
{
    const int64_t cols = (d.N >> d.l0) * (nv / TN);
    const size_t shm = size_t(1 << d.l0) * 32 * TN * sizeof(float2);
    auto kern = s0_kernel<R, TN>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm));
    if (e != cudaSuccess) return e;
    kern<<<unsigned((cols + 31) / 32), 256, shm, s>>>(F, ldf, ampb, V0, out, d.LN, d.l0, d.n_amp, nv);
    return cudaGetLastError();
}

template <int R, bool SW, int TN>
static cudaError_t xfer_go(const Dims& d, int l, const float2* in, float2* out, const float2* W, const float2* Sw, int nv,
                           cudaStream_t s)
{
    const int64_t threads = (d.N / 2) * (nv / TN);
    xfer_kernel<R, TN, SW><<<unsigned((threads + 127) / 128), 128, 0, s>>>(in, out, W, Sw, d.LN, l, nv);
    return cudaGetLastError();
}

template <int R, int TN>
static cudaError_t sw_go(const Dims& d, const float2* in, float2* out, const float2* Sw, int nv, cudaStream_t s)
{
    const int64_t threads = d.N * (nv / TN);
    switch_kernel<R, TN><<<unsigned((threads + 127) / 128), 128, 0, s>>>(in, out, Sw, d.LN, nv);
    return cudaGetLastError();
}

template <int R, int TN, int NA>
static cudaError_t sl_go(const Dims& d, const float2* in, const float2* U, const float2* ampa, float2* G, int64_t ldg,
                         int nv, cudaStream_t s)
{
    constexpr int JT = 8;
    const int n0 = 1 << d.l0;
    const int64_t cols = (d.N >> d.l0) * (nv / TN);
    sl_kernel<R, TN, JT, NA><<<unsigned((cols + 31) / 32), 32 * (n0 / JT), 0, s>>>(in, U, ampa, G, ldg, d.LN, d.l0, nv);
    return cudaGetLastError();
}

#define BF_DISPATCH_R(R, CALL)                                                                                         \
    switch (R) {                                                                                                       \
    case 6: { constexpr int RR = 6; return CALL; }                                                                     \
    case 8: { constexpr int RR = 8; return CALL; }                                                                     \
    case 10: { constexpr int RR = 10; return CALL; }                                                                   \
    case 12: { constexpr int RR = 12; return CALL; }                                                                   \
    case 14: { constexpr int RR = 14; return CALL; }                                                                   \
    case 16: { constexpr int RR = 16; return CALL; }                                                                   \
    default: return cudaErrorInvalidValue;                                                                             \
    }

cudaError_t launch_s0(const Dims& d, const float2* F, int64_t ldf, const float2* ampb, const float2* V0, float2* out,
                      int nv, cudaStream_t s)
{
    const int tn = pick_tn(nv, 4);
    if (tn == 4) BF_DISPATCH_R(d.R, (s0_go<RR, 4>(d, F, ldf, ampb, V0, out, nv, s)))
    if (tn == 2) BF_DISPATCH_R(d.R, (s0_go<RR, 2>(d, F, ldf, ampb, V0, out, nv, s)))
    BF_DISPATCH_R(d.R, (s0_go<RR, 1>(d, F, ldf, ampb, V0, out, nv, s)))
}

cudaError_t launch_xfer(const Dims& d, int l, const float2* in, float2* out, const float2* W, const float2* Sw, int nv,
                        cudaStream_t s)
{
    const int tn = pick_tn(nv, 2);
    if (Sw) {
        if (tn == 2) BF_DISPATCH_R(d.R, (xfer_go<RR, true, 2>(d, l, in, out, W, Sw, nv, s)))
        BF_DISPATCH_R(d.R, (xfer_go<RR, true, 1>(d, l, in, out, W, Sw, nv, s)))
    }
    if (tn == 2) BF_DISPATCH_R(d.R, (xfer_go<RR, false, 2>(d, l, in, out, W, Sw, nv, s)))
    BF_DISPATCH_R(d.R, (xfer_go<RR, false, 1>(d, l, in, out, W, Sw, nv, s)))
}

cudaError_t launch_switch(const Dims& d, const float2* in, float2* out, const float2* Sw, int nv, cudaStream_t s)
{
    const int tn = pick_tn(nv, 2);
    if (tn == 2) BF_DISPATCH_R(d.R, (sw_go<RR, 2>(d, in, out, Sw, nv, s)))
    BF_DISPATCH_R(d.R, (sw_go<RR, 1>(d, in, out, Sw, nv, s)))
}

cudaError_t launch_sl(const Dims& d, const float2* in, const float2* U, const float2* ampa, float2* G, int64_t ldg,
                      int nv, cudaStream_t s)
{
    // a thread must own whole RHS columns (all n_amp terms of a column): TN % n_amp == 0
    int tn = pick_tn(nv, 4);
    if (tn % d.n_amp != 0) tn = d.n_amp;
    if (d.n_amp == 4) BF_DISPATCH_R(d.R, (sl_go<RR, 4, 4>(d, in, U, ampa, G, ldg, nv, s)))
    if (d.n_amp == 2) {
        if (tn == 4) BF_DISPATCH_R(d.R, (sl_go<RR, 4, 2>(d, in, U, ampa, G, ldg, nv, s)))
        BF_DISPATCH_R(d.R, (sl_go<RR, 2, 2>(d, in, U, ampa, G, ldg, nv, s)))
    }
    if (tn == 4) BF_DISPATCH_R(d.R, (sl_go<RR, 4, 1>(d, in, U, ampa, G, ldg, nv, s)))
    if (tn == 2) BF_DISPATCH_R(d.R, (sl_go<RR, 2, 1>(d, in, U, ampa, G, ldg, nv, s)))
    BF_DISPATCH_R(d.R, (sl_go<RR, 1, 1>(d, in, U, ampa, G, ldg, nv, s)))
}

}  // namespace bfk
