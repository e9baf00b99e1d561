// bf_struct.cu -- the apply on STRUCTURED interpolative factors (include/bf.h "structured
// plans").  Every interpolative block of Algorithm 4.1 is diag(phases) . L . diag(phases) with the Lagrange
// matrix L shared by the whole level, because the Mock-Chebyshev grids of a level are translates of each other
// (eqn:gdA/gdB P:214-226, "simply shift the grid points" P:213).  The plan stores per pair only the merged
// phase diagonal of each level (bf_build.cpp) and per level one real matrix:
//   S0      eta[p](t)       = sum_j L0(t, j) omega[p][j] y_b[j],            y_b[j] = b_k(x) F[x, c], x = b n0 + j
//   first   eta_l[p](t)     = sum_{c,s} L1(t, c r + s) psi[p][c r + s] eta_{l-1}[q_c](s)           (eqn:2)
//   second  zeta_l[p](t)    = sum_c chi[p][c r + t] sum_s L2_{a&1}(t, s) zeta_{l-1}[q_c](s)        (eqn:3)
//   SL      G[a n0 + j, c]  = sum_k a_k(x) sum_{b<n0} Omega[a n0 + b][j] sum_t Lsl(j, t) zeta_D[a n0 + b](t)
// with q_c = (a >> 1) 2^(LN-l+1) + 2b + c the input pairs of p = a 2^(LN-l) + b.  A complex x real product is 2
// FMAs against 4 for the dense complex block, and the factor stream per level drops from 2r^2 to 2r complex per
// pair.  Level h (switch P:755-766 with both neighbouring phase diagonals) stays a dense block (bf_kernels.cu).
//
// This file holds the GENERIC kernels (any nv, one level per launch; a thread owns one (pair, vector) and all r
// outputs, L staged in shared memory and read as warp-uniform broadcasts) and the expansion of structured
// factors into dense blocks for the tensor-core path (plan finalization).
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>

#include "bf_internal.h"

namespace bfk {

namespace {

__device__ __forceinline__ float2 cmul(const float2 a, const float2 b)
{
    return make_float2(fmaf(a.x, b.x, -(a.y * b.y)), fmaf(a.x, b.y, a.y * b.x));
}

unsigned grid_of(int64_t n, int block) { return unsigned((n + block - 1) / block); }

// ---- S0: CTA = (leaf b, chunk of VC vectors); y_b staged in shared memory; thread = (a, vector) ----
constexpr int S0_VC = 32;

template <int R>
__global__ void __launch_bounds__(256) s0_st_kernel(const float2* __restrict__ F, int64_t ldf,
                                                    const float2* __restrict__ ampb, const float* __restrict__ L0,
                                                    const float2* __restrict__ om, float2* __restrict__ out, int LN,
                                                    int l0, int n_amp, int nv)
{
    extern __shared__ __align__(16) unsigned char st_smem[];
    const int n0 = 1 << l0;
    const int64_t N = int64_t(1) << LN, nleaf = N >> l0;
    float* Ls = reinterpret_cast<float*>(st_smem);                 // [n0][R]
    float2* Y = reinterpret_cast<float2*>(st_smem + ((R * n0 * 4 + 15) / 16) * 16);   // [n0][VC]
    const int64_t b = blockIdx.x;
    const int v0 = blockIdx.y * S0_VC, vc = min(S0_VC, nv - v0);
    for (int i = threadIdx.x; i < R * n0; i += blockDim.x) Ls[i] = L0[i];
    for (int i = threadIdx.x; i < n0 * vc; i += blockDim.x) {
        const int j = i % n0, vl = i / n0, v = v0 + vl;
        const int64_t x = b * n0 + j;
        Y[j * S0_VC + vl] = cmul(__ldg(ampb + int64_t(v % n_amp) * N + x), __ldg(F + x + int64_t(v / n_amp) * ldf));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n0 * vc; i += blockDim.x) {
        const int vl = i % vc, a = i / vc;
        const int64_t p = int64_t(a) * nleaf + b;
        const float2* o = om + p * n0;
        float2 acc[R];
#pragma unroll
        for (int t = 0; t < R; t++) acc[t] = make_float2(0.f, 0.f);
        for (int j = 0; j < n0; j++) {
            const float2 z = cmul(__ldg(o + j), Y[j * S0_VC + vl]);
#pragma unroll
            for (int t = 0; t < R; t++) {
                const float w = Ls[j * R + t];
                acc[t].x = fmaf(w, z.x, acc[t].x);
                acc[t].y = fmaf(w, z.y, acc[t].y);
            }
        }
        float2* dst = out + p * R * nv + v0 + vl;
#pragma unroll
        for (int t = 0; t < R; t++) dst[int64_t(t) * nv] = acc[t];
    }
}

// ---- one transfer level: thread = (output pair p, vector v) ----
template <int R, int KIND>
__global__ void __launch_bounds__(256) xfer_st_kernel(const float* __restrict__ L, const float2* __restrict__ ph,
                                                      const float2* __restrict__ in, float2* __restrict__ out, int LN,
                                                      int l, int nv, int64_t total)
{
    __shared__ float Ls[2 * R * R];
    for (int i = threadIdx.x; i < 2 * R * R; i += blockDim.x) Ls[i] = L[i];
    __syncthreads();
    const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g >= total) return;
    const int64_t p = g / nv;
    const int v = int(g % nv);
    const int sh = LN - l;
    const int64_t a = p >> sh, b = p & ((int64_t(1) << sh) - 1);
    const int64_t q0 = ((a >> 1) << (sh + 1)) + 2 * b;   // input pairs q0, q0 + 1 at level l - 1
    const float2* php = ph + p * 2 * R;
    float2 acc[R];
#pragma unroll
    for (int t = 0; t < R; t++) acc[t] = make_float2(0.f, 0.f);
#pragma unroll
    for (int c = 0; c < 2; c++) {
        const float2* x = in + (q0 + c) * R * nv + v;
        if (KIND == 1) {   // first half: phases on the inputs, then L1
#pragma unroll
            for (int s = 0; s < R; s++) {
                const float2 y = cmul(__ldg(php + c * R + s), __ldg(x + int64_t(s) * nv));
#pragma unroll
                for (int t = 0; t < R; t++) {
                    const float w = Ls[(c * R + s) * R + t];
                    acc[t].x = fmaf(w, y.x, acc[t].x);
                    acc[t].y = fmaf(w, y.y, acc[t].y);
                }
            }
        } else {           // second half: L2_e on each input, phases on the outputs
            const float* Le = Ls + int(a & 1) * R * R;
            float2 z[R];
#pragma unroll
            for (int t = 0; t < R; t++) z[t] = make_float2(0.f, 0.f);
#pragma unroll
            for (int s = 0; s < R; s++) {
                const float2 y = __ldg(x + int64_t(s) * nv);
#pragma unroll
                for (int t = 0; t < R; t++) {
                    const float w = Le[s * R + t];
                    z[t].x = fmaf(w, y.x, z[t].x);
                    z[t].y = fmaf(w, y.y, z[t].y);
                }
            }
#pragma unroll
            for (int t = 0; t < R; t++) {
                const float2 f = __ldg(php + c * R + t);
                acc[t].x = fmaf(f.x, z[t].x, acc[t].x);
                acc[t].x = fmaf(-f.y, z[t].y, acc[t].x);
                acc[t].y = fmaf(f.x, z[t].y, acc[t].y);
                acc[t].y = fmaf(f.y, z[t].x, acc[t].y);
            }
        }
    }
    float2* dst = out + p * R * nv + v;
#pragma unroll
    for (int t = 0; t < R; t++) dst[int64_t(t) * nv] = acc[t];
}

// ---- SL: CTA = (T_X leaf a, chunk of columns); thread = (row j, column c), the sum over k and b in registers
constexpr int SL_CC = 4;

template <int R>
__global__ void __launch_bounds__(256) sl_st_kernel(const float2* __restrict__ in, const float* __restrict__ Lsl,
                                                    const float2* __restrict__ Om, const float2* __restrict__ ampa,
                                                    float2* __restrict__ G, int64_t ldg, int LN, int l0, int n_amp,
                                                    int nrhs)
{
    extern __shared__ __align__(16) unsigned char st_smem[];
    const int n0 = 1 << l0;
    const int64_t N = int64_t(1) << LN;
    const int nv = nrhs * n_amp;
    float* Ls = reinterpret_cast<float*>(st_smem);   // [R][n0]
    for (int i = threadIdx.x; i < R * n0; i += blockDim.x) Ls[i] = Lsl[i];
    __syncthreads();
    const int64_t a = blockIdx.x;
    const int c0 = blockIdx.y * SL_CC, cc = min(SL_CC, nrhs - c0);
    for (int i = threadIdx.x; i < n0 * cc; i += blockDim.x) {
        const int j = i % n0, c = c0 + i / n0;
        const int64_t x = a * n0 + j;
        float2 g = make_float2(0.f, 0.f);
        for (int k = 0; k < n_amp; k++) {
            const int v = c * n_amp + k;
            float2 u = make_float2(0.f, 0.f);
            for (int b = 0; b < n0; b++) {
                const int64_t p = a * n0 + b;
                const float2* z = in + p * R * nv + v;
                float2 s = make_float2(0.f, 0.f);
#pragma unroll
                for (int t = 0; t < R; t++) {
                    const float2 y = __ldg(z + int64_t(t) * nv);
                    const float w = Ls[t * n0 + j];
                    s.x = fmaf(w, y.x, s.x);
                    s.y = fmaf(w, y.y, s.y);
                }
                const float2 f = __ldg(Om + p * n0 + j);
                u.x = fmaf(f.x, s.x, u.x);
                u.x = fmaf(-f.y, s.y, u.x);
                u.y = fmaf(f.x, s.y, u.y);
                u.y = fmaf(f.y, s.x, u.y);
            }
            const float2 am = __ldg(ampa + int64_t(k) * N + x);
            g.x = fmaf(am.x, u.x, g.x);
            g.x = fmaf(-am.y, u.y, g.x);
            g.y = fmaf(am.x, u.y, g.y);
            g.y = fmaf(am.y, u.x, g.y);
        }
        G[x + int64_t(c) * ldg] = g;
    }
}

// ---- dense expansion (plan finalization, for the kernels that take dense blocks: the tensor-core path) ----
// kind 0 (S0):     V[p](t, j)      = L0(t, j) omega[p][j]                 (r x n0 column-major)
// kind 1 (first):  W[p](t, k)      = L1(t, k) psi[p][k]                   (r x 2r)
// kind 2 (second): W[p](t, c r+s)  = chi[p][c r + t] L2_{a&1}(t, s)       (r x 2r)
// kind 3 (SL):     U[p](j, t)      = Omega[p][j] Lsl(j, t)                (n0 x r column-major)
__global__ void expand_st_kernel(const float* __restrict__ L, const float2* __restrict__ ph, float2* __restrict__ out,
                                 int kind, int R, int n0, int sh, int64_t total)
{
    for (int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < total; g += int64_t(gridDim.x) * blockDim.x) {
        const int per = (kind == 1 || kind == 2) ? 2 * R * R : R * n0;
        const int64_t p = g / per;
        const int e = int(g % per);
        float w;
        float2 f;
        if (kind == 0) {
            const int j = e / R;
            w = L[e];
            f = ph[p * n0 + j];
        } else if (kind == 1) {
            w = L[e];
            f = ph[p * 2 * R + e / R];
        } else if (kind == 2) {
            const int t = e % R, col = e / R, c = col / R, s = col % R;
            w = L[int((p >> sh) & 1) * R * R + s * R + t];
            f = ph[p * 2 * R + c * R + t];
        } else {
            const int j = e % n0;
            w = L[e];
            f = ph[p * n0 + j];
        }
        out[g] = make_float2(w * f.x, w * f.y);
    }
}

}  // namespace

#define ST_R(R_, CALL)            \
    switch (R_) {                 \
    case 6: CALL(6); break;       \
    case 8: CALL(8); break;       \
    case 10: CALL(10); break;     \
    case 12: CALL(12); break;     \
    case 14: CALL(14); break;     \
    case 16: CALL(16); break;     \
    default: return cudaErrorInvalidValue; \
    }

cudaError_t launch_s0_st(const Dims& d, const float2* F, int64_t ldf, const float2* ampb, const float* L0,
                         const float2* om, float2* out, int nv, cudaStream_t s)
{
    const int n0 = 1 << d.l0;
    const size_t shm = size_t((d.R * n0 * 4 + 15) / 16) * 16 + size_t(n0) * S0_VC * 8;
    const dim3 grid(unsigned(d.N >> d.l0), unsigned((nv + S0_VC - 1) / S0_VC));
#define S0_CALL(R)                                                                                        \
    {                                                                                                     \
        cudaFuncSetAttribute(s0_st_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm));     \
        s0_st_kernel<R><<<grid, 256, shm, s>>>(F, ldf, ampb, L0, om, out, d.LN, d.l0, d.n_amp, nv);        \
    }
    ST_R(d.R, S0_CALL)
#undef S0_CALL
    return cudaGetLastError();
}

cudaError_t launch_xfer_st(const Dims& d, int l, int kind, const float* L, const float2* ph, const float2* in,
                           float2* out, int nv, cudaStream_t s)
{
    const int64_t total = d.N * nv;
    if (kind != 1 && kind != 2) return cudaErrorInvalidValue;
#define X_CALL(R)                                                                                                 \
    {                                                                                                             \
        if (kind == 1) xfer_st_kernel<R, 1><<<grid_of(total, 256), 256, 0, s>>>(L, ph, in, out, d.LN, l, nv, total); \
        else xfer_st_kernel<R, 2><<<grid_of(total, 256), 256, 0, s>>>(L, ph, in, out, d.LN, l, nv, total);          \
    }
    ST_R(d.R, X_CALL)
#undef X_CALL
    return cudaGetLastError();
}

cudaError_t launch_sl_st(const Dims& d, const float2* in, const float* Lsl, const float2* Om, const float2* ampa,
                         float2* G, int64_t ldg, int nv, cudaStream_t s)
{
    const int n0 = 1 << d.l0, nrhs = nv / d.n_amp;
    const size_t shm = size_t(d.R) * n0 * 4;
    const dim3 grid(unsigned(d.N >> d.l0), unsigned((nrhs + SL_CC - 1) / SL_CC));
    const int threads = std::min(256, ((n0 * std::min(SL_CC, nrhs) + 31) / 32) * 32);
#define SL_CALL(R) \
    sl_st_kernel<R><<<grid, threads, shm, s>>>(in, Lsl, Om, ampa, G, ldg, d.LN, d.l0, d.n_amp, nrhs);
    ST_R(d.R, SL_CALL)
#undef SL_CALL
    return cudaGetLastError();
}

cudaError_t launch_expand_st(const Dims& d, int kind, int l, const float* L, const float2* ph, float2* out,
                             cudaStream_t s)
{
    const int n0 = 1 << d.l0;
    const int64_t per = (kind == 1 || kind == 2) ? 2 * int64_t(d.R) * d.R : int64_t(d.R) * n0;
    const int64_t total = d.N * per;
    const unsigned grid = unsigned(std::min<int64_t>((total + 255) / 256, int64_t(148) * 32));
    expand_st_kernel<<<grid, 256, 0, s>>>(L, ph, out, kind, d.R, n0, d.LN - l, total);
    return cudaGetLastError();
}

#undef ST_R

}  // namespace bfk
