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
// This file holds the kernels for any vector batch (one level per launch; a thread owns one (pair, vector) and
// all r outputs, or one output row of SL) and the expansion of structured factors into dense blocks for the
// tensor-core path (plan finalization).
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

// The Lagrange matrix of a stage travels BY VALUE in the kernel parameters (constant bank 0): with the loops over
// its rows and columns fully unrolled every weight is a compile-time constant-bank operand of its FFMA -- no load
// instruction at all (a shared-memory copy cost one LDS per two FMAs and made the first version LDS-bound).

__device__ __forceinline__ void rmac(float2& acc, const float w, const float2 x)
{
    acc.x = fmaf(w, x.x, acc.x);
    acc.y = fmaf(w, x.y, acc.y);
}

__device__ __forceinline__ void cmac(float2& acc, const float2 f, const float2 x)
{
    acc.x = fmaf(f.x, x.x, acc.x);
    acc.x = fmaf(-f.y, x.y, acc.x);
    acc.y = fmaf(f.x, x.y, acc.y);
    acc.y = fmaf(f.y, x.x, acc.y);
}

// ---- S0: CTA = (leaf b, chunk of VC vectors); y_b staged in shared memory; thread = (a, vector) ----
constexpr int S0_VC = 32;

template <int R, int N0>
__global__ void __launch_bounds__(256) s0_st_kernel(const float2* __restrict__ F, int64_t ldf,
                                                    const float2* __restrict__ ampb, const __grid_constant__ LagP L0,
                                                    const float2* __restrict__ om, float2* __restrict__ out, int LN,
                                                    int n_amp, int nv)
{
    __shared__ float2 Y[N0 * S0_VC];   // [j][vl]
    const int64_t N = int64_t(1) << LN, nleaf = N / N0;
    const int64_t b = blockIdx.x;
    const int v0 = blockIdx.y * S0_VC, vc = min(S0_VC, nv - v0);
    for (int i = threadIdx.x; i < N0 * vc; i += blockDim.x) {
        const int j = i % N0, vl = i / N0, v = v0 + vl;
        const int64_t x = b * N0 + j;
        Y[j * S0_VC + vl] = cmul(__ldg(ampb + int64_t(v % n_amp) * N + x), __ldg(F + x + int64_t(v / n_amp) * ldf));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < N0 * vc; i += blockDim.x) {
        const int vl = i % vc, a = i / vc;
        const int64_t p = int64_t(a) * nleaf + b;
        const float2* o = om + p * N0;
        float2 acc[R];
#pragma unroll
        for (int t = 0; t < R; t++) acc[t] = make_float2(0.f, 0.f);
#pragma unroll
        for (int j = 0; j < N0; j++) {
            const float2 z = cmul(__ldg(o + j), Y[j * S0_VC + vl]);
#pragma unroll
            for (int t = 0; t < R; t++) rmac(acc[t], L0.v[j * R + t], z);
        }
        float2* dst = out + p * R * nv + v0 + vl;
#pragma unroll
        for (int t = 0; t < R; t++) dst[int64_t(t) * nv] = acc[t];
    }
}

// ---- one transfer level: thread = (output pair p, vector v) ----
template <int R, int E>
__device__ __forceinline__ void second_half(const LagP& L, const float2* __restrict__ php, const float2* __restrict__ x0,
                                            const float2* __restrict__ x1, int nv, float2 (&acc)[R])
{
#pragma unroll
    for (int c = 0; c < 2; c++) {
        const float2* x = c ? x1 : x0;
        float2 xs[R], z[R];
#pragma unroll
        for (int s = 0; s < R; s++) xs[s] = __ldg(x + int64_t(s) * nv);
#pragma unroll
        for (int t = 0; t < R; t++) z[t] = make_float2(0.f, 0.f);
#pragma unroll
        for (int s = 0; s < R; s++)
#pragma unroll
            for (int t = 0; t < R; t++) rmac(z[t], L.v[E * R * R + s * R + t], xs[s]);
#pragma unroll
        for (int t = 0; t < R; t++) cmac(acc[t], __ldg(php + c * R + t), z[t]);
    }
}

template <int R, int KIND>
__global__ void __launch_bounds__(256) xfer_st_kernel(const __grid_constant__ LagP L, const float2* __restrict__ ph,
                                                      const float2* __restrict__ in, float2* __restrict__ out, int LN,
                                                      int l, int nv, int64_t total)
{
    const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g >= total) return;
    const int64_t p = g / nv;
    const int v = int(g % nv);
    const int sh = LN - l;
    const int64_t a = p >> sh, b = p & ((int64_t(1) << sh) - 1);
    const int64_t q0 = ((a >> 1) << (sh + 1)) + 2 * b;   // input pairs q0, q0 + 1 at level l - 1
    const float2* php = ph + p * 2 * R;
    const float2* x0 = in + q0 * R * nv + v;
    const float2* x1 = x0 + int64_t(R) * nv;
    float2 acc[R];
#pragma unroll
    for (int t = 0; t < R; t++) acc[t] = make_float2(0.f, 0.f);
    if (KIND == 1 || KIND == 3) {   // first half: phases on the inputs, then L1 (then the switch: KIND 3)
        const float2* pc = ph + p * (KIND == 3 ? 2 * R + R * R : 2 * R);
#pragma unroll
        for (int c = 0; c < 2; c++) {
            const float2* x = c ? x1 : x0;
            float2 y[R];
#pragma unroll
            for (int s = 0; s < R; s++) y[s] = cmul(__ldg(pc + c * R + s), __ldg(x + int64_t(s) * nv));
#pragma unroll
            for (int s = 0; s < R; s++)
#pragma unroll
                for (int t = 0; t < R; t++) rmac(acc[t], L.v[(c * R + s) * R + t], y[s]);
        }
        if (KIND == 3) {
            float2 y[R];
#pragma unroll
            for (int t = 0; t < R; t++) {
                y[t] = acc[t];
                acc[t] = make_float2(0.f, 0.f);
            }
#pragma unroll
            for (int s = 0; s < R; s++)
#pragma unroll
                for (int t = 0; t < R; t++) cmac(acc[t], __ldg(pc + 2 * R + s * R + t), y[s]);
        }
    } else {           // second half: L2_e on each input, phases on the outputs (e uniform over a warp's pairs
                       // whenever 2^(LN-l) >= 32 / nv)
        if (a & 1) second_half<R, 1>(L, php, x0, x1, nv, acc);
        else second_half<R, 0>(L, php, x0, x1, nv, acc);
    }
    float2* dst = out + p * R * nv + v;
#pragma unroll
    for (int t = 0; t < R; t++) dst[int64_t(t) * nv] = acc[t];
}

// ---- two transfer levels per launch (l, l+1): a JOB is 4 consecutive input pairs 4j .. 4j+3 of level l-1,
// closed under the two levels (SURVEY 8(a) fusion geometry; the slot algebra of band_sv_kernel in bf_small.cu):
// level-l output (u, e) is pair ((2 a0 + e) << (LN - l)) + 2 bq + u, reading input slots 2u + c; level-(l+1)
// output (u, e) is pair ((4 a0 + 2u + e) << shg) + bq, reading level-l slots 2c + u.  Thread = (job, output slot,
// vector); level l reads its inputs from global memory (each input feeds two threads' pairs: the second read
// hits L1), keeps its outputs in shared memory, level l+1 writes HBM.  Per level: kind 1 first half, 2 second
// half, 0 dense block (the level carrying the switch).  L of level l at L.v[0], of level l+1 at L.v[512].
template <int R, int KIND>
__device__ __forceinline__ void level_out(const float* __restrict__ Lv, const float2* __restrict__ wp, int e,
                                          const float2* __restrict__ x0, const float2* __restrict__ x1, int64_t sx,
                                          float2 (&acc)[R])
{
#pragma unroll
    for (int t = 0; t < R; t++) acc[t] = make_float2(0.f, 0.f);
#pragma unroll
    for (int c = 0; c < 2; c++) {
        const float2* x = c ? x1 : x0;
        float2 xs[R];
#pragma unroll
        for (int s = 0; s < R; s++) xs[s] = x[s * sx];
        if (KIND == 1 || KIND == 3) {
#pragma unroll
            for (int s = 0; s < R; s++) {
                const float2 y = cmul(wp[c * R + s], xs[s]);
#pragma unroll
                for (int t = 0; t < R; t++) rmac(acc[t], Lv[(c * R + s) * R + t], y);
            }
        } else if (KIND == 2) {
            float2 z[R];
#pragma unroll
            for (int t = 0; t < R; t++) z[t] = make_float2(0.f, 0.f);
            if (e) {
#pragma unroll
                for (int s = 0; s < R; s++)
#pragma unroll
                    for (int t = 0; t < R; t++) rmac(z[t], Lv[R * R + s * R + t], xs[s]);
            } else {
#pragma unroll
                for (int s = 0; s < R; s++)
#pragma unroll
                    for (int t = 0; t < R; t++) rmac(z[t], Lv[s * R + t], xs[s]);
            }
#pragma unroll
            for (int t = 0; t < R; t++) cmac(acc[t], wp[c * R + t], z[t]);
        } else {   // dense r x 2r block, column-major
#pragma unroll
            for (int s = 0; s < R; s++)
#pragma unroll
                for (int t = 0; t < R; t++) cmac(acc[t], wp[(c * R + s) * R + t], xs[s]);
        }
    }
    if (KIND == 3) {   // the switch with its phases: acc <- Sw' acc (Sw' column-major after the 2r phases)
        float2 y[R];
#pragma unroll
        for (int t = 0; t < R; t++) {
            y[t] = acc[t];
            acc[t] = make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int s = 0; s < R; s++)
#pragma unroll
            for (int t = 0; t < R; t++) cmac(acc[t], wp[2 * R + s * R + t], y[s]);
    }
}

// The CTA takes jobs_cta consecutive jobs per iteration; their inputs (contiguous), the per-pair data of both
// levels and (next iteration) are staged with cp.async into a 2-deep ring while the current iteration computes,
// so every thread has a whole iteration of copies in flight (the unpipelined version, which loaded its inputs
// from global memory inside the level-l loop, ran at 0.27 of HBM).
__device__ __forceinline__ void cp_async16_g(void* smem, const void* gmem)
{
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}

template <int R, int K1, int K2>
__global__ void __launch_bounds__(256) band_st_kernel(const __grid_constant__ LagP L, const float2* __restrict__ w1,
                                                      const float2* __restrict__ w2, const float2* __restrict__ in,
                                                      float2* __restrict__ out, int LN, int l, int nv, int64_t njobs,
                                                      int jobs_cta)
{
    extern __shared__ __align__(16) unsigned char st_smem[];
    constexpr int WS1 = K1 == 0 ? 2 * R * R : (K1 == 3 ? 2 * R + R * R : 2 * R);
    constexpr int WS2 = K2 == 0 ? 2 * R * R : (K2 == 3 ? 2 * R + R * R : 2 * R);
    const int per_job = 4 * nv;
    // thread = (job, e, u, vector): with nv >= 16 a warp's threads share e (the second-half Lagrange matrix)
    const int jl = threadIdx.x / per_job, v = threadIdx.x % nv;
    const int u = (threadIdx.x / nv) & 1, e = (threadIdx.x / (2 * nv)) & 1, os = 2 * u + e;
    const int shg = LN - l - 1;
    const int xin = jobs_cta * 4 * R * nv;   // complex per input buffer
    float2* X0 = reinterpret_cast<float2*>(st_smem);          // [2][jobs][4 slots][R][nv]
    float2* X1 = X0 + 2 * xin;                                 // [jobs][4][R][nv]
    float2* P1 = X1 + xin;                                     // [2][jobs][4][WS1]
    float2* P2 = P1 + 2 * jobs_cta * 4 * WS1;                  // [2][jobs][4][WS2]
    const int64_t stride = int64_t(gridDim.x) * jobs_cta;
    auto pair1 = [&](int64_t j, int uu, int ee) {
        const int64_t a0 = j >> shg, bq = j & ((int64_t(1) << shg) - 1);
        return (((a0 << 1) + ee) << (LN - l)) + (bq << 1) + uu;
    };
    auto pair2 = [&](int64_t j, int uu, int ee) {
        const int64_t a0 = j >> shg, bq = j & ((int64_t(1) << shg) - 1);
        return (((a0 << 2) + 2 * uu + ee) << shg) + bq;
    };
    auto issue = [&](int64_t j0, int buf) {
        const int64_t nj = njobs - j0 < jobs_cta ? njobs - j0 : jobs_cta;
        const int pieces = int(nj) * 4 * R * nv / 2;   // 16-byte pieces of the inputs (nv even)
        const float2* src = in + 4 * j0 * R * int64_t(nv);
        float2* dst = X0 + buf * xin;
        for (int i = threadIdx.x; i < pieces; i += blockDim.x) cp_async16_g(dst + 2 * i, src + 2 * i);
        const int p1n = int(nj) * 4 * (WS1 / 2), p2n = int(nj) * 4 * (WS2 / 2);
        for (int i = threadIdx.x; i < p1n; i += blockDim.x) {
            const int q = i / (WS1 / 2), k = i % (WS1 / 2), jj = q / 4, o = q % 4;
            cp_async16_g(P1 + ((buf * jobs_cta + jj) * 4 + o) * WS1 + 2 * k, w1 + pair1(j0 + jj, o >> 1, o & 1) * WS1 + 2 * k);
        }
        for (int i = threadIdx.x; i < p2n; i += blockDim.x) {
            const int q = i / (WS2 / 2), k = i % (WS2 / 2), jj = q / 4, o = q % 4;
            cp_async16_g(P2 + ((buf * jobs_cta + jj) * 4 + o) * WS2 + 2 * k, w2 + pair2(j0 + jj, o >> 1, o & 1) * WS2 + 2 * k);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    int64_t j0 = int64_t(blockIdx.x) * jobs_cta;
    if (j0 < njobs) issue(j0, 0);
    for (int it = 0; j0 < njobs; it++, j0 += stride) {
        const int buf = it & 1;
        if (j0 + stride < njobs) {
            issue(j0 + stride, buf ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const int64_t j = j0 + jl;
        const bool live = jl < jobs_cta && j < njobs;
        float2 acc[R];
        if (live) {   // level l: output (u, e) from input slots 2u, 2u + 1
            const float2* x0 = X0 + buf * xin + ((jl * 4) + 2 * u) * R * nv + v;
            level_out<R, K1>(L.v, P1 + ((buf * jobs_cta + jl) * 4 + os) * WS1, e, x0, x0 + R * nv, nv, acc);
            float2* d = X1 + (jl * 4 + os) * R * nv + v;
#pragma unroll
            for (int t = 0; t < R; t++) d[t * nv] = acc[t];
        }
        __syncthreads();
        if (live) {   // level l + 1: output (u, e) from level-l slots u (c = 0) and u + 2 (c = 1)
            const float2* x0 = X1 + (jl * 4 + u) * R * nv + v;
            level_out<R, K2>(L.v + 512, P2 + ((buf * jobs_cta + jl) * 4 + os) * WS2, e, x0, x0 + 2 * R * nv, nv, acc);
            float2* d = out + pair2(j, u, e) * R * int64_t(nv) + v;
#pragma unroll
            for (int t = 0; t < R; t++) d[int64_t(t) * nv] = acc[t];
        }
        __syncthreads();   // buffer `buf` and X1 are free for the copies issued next iteration
    }
}

// ---- SL: CTA = (T_X leaf a, chunk of VC = VG VPT vectors).  The leaf's coefficients zeta[a n0 + b](t)[chunk]
// (n0 r VC complex) and phases Omega[a n0 + b][j] (n0^2 complex) are staged in shared memory with cp.async by
// every thread (high memory-level parallelism: the first version streamed them per warp from L2 and was latency-
// bound); thread = (row j, vector group) holds its r weights Lsl(j, .) in registers and VPT accumulators; the
// coefficient loads are broadcasts (all rows of a warp read the same address) ----
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem)
{
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}

// The leaf is streamed in chunks of BC b's through two shared-memory stages (cp.async, double-buffered): the copies of
// chunk c + 1 overlap the MACs of chunk c, and the smaller footprint lets more CTAs share an SM (the whole-leaf version
// waited for all its copies before the first MAC: 0.37 of the FP32 peak at cfg5).
template <int R, int VPT>
__global__ void __launch_bounds__(256) sl_st_kernel(const float2* __restrict__ in, const float* __restrict__ Lsl,
                                                    const float2* __restrict__ Om, const float2* __restrict__ ampa,
                                                    float2* __restrict__ G, int64_t ldg, int LN, int l0, int n_amp,
                                                    int nv, int VG, int BC)
{
    extern __shared__ __align__(16) unsigned char st_smem[];
    const int64_t N = int64_t(1) << LN;
    const int n0 = 1 << l0, VC = VG * VPT;
    const int zst = BC * R * VC, ost = BC * n0;               // complex per stage
    float2* Zs = reinterpret_cast<float2*>(st_smem);          // [2][BC][t][VC]
    float2* Oss = Zs + 2 * zst;                               // [2][BC][j]
    const int64_t a = blockIdx.x;
    const int v0 = blockIdx.y * VC;
    const float2* zsrc = in + a * n0 * R * int64_t(nv) + v0;
    const float2* osrc = Om + a * n0 * int64_t(n0);
    const int nch = n0 / BC;
    auto stage = [&](int c) {   // chunk c -> stage c & 1
        float2* Z = Zs + (c & 1) * zst;
        float2* O = Oss + (c & 1) * ost;
        const float2* zc = zsrc + int64_t(c) * BC * R * nv;
        if (VPT >= 2) {   // 16-byte pieces: nv and v0 even
            const int pr = VC / 2;
            for (int i = threadIdx.x; i < BC * R * pr; i += blockDim.x) {
                const int row = i / pr, q = i % pr;
                cp_async16(Z + row * VC + 2 * q, zc + int64_t(row) * nv + 2 * q);
            }
        } else {
            for (int i = threadIdx.x; i < BC * R * VC; i += blockDim.x) Z[i] = __ldg(zc + int64_t(i / VC) * nv + i % VC);
        }
        const float2* oc = osrc + int64_t(c) * BC * n0;
        for (int i = threadIdx.x; i < BC * n0 / 2; i += blockDim.x) cp_async16(O + 2 * i, oc + 2 * i);
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    const int j = threadIdx.x % n0, vg = threadIdx.x / n0;
    const bool active = vg < VG;
    const int64_t x = a * n0 + j;
    float Lr[R];
#pragma unroll
    for (int t = 0; t < R; t++) Lr[t] = active ? __ldg(Lsl + t * n0 + j) : 0.f;
    float2 acc[VPT];
#pragma unroll
    for (int q = 0; q < VPT; q++) acc[q] = make_float2(0.f, 0.f);
    stage(0);
    for (int c = 0; c < nch; c++) {
        if (c + 1 < nch) {
            stage(c + 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        if (active) {
            const float2* Zc = Zs + (c & 1) * zst;
            const float2* Oc = Oss + (c & 1) * ost;
            for (int bb = 0; bb < BC; bb++) {
                const float2* z = Zc + (bb * R) * VC + vg * VPT;
                float2 sacc[VPT];
#pragma unroll
                for (int q = 0; q < VPT; q++) sacc[q] = make_float2(0.f, 0.f);
#pragma unroll
                for (int t = 0; t < R; t++) {
                    float2 zt[VPT];
                    if constexpr (VPT == 1) {
                        zt[0] = z[t * VC];
                    } else {
#pragma unroll
                        for (int q = 0; q < VPT / 2; q++) {
                            const float4 f = reinterpret_cast<const float4*>(z + t * VC)[q];
                            zt[2 * q] = make_float2(f.x, f.y);
                            zt[2 * q + 1] = make_float2(f.z, f.w);
                        }
                    }
#pragma unroll
                    for (int q = 0; q < VPT; q++) rmac(sacc[q], Lr[t], zt[q]);
                }
                const float2 f = Oc[bb * n0 + j];
#pragma unroll
                for (int q = 0; q < VPT; q++) cmac(acc[q], f, sacc[q]);
            }
        }
        __syncthreads();   // stage c & 1 is refilled by the copies of chunk c + 2, issued next iteration
    }
    if (!active) return;
    // a_k(x) and the sum over the n_amp vectors of each column (consecutive within the thread)
    const int vb = v0 + vg * VPT;
    float2 g = make_float2(0.f, 0.f);
#pragma unroll
    for (int q = 0; q < VPT; q++) {
        const int k = q % n_amp;
        cmac(g, __ldg(ampa + int64_t(k) * N + x), acc[q]);
        if (k == n_amp - 1) {
            G[x + int64_t((vb + q) / n_amp) * ldg] = g;
            g = make_float2(0.f, 0.f);
        }
    }
}

// ---- dense expansion (plan finalization, for the kernels that take dense blocks: the tensor-core path) ----
// kind 0 (S0):     V[p](t, j)      = L0(t, j) omega[p][j]                 (r x n0 column-major)
// kind 1 (first):  W[p](t, k)      = L1(t, k) psi[p][k]                   (r x 2r)
// kind 2 (second): W[p](t, c r+s)  = chi[p][c r + t] L2_{a&1}(t, s)       (r x 2r)
// kind 3 (switch): W[p](t, k)      = sum_s Sw'[p](t, s) L1(s, k) psi[p][k] (r x 2r)
// kind 4 (SL):     U[p](j, t)      = Omega[p][j] Lsl(j, t)                (n0 x r column-major)
__global__ void expand_st_kernel(const float* __restrict__ L, const float2* __restrict__ ph, float2* __restrict__ out,
                                 int kind, int R, int n0, int sh, int64_t total)
{
    for (int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < total; g += int64_t(gridDim.x) * blockDim.x) {
        const int per = (kind == 1 || kind == 2 || kind == 3) ? 2 * R * R : R * n0;
        const int64_t p = g / per;
        const int e = int(g % per);
        float w;
        float2 f;
        if (kind == 0) {
            w = L[e];
            f = ph[p * n0 + e / R];
        } else if (kind == 1) {
            w = L[e];
            f = ph[p * 2 * R + e / R];
        } else if (kind == 2) {
            const int t = e % R, col = e / R, c = col / R, s = col % R;
            w = L[int((p >> sh) & 1) * R * R + s * R + t];
            f = ph[p * 2 * R + c * R + t];
        } else if (kind == 3) {
            const int t = e % R, k = e / R;
            const float2* pp = ph + p * (2 * R + R * R);
            float2 acc = make_float2(0.f, 0.f);
            for (int s = 0; s < R; s++) {
                const float2 sw = pp[2 * R + s * R + t];
                const float lw = L[k * R + s];
                acc.x = fmaf(sw.x, lw, acc.x);
                acc.y = fmaf(sw.y, lw, acc.y);
            }
            out[g] = cmul(acc, pp[k]);
            continue;
        } else {
            w = L[e];
            f = ph[p * n0 + e % n0];
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
#define ST_N0(N0_, R, CALL)       \
    switch (N0_) {                \
    case 8: CALL(R, 8); break;    \
    case 16: CALL(R, 16); break;  \
    case 32: CALL(R, 32); break;  \
    case 64: CALL(R, 64); break;  \
    default: return cudaErrorInvalidValue; \
    }

cudaError_t launch_s0_st(const Dims& d, const float2* F, int64_t ldf, const float2* ampb, const LagP& L0,
                         const float2* om, float2* out, int nv, cudaStream_t s)
{
    const int n0 = 1 << d.l0;
    const dim3 grid(unsigned(d.N >> d.l0), unsigned((nv + S0_VC - 1) / S0_VC));
    const int threads = std::min(256, ((n0 * std::min(nv, S0_VC) + 31) / 32) * 32);
#define S0_CALL(R, N0) s0_st_kernel<R, N0><<<grid, threads, 0, s>>>(F, ldf, ampb, L0, om, out, d.LN, d.n_amp, nv)
#define S0_N(R) ST_N0(n0, R, S0_CALL)
    ST_R(d.R, S0_N)
#undef S0_N
#undef S0_CALL
    return cudaGetLastError();
}

cudaError_t launch_xfer_st(const Dims& d, int l, int kind, const LagP& L, const float2* ph, const float2* in,
                           float2* out, int nv, cudaStream_t s)
{
    const int64_t total = d.N * nv;
    if (kind != 1 && kind != 2 && kind != 3) return cudaErrorInvalidValue;
#define X_CALL(R)                                                                                                 \
    {                                                                                                             \
        if (kind == 1) xfer_st_kernel<R, 1><<<grid_of(total, 256), 256, 0, s>>>(L, ph, in, out, d.LN, l, nv, total); \
        else if (kind == 3)                                                                                       \
            xfer_st_kernel<R, 3><<<grid_of(total, 256), 256, 0, s>>>(L, ph, in, out, d.LN, l, nv, total);          \
        else xfer_st_kernel<R, 2><<<grid_of(total, 256), 256, 0, s>>>(L, ph, in, out, d.LN, l, nv, total);          \
    }
    ST_R(d.R, X_CALL)
#undef X_CALL
    return cudaGetLastError();
}

cudaError_t launch_sl_st(const Dims& d, const float2* in, const float* Lsl, const float2* Om, const float2* ampa,
                         float2* G, int64_t ldg, int nv, cudaStream_t s)
{
    const int n0 = 1 << d.l0;
    int vpt = 8;   // vectors per thread: a power of two dividing nv and a multiple of n_amp
    while (vpt > 1 && (nv % vpt || vpt % d.n_amp)) vpt >>= 1;
    if (vpt % d.n_amp) return cudaErrorInvalidValue;
    int vg = 1;    // vector groups per CTA: up to 256 threads, at most ~100 KB of staged coefficients
    while (vg < 4 && nv % (2 * vg * vpt) == 0 && n0 * 2 * vg <= 256 &&
           size_t(n0) * d.R * 2 * vg * vpt * 8 <= 96 * 1024)
        vg *= 2;
    const int vc = vg * vpt;
    const int bc = n0 >= 8 ? 8 : n0;     // b's per pipeline chunk (8 / 16 / 32 measured: cfg5 5.96 / 5.95 / 6.44 ms, cfg2 0.112 / 0.132 / 0.189 ms)
    const size_t shm = 2 * (size_t(bc) * d.R * vc + size_t(bc) * n0) * 8;
    const dim3 grid(unsigned(d.N >> d.l0), unsigned(nv / vc));
    const int threads = n0 * vg < 32 ? 32 : n0 * vg;
#define SL_GO(R, V)                                                                                                \
    {                                                                                                              \
        cudaFuncSetAttribute(sl_st_kernel<R, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm));          \
        sl_st_kernel<R, V><<<grid, threads, shm, s>>>(in, Lsl, Om, ampa, G, ldg, d.LN, d.l0, d.n_amp, nv, vg, bc); \
    }
#define SL_CALL(R)                      \
    switch (vpt) {                      \
    case 8: SL_GO(R, 8) break;          \
    case 4: SL_GO(R, 4) break;          \
    case 2: SL_GO(R, 2) break;          \
    default: SL_GO(R, 1) break;         \
    }
    ST_R(d.R, SL_CALL)
#undef SL_CALL
#undef SL_GO
    return cudaGetLastError();
}

bool band_st_supported(const Dims& d, int nv) { return nv >= 2 && nv % 2 == 0 && 4 * nv <= 256 && d.R <= 16; }

bool band_st_kinds(int k1, int k2)
{
    const int kk = k1 * 4 + k2;
    return kk == 1 * 4 + 1 || kk == 2 * 4 + 2 || kk == 1 * 4 + 3 || kk == 3 * 4 + 2 || kk == 1 * 4 + 0 ||
           kk == 0 * 4 + 2 || kk == 0 * 4 + 0;
}

cudaError_t launch_band_st(const Dims& d, int l, int k1, int k2, const LagP& L, const float2* w1, const float2* w2,
                           const float2* in, float2* out, int nv, cudaStream_t s)
{
    if (!band_st_supported(d, nv)) return cudaErrorInvalidValue;
    auto ws = [&](int k) { return k == 0 ? 2 * d.R * d.R : (k == 3 ? 2 * d.R + d.R * d.R : 2 * d.R); };
    const int ws1 = ws(k1), ws2 = ws(k2);
    const size_t per_job = size_t(4) * (3 * size_t(d.R) * nv + 2 * ws1 + 2 * ws2) * 8;
    // up to 256 threads, and at most ~100 KB of shared memory (two CTAs per SM)
    const int jobs_cta = int(std::max<size_t>(1, std::min<size_t>(256 / (4 * nv), (100 << 10) / per_job)));
    const int threads = jobs_cta * 4 * nv;
    const size_t shm = size_t(jobs_cta) * per_job;
    const int64_t njobs = d.N / 4;
    const int kk = k1 * 4 + k2;
    // persistent grid = the CTAs that are resident at once (occupancy), not a fixed 4 per SM: a CTA that does not fit
    // would start after a resident one finishes and, with an equal share of the jobs, double the kernel's time
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
#define B_GO(R, A, B)                                                                                              \
    {                                                                                                              \
        cudaFuncSetAttribute(band_st_kernel<R, A, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm));     \
        int occ = 1;                                                                                               \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, band_st_kernel<R, A, B>, threads, shm);                \
        const unsigned grid = unsigned(std::min<int64_t>((njobs + jobs_cta - 1) / jobs_cta,                        \
                                                         int64_t(nsm) * std::max(1, occ)));                        \
        band_st_kernel<R, A, B><<<grid, threads, shm, s>>>(L, w1, w2, in, out, d.LN, l, nv, njobs, jobs_cta);      \
    }
#define B_CALL(R)                                      \
    switch (kk) {                                      \
    case 1 * 4 + 1: B_GO(R, 1, 1); break;              \
    case 2 * 4 + 2: B_GO(R, 2, 2); break;              \
    case 1 * 4 + 3: B_GO(R, 1, 3); break;              \
    case 3 * 4 + 2: B_GO(R, 3, 2); break;              \
    case 1 * 4 + 0: B_GO(R, 1, 0); break;              \
    case 0 * 4 + 2: B_GO(R, 0, 2); break;              \
    case 0 * 4 + 0: B_GO(R, 0, 0); break;              \
    default: return cudaErrorInvalidValue;             \
    }
    ST_R(d.R, B_CALL)
#undef B_CALL
#undef B_GO
    return cudaGetLastError();
}

cudaError_t launch_expand_st(const Dims& d, int kind, int l, const float* L, const float2* ph, float2* out,
                             cudaStream_t s)
{
    const int n0 = 1 << d.l0;
    const int64_t per = (kind == 1 || kind == 2 || kind == 3) ? 2 * int64_t(d.R) * d.R : int64_t(d.R) * n0;
    const int64_t total = d.N * per;
    const unsigned grid = unsigned(std::min<int64_t>((total + 255) / 256, int64_t(148) * 32));
    expand_st_kernel<<<grid, 256, 0, s>>>(L, ph, out, kind, d.R, n0, d.LN - l, total);
    return cudaGetLastError();
}

#undef ST_R
#undef ST_N0

}  // namespace bfk
