// bf_nufft.cu -- the NUFFT path of the unified framework (include/bf_nufft.h, eqn:tg3):
// per frequency submatrix s a one-dimensional type-2 NUFFT (uniform frequencies, non-uniform targets t_s(x_i)),
// for every amplitude term k and RHS column c, summed into G.  Three launches per chunk:
//   place_kernel       h[s][v][kappa mod n_f] = b_k(xi) F[xi, c] / phi^(kappa), the zeros elsewhere written once at
//                      plan creation                                                          (v = c n_amp + k)
//   cuFFT              one batched inverse C2C FFT of size n_f over the n_sub n_amp nrhs grids (out of place)
//   interp_win_kernel  G[i, c] = sum_k a_k(x_i) sum_s e^{2 pi i t_s xi_c} sum_m phi(z_m) u[s][v][(l_s + m) mod n_f]
// with the w-point ES kernel phi(z) = e^{beta (sqrt(1 - z^2) - 1)}, z_m = (l_s + m - n_f t_s) / (w / 2).
// Memory-bound at cfg4 sizes: the grids (2 n_sub n_amp nrhs N complex64) are written
// once, transformed by cuFFT, read once.
#include <cuda_runtime.h>
#include <cufft.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../include/bf.h"
#include "../../include/bf_nufft.h"
#include "bf_plan_internal.h"

struct bf_nufft_s {
    int device = 0;
    int LN = 0, n_amp = 0, n_sub = 0, w = 0;
    int64_t N = 0, M = 0, nf = 0, max_chunk = 0;
    double beta = 0;
    float2* amp_a = nullptr;   // [n_amp][N]
    float2* amp_b = nullptr;   // [n_amp][N]
    float* deconv = nullptr;   // [M] 1 / phi^(kappa), kappa = -M/2 .. M/2-1
    int* l0 = nullptr;         // [n_sub][N] first grid point of target i
    float* off = nullptr;      // [n_sub][N] n_f t - l0 (FP64 -> FP32 once), in [w/2 - 1, w/2)
    float2* ph = nullptr;      // [n_sub][N] e^{2 pi i t_s(x_i) xi_c(s)}
    float2* grid = nullptr;    // [n_sub][nv][n_f] placed coefficients of one chunk (zero outside the M frequencies)
    float2* gout = nullptr;    // [n_sub][nv][n_f] their inverse FFTs (out of place: the zeros of `grid` are written
                               // once at creation, so the placement writes only the M frequencies)
    cufftHandle fft = 0;
    bool fft_ok = false;
    int fft_batch = 0;
};

namespace {

bf_status_t nf_fail(bf_status_t s, const char* what) { return bfp_fail(s, what); }
bf_status_t nf_cuda(cudaError_t e, const char* what)
{
    char m[256];
    snprintf(m, sizeof m, "%s: %s", what, cudaGetErrorString(e));
    return bfp_fail(BF_ERR_CUDA, m);
}

struct Guard {
    int prev = -1;
    explicit Guard(int d)
    {
        cudaGetDevice(&prev);
        if (prev != d) cudaSetDevice(d);
    }
    ~Guard()
    {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// ES kernel in grid units y (|y| <= w/2)
inline double es(double y, int w, double beta)
{
    const double z = 2.0 * y / w;
    return (std::fabs(z) >= 1.0) ? 0.0 : std::exp(beta * (std::sqrt(1.0 - z * z) - 1.0));
}

// phi^(kappa) = int phi(y) cos(2 pi kappa y / n_f) dy over |y| <= w/2, Gauss-Legendre (FP64)
void deconv_factors(int w, double beta, int64_t M, int64_t nf, std::vector<float>& out)
{
    constexpr int Q = 96;
    std::vector<double> x(Q), wq(Q);
    for (int i = 0; i < Q; i++) {   // Gauss-Legendre nodes by Newton on P_Q
        double z = std::cos(M_PI * (i + 0.75) / (Q + 0.5)), pp = 0;
        for (int it = 0; it < 100; it++) {
            double p1 = 1, p2 = 0;
            for (int j = 1; j <= Q; j++) {
                const double p3 = p2;
                p2 = p1;
                p1 = ((2.0 * j - 1.0) * z * p2 - (j - 1.0) * p3) / j;
            }
            pp = Q * (z * p1 - p2) / (z * z - 1.0);
            const double dz = p1 / pp;
            z -= dz;
            if (std::fabs(dz) < 1e-16) break;
        }
        x[i] = z;
        wq[i] = 2.0 / ((1.0 - z * z) * pp * pp);
    }
    out.resize(size_t(M));
    const double h = 0.5 * w;
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < M; k++) {
        const double kap = double(k - M / 2);
        double s = 0;
        for (int i = 0; i < Q; i++) {
            const double y = h * x[i];
            s += wq[i] * es(y, w, beta) * std::cos(2.0 * M_PI * kap * y / double(nf));
        }
        out[size_t(k)] = float(1.0 / (h * s));
    }
}

// h[s][v][kappa mod n_f] for the M frequencies of (s, v) (the rest of the grid stays zero from creation): one
// thread per frequency, v = c n_amp + k.  Frequencies of submatrix s are the F rows [s M, (s+1) M); kappa =
// j - s M - M/2.
__global__ void place_kernel(const float2* __restrict__ F, int64_t ldf, const float2* __restrict__ ampb,
                             const float* __restrict__ deconv, float2* __restrict__ grid, int64_t N, int64_t M,
                             int64_t nf, int n_amp, int nv)
{
    // two consecutive frequencies per thread (16-byte loads and stores: M/2 is even, so a pair never straddles the
    // kappa = -1 / 0 wrap of the grid)
    const int64_t q = 2 * (int64_t(blockIdx.x) * blockDim.x + threadIdx.x);   // 0 .. M-2
    if (q >= M) return;
    const int v = blockIdx.y, s = blockIdx.z;
    const int c = v / n_amp, k = v - c * n_amp;
    const int64_t kap = q - M / 2;
    const int64_t j = s * M + q;   // F row
    const float4 f = *reinterpret_cast<const float4*>(F + int64_t(c) * ldf + j);
    const float4 b = __ldg(reinterpret_cast<const float4*>(ampb + int64_t(k) * N + j));
    const float2 d = __ldg(reinterpret_cast<const float2*>(deconv + q));
    const int64_t l = kap < 0 ? kap + nf : kap;
    *reinterpret_cast<float4*>(grid + (int64_t(s) * nv + v) * nf + l) =
        make_float4((b.x * f.x - b.y * f.y) * d.x, (b.x * f.y + b.y * f.x) * d.x, (b.z * f.z - b.w * f.w) * d.y,
                    (b.z * f.w + b.w * f.z) * d.y);
}

// Interpolation with the grid window of a block in shared memory: 256 consecutive targets of a submatrix touch
// the grid points [min l0, max l0 + w) -- about 1.4 x 256 + w for the configs' monotone targets -- so the block
// stages that window of each of its RW grid rows (coalesced, once) and every thread reads its w taps from shared
// memory (the direct version issued w global loads per target, row and submatrix: 0.18 of HBM).  Targets whose
// window exceeds LWMAX (non-monotone or widely spread targets) take the direct path for that block.
constexpr int kRW = 16;       // grid rows (vectors) per block: CB = kRW / n_amp RHS columns
constexpr int kLWMAX = 384;   // window points per row staged in shared memory (256 x 1.4 + w for the configs)

template <int W>
__global__ void __launch_bounds__(256) interp_win_kernel(const float2* __restrict__ grid, const int* __restrict__ l0,
                                                         const float* __restrict__ off, const float2* __restrict__ ph,
                                                         const float2* __restrict__ ampa, float2* __restrict__ G,
                                                         int64_t ldg, int64_t N, int64_t nf, int n_sub, int n_amp,
                                                         int nv, int nrhs, float beta)
{
    extern __shared__ float2 win[];   // [kRW][kLWMAX]
    __shared__ int red[2][8];
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + tid;
    const bool ok = i < N;
    const int cb = kRW / n_amp;
    const int c0 = blockIdx.y * cb;
    const int nc = min(cb, nrhs - c0), nrow = nc * n_amp;
    float2 acc[kRW];
#pragma unroll
    for (int q = 0; q < kRW; q++) acc[q] = make_float2(0.f, 0.f);
    for (int s = 0; s < n_sub; s++) {
        const int64_t idx = int64_t(s) * N + (ok ? i : 0);
        const int lb = l0[idx];
        const float o = off[idx];
        const float2 e = ph[idx];
        float wt[W];
#pragma unroll
        for (int m = 0; m < W; m++) {
            const float z = (float(m) - o) * (2.0f / W);
            wt[m] = __expf(beta * (sqrtf(fmaxf(1.f - z * z, 0.f)) - 1.f));
        }
        // block min / max of the first grid points
        int mn = ok ? lb : 0x7fffffff, mx = ok ? lb : -0x7fffffff;
#pragma unroll
        for (int d = 16; d; d >>= 1) {
            mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, d));
            mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d));
        }
        if (lane == 0) {
            red[0][wp] = mn;
            red[1][wp] = mx;
        }
        __syncthreads();
        mn = red[0][0];
        mx = red[1][0];
#pragma unroll
        for (int q = 1; q < 8; q++) {
            mn = min(mn, red[0][q]);
            mx = max(mx, red[1][q]);
        }
        const int mn2 = mn & ~1;                       // 16-byte aligned pairs (n_f is even: no pair wraps)
        const int lw = mx - mn2 + W;
        const int np = (lw + 1) >> 1;                  // pairs per row
        const float2* gs = grid + (int64_t(s) * nv + int64_t(c0) * n_amp) * nf;
        if (2 * np <= kLWMAX) {
            // every row's window with asynchronous 16-byte copies, all in flight at once (one load round trip
            // per block instead of one per row and pass)
            for (int t = tid; t < np; t += 256) {   // a thread copies pair t of every row (no index division)
                int l = mn2 + 2 * t;
                l = l < 0 ? l + int(nf) : (l >= int(nf) ? l - int(nf) : l);
                const uint32_t dst = uint32_t(__cvta_generic_to_shared(win + 2 * t));
                const float2* src = gs + l;
                for (int r = 0; r < nrow; r++)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + uint32_t(r * kLWMAX * 8)),
                                 "l"(src + int64_t(r) * nf)
                                 : "memory");
            }
            asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
            __syncthreads();
            if (ok) {
                const int rel = lb - mn2;
                for (int k = 0; k < n_amp; k++) {
                    const float2 a = ampa[int64_t(k) * N + i];
                    const float2 ea = make_float2(a.x * e.x - a.y * e.y, a.x * e.y + a.y * e.x);
#pragma unroll
                    for (int q = 0; q < kRW; q++) {
                        if (q >= nc) break;
                        const float2* wr = win + (q * n_amp + k) * kLWMAX + rel;
                        float2 u = make_float2(0.f, 0.f);
#pragma unroll
                        for (int m = 0; m < W; m++) {
                            const float2 x = wr[m];
                            u.x = fmaf(wt[m], x.x, u.x);
                            u.y = fmaf(wt[m], x.y, u.y);
                        }
                        acc[q].x += ea.x * u.x - ea.y * u.y;
                        acc[q].y += ea.x * u.y + ea.y * u.x;
                    }
                }
            }
        } else if (ok) {   // direct path: w global loads per target and row
            for (int k = 0; k < n_amp; k++) {
                const float2 a = ampa[int64_t(k) * N + i];
                const float2 ea = make_float2(a.x * e.x - a.y * e.y, a.x * e.y + a.y * e.x);
#pragma unroll
                for (int q = 0; q < kRW; q++) {
                    if (q >= nc) break;
                    const float2* gv = gs + int64_t(q * n_amp + k) * nf;
                    float2 u = make_float2(0.f, 0.f);
#pragma unroll
                    for (int m = 0; m < W; m++) {
                        int l = lb + m;
                        l = l < 0 ? l + int(nf) : (l >= int(nf) ? l - int(nf) : l);
                        const float2 x = __ldg(gv + l);
                        u.x = fmaf(wt[m], x.x, u.x);
                        u.y = fmaf(wt[m], x.y, u.y);
                    }
                    acc[q].x += ea.x * u.x - ea.y * u.y;
                    acc[q].y += ea.x * u.y + ea.y * u.x;
                }
            }
        }
        __syncthreads();   // the window and red[] are reused by the next submatrix
    }
    if (ok)
#pragma unroll
        for (int q = 0; q < kRW; q++)
            if (q < nc) G[int64_t(c0 + q) * ldg + i] = acc[q];
}

template <int W>
cudaError_t launch_interp(const bf_nufft_s* p, float2* G, int64_t ldg, int nv, int nrhs, cudaStream_t st)
{
    auto kern = interp_win_kernel<W>;
    const size_t smem = size_t(kRW) * kLWMAX * sizeof(float2);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    const int cb = kRW / p->n_amp;
    dim3 grid(unsigned((p->N + 255) / 256), unsigned((nrhs + cb - 1) / cb));
    kern<<<grid, 256, smem, st>>>(p->gout, p->l0, p->off, p->ph, p->amp_a, G, ldg, p->N, p->nf, p->n_sub, p->n_amp,
                                  nv, nrhs, float(p->beta));
    return cudaGetLastError();
}

cudaError_t interp(const bf_nufft_s* p, float2* G, int64_t ldg, int nv, int nrhs, cudaStream_t st)
{
    switch (p->w) {
    case 4: return launch_interp<4>(p, G, ldg, nv, nrhs, st);
    case 5: return launch_interp<5>(p, G, ldg, nv, nrhs, st);
    case 6: return launch_interp<6>(p, G, ldg, nv, nrhs, st);
    case 7: return launch_interp<7>(p, G, ldg, nv, nrhs, st);
    case 8: return launch_interp<8>(p, G, ldg, nv, nrhs, st);
    case 9: return launch_interp<9>(p, G, ldg, nv, nrhs, st);
    case 10: return launch_interp<10>(p, G, ldg, nv, nrhs, st);
    case 11: return launch_interp<11>(p, G, ldg, nv, nrhs, st);
    case 12: return launch_interp<12>(p, G, ldg, nv, nrhs, st);
    case 13: return launch_interp<13>(p, G, ldg, nv, nrhs, st);
    case 14: return launch_interp<14>(p, G, ldg, nv, nrhs, st);
    default: return cudaErrorInvalidValue;
    }
}

void free_plan(bf_nufft_s* p)
{
    if (!p) return;
    Guard g(p->device);
    if (p->fft_ok) cufftDestroy(p->fft);
    cudaFree(p->amp_a);
    cudaFree(p->amp_b);
    cudaFree(p->deconv);
    cudaFree(p->l0);
    cudaFree(p->off);
    cudaFree(p->ph);
    cudaFree(p->grid);
    cudaFree(p->gout);
    delete p;
}

template <class T>
bf_status_t upload(T** dst, const void* src, size_t bytes, const char* what)
{
    if (cudaMalloc(dst, bytes) != cudaSuccess) {
        cudaGetLastError();
        return nf_fail(BF_ERR_OOM, what);
    }
    const cudaError_t e = cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
    return e == cudaSuccess ? BF_OK : nf_cuda(e, what);
}

}  // namespace

extern "C" bf_status_t bf_nufft_create(const bf_nufft_desc_t* d, int device, int64_t max_nrhs_chunk, bf_nufft_t* out)
{
    if (!d || !out || !d->targets || !d->amp_a || !d->amp_b) return nf_fail(BF_ERR_INVALID_ARG, "bf_nufft_create: null");
    *out = nullptr;
    if (d->abi_version != BF_ABI_VERSION) return nf_fail(BF_ERR_INVALID_ARG, "bf_nufft_create: abi_version");
    if (d->log2n < 4 || d->log2n > 26 || d->n_amp < 1 || d->n_amp > 8 || (d->n_sub != 1 && d->n_sub != 2) ||
        !(d->eps >= 1e-12 && d->eps <= 1e-2) || max_nrhs_chunk < 1)
        return nf_fail(BF_ERR_SHAPE, "bf_nufft_create: log2n 4..26, n_amp 1..8, n_sub 1|2, eps 1e-12..1e-2, chunk >= 1");
    auto* p = new bf_nufft_s;
    p->device = device;
    p->LN = d->log2n;
    p->n_amp = d->n_amp;
    p->n_sub = d->n_sub;
    p->N = int64_t(1) << d->log2n;
    p->M = p->N / d->n_sub;
    p->nf = 2 * p->M;
    p->w = std::min(14, std::max(4, int(std::ceil(-std::log10(d->eps))) + 2));
    p->beta = 2.30 * p->w;
    const int64_t nv = max_nrhs_chunk * d->n_amp;
    if (int64_t(d->n_sub) * nv > (int64_t(1) << 30) / 1) {
        delete p;
        return nf_fail(BF_ERR_SHAPE, "bf_nufft_create: too many grids per chunk");
    }
    p->max_chunk = max_nrhs_chunk;
    Guard g(device);
    const size_t c8 = sizeof(float2);
    bf_status_t st;
    if ((st = upload(&p->amp_a, d->amp_a, size_t(d->n_amp) * p->N * c8, "amp_a")) != BF_OK ||
        (st = upload(&p->amp_b, d->amp_b, size_t(d->n_amp) * p->N * c8, "amp_b")) != BF_OK) {
        free_plan(p);
        return st;
    }
    std::vector<float> dc;
    deconv_factors(p->w, p->beta, p->M, p->nf, dc);
    // per target and submatrix: first grid point, offset, phase e^{2 pi i t xi_c} -- FP64, rounded once
    const int64_t NT = int64_t(d->n_sub) * p->N;
    std::vector<int> l0(static_cast<size_t>(NT));
    std::vector<float> off(static_cast<size_t>(NT));
    std::vector<float2> ph(static_cast<size_t>(NT));
    const double half = 0.5 * p->w;
#pragma omp parallel for schedule(static)
    for (int64_t idx = 0; idx < NT; idx++) {
        const int s = int(idx / p->N);
        const double t = d->targets[idx];
        const double tf = t - std::floor(t);                      // the sums are 1-periodic in t (integer xi)
        const double pos = tf * double(p->nf);
        const double lb = std::ceil(pos - half);
        l0[size_t(idx)] = int(lb);
        off[size_t(idx)] = float(pos - lb);
        const double xic = double(int64_t(s) * p->M + p->M / 2 - p->N / 2);   // centre frequency of X_s
        // t xi_c mod 1 with xi_c an integer: split t into integer and fraction first (t xi_c can exceed 2^20)
        double fr = tf * xic;
        fr -= std::floor(fr);
        double sn, cs;
        sincos(2.0 * M_PI * fr, &sn, &cs);
        ph[size_t(idx)] = make_float2(float(cs), float(sn));
    }
    if ((st = upload(&p->deconv, dc.data(), dc.size() * sizeof(float), "deconv")) != BF_OK ||
        (st = upload(&p->l0, l0.data(), l0.size() * sizeof(int), "l0")) != BF_OK ||
        (st = upload(&p->off, off.data(), off.size() * sizeof(float), "off")) != BF_OK ||
        (st = upload(&p->ph, ph.data(), ph.size() * c8, "phase")) != BF_OK) {
        free_plan(p);
        return st;
    }
    const size_t gbytes = size_t(d->n_sub) * size_t(nv) * size_t(p->nf) * c8;
    if (cudaMalloc(&p->grid, gbytes) != cudaSuccess || cudaMalloc(&p->gout, gbytes) != cudaSuccess) {
        cudaGetLastError();
        free_plan(p);
        return nf_fail(BF_ERR_OOM, "bf_nufft_create: fine grids");
    }
    if (cudaError_t e = cudaMemset(p->grid, 0, gbytes); e != cudaSuccess) {   // the zero padding, once
        free_plan(p);
        return nf_cuda(e, "bf_nufft_create: grid zero");
    }
    int n = int(p->nf);
    p->fft_batch = int(d->n_sub * nv);
    if (cufftPlanMany(&p->fft, 1, &n, nullptr, 1, n, nullptr, 1, n, CUFFT_C2C, p->fft_batch) != CUFFT_SUCCESS) {
        free_plan(p);
        return nf_fail(BF_ERR_CUDA, "bf_nufft_create: cufftPlanMany");
    }
    p->fft_ok = true;
    *out = p;
    return BF_OK;
}

extern "C" bf_status_t bf_nufft_apply(bf_nufft_t p, const bf_c64* Fc, int64_t ldf, bf_c64* Gc, int64_t ldg, int64_t nrhs,
                                      void* stream)
{
    if (!p) return nf_fail(BF_ERR_INVALID_ARG, "bf_nufft_apply: plan is NULL");
    if (nrhs < 0) return nf_fail(BF_ERR_INVALID_ARG, "bf_nufft_apply: nrhs < 0");
    if (nrhs == 0) return BF_OK;
    if (!Fc || !Gc) return nf_fail(BF_ERR_INVALID_ARG, "bf_nufft_apply: F or G is NULL");
    if (ldf < p->N || ldg < p->N) return nf_fail(BF_ERR_SHAPE, "bf_nufft_apply: ld < N");
    if ((reinterpret_cast<uintptr_t>(Fc) & 15) | (reinterpret_cast<uintptr_t>(Gc) & 7) | (ldf & 1))
        return nf_fail(BF_ERR_ALIGNMENT, "bf_nufft_apply: F not 16-byte aligned, odd ldf, or G not 8-byte aligned");
    const float2* F = reinterpret_cast<const float2*>(Fc);
    float2* G = reinterpret_cast<float2*>(Gc);
    if (F < G + ldg * nrhs && G < F + ldf * nrhs) return nf_fail(BF_ERR_INVALID_ARG, "bf_nufft_apply: F and G alias");
    Guard g(p->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (cufftSetStream(p->fft, st) != CUFFT_SUCCESS) return nf_fail(BF_ERR_CUDA, "cufftSetStream");
    for (int64_t c0 = 0; c0 < nrhs; c0 += p->max_chunk) {
        const int cn = int(std::min<int64_t>(p->max_chunk, nrhs - c0));
        const int nv = cn * p->n_amp, nvf = int(p->max_chunk) * p->n_amp;
        // the grids of a short chunk keep the full chunk's layout (the FFT plan's batch is fixed; the unused
        // grids hold an earlier chunk's finite values or zeros, and their transforms are not read)
        dim3 pg(unsigned((p->M / 2 + 255) / 256), unsigned(nv), unsigned(p->n_sub));
        place_kernel<<<pg, 256, 0, st>>>(F + c0 * ldf, ldf, p->amp_b, p->deconv, p->grid, p->N, p->M, p->nf, p->n_amp,
                                         nvf);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return nf_cuda(e, "bf_nufft_apply: place");
        if (cufftExecC2C(p->fft, reinterpret_cast<cufftComplex*>(p->grid), reinterpret_cast<cufftComplex*>(p->gout),
                         CUFFT_INVERSE) != CUFFT_SUCCESS)
            return nf_fail(BF_ERR_CUDA, "bf_nufft_apply: cufftExecC2C");
        e = interp(p, G + c0 * ldg, ldg, nvf, cn, st);
        if (e != cudaSuccess) return nf_cuda(e, "bf_nufft_apply: interp");
    }
    return BF_OK;
}

extern "C" bf_status_t bf_nufft_get_info(bf_nufft_t p, bf_nufft_info_t* info)
{
    if (!p || !info) return nf_fail(BF_ERR_INVALID_ARG, "bf_nufft_get_info: null");
    info->n = p->N;
    info->width = p->w;
    info->beta = p->beta;
    info->grid = p->nf;
    info->workspace_bytes = 2 * int64_t(p->n_sub) * p->max_chunk * p->n_amp * p->nf * int64_t(sizeof(float2));
    info->launches_per_chunk = 2;
    return BF_OK;
}

extern "C" bf_status_t bf_nufft_destroy(bf_nufft_t p)
{
    if (!p) return BF_OK;
    {
        Guard g(p->device);
        cudaDeviceSynchronize();
    }
    free_plan(p);
    return BF_OK;
}
