// tc_probe_f16.cu -- design questions for a kind::f16 leaf path (item 1):
//   (1) tcgen05.mma kind::f16 with A in TMEM (two f16 per 32-bit column) and B in shared memory (K-major,
//       SWIZZLE_NONE, 8 rows x 16 B core matrices), M = 128: correctness and the packing order of A
//   (2) issue cost per MMA (M = 128, N = 128, K = 16) back to back, A from TMEM -- the rate versus the
//       kind::tf32 MMA (K = 8) of the current kernels
//   (3) precision of the 3-pass split (hi hi + lo hi + hi lo) in FP16 with power-of-two scaling of every
//       A row and B row to max |x| in [0.5, 1), versus the 3-pass TF32 split, for a long K chain
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_probe_f16 tools/tc_probe_f16.cu
#include <cuda_fp16.h>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "../paper_1803_04128_b200/csrc/tc_sm100.cuh"

constexpr int M = 128;

__host__ __device__ constexpr uint32_t idesc_f16(int m, int n)
{
    return (1u << 4) | (0u << 7) | (0u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}
__host__ __device__ constexpr uint32_t kmaj_off16(int row, int k, int rows)
{
    return uint32_t((k >> 3) * (rows >> 3) * 128 + (row >> 3) * 128 + (row & 7) * 16 + (k & 7) * 2);
}
__device__ __forceinline__ void mma_f16_ts(uint32_t d, uint32_t a_tmem, uint64_t db, uint32_t idesc, uint32_t acc)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
        "r"(a_tmem), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ uint32_t pack2(__half lo, __half hi)
{
    return uint32_t(__half_as_ushort(lo)) | (uint32_t(__half_as_ushort(hi)) << 16);
}

// D[M][N] = sum_k A[M][K] B[N][K]; A, B given as f16 (row-major [.][K]); K multiple of 16, N <= 256.
// swap = 1 packs k = 2c into the HIGH half (tests the packing order).
template <int N, int K>
__global__ void check_kernel(const __half* A, const __half* B, float* D, int swap)
{
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < N * K; i += blockDim.x) {
        const int r = i / K, k = i % K;
        *reinterpret_cast<__half*>(smem + kmaj_off16(r, k, N)) = B[i];
    }
    if (warp == 0) tc::tmem_alloc<512>(&tbase);
    if (tid == 0) {
        tc::mbar_init(&bar, 1);
        tc::mbar_fence_init();
    }
    tc::fence_proxy_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = tbase, a_tm = tm + 256;
    {
        uint32_t w[K / 2];
        for (int c = 0; c < K / 2; c++) {
            const __half e0 = A[tid * K + 2 * c], e1 = A[tid * K + 2 * c + 1];
            w[c] = swap ? pack2(e1, e0) : pack2(e0, e1);
        }
        const uint32_t ta = a_tm + (uint32_t(warp * 32) << 16);
        for (int c = 0; c < K / 2; c += 4) tc::tmem_st4(ta + c, reinterpret_cast<const float*>(w + c));
        tc::tmem_wait_st();
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (tid == 0) {
        constexpr uint32_t LBO = (N / 8) * 128;
        for (int ks = 0; ks < K / 16; ks++)
            mma_f16_ts(tm, a_tm + ks * 8, tc::desc_kmajor(tc::smem_u32(smem) + ks * 2 * LBO, LBO), idesc_f16(M, N),
                       ks ? 1u : 0u);
        tc::commit(&bar);
    }
    tc::mbar_wait(&bar, 0);
    tc::fence_after_sync();
    for (int c0 = 0; c0 < N; c0 += 8) {
        float v[8];
        tc::tmem_ld8(tm + (uint32_t(warp * 32) << 16) + c0, v);
        tc::tmem_wait_ld();
        for (int j = 0; j < 8; j++) D[tid * N + c0 + j] = v[j];
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<512>(tm);
}

template <int N, int K>
int check(int swap)
{
    std::mt19937 g(7);
    std::uniform_int_distribution<int> u(-8, 8);
    std::vector<__half> A(M * K), B(N * K);
    std::vector<float> Af(M * K), Bf(N * K);
    for (int i = 0; i < M * K; i++) { Af[i] = u(g) / 4.0f; A[i] = __float2half(Af[i]); }
    for (int i = 0; i < N * K; i++) { Bf[i] = u(g) / 4.0f; B[i] = __float2half(Bf[i]); }
    __half *dA, *dB;
    float* dD;
    cudaMalloc(&dA, A.size() * 2);
    cudaMalloc(&dB, B.size() * 2);
    cudaMalloc(&dD, M * N * 4);
    cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
    const int sm = N * K * 2;
    cudaFuncSetAttribute(check_kernel<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    check_kernel<N, K><<<1, 128, sm>>>(dA, dB, dD, swap);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> D(M * N);
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int r = 0; r < M; r++)
        for (int n = 0; n < N; n++) {
            double s = 0;
            for (int k = 0; k < K; k++) s += double(Af[r * K + k]) * Bf[n * K + k];
            maxerr = std::fmax(maxerr, std::fabs(s - D[r * N + n]));
        }
    printf("f16 TS check N=%d K=%d packing %s: max|err| = %g (%s)\n", N, K, swap ? "k=2c HIGH" : "k=2c LOW", maxerr,
           e == cudaSuccess ? "ok" : cudaGetErrorString(e));
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
    return maxerr == 0 ? 0 : 1;
}

// issue rate: `iters` MMAs (M = 128, N, K = 16) back to back, A from TMEM
template <int N>
__global__ void rate_kernel(int iters, long long* out)
{
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < N * 16; i += blockDim.x) *reinterpret_cast<__half*>(smem + 2 * i) = __float2half(0.001f);
    if (warp == 0) tc::tmem_alloc<512>(&tbase);
    if (tid == 0) {
        tc::mbar_init(&bar, 1);
        tc::mbar_fence_init();
    }
    tc::fence_proxy_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = tbase;
    if (tid == 0) {
        constexpr uint32_t LBO = (N / 8) * 128;
        const uint64_t db = tc::desc_kmajor(tc::smem_u32(smem), LBO);
        const long long t0 = clock64();
        for (int i = 0; i < iters; i++) mma_f16_ts(tm, tm + 384, db, idesc_f16(M, N), 1u);
        tc::commit(&bar);
        tc::mbar_wait(&bar, 0);
        out[0] = clock64() - t0;
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<512>(tm);
}

template <int N>
void rate(int iters)
{
    long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(rate_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, N * 32);
    rate_kernel<N><<<1, 128, N * 32>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("f16 TS rate N=%3d: %.1f clk per MMA (M=128, K=16) -> %.0f MAC/clk (%s)\n", N, double(c) / iters,
           128.0 * N * 16 / (double(c) / iters), e == cudaSuccess ? "ok" : cudaGetErrorString(e));
    cudaFree(d);
}

// ---- (3) precision: host model of the two 3-pass splits against FP64 ----
// The tensor core multiplies f16 x f16 exactly and accumulates in FP32; this host model accumulates the
// same products in FP32 in chains of `seg` K-steps of 16 (summed in FP32 like the kernels' segments).
static double rel_err(const std::vector<double>& ref, const std::vector<double>& got)
{
    double n = 0, d = 0;
    for (size_t i = 0; i < ref.size(); i++) {
        n += (ref[i] - got[i]) * (ref[i] - got[i]);
        d += ref[i] * ref[i];
    }
    return std::sqrt(n / d);
}
static float tf32_rna(float x)
{
    uint32_t u;
    memcpy(&u, &x, 4);
    u = (u + 0x1000u) & 0xffffe000u;
    float y;
    memcpy(&y, &u, 4);
    return y;
}
static float tf32_trunc(float x)
{
    uint32_t u;
    memcpy(&u, &x, 4);
    u &= 0xffffe000u;
    float y;
    memcpy(&y, &u, 4);
    return y;
}
void precision(int K, double spread)
{
    std::mt19937 g(11);
    std::normal_distribution<double> nd(0, 1);
    std::uniform_real_distribution<double> ud(-spread, spread);
    const int R = 64, C = 64;
    std::vector<double> a(R * K), b(C * K), ref(R * C), g16(R * C), g32(R * C);
    for (auto& x : a) x = nd(g) * std::pow(10.0, ud(g));
    for (auto& x : b) x = nd(g) * std::pow(10.0, ud(g));
    // per-row scales (power of two, max |x| in [0.5, 1))
    auto rscale = [&](const std::vector<double>& m, int r) {
        double mx = 0;
        for (int k = 0; k < K; k++) mx = std::fmax(mx, std::fabs(m[r * K + k]));
        int e;
        std::frexp(mx, &e);
        return -e;   // x 2^-e in [0.5, 1)
    };
    for (int r = 0; r < R; r++) {
        const int ea = rscale(a, r);
        for (int c = 0; c < C; c++) {
            const int eb = rscale(b, c);
            double s = 0;
            float acc16 = 0, acc32 = 0;
            for (int k = 0; k < K; k++) {
                const double x = a[r * K + k], y = b[c * K + k];
                s += x * y;
                // f16 split of the scaled values
                const float xs = float(std::ldexp(x, ea)), ys = float(std::ldexp(y, eb));
                const __half xh = __float2half_rn(xs), yh = __float2half_rn(ys);
                const __half xl = __float2half_rn(xs - __half2float(xh)), yl = __float2half_rn(ys - __half2float(yh));
                acc16 += __half2float(xh) * __half2float(yh) + __half2float(xl) * __half2float(yh) +
                         __half2float(xh) * __half2float(yl);
                // tf32 split (hi = rna, lo = exact residual truncated by the tensor core)
                const float xf = float(x), yf = float(y);
                const float xhi = tf32_rna(xf), yhi = tf32_rna(yf);
                const float xlo = tf32_trunc(xf - xhi), ylo = tf32_trunc(yf - yhi);
                acc32 += xhi * yhi + xlo * yhi + xhi * ylo;
            }
            ref[r * C + c] = s;
            g16[r * C + c] = std::ldexp(double(acc16), -ea - eb);
            g32[r * C + c] = acc32;
        }
    }
    printf("3-pass split precision, K=%4d, magnitude spread 10^+-%.0f: f16 (row-scaled) %.2e   tf32 %.2e\n", K, spread,
           rel_err(ref, g16), rel_err(ref, g32));
}

int main()
{
    int fails = 0;
    fails += check<128, 32>(0);
    check<128, 32>(1);
    fails += check<80, 64>(0);
    rate<64>(4096);
    rate<128>(4096);
    rate<256>(4096);
    precision(128, 0);
    precision(128, 2);
    precision(1280, 0);
    precision(1280, 2);
    printf(fails ? "TC PROBE F16: %d FAILED\n" : "TC PROBE F16 OK\n", fails);
    return 0;
}
