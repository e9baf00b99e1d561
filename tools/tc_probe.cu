// tc_probe.cu -- validates the tcgen05 building blocks used by the tensor-core kernels:
// kind::tf32 MMA with K-major SWIZZLE_NONE shared-memory descriptors, TMEM allocation,
// tcgen05.commit -> mbarrier, tcgen05.ld 32x32b readback, and the 3xTF32 split
// D = Ahi Bhi + Alo Bhi + Ahi Blo.  One CTA computes D[128][N] = A[128][K] B[K][N]
// (B given as Bt[N][K], i.e. both operands K-major) and the host compares with FP64.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_probe tools/tc_probe.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <vector>

constexpr int M = 128, N = 40, K = 48;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

// K-major, no swizzle canonical layout (CUTLASS make_umma_desc<K>, INTERLEAVE): core matrix = 8 rows x 16 B
// (4 tf32) contiguous; the 2 core matrices of one MMA's K (= 8 tf32) LBO bytes apart; 8-row groups SBO
// bytes apart.  Our tile: [kcore][rowgroup][8 rows][16 B]  ->  LBO = (rows/8) * 128, SBO = 128.
__device__ __forceinline__ uint32_t off_kmajor(int row, int k, int rows)
{
    return uint32_t(((k >> 2) * (rows >> 3) + (row >> 3)) * 128 + (row & 7) * 16 + (k & 3) * 4);
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo)
{
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFF);
    d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
    d |= uint64_t(1) << 46;   // version 1 (sm_100)
    // base offset 0, lbo mode 0, layout type 0 = SWIZZLE_NONE
    return d;
}

// instruction descriptor: D f32, A/B tf32, K-major both, N>>3, M>>4
__host__ __device__ constexpr uint32_t make_idesc(int m, int n)
{
    return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}

__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo)
{
    uint32_t h;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
    hi = __uint_as_float(h);
    lo = x - hi;   // exact in FP32; the MMA truncates lo to tf32 (its own 10-bit mantissa)
}

__global__ void tc_probe_kernel(const float* A, const float* Bt, float* D, int mode)
{
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* a_hi = smem;
    uint8_t* a_lo = a_hi + M * K * 4;
    uint8_t* b_hi = a_lo + M * K * 4;
    uint8_t* b_lo = b_hi + N * K * 4;
    __shared__ uint64_t mbar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    for (int i = tid; i < M * K; i += blockDim.x) {
        const int r = i / K, k = i % K;
        float hi, lo;
        split_tf32(A[i], hi, lo);
        *reinterpret_cast<float*>(a_hi + off_kmajor(r, k, M)) = hi;
        *reinterpret_cast<float*>(a_lo + off_kmajor(r, k, M)) = lo;
    }
    for (int i = tid; i < N * K; i += blockDim.x) {
        const int r = i / K, k = i % K;
        float hi, lo;
        split_tf32(Bt[i], hi, lo);
        *reinterpret_cast<float*>(b_hi + off_kmajor(r, k, N)) = hi;
        *reinterpret_cast<float*>(b_lo + off_kmajor(r, k, N)) = lo;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                     "r"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");   // generic-proxy smem writes -> visible to the tensor core
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;

    if (tid == 0) {
        const uint32_t idesc = make_idesc(M, N);
        const uint32_t lboA = (M / 8) * 128, lboB = (N / 8) * 128;
        const int npass = mode == 0 ? 1 : 3;
        int first = 1;
        for (int pass = 0; pass < npass; pass++) {
            const uint8_t* a = (pass == 1) ? a_lo : a_hi;
            const uint8_t* b = (pass == 2) ? b_lo : b_hi;
            for (int kk = 0; kk < K / 8; kk++) {
                // K step of 8 tf32 = 2 core columns = 2 * LBO bytes
                const uint64_t da = make_desc(smem_u32(a) + kk * 2 * lboA, lboA, 128);
                const uint64_t db = make_desc(smem_u32(b) + kk * 2 * lboB, lboB, 128);
                const uint32_t acc = first ? 0u : 1u;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                    "l"(da), "l"(db), "r"(idesc), "r"(acc));
                first = 0;
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&mbar)));
    }
    // wait for the MMAs (phase 0)
    {
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                : "=r"(done)
                : "r"(smem_u32(&mbar)), "r"(0));
        }
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    // each warp reads its 32 TMEM lanes (rows 32w..32w+31), 8 columns at a time
    for (int c0 = 0; c0 < N; c0 += 8) {
        uint32_t v[8];
        const uint32_t taddr = tmem + (uint32_t(warp * 32) << 16) + c0;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 8; j++) D[(warp * 32 + lane) * N + c0 + j] = __uint_as_float(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
}

int main()
{
    std::vector<float> A(M * K), Bt(N * K), D(M * N);
    srand(1);
    for (auto& x : A) x = float(rand()) / RAND_MAX * 2 - 1;
    for (auto& x : Bt) x = float(rand()) / RAND_MAX * 2 - 1;
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, Bt.size() * 4);
    cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, Bt.data(), Bt.size() * 4, cudaMemcpyHostToDevice);
    const int smem = 2 * M * K * 4 + 2 * N * K * 4;
    cudaFuncSetAttribute(tc_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int fails = 0;
    for (int mode = 0; mode < 2; mode++) {
        cudaMemset(dD, 0, D.size() * 4);
        tc_probe_kernel<<<1, 128, smem>>>(dA, dB, dD, mode);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("mode %d: CUDA error %s\n", mode, cudaGetErrorString(e));
            return 1;
        }
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double num = 0, den = 0, maxrel = 0;
        for (int i = 0; i < M; i++)
            for (int j = 0; j < N; j++) {
                double ref = 0;
                for (int k = 0; k < K; k++) ref += double(A[i * K + k]) * Bt[j * K + k];
                num += (D[i * N + j] - ref) * (D[i * N + j] - ref);
                den += ref * ref;
                maxrel = fmax(maxrel, fabs(D[i * N + j] - ref));
            }
        const double rel = sqrt(num / den);
        printf("mode %s: rel l2 error vs FP64 = %.3e (max abs %.3e)  D[0]=%f D[last]=%f\n",
               mode ? "3xTF32" : "1xTF32", rel, maxrel, D[0], D[M * N - 1]);
        if (mode == 0 && !(rel < 2e-3)) fails++;
        if (mode == 1 && !(rel < 2e-6)) fails++;
    }
    printf(fails ? "TC PROBE FAILED\n" : "TC PROBE OK\n");
    return fails;
}
