// sustained_peaks.cu -- sustained (>= 4 s, every SM) device rates the roofline denominators of bench.py compare with:
//   ffma : FP32 FFMA throughput (8 independent chains per thread, 148 x 8 CTAs of 256 threads)
//   tf32 : kind::tf32 tcgen05.mma throughput (M = 128, N = 256, K = 8; A and B in shared memory; one CTA per SM,
//          one elected thread issuing into two alternating TMEM accumulators, a commit + wait every 32 MMAs)
// Prints one JSON object.  The rates are the hardware's under the 1 kW power cap, i.e. what a kernel that keeps the
// pipe busy for seconds can get; bench.py reports its tensor / alu fractions against them beside the nominal peaks.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/sustained_peaks tools/sustained_peaks.cu
#include <cstdint>
#include <cstdio>

#include "../paper_1803_04128_b200/csrc/tc_sm100.cuh"

__global__ void __launch_bounds__(256) ffma_kernel(float* out, long long iters, float a, float b)
{
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 1e-3f + i;
    for (long long it = 0; it < iters; it++) {
#pragma unroll
        for (int r = 0; r < 16; r++)
#pragma unroll
            for (int i = 0; i < 8; i++) x[i] = fmaf(x[i], a, b);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) s += x[i];
    if (s == 1234.5f) out[blockIdx.x] = s;   // keep the chains alive
}

constexpr int TM = 128, TN = 256, TK = 8;

__global__ void __launch_bounds__(128, 1) tf32_kernel(float* out, long long iters)
{
    extern __shared__ __align__(128) uint8_t sm[];
    uint8_t* a_s = sm;                 // 128 x 8 tf32, K-major
    uint8_t* b_s = sm + TM * TK * 4;   // 256 x 8
    __shared__ uint64_t bar[2];
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < TM * TK; i += blockDim.x)
        *reinterpret_cast<float*>(a_s + tc::kmaj_off(i / TK, i % TK, TM)) = 1e-3f * (i % 7);
    for (int i = tid; i < TN * TK; i += blockDim.x)
        *reinterpret_cast<float*>(b_s + tc::kmaj_off(i / TK, i % TK, TN)) = 1e-3f * (i % 5);
    if (warp == 0) tc::tmem_alloc<512>(&tbase);
    if (tid == 0) {
        tc::mbar_init(&bar[0], 1);
        tc::mbar_init(&bar[1], 1);
        tc::mbar_fence_init();
    }
    tc::fence_proxy_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tbase;
    if (warp == 0) {
        constexpr uint32_t idesc = tc::idesc_tf32(TM, TN);
        const uint64_t da = tc::desc_kmajor(tc::smem_u32(a_s), (TM / 8) * 128);
        const uint64_t db = tc::desc_kmajor(tc::smem_u32(b_s), (TN / 8) * 128);
        // groups of 32 MMAs, each committed to its own barrier; before issuing group g + 1 the issuer waits for group
        // g - 1, so one group is always queued behind the executing one (the pipe never drains)
        long long g = 0;
        for (long long it = 0; it < iters; it += 32, g++) {
#pragma unroll
            for (int q = 0; q < 32; q++)
                tc::mma_tf32_warp(tmem + uint32_t((q & 1) * TN), da, db, idesc, (it > 0 || q >= 2) ? 1u : 0u);
            tc::commit_warp(&bar[g & 1]);
            if (g >= 1) tc::mbar_wait(&bar[(g - 1) & 1], uint32_t((g - 1) >> 1) & 1);
        }
        if (g >= 1) tc::mbar_wait(&bar[(g - 1) & 1], uint32_t((g - 1) >> 1) & 1);
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) {
        tc::fence_after_sync();
        float v[4];
        tc::tmem_ld_cols<4>(tmem, v);
        tc::tmem_wait_ld();
        if (v[0] == 1234.5f) out[blockIdx.x] = v[1];
        tc::tmem_dealloc<512>(tmem);
    }
}

int main()
{
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    cudaMalloc(&out, 1 << 20);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms = 0;
    // ---- FFMA: calibrate, then run >= 4 s ----
    const int fblocks = nsm * 8;
    long long fit = 1000;
    for (;;) {
        cudaEventRecord(e0);
        ffma_kernel<<<fblocks, 256>>>(out, fit, 0.999999f, 1e-7f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms > 4000.f) break;
        fit = (long long)(fit * (ms < 10.f ? 20.0 : 4200.0 / ms)) + 1;
    }
    const double ffma_tf = 2.0 * 16 * 8 * double(fit) * fblocks * 256 / (ms * 1e-3) / 1e12;
    const float ffma_ms = ms;
    // ---- TF32 MMA ----
    const size_t smem = (TM + TN) * TK * 4;
    cudaFuncSetAttribute(tf32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    long long tit = 3200;
    for (;;) {
        cudaEventRecord(e0);
        tf32_kernel<<<nsm, 128, smem>>>(out, tit);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms > 4000.f) break;
        tit = ((long long)(tit * (ms < 10.f ? 20.0 : 4200.0 / ms)) / 32 + 1) * 32;
    }
    const cudaError_t err = cudaGetLastError();
    const double tf32_tf = 2.0 * TM * TN * TK * double(tit) * nsm / (ms * 1e-3) / 1e12;
    printf("{\"ffma_tflops_sustained\": %.2f, \"ffma_seconds\": %.2f, \"tf32_tflops_sustained\": %.2f, "
           "\"tf32_seconds\": %.2f, \"tf32_mma\": \"kind::tf32 M=128 N=256 K=8, A and B in SMEM, one issuing thread "
           "per SM\", \"sms\": %d, \"status\": \"%s\"}\n",
           ffma_tf, ffma_ms / 1e3, tf32_tf, ms / 1e3, nsm, cudaGetErrorString(err));
    return err == cudaSuccess ? 0 : 1;
}
