// cmac_bench.cu -- FP32 FFMA throughput microbenchmarks on B200 (the "alu" roofline and the
// register-bank question of DESIGN.md section 5).
//   ffma_peak      : 8 independent FFMA chains per thread (upper bound of the FP32 pipe)
//   cmac_inter<R>  : the S0/band inner loop (R rows x 4 vectors complex outer product) with operands
//                    loaded from shared memory as interleaved complex {re,im} (LDS.128)
//   cmac_planar<R> : the same loop with the vector operand stored planar (4 re, then 4 im)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cmac_bench tools/cmac_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void ffma_peak(float* out, int iters)
{
    float a[8];
    for (int i = 0; i < 8; i++) a[i] = threadIdx.x * 1e-7f + i;
    const float b = 0.999999f, c = 1e-7f;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 16; k++)
#pragma unroll
            for (int i = 0; i < 8; i++) a[i] = fmaf(a[i], b, c);
    }
    float s = 0;
    for (int i = 0; i < 8; i++) s += a[i];
    if (s == 1234.5f) out[0] = s;
}

// the same with packed FP32 pairs (sm_100a FFMA2): 8 independent chains of 2-wide FMAs
__global__ void ffma2_peak(float* out, int iters)
{
    unsigned long long a[8];
    for (int i = 0; i < 8; i++) {
        const float lo = threadIdx.x * 1e-7f + i, hi = lo + 0.5f;
        asm("mov.b64 %0, {%1, %2};" : "=l"(a[i]) : "f"(lo), "f"(hi));
    }
    unsigned long long b, c;
    asm("mov.b64 %0, {%1, %1};" : "=l"(b) : "f"(0.999999f));
    asm("mov.b64 %0, {%1, %1};" : "=l"(c) : "f"(1e-7f));
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 16; k++)
#pragma unroll
            for (int i = 0; i < 8; i++) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[i]) : "l"(b), "l"(c));
    }
    float s = 0;
    for (int i = 0; i < 8; i++) {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a[i]));
        s += lo + hi;
    }
    if (s == 1234.5f) out[0] = s;
}

__device__ __forceinline__ void cmac(float2& acc, float2 w, float2 v)
{
    acc.x = fmaf(w.x, v.x, acc.x);
    acc.x = fmaf(-w.y, v.y, acc.x);
    acc.y = fmaf(w.x, v.y, acc.y);
    acc.y = fmaf(w.y, v.x, acc.y);
}

template <int R>
__global__ void __launch_bounds__(256, 2) cmac_inter(float* out, int iters)
{
    __shared__ float4 Ys[32 * 64];   // [j][32 lanes x 2 float4] interleaved: 4 complex per lane
    __shared__ float4 Ws[64 * R / 2];
    for (int i = threadIdx.x; i < 32 * 64; i += blockDim.x) Ys[i] = make_float4(1e-3f * i, 1, 2, 3);
    for (int i = threadIdx.x; i < 64 * R / 2; i += blockDim.x) Ws[i] = make_float4(1e-4f * i, .5f, .25f, .125f);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    float2 acc[R][4];
#pragma unroll
    for (int t = 0; t < R; t++)
#pragma unroll
        for (int i = 0; i < 4; i++) acc[t][i] = make_float2(0, 0);
    for (int it = 0; it < iters; it++) {
#pragma unroll 2
        for (int j = 0; j < 64; j++) {
            float4 y0 = Ys[(j & 31) * 64 + lane * 2], y1 = Ys[(j & 31) * 64 + lane * 2 + 1];
            float2 y[4] = {make_float2(y0.x, y0.y), make_float2(y0.z, y0.w), make_float2(y1.x, y1.y),
                           make_float2(y1.z, y1.w)};
            float2 w[R];
#pragma unroll
            for (int q = 0; q < R / 2; q++) {
                float4 ww = Ws[j * R / 2 + q];
                w[2 * q] = make_float2(ww.x, ww.y);
                w[2 * q + 1] = make_float2(ww.z, ww.w);
            }
#pragma unroll
            for (int t = 0; t < R; t++)
#pragma unroll
                for (int i = 0; i < 4; i++) cmac(acc[t][i], w[t], y[i]);
        }
    }
    float s = 0;
#pragma unroll
    for (int t = 0; t < R; t++)
#pragma unroll
        for (int i = 0; i < 4; i++) s += acc[t][i].x + acc[t][i].y;
    if (s == 1234.5f) out[0] = s;
}

template <int R>
__global__ void __launch_bounds__(256, 2) cmac_planar(float* out, int iters)
{
    __shared__ float4 Ys[32 * 64];   // [j][lane][re4 | im4]
    __shared__ float4 Ws[64 * R / 2];
    for (int i = threadIdx.x; i < 32 * 64; i += blockDim.x) Ys[i] = make_float4(1e-3f * i, 1, 2, 3);
    for (int i = threadIdx.x; i < 64 * R / 2; i += blockDim.x) Ws[i] = make_float4(1e-4f * i, .5f, .25f, .125f);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    float ar[R][4], ai[R][4];
#pragma unroll
    for (int t = 0; t < R; t++)
#pragma unroll
        for (int i = 0; i < 4; i++) ar[t][i] = ai[t][i] = 0;
    for (int it = 0; it < iters; it++) {
#pragma unroll 2
        for (int j = 0; j < 64; j++) {
            float4 yr4 = Ys[(j & 31) * 64 + lane * 2], yi4 = Ys[(j & 31) * 64 + lane * 2 + 1];
            float yr[4] = {yr4.x, yr4.y, yr4.z, yr4.w}, yi[4] = {yi4.x, yi4.y, yi4.z, yi4.w};
            float2 w[R];
#pragma unroll
            for (int q = 0; q < R / 2; q++) {
                float4 ww = Ws[j * R / 2 + q];
                w[2 * q] = make_float2(ww.x, ww.y);
                w[2 * q + 1] = make_float2(ww.z, ww.w);
            }
#pragma unroll
            for (int t = 0; t < R; t++)
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    ar[t][i] = fmaf(w[t].x, yr[i], ar[t][i]);
                    ar[t][i] = fmaf(-w[t].y, yi[i], ar[t][i]);
                    ai[t][i] = fmaf(w[t].x, yi[i], ai[t][i]);
                    ai[t][i] = fmaf(w[t].y, yr[i], ai[t][i]);
                }
        }
    }
    float s = 0;
#pragma unroll
    for (int t = 0; t < R; t++)
#pragma unroll
        for (int i = 0; i < 4; i++) s += ar[t][i] + ai[t][i];
    if (s == 1234.5f) out[0] = s;
}

template <class K>
static void run(const char* name, K kern, int blocks, int threads, int iters, double flops_per_thread_iter)
{
    float* out;
    cudaMalloc(&out, 4);
    kern<<<blocks, threads>>>(out, 1);
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<blocks, threads>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double fl = double(blocks) * threads * iters * flops_per_thread_iter;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);   // kHz
    printf("%-16s %8.3f ms  %7.2f TFLOP/s  (%.1f%% of 148x128x2x%.3f GHz)\n", name, ms, fl / ms / 1e9,
           100.0 * fl / ms / 1e9 / (148 * 128 * 2 * clk * 1e-6), clk * 1e-6);
    cudaFree(out);
}

int main()
{
    const int blocks = 148 * 8;
    run("ffma_peak", ffma_peak, blocks, 256, 20000, 16.0 * 8 * 2);
    run("ffma2_peak", ffma2_peak, blocks, 256, 20000, 16.0 * 8 * 4);
    // low occupancy: 8 warps per SM (2 per sub-partition), as the persistent small-batch band runs
    run("ffma_8w", ffma_peak, 148, 256, 20000, 16.0 * 8 * 2);
    run("ffma2_8w", ffma2_peak, 148, 256, 20000, 16.0 * 8 * 4);
    run("ffma_4w", ffma_peak, 148, 128, 20000, 16.0 * 8 * 2);
    run("ffma2_4w", ffma2_peak, 148, 128, 20000, 16.0 * 8 * 4);
    run("cmac_inter<10>", cmac_inter<10>, 148 * 2 * 8, 256, 400, 64.0 * 10 * 4 * 8);
    run("cmac_planar<10>", cmac_planar<10>, 148 * 2 * 8, 256, 400, 64.0 * 10 * 4 * 8);
    run("cmac_inter<8>", cmac_inter<8>, 148 * 2 * 8, 256, 400, 64.0 * 8 * 4 * 8);
    run("cmac_planar<8>", cmac_planar<8>, 148 * 2 * 8, 256, 400, 64.0 * 8 * 4 * 8);
    return 0;
}
