// tc_probe2.cu -- answers the design questions of the tensor-core kernels:
//   (1) kind::tf32 SS MMA (both operands in shared memory, K-major SWIZZLE_NONE), M=128 N=48
//   (2) the "negate B" instruction-descriptor bit (bit 14) with kind::tf32
//   (3) A operand in TMEM (tcgen05.st, then tcgen05.mma [d], [a_tmem], b_desc) with kind::tf32
//   (4) MMA issue cost per instruction (clock64 over a long chain) for N in {48, 80, 160, 256},
//       A from SMEM vs from TMEM -- whether small-N tf32 MMAs are operand-bandwidth bound
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_probe2 tools/tc_probe2.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1803_04128_b200/csrc/tc_sm100.cuh"

constexpr int M = 128, K = 16;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t db, uint32_t idesc, uint32_t acc)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
        "r"(a_tmem), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float* v)
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
                 "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
                 "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
                 "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
                 : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// mode 0: SS, mode 1: SS with negate-B, mode 2: A from TMEM.  D[M][N] = A[M][K] Bt[N][K]^T (K=16, 2 steps)
template <int N>
__global__ void probe_kernel(const float* A, const float* Bt, float* D, int mode)
{
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* a_s = smem;
    uint8_t* b_s = smem + M * K * 4;
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < M * K; i += blockDim.x) {
        const int r = i / K, k = i % K;
        *reinterpret_cast<float*>(a_s + tc::kmaj_off(r, k, M)) = A[i];
    }
    for (int i = tid; i < N * K; i += blockDim.x) {
        const int r = i / K, k = i % K;
        *reinterpret_cast<float*>(b_s + tc::kmaj_off(r, k, N)) = Bt[i];
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
    const uint32_t tm = tbase;
    const uint32_t a_tm = tm + 256;   // A in TMEM at columns 256..256+K
    if (mode == 2) {
        // thread = row (warp w owns lanes 32w..): columns k of its row
        float v[K];
        for (int k = 0; k < K; k++) v[k] = A[tid * K + k];
        const uint32_t ta = a_tm + (uint32_t(warp * 32) << 16);
        tmem_st8(ta, v);
        tmem_st8(ta + 8, v + 8);
        tmem_wait_st();
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (tid == 0) {
        uint32_t idesc = tc::idesc_tf32(M, N);
        if (mode == 1) idesc |= 1u << 14;
        constexpr uint32_t LBOA = (M / 8) * 128, LBOB = (N / 8) * 128;
        for (int ks = 0; ks < K / 8; ks++) {
            const uint64_t db = tc::desc_kmajor(tc::smem_u32(b_s) + ks * 2 * LBOB, LBOB);
            if (mode == 2)
                mma_ts(tm, a_tm + ks * 8, db, idesc, ks ? 1u : 0u);
            else
                tc::mma_tf32(tm, tc::desc_kmajor(tc::smem_u32(a_s) + ks * 2 * LBOA, LBOA), db, idesc, ks ? 1u : 0u);
        }
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

// throughput: one thread issues `iters` MMAs (M=128, N, K=8) back to back into one accumulator
template <int N>
__global__ void rate_kernel(int iters, int a_in_tmem, long long* cycles)
{
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < (M + N) * 8; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.5f;
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
        const uint32_t idesc = tc::idesc_tf32(M, N);
        const uint64_t da = tc::desc_kmajor(tc::smem_u32(smem), (M / 8) * 128);
        const uint64_t db = tc::desc_kmajor(tc::smem_u32(smem + M * 8 * 4), (N / 8) * 128);
        const long long t0 = clock64();
        for (int i = 0; i < iters; i++) {
            if (a_in_tmem)
                mma_ts(tm, tm + 256, db, idesc, 1u);
            else
                tc::mma_tf32(tm, da, db, idesc, 1u);
        }
        tc::commit(&bar);
        tc::mbar_wait(&bar, 0);
        cycles[0] = clock64() - t0;
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<512>(tm);
}

// NACC independent accumulators round-robin (D at column offsets acc * N)
template <int N, int NACC, bool TS = false>
__global__ void rate_multi_kernel(int iters, long long* cycles)
{
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < (M + N) * 8; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.5f;
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
        const uint32_t idesc = tc::idesc_tf32(M, N);
        const uint64_t da = tc::desc_kmajor(tc::smem_u32(smem), (M / 8) * 128);
        const uint64_t db = tc::desc_kmajor(tc::smem_u32(smem + M * 8 * 4), (N / 8) * 128);
        const long long t0 = clock64();
        for (int i = 0; i < iters; i += NACC) {
#pragma unroll
            for (int a = 0; a < NACC; a++) {
                if constexpr (TS)
                    mma_ts(tm + a * N, tm + 480, db, idesc, 1u);
                else
                    tc::mma_tf32(tm + a * N, da, db, idesc, 1u);
            }
        }
        tc::commit(&bar);
        tc::mbar_wait(&bar, 0);
        cycles[0] = clock64() - t0;
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<512>(tm);
}

template <int N, int NACC, bool TS = false>
void rate_multi()
{
    long long* dc;
    cudaMalloc(&dc, 8);
    const int sm = (M + N) * 8 * 4;
    cudaFuncSetAttribute(rate_multi_kernel<N, NACC, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    const int iters = 4096;
    rate_multi_kernel<N, NACC, TS><<<1, 128, sm>>>(iters, dc);
    rate_multi_kernel<N, NACC, TS><<<1, 128, sm>>>(iters, dc);
    cudaError_t e = cudaDeviceSynchronize();
    long long c = 0;
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    const double per = double(c) / iters;
    printf("rate N=%3d x %d accumulators, A in %s: %.1f cycles per MMA -> %.0f MAC/clk/SM (%s)\n", N, NACC,
           TS ? "TMEM" : "SMEM", per,
           128.0 * N * 8 / per, e == cudaSuccess ? "ok" : cudaGetErrorString(e));
    cudaFree(dc);
}

// MMA rate (N=48, A in TMEM or SMEM) while 4 other warps stream tcgen05.st / tcgen05.ld traffic to other
// TMEM columns (the band kernel's split / epilogue load) -- is the MMA slowed by TMEM contention?
template <bool TS, int MODE>   // MODE 0: none, 1: st, 2: ld, 3: st+ld heavy (8 warps), 4: LDS, 5: STG
__global__ void contention_kernel(int iters, long long* cycles, float2* gbuf)
{
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    __shared__ volatile int stop;
    constexpr int N = 48;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < (M + N) * 8; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.5f;
    if (warp == 0) tc::tmem_alloc<512>(&tbase);
    if (tid == 0) {
        tc::mbar_init(&bar, 1);
        tc::mbar_fence_init();
        stop = 0;
    }
    tc::fence_proxy_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = tbase;
    if (warp == 0) {
        if (lane == 0) {
            const uint32_t idesc = tc::idesc_tf32(M, N);
            const uint64_t da = tc::desc_kmajor(tc::smem_u32(smem), (M / 8) * 128);
            const uint64_t db = tc::desc_kmajor(tc::smem_u32(smem + M * 8 * 4), (N / 8) * 128);
            const long long t0 = clock64();
            for (int i = 0; i < iters; i += 2) {
                if constexpr (TS) {
                    mma_ts(tm, tm + 200, db, idesc, 1u);
                    mma_ts(tm + 48, tm + 208, db, idesc, 1u);
                } else {
                    tc::mma_tf32(tm, da, db, idesc, 1u);
                    tc::mma_tf32(tm + 48, da, db, idesc, 1u);
                }
            }
            tc::commit(&bar);
            tc::mbar_wait(&bar, 0);
            cycles[0] = clock64() - t0;
            stop = 1;
        }
        __syncwarp();
    } else if (MODE > 0) {
        const uint32_t ta = tm + (uint32_t((warp & 3) * 32) << 16) + 256;
        float v[16];
        for (int i = 0; i < 16; i++) v[i] = float(i);
        float acc = 0.f;
        int it = 0;
        while (!stop) {
            if constexpr (MODE == 1 || MODE == 2) {
                for (int r = 0; r < 8; r++) {
                    if constexpr (MODE == 1) tc::tmem_st16(ta + r * 16, v); else tc::tmem_ld16(ta + r * 16, v);
                }
                if constexpr (MODE == 1) tc::tmem_wait_st(); else tc::tmem_wait_ld();
            } else if constexpr (MODE == 3) {
                for (int r = 0; r < 10; r++) tc::tmem_st16(ta + r * 16, v);
                for (int r = 0; r < 5; r++) tc::tmem_ld16(ta + 160 + r * 16, v);
                tc::tmem_wait_st();
                tc::tmem_wait_ld();
            } else if constexpr (MODE == 4) {
                const float4* sp = reinterpret_cast<const float4*>(smem);
                for (int r = 0; r < 16; r++) {
                    const float4 q = sp[(r * 256 + threadIdx.x) % 352];
                    acc += q.x + q.w;
                }
            } else {
                for (int r = 0; r < 16; r++) gbuf[(int64_t(it) * 16 + r) * 512 % (1 << 24) + threadIdx.x] = make_float2(acc, 1.f);
                it++;
            }
        }
        if (v[3] == 12345.f || acc == 12345.f) cycles[1] = 1;
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<512>(tm);
}

template <bool TS, int MODE>
void contention()
{
    long long* dc;
    cudaMalloc(&dc, 16);
    const int sm = (M + 48) * 8 * 4;
    cudaFuncSetAttribute(contention_kernel<TS, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    float2* gb;
    cudaMalloc(&gb, (size_t(1) << 24) * 8 + 4096 * 8);
    const int threads = MODE >= 3 ? 288 : 160;
    contention_kernel<TS, MODE><<<1, threads, sm>>>(4096, dc, gb);
    contention_kernel<TS, MODE><<<1, threads, sm>>>(4096, dc, gb);
    cudaError_t e = cudaDeviceSynchronize();
    long long c = 0;
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    printf("contention: N=48 A in %s, other warps %s: %.1f cycles per MMA (%s)\n", TS ? "TMEM" : "SMEM",
           MODE == 0 ? "idle" : MODE == 1 ? "tcgen05.st" : MODE == 2 ? "tcgen05.ld" : MODE == 3 ? "st+ld x8 warps" : MODE == 4 ? "LDS x8 warps" : "STG x8 warps", double(c) / 4096,
           e == cudaSuccess ? "ok" : cudaGetErrorString(e));
    cudaFree(dc);
}

// The band kernel's exact MMA sequence (r = 10): per level 2 units x 3 passes x 5 K steps, A in TMEM
// (hi slots at +0, lo at +80), B = 4 distinct 48 x 40 K-major tiles in smem.  VARIANT 0: as the band;
// 1: B always tile 0; 2: A always columns 0..7; 3: B tiles in SWIZZLE_NONE but N=48 rows padded to 64.
template <int VARIANT>
__global__ void bandseq_kernel(int reps, long long* cycles)
{
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    constexpr int NB = VARIANT == 3 ? 64 : 48, KU = 40;
    constexpr uint32_t WT = NB * KU * 4;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 4 * NB * KU; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.001f * (i % 97);
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
        constexpr uint32_t idesc = tc::idesc_tf32(128, NB);
        constexpr uint32_t LBO_B = (NB / 8) * 128;
        const uint64_t dW = tc::desc_kmajor(tc::smem_u32(smem), LBO_B);
        const long long t0 = clock64();
        for (int r = 0; r < reps; r++) {
#pragma unroll
            for (int u = 0; u < 2; u++) {
                const uint32_t d = tm + 160 + u * NB;
                const uint32_t ahi = tm + (VARIANT == 2 ? 0 : 2 * u * 20);
                const uint64_t bhi = tc::desc_add(dW, (VARIANT == 1 ? 0 : u * 2) * WT);
#pragma unroll
                for (int q = 0; q < 3; q++) {
                    const int pass = q == 0 ? 1 : q == 1 ? 2 : 0;
                    const uint32_t a = ahi + (pass == 1 && VARIANT != 2 ? 80 : 0);
                    const uint64_t b = pass == 2 && VARIANT != 1 ? tc::desc_add(bhi, WT) : bhi;
#pragma unroll
                    for (int ks = 0; ks < KU / 8; ks++)
                        mma_ts(d, a + (VARIANT == 2 ? 0 : ks * 8), tc::desc_add(b, ks * 2 * LBO_B), idesc, (q | ks) ? 1u : 0u);
                }
            }
        }
        tc::commit(&bar);
        tc::mbar_wait(&bar, 0);
        cycles[0] = clock64() - t0;
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<512>(tm);
}

template <int VARIANT>
void bandseq()
{
    long long* dc;
    cudaMalloc(&dc, 8);
    const int sm = 4 * 64 * 40 * 4;
    cudaFuncSetAttribute(bandseq_kernel<VARIANT>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    bandseq_kernel<VARIANT><<<1, 128, sm>>>(200, dc);
    bandseq_kernel<VARIANT><<<1, 128, sm>>>(200, dc);
    cudaError_t e = cudaDeviceSynchronize();
    long long c = 0;
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    printf("bandseq variant %d: %.1f cycles per MMA (%s)\n", VARIANT, double(c) / (200 * 30),
           e == cudaSuccess ? "ok" : cudaGetErrorString(e));
    cudaFree(dc);
}

// precision of a long 3xTF32 accumulation chain: D[128][32] = sum over S K-steps (K = 8 S) of random
// FP32 A B, one accumulator (seg = S) or fresh accumulators every `seg` steps summed in FP32 registers
constexpr int PN = 32;
__global__ void prec_kernel(const float* A, const float* Bt, float* D, int S, int seg)
{
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr int SP = 16;                    // stored steps (the K data repeats with period 8 SP)
    uint8_t* ah = smem;                       // [SP][128 x 8] canonical, step-major
    uint8_t* al = ah + SP * M * 8 * 4;
    uint8_t* bh = al + SP * M * 8 * 4;
    uint8_t* bl = bh + SP * PN * 8 * 4;
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int K = 8 * SP;
    for (int i = tid; i < M * K; i += blockDim.x) {
        const int r = i / K, k = i % K, st = k / 8;
        float h, l;
        tc::split(A[i], h, l);
        *reinterpret_cast<float*>(ah + st * M * 32 + tc::kmaj_off(r, k % 8, M)) = h;
        *reinterpret_cast<float*>(al + st * M * 32 + tc::kmaj_off(r, k % 8, M)) = l;
    }
    for (int i = tid; i < PN * K; i += blockDim.x) {
        const int r = i / K, k = i % K, st = k / 8;
        float h, l;
        tc::split(Bt[i], h, l);
        *reinterpret_cast<float*>(bh + st * PN * 32 + tc::kmaj_off(r, k % 8, PN)) = h;
        *reinterpret_cast<float*>(bl + st * PN * 32 + tc::kmaj_off(r, k % 8, PN)) = l;
    }
    if (warp == 0) tc::tmem_alloc<64>(&tbase);
    if (tid == 0) {
        tc::mbar_init(&bar, 1);
        tc::mbar_fence_init();
    }
    tc::fence_proxy_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = tbase;
    float acc[PN];
    for (int j = 0; j < PN; j++) acc[j] = 0.f;
    int phase = 0;
    for (int s0 = 0; s0 < S; s0 += seg) {
        if (tid == 0) {
            const uint32_t idesc = tc::idesc_tf32(M, PN);
            for (int st = s0; st < s0 + seg; st++)
                for (int pass = 0; pass < 3; pass++) {
                    const uint8_t* a = pass == 1 ? al : ah;
                    const uint8_t* b = pass == 2 ? bl : bh;
                    tc::mma_tf32(tm, tc::desc_kmajor(tc::smem_u32(a + (st % SP) * M * 32), (M / 8) * 128),
                                 tc::desc_kmajor(tc::smem_u32(b + (st % SP) * PN * 32), (PN / 8) * 128), idesc,
                                 (st > s0 || pass) ? 1u : 0u);
                }
            tc::commit(&bar);
        }
        tc::mbar_wait(&bar, phase);
        phase ^= 1;
        tc::fence_after_sync();
        for (int c0 = 0; c0 < PN; c0 += 8) {
            float v[8];
            tc::tmem_ld8(tm + (uint32_t(warp * 32) << 16) + c0, v);
            tc::tmem_wait_ld();
            for (int j = 0; j < 8; j++) acc[c0 + j] += v[j];
        }
        tc::fence_before_sync();
        __syncthreads();
        tc::fence_after_sync();
    }
    for (int j = 0; j < PN; j++) D[tid * PN + j] = acc[j];
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<64>(tm);
}

void prec(int S, int seg)
{
    const int K = 8 * S, KP = 128;   // device holds K period KP
    std::vector<float> Ap(M * KP), Btp(PN * KP), A(M * K), Bt(PN * K), D(M * PN);
    srand(11);
    for (auto& x : Ap) x = float(rand()) / RAND_MAX * 2 - 1;
    for (auto& x : Btp) x = float(rand()) / RAND_MAX * 2 - 1;
    for (int i = 0; i < M; i++)
        for (int k = 0; k < K; k++) A[i * K + k] = Ap[i * KP + k % KP];
    for (int i = 0; i < PN; i++)
        for (int k = 0; k < K; k++) Bt[i * K + k] = Btp[i * KP + k % KP];
    float *dA, *dB, *dD;
    cudaMalloc(&dA, Ap.size() * 4);
    cudaMalloc(&dB, Btp.size() * 4);
    cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, Ap.data(), Ap.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, Btp.data(), Btp.size() * 4, cudaMemcpyHostToDevice);
    const int sm = 2 * 16 * (M + PN) * 8 * 4;
    cudaFuncSetAttribute(prec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    prec_kernel<<<1, 128, sm>>>(dA, dB, dD, S, seg);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double num = 0, den = 0, num32 = 0;
    for (int i = 0; i < M; i++)
        for (int j = 0; j < PN; j++) {
            double ref = 0;
            float r32 = 0;
            for (int k = 0; k < K; k++) {
                ref += double(A[i * K + k]) * Bt[j * K + k];
                r32 = fmaf(A[i * K + k], Bt[j * K + k], r32);
            }
            num += (D[i * PN + j] - ref) * (D[i * PN + j] - ref);
            num32 += (r32 - ref) * (r32 - ref);
            den += ref * ref;
        }
    printf("prec K=%5d (S=%3d MMA steps x3) seg=%3d: 3xTF32 rel l2 %.2e   (sequential FP32 FFMA: %.2e) %s\n", K, S,
           seg, sqrt(num / den), sqrt(num32 / den), e == cudaSuccess ? "" : cudaGetErrorString(e));
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
}

template <int N>
int check(int mode)
{
    std::vector<float> A(M * K), Bt(N * K), D(M * N);
    srand(3 + mode);
    for (auto& x : A) x = float(rand() % 64 - 32) / 16.f;   // exactly representable in tf32
    for (auto& x : Bt) x = float(rand() % 64 - 32) / 16.f;
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, Bt.size() * 4);
    cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, Bt.data(), Bt.size() * 4, cudaMemcpyHostToDevice);
    const int sm = (M + N) * K * 4;
    cudaFuncSetAttribute(probe_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    probe_kernel<N><<<1, 128, sm>>>(dA, dB, dD, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("probe N=%d mode %d: CUDA error %s\n", N, mode, cudaGetErrorString(e));
        return 1;
    }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int i = 0; i < M; i++)
        for (int j = 0; j < N; j++) {
            double ref = 0;
            for (int k = 0; k < K; k++) ref += double(A[i * K + k]) * Bt[j * K + k];
            if (mode == 1) ref = -ref;
            maxerr = fmax(maxerr, fabs(D[i * N + j] - ref));
        }
    printf("probe N=%d mode %s: max abs err %.3e -> %s\n", N, mode == 0 ? "SS" : mode == 1 ? "SS negB" : "TS (A in TMEM)",
           maxerr, maxerr == 0 ? "EXACT" : "WRONG");
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
    return maxerr == 0 ? 0 : 1;
}

template <int N>
void rate(int ts)
{
    long long* dc;
    cudaMalloc(&dc, 8);
    const int sm = (M + N) * 8 * 4;
    cudaFuncSetAttribute(rate_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    const int iters = 4096;
    rate_kernel<N><<<1, 128, sm>>>(iters, ts, dc);
    rate_kernel<N><<<1, 128, sm>>>(iters, ts, dc);
    cudaError_t e = cudaDeviceSynchronize();
    long long c = 0;
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    const double per = double(c) / iters;
    printf("rate N=%3d A in %s: %.1f cycles per 128x%dx8 MMA -> %.0f MAC/clk/SM (%s)\n", N, ts ? "TMEM" : "SMEM", per,
           N, 128.0 * N * 8 / per, e == cudaSuccess ? "ok" : cudaGetErrorString(e));
    cudaFree(dc);
}

// How does kind::tf32 consume an FP32 operand: truncation or round-to-nearest of the low 13 bits?
// A = 1 + 3 2^-12 (0.75 tf32 ulp above 1), B = 1 (K = 8, one nonzero term): D = 1 (truncate) or 1 + 2^-10 (round).
__global__ void tf32_rounding_kernel(float* out)
{
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < (M + 32) * 8; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.f;
    __syncthreads();
    if (tid == 0) {
        *reinterpret_cast<float*>(smem + tc::kmaj_off(0, 0, M)) = 1.0f + 3.0f / 4096.0f;            // A[0][0]
        *reinterpret_cast<float*>(smem + M * 8 * 4 + tc::kmaj_off(0, 0, 32)) = 1.0f;                // B[0][0]
        *reinterpret_cast<float*>(smem + tc::kmaj_off(1, 0, M)) = -(1.0f + 3.0f / 4096.0f);         // A[1][0]
        *reinterpret_cast<float*>(smem + tc::kmaj_off(2, 0, M)) = 1.0f + 1.0f / 4096.0f;            // 0.25 ulp
    }
    if (warp == 0) tc::tmem_alloc<32>(&tbase);
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
        tc::mma_tf32(tm, tc::desc_kmajor(tc::smem_u32(smem), (M / 8) * 128),
                     tc::desc_kmajor(tc::smem_u32(smem + M * 8 * 4), (32 / 8) * 128), tc::idesc_tf32(M, 32), 0u);
        tc::commit(&bar);
    }
    tc::mbar_wait(&bar, 0);
    tc::fence_after_sync();
    float v[8];
    tc::tmem_ld8(tm + (uint32_t(warp * 32) << 16), v);
    tc::tmem_wait_ld();
    if (tid < 3) out[tid] = v[0];
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<32>(tm);
}

int main()
{
    int fails = 0;
    {
        float* d;
        cudaMalloc(&d, 16);
        cudaFuncSetAttribute(tf32_rounding_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (M + 32) * 32);
        tf32_rounding_kernel<<<1, 128, (M + 32) * 32>>>(d);
        float h[3] = {0, 0, 0};
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, 12, cudaMemcpyDeviceToHost);
        printf("tf32 operand conversion: 1+0.75ulp -> %.9g, -(1+0.75ulp) -> %.9g, 1+0.25ulp -> %.9g  => %s (%s)\n", h[0],
               h[1], h[2], h[0] == 1.0f ? "TRUNCATION" : (h[0] == 1.0f + 1.0f / 1024 ? "ROUND-TO-NEAREST" : "?"),
               e == cudaSuccess ? "ok" : cudaGetErrorString(e));
        cudaFree(d);
    }
    fails += check<48>(0);
    fails += check<48>(1);
    fails += check<48>(2);
    fails += check<160>(0);
    fails += check<256>(2);
    for (int ts = 0; ts < 2; ts++) {
        rate<32>(ts);
        rate<48>(ts);
        rate<80>(ts);
        rate<128>(ts);
        rate<160>(ts);
        rate<256>(ts);
    }
    rate_multi<32, 1>();
    rate_multi<32, 4>();
    rate_multi<64, 1>();
    rate_multi<64, 2>();
    rate_multi<64, 4>();
    rate_multi<128, 2>();
    rate_multi<128, 4>();
    rate_multi<256, 2>();
    rate_multi<48, 1, true>();
    rate_multi<48, 2, true>();
    rate_multi<64, 1, true>();
    rate_multi<128, 2, true>();
    rate_multi<48, 2>();
    bandseq<0>();
    bandseq<1>();
    bandseq<2>();
    bandseq<3>();
    contention<true, 0>();
    contention<true, 1>();
    contention<true, 2>();
    contention<false, 0>();
    contention<false, 1>();
    contention<false, 2>();
    contention<true, 3>();
    contention<true, 4>();
    contention<true, 5>();
    for (int S : {16, 64, 256}) {
        prec(S, S);
        prec(S, 4);
        prec(S, 1);
    }
    printf(fails ? "TC PROBE2: %d FAILED\n" : "TC PROBE2 OK\n", fails);
    return 0;
}
