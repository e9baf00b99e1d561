// bf_tc.cu -- tensor-core (tcgen05, 3xTF32) kernels of the IBF-MAT apply for large
// vector batches (north_star: "Use tensor cores only where nrhs makes a level a real
// dense contraction, and only if a 3xTF32 ... path keeps the error bound").
//
// Orientation: every stage is written as D[v][n] = sum_k A[v][k] B[n][k] with the
// M = 128 rows of the MMA the VECTORS of one tile (v = c n_amp + k), so that the
// accumulator row a thread reads back from TMEM (lane = v) is exactly one vector's
// output coefficients and is stored to the coefficient array delta[pair][t][v] with
// warp-coalesced 8-byte stores.  Complex products are real-embedded on the weight
// side:  A[v][2s + c] = (x_s).c,  B[2t + c'][2s + c] = [[Wr, -Wi], [Wi, Wr]](c', c),
// so D[v][2t + c'] = (W x)_t.c'.
//
// Leaf stages (S0, SL): the weights are used by every vector tile, so the plan expands
// them ONCE at finalization (expand_leaf_weights) into the exact shared-memory image the
// MMA reads -- real-embedded, split hi/lo, canonical K-major tiles -- and the kernels move
// them with 1-D bulk copies (TMA engine).  Activations are split hi/lo by SIMT warps.
//
// Measured on B200 (tools/tc_probe2.cu, profiles/r1_tc_probe2.txt): a kind::tf32 MMA
// (M=128, K=8) costs max(~45 clk, N/2 clk), so N >= 128 reaches 2048 MAC/clk/SM; and a
// long accumulation chain in TMEM loses precision (768 chained MMAs: 1.3e-5 relative,
// versus 3.7e-7 when the chain is cut every 12 MMAs and the partial sums are added in
// FP32 registers).  Hence N = 128 tiles, accumulation chains of <= 24 MMAs (at most 8 of them
// the large Ahi Bhi products, issued last) and FP32 register sums across chains here.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <algorithm>
#include <cstdint>

#include "bf_internal.h"
#include "bf_shard.h"
#include "tc_sm100.cuh"

namespace bfk {

namespace {

__device__ __forceinline__ float2 cmul_tc(const float2 a, const float2 b)
{
    return make_float2(fmaf(a.x, b.x, -(a.y * b.y)), fmaf(a.x, b.y, a.y * b.x));
}

__device__ __forceinline__ void st_f4(uint8_t* base, uint32_t off, float4 v) { *reinterpret_cast<float4*>(base + off) = v; }

template <int NCOLS>
__host__ __device__ constexpr int tmem_cols_pow2()
{
    return NCOLS <= 32 ? 32 : NCOLS <= 64 ? 64 : NCOLS <= 128 ? 128 : NCOLS <= 256 ? 256 : 512;
}

// 3xTF32 pass order of every accumulation chain: the two small correction products (Alo Bhi,
// Ahi Blo) first, while the accumulator is still small, then Ahi Bhi.  The tensor core's FP32
// accumulation truncates; its error grows with the number of large partial sums added, so the
// corrections-first order cuts the effective chain length to the Ahi Bhi steps.
__device__ constexpr int kPassOrder[3] = {1, 2, 0};

// real embedding of complex w for output part cp (0 = re, 1 = im) and input part c
__device__ __forceinline__ float embed(float2 w, int cp, int c)
{
    return cp == 0 ? (c == 0 ? w.x : -w.y) : (c == 0 ? w.y : w.x);
}

}  // namespace

// Tensor map of a coefficient array viewed as a 2-D FP32 tensor [rows][2 nv] (row = (pair, t), nv vectors of
// 8 bytes), box = 2 * 128 floats x box_rows rows: one TMA request moves a job's rows of one vector tile.
// The driver entry point is resolved once through the runtime (the library links no libcuda).
static cudaError_t make_rows_tmap(CUtensorMap* m, const float2* base, int64_t rows, int nv, int box_rows)
{
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return cudaErrorNotSupported;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t dims[2] = {cuuint64_t(2 * nv), cuuint64_t(rows)};
    const cuuint64_t strides[1] = {cuuint64_t(nv) * 8};
    const cuuint32_t box[2] = {256, cuuint32_t(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float2*>(base), dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// =============================================================================================
// Expanded leaf weights (plan finalization)
// =============================================================================================
// S0: per leaf b the B matrix has rows n = (a, t, c') (n0 2r of them) and K = (j, c) (2 n0).  It is
// stored as [leaf][n chunk of 128 rows][K chunk of 32][hi | lo][canonical K-major 128 x 32 tile].
constexpr int S0X_NC = 128, S0X_KC = 32;
constexpr int64_t S0X_TILE_FLOATS = int64_t(S0X_NC) * S0X_KC;

int64_t leafx_floats(const Dims& d) { return d.N * int64_t(2 * d.R) * int64_t(2 << d.l0) * 2; }

__global__ void expand_s0_kernel(const float2* __restrict__ V0, float* __restrict__ X, int LN, int l0, int R)
{
    const int n0 = 1 << l0;
    const int64_t nleaf = (int64_t(1) << LN) >> l0;
    const int rows = n0 * 2 * R, K = 2 * n0;
    const int nch = rows / S0X_NC, kch = K / S0X_KC;
    const int64_t total = nleaf * rows * int64_t(K);
    for (int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < total; g += int64_t(gridDim.x) * blockDim.x) {
        const int64_t b = g / (int64_t(rows) * K);
        const int rem = int(g - b * rows * K);
        const int n = rem / K, k = rem - n * K;
        const int a = n / (2 * R), t = (n / 2) % R, cp = n & 1, j = k >> 1, c = k & 1;
        const float2 w = V0[(int64_t(a) * nleaf + b) * (n0 * R) + int64_t(j) * R + t];
        float hi, lo;
        tc::split(embed(w, cp, c), hi, lo);
        const int nc = n / S0X_NC, kc = k / S0X_KC;
        float* tile = X + ((b * nch + nc) * kch + kc) * 2 * S0X_TILE_FLOATS;
        const uint32_t off = tc::kmaj_off(n % S0X_NC, k % S0X_KC, S0X_NC) / 4;
        tile[off] = hi;
        tile[S0X_TILE_FLOATS + off] = lo;
    }
}

// SL: per T_X leaf a the B matrix has rows n = (j, c') (2 n0) and K = (b, t, c) (n0 2r), stored as
// [leaf][K chunk of KP pairs][hi | lo][canonical K-major 2 n0 x KP 2r tile].
static int sl_kp(int R) { return R >= 12 ? 1 : 2; }

__global__ void expand_sl_kernel(const float2* __restrict__ U, float* __restrict__ X, int LN, int l0, int R, int KP)
{
    const int n0 = 1 << l0;
    const int64_t nleaf = (int64_t(1) << LN) >> l0;
    const int rows = 2 * n0, K = n0 * 2 * R, KC = KP * 2 * R;
    const int nch = n0 / KP;
    const int64_t tile = int64_t(rows) * KC;
    const int64_t total = nleaf * rows * int64_t(K);
    for (int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < total; g += int64_t(gridDim.x) * blockDim.x) {
        const int64_t a = g / (int64_t(rows) * K);
        const int rem = int(g - a * rows * K);
        const int n = rem / K, k = rem - n * K;
        const int j = n >> 1, cp = n & 1, b = k / (2 * R), t = (k / 2) % R, c = k & 1;
        const float2 w = U[(a * n0 + b) * (n0 * R) + int64_t(t) * n0 + j];
        float hi, lo;
        tc::split(embed(w, cp, c), hi, lo);
        const int ch = b / KP, kk = k - ch * KC;
        float* tl = X + ((a * nch + ch) * 2) * tile;
        const uint32_t off = tc::kmaj_off(n, kk, rows) / 4;
        tl[off] = hi;
        tl[tile + off] = lo;
    }
}

bool leaf_tc_shape(const Dims& d)
{
    const int n0 = 1 << d.l0;
    return (n0 == 32 || n0 == 64) && (d.R == 6 || d.R == 8 || d.R == 10 || d.R == 12 || d.R == 16) &&
           (d.n_amp == 1 || d.n_amp == 2 || d.n_amp == 4);
}

cudaError_t expand_leaf_weights(const Dims& d, const float2* V0, const float2* U, float* V0x, float* Ux, cudaStream_t s)
{
    if (!leaf_tc_shape(d)) return cudaErrorInvalidValue;
    const unsigned grid = 148 * 16;
    if (V0x) {
        expand_s0_kernel<<<grid, 256, 0, s>>>(V0, V0x, d.LN, d.l0, d.R);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    if (Ux) expand_sl_kernel<<<grid, 256, 0, s>>>(U, Ux, d.LN, d.l0, d.R, sl_kp(d.R));
    return cudaGetLastError();
}

// =============================================================================================
// S0 (eqn:1 P:698-702, amplitude pre-scale eqn:tg P:24-28) on the tensor cores, persistent.
// A job = one leaf b x one tile of 128 vectors (vector tile fastest, so the CTAs working at the same
// time share each leaf's weights in L2).  D[v][n] = sum_k A[v][k] B[n][k] with A = Y^T,
// Y[j][v] = b_k(x) F[x, c] (x = b n0 + j, K = 2 n0) split hi/lo into TMEM, and B = the expanded V0
// tiles of the leaf (n = (a, t, c'), swept in chunks of 128 = MMA N).  Each chunk is one accumulation
// chain over its K tiles of 32, each tile's passes ordered corrections first;
// a tile is released as soon as its passes are issued, so the ring streams KS + 1 tiles ahead.
// Warp roles:
//   warp 4 (one thread)  bulk-copies the job's F columns + b_k rows into a padded staging tile, and
//                        streams the weight tiles (ring),
//   warps 0-3            build A in TMEM (lane = vector) from the staging tile,
//   warp 5               issues the MMAs (elected lane) into one of two TMEM accumulators,
//   warps 6-13           epilogue: lane quarter = vectors, half the columns of a chunk each; store
//                        delta_l0[a N/n0 + b][t][v] (coalesced over v).
// =============================================================================================
static int sm_count()
{
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    }
    return n;
}

template <int R, int N0>
struct S0TC {
    static constexpr int K = 2 * N0;
    static constexpr int KS = K / S0X_KC;                 // 32-wide K tiles per chunk (2 or 4)
    static constexpr int NCH = N0 * 2 * R / S0X_NC;       // 128-row N chunks per job
    static constexpr int NSTAGE = KS + 1;                 // weight ring depth (32 KB tiles)
    static constexpr uint32_t TILE = S0X_TILE_FLOATS * 4;  // 16 KB
    static constexpr uint32_t STAGE = 2 * TILE;            // hi + lo
    // staging row stride (complex): padded (bank spread) where shared memory allows, else dense
    static constexpr int FS = (N0 == 64) ? N0 : N0 + 2;
    static constexpr uint32_t FBYTES = 128u * FS * 8;      // up to 128 F columns (n_amp = 1)
    static constexpr uint32_t OFF_F = NSTAGE * STAGE, OFF_BK = OFF_F + FBYTES;
    static constexpr size_t SMEM = size_t(OFF_BK) + 4 * N0 * 8;
    static constexpr int A_COLS = K;                       // hi at +0, lo at +K
    static constexpr int D_OFF = 2 * K;                    // two accumulators of 128 columns
    static constexpr int TMEM_COLS = tmem_cols_pow2<D_OFF + 2 * S0X_NC>();
    static_assert((N0 * 2 * R) % S0X_NC == 0 && KS >= 2, "tiling");
    static_assert(SMEM <= 232448 - 1024 && D_OFF + 2 * S0X_NC <= 512, "budget");
};

// CL = 2: clusters of two CTAs on the two halves of a leaf's vector tiles at the same time; each CTA bulk-copies
// one of the two 16 KB tiles (hi or lo) of every V0x stage and multicasts it to both (half the L2 -> SM
// traffic of the 1.3 MB-per-job weight stream); cluster-multicast MMA commits release a stage in both CTAs.
template <int R, int N0, int CL>
__global__ void __launch_bounds__(448, 1)
    s0_tc_kernel(const float2* __restrict__ F, int64_t ldf, const float2* __restrict__ ampb,
                 const float* __restrict__ V0x, float2* __restrict__ out, int LN, int n_amp, int nv, int nvt)
{
    using C = S0TC<R, N0>;
    extern __shared__ __align__(128) uint8_t sm_s0tc[];
    uint8_t* ring = sm_s0tc;
    float2* Fs = reinterpret_cast<float2*>(sm_s0tc + C::OFF_F);    // [column][FS]
    float2* Bk = reinterpret_cast<float2*>(sm_s0tc + C::OFF_BK);   // [k][N0] b_k(x)
    // A is built and released per 32-wide K tile (a_full / a_free per tile): the next job's split of tile kt
    // overlaps the current job's last chunk on tiles > kt (a single A buffer fills TMEM with the accumulators)
    __shared__ uint64_t full[C::NSTAGE], empty[C::NSTAGE], dfull[2], dempty[2], f_full, f_empty, a_full[4], a_free[4];
    __shared__ uint32_t tmem_base;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t N = int64_t(1) << LN;
    const int64_t nleaf = N / N0;
    const int cr = CL == 2 ? int(blockIdx.x & 1) : 0;
    const int64_t cid = CL == 2 ? int64_t(blockIdx.x >> 1) : int64_t(blockIdx.x);
    const int64_t ncl = CL == 2 ? int64_t(gridDim.x >> 1) : int64_t(gridDim.x);
    const int per = CL == 2 ? nvt / 2 : nvt;
    const int64_t njobs = (nleaf * per - cid + ncl - 1) / ncl;
    auto job_of = [&](int64_t jl, int64_t& b, int& v0) {   // job jl of this CTA -> (leaf b, first vector v0)
        const int64_t u = cid + jl * ncl;
        b = u / per;
        v0 = (CL == 2 ? int(u % per) * 2 + cr : int(u % per)) * 128;
    };

    if (warp == 0) tc::tmem_alloc<C::TMEM_COLS>(&tmem_base);
    if (tid == 0) {
        for (int i = 0; i < C::NSTAGE; i++) {
            tc::mbar_init(&full[i], 1);
            tc::mbar_init(&empty[i], CL);
        }
        for (int i = 0; i < 2; i++) {
            tc::mbar_init(&dfull[i], 1);
            tc::mbar_init(&dempty[i], 256);
        }
        tc::mbar_init(&f_full, 1);
        tc::mbar_init(&f_empty, 128);
        for (int i = 0; i < C::KS; i++) {
            tc::mbar_init(&a_full[i], 128);
            tc::mbar_init(&a_free[i], 1);
        }
        tc::mbar_fence_init();
    }
    tc::fence_before_sync();
    __syncthreads();
    if constexpr (CL == 2) tc::cluster_sync();
    tc::fence_after_sync();
    const uint32_t tmem = tmem_base;

    if (warp == 4) {
        // ---- loader: per job the F staging tile, and the weight ring (all jobs, in order).  The next job's F
        //      tile is issued a few weight tiles into the current job (as soon as the split has released the
        //      staging tile), so its latency hides behind the current job's MMAs ----
        if (lane == 0) {
            auto issue_f = [&](int64_t jl) {
                int64_t b;
                int v0;
                job_of(jl, b, v0);
                const int vw = min(128, nv - v0);
                const int c0 = v0 / n_amp, cw = (vw + n_amp - 1) / n_amp;
                if (jl > 0) tc::mbar_wait(&f_empty, uint32_t(jl - 1) & 1);
                tc::mbar_arrive_expect_tx(&f_full, uint32_t(cw) * N0 * 8 + uint32_t(n_amp) * N0 * 8);
                for (int cl = 0; cl < cw; cl++)
                    tc::bulk_g2s(Fs + cl * C::FS, F + b * N0 + int64_t(c0 + cl) * ldf, N0 * 8, &f_full);
                for (int k = 0; k < n_amp; k++) tc::bulk_g2s(Bk + k * N0, ampb + k * N + b * N0, N0 * 8, &f_full);
            };
            constexpr int WPJ = C::NCH * C::KS;                       // weight tiles per job
            constexpr int F_AT = C::NSTAGE < WPJ - 1 ? C::NSTAGE : WPJ - 1;
            if (njobs > 0) issue_f(0);
            int64_t it = 0;
            for (int64_t jl = 0; jl < njobs; jl++) {
                int64_t b;
                int v0j;
                job_of(jl, b, v0j);
                for (int w = 0; w < WPJ; w++, it++) {
                    const int st = int(it % C::NSTAGE);
                    if (it >= C::NSTAGE) tc::mbar_wait(&empty[st], uint32_t(it / C::NSTAGE - 1) & 1);
                    tc::mbar_arrive_expect_tx(&full[st], C::STAGE);   // both tiles land here
                    const float* src = V0x + (b * WPJ + w) * 2 * S0X_TILE_FLOATS;
                    if constexpr (CL == 2)
                        tc::bulk_g2s_mc(ring + st * C::STAGE + cr * C::TILE, src + cr * S0X_TILE_FLOATS, C::TILE,
                                        &full[st], uint16_t(3));
                    else
                        tc::bulk_g2s(ring + st * C::STAGE, src, C::STAGE, &full[st]);
                    if (w == F_AT && jl + 1 < njobs) issue_f(jl + 1);
                }
            }
        }
    } else if (warp < 4) {
        // ---- A = Y^T (hi, lo) into TMEM; thread = vector ----
        const int v = tid;
        const uint32_t lb = uint32_t(warp * 32) << 16;
        for (int64_t jl = 0; jl < njobs; jl++) {
            int64_t bj;
            int v0;
            job_of(jl, bj, v0);
            const int vg = v0 + v;
            const int c0 = v0 / n_amp;
            tc::mbar_wait(&f_full, uint32_t(jl & 1));
            const bool ok = vg < nv;
            const int cl = ok ? vg / n_amp - c0 : 0, k = ok ? vg % n_amp : 0;
            const float2* fc = Fs + cl * C::FS;
            const float2* bk = Bk + k * N0;
#pragma unroll 1
            for (int j0 = 0; j0 < N0; j0 += 8) {
                const int kt = j0 / (S0X_KC / 2);   // 32-wide K tile = 16 complex j
                if ((j0 % (S0X_KC / 2)) == 0) {
                    if (jl > 0) tc::mbar_wait(&a_free[kt], uint32_t(jl - 1) & 1);
                    tc::fence_after_sync();
                }
                float hi[16], lo[16];
#pragma unroll
                for (int jj = 0; jj < 8; jj += 2) {
                    const float4 f = *reinterpret_cast<const float4*>(fc + j0 + jj);
                    const float4 a = *reinterpret_cast<const float4*>(bk + j0 + jj);
                    float2 y0 = cmul_tc(make_float2(a.x, a.y), make_float2(f.x, f.y));
                    float2 y1 = cmul_tc(make_float2(a.z, a.w), make_float2(f.z, f.w));
                    if (!ok) y0 = y1 = make_float2(0.f, 0.f);
                    tc::split(y0.x, hi[2 * jj], lo[2 * jj]);
                    tc::split(y0.y, hi[2 * jj + 1], lo[2 * jj + 1]);
                    tc::split(y1.x, hi[2 * jj + 2], lo[2 * jj + 2]);
                    tc::split(y1.y, hi[2 * jj + 3], lo[2 * jj + 3]);
                }
                tc::tmem_st16(tmem + lb + uint32_t(2 * j0), hi);
                tc::tmem_st16(tmem + lb + uint32_t(C::A_COLS + 2 * j0), lo);
                if ((j0 + 8) % (S0X_KC / 2) == 0) {
                    tc::tmem_wait_st();
                    tc::fence_before_sync();
                    tc::mbar_arrive(&a_full[kt]);
                }
            }
            tc::mbar_arrive(&f_empty);   // the staging tile may be refilled for the next job
        }
    } else if (warp == 5) {
        // ---- MMA issuer (whole warp, one elected lane issues) ----
        constexpr uint32_t idesc = tc::idesc_tf32(128, S0X_NC);
        constexpr uint32_t LBO_B = (S0X_NC / 8) * 128;
        const uint64_t dB0 = tc::desc_kmajor(tc::smem_u32(ring), LBO_B);
        int64_t gc = 0;   // global chunk counter (accumulator slots alternate across jobs)
        for (int64_t jl = 0; jl < njobs; jl++) {
            for (int nc = 0; nc < C::NCH; nc++, gc++) {
                const int slot = int(gc & 1);
                if (gc >= 2) tc::mbar_wait(&dempty[slot], uint32_t((gc >> 1) - 1) & 1);
                const int64_t it0 = gc * C::KS;
                const uint32_t d = tmem + uint32_t(C::D_OFF + slot * S0X_NC);
                for (int ks = 0; ks < C::KS; ks++) {
                    const int st = int((it0 + ks) % C::NSTAGE);
                    if (nc == 0) tc::mbar_wait(&a_full[ks], uint32_t(jl & 1));
                    tc::mbar_wait(&full[st], uint32_t((it0 + ks) / C::NSTAGE) & 1);
                    tc::fence_after_sync();
#pragma unroll
                    for (int q = 0; q < 3; q++) {
                        const int pass = kPassOrder[q];
                        const uint64_t b = tc::desc_add(dB0, st * C::STAGE + (pass == 2 ? C::TILE : 0));
                        const uint32_t a = tmem + uint32_t((pass == 1 ? C::A_COLS : 0) + ks * S0X_KC);
#pragma unroll
                        for (int kk = 0; kk < S0X_KC / 8; kk++)
                            tc::mma_tf32_ts_warp(d, a + kk * 8, tc::desc_add(b, kk * 2 * LBO_B), idesc,
                                                 (q | ks | kk) ? 1u : 0u);
                    }
                    if constexpr (CL == 2)
                        tc::commit_mc_warp(&empty[st], uint16_t(3));   // free in both CTAs of the cluster
                    else
                        tc::commit_warp(&empty[st]);   // the tile is free once its 3 passes are done
                    if (nc == C::NCH - 1) tc::commit_warp(&a_free[ks]);   // A tile ks: last use in this job
                }
                tc::commit_warp(&dfull[slot]);
                __syncwarp();
            }
        }
    } else {
        // ---- epilogue (warps 6-13): lane quarter warp % 4 = vectors, column half (warp - 6) / 4; output rows
        //      advance incrementally (t, then pair a at stride nleaf R nv) ----
        const int q4 = warp & 3, cbase = ((warp - 6) >> 2) * 64;
        const int64_t strideA = nleaf * R * int64_t(nv), jumpA = strideA - int64_t(R) * nv;
        int64_t gc = 0;
        for (int64_t jl = 0; jl < njobs; jl++) {
            int64_t b;
            int v0;
            job_of(jl, b, v0);
            const int vg = v0 + q4 * 32 + lane;
            float2* const obase = out + b * R * int64_t(nv) + vg;
            for (int nc = 0; nc < C::NCH; nc++, gc++) {
                const int slot = int(gc & 1);
                tc::mbar_wait(&dfull[slot], uint32_t(gc >> 1) & 1);
                tc::fence_after_sync();
                const uint32_t taddr = tmem + (uint32_t(q4 * 32) << 16) + uint32_t(C::D_OFF + slot * S0X_NC + cbase);
                const int q0 = (nc * S0X_NC + cbase) >> 1;
                int t = q0 % R;
                float2* o = obase + int64_t(q0 / R) * strideA + int64_t(t) * nv;
#pragma unroll
                for (int c0 = 0; c0 < 64; c0 += 32) {
                    float x[32];
                    tc::tmem_ld16(taddr + c0, x);
                    tc::tmem_ld16(taddr + c0 + 16, x + 16);
                    tc::tmem_wait_ld();
                    if (c0 == 32) {
                        tc::fence_before_sync();
                        tc::mbar_arrive(&dempty[slot]);
                    }
#pragma unroll
                    for (int i = 0; i < 16; i++) {
                        if (vg < nv) *o = make_float2(x[2 * i], x[2 * i + 1]);
                        o += nv;
                        if (++t == R) {
                            t = 0;
                            o += jumpA;
                        }
                    }
                }
            }
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if constexpr (CL == 2) tc::cluster_sync();
    if (warp == 0) {
        tc::fence_after_sync();
        tc::tmem_dealloc<C::TMEM_COLS>(tmem);
    }
}

template <int R, int N0>
static cudaError_t s0_tc_go(const Dims& d, const float2* F, int64_t ldf, const float2* ampb, const float* V0x,
                            float2* out, int nv, cudaStream_t s, bool multicast)
{
    using C = S0TC<R, N0>;
    const int nvt = (nv + 127) / 128;
    const int64_t leaves = d.N / N0;
    cudaError_t e;
    if (multicast && nvt % 2 == 0 && sm_count() >= 2) {
        auto kern = s0_tc_kernel<R, N0, 2>;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
        if (e != cudaSuccess) return e;
        const int64_t ncl = std::min<int64_t>(leaves * (nvt / 2), sm_count() / 2);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(unsigned(2 * ncl));
        cfg.blockDim = dim3(448);
        cfg.dynamicSmemBytes = C::SMEM;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kern, F, ldf, ampb, V0x, out, d.LN, d.n_amp, nv, nvt);
    }
    auto kern = s0_tc_kernel<R, N0, 1>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
    if (e != cudaSuccess) return e;
    const int64_t jobs = leaves * nvt;
    const unsigned grid = unsigned(jobs < sm_count() ? jobs : sm_count());
    kern<<<grid, 448, C::SMEM, s>>>(F, ldf, ampb, V0x, out, d.LN, d.n_amp, nv, nvt);
    return cudaGetLastError();
}

bool s0_tc_supported(const Dims& d, int nv, int64_t ldf) { return leaf_tc_shape(d) && nv >= 64 && (ldf % 2) == 0; }

cudaError_t launch_s0_tc(const Dims& d, const float2* F, int64_t ldf, const float2* ampb, const float* V0x, float2* out,
                         int nv, cudaStream_t s, bool multicast)
{
    const int n0 = 1 << d.l0;
#define S0TC_CASE(RR)                                                                                      \
    if (d.R == RR)                                                                                         \
        return n0 == 64 ? s0_tc_go<RR, 64>(d, F, ldf, ampb, V0x, out, nv, s, multicast)                               \
                        : s0_tc_go<RR, 32>(d, F, ldf, ampb, V0x, out, nv, s, multicast);
    S0TC_CASE(6) S0TC_CASE(8) S0TC_CASE(10) S0TC_CASE(12) S0TC_CASE(16)
#undef S0TC_CASE
    return cudaErrorInvalidValue;
}


// =============================================================================================
// S0 in FP16 passes (BF_OPT_LEAF_F16 = 1, the default).  Same job structure as s0_tc_kernel, but every
// operand is split into FP16 hi + lo after a power-of-two scaling that brings each A row (one vector's
// b_k F values of the leaf) and each B row (one output coefficient's V0 row) to max |x| in [0.5, 1):
// hi = fp16(x), lo = fp16(x - hi), and D = Ahi Bhi + Alo Bhi + Ahi Blo accumulates in FP32 with
// kind::f16 MMAs (K = 16 per instruction: twice the MAC rate of kind::tf32, tools/tc_probe_f16.cu).
// The hi parts carry 11 significant bits like TF32, and the scaling keeps every value of interest in
// FP16's normal range, so the product error matches the 3xTF32 split (measured model in the probe);
// values below 2^-14 of their row's maximum go subnormal with an absolute error <= 2^-25 of that
// maximum.  The epilogue multiplies by 2^{e_v} 2^{f_n}.  The weight image is half the bytes of the TF32
// image (plus one FP32 scale per row).
// =============================================================================================
constexpr uint32_t S0H_TILE = uint32_t(S0X_NC) * S0X_KC * 2;   // one 128 x 32 FP16 tile (8 KB)

int64_t leafh_rows(const Dims& d) { return d.N * int64_t(d.R); }   // biased exponents, one per complex output row

__global__ void expand_s0_h16_kernel(const float2* __restrict__ V0, __half* __restrict__ X, uint8_t* __restrict__ S,
                                     int LN, int l0, int R)
{
    const int n0 = 1 << l0;
    const int64_t nleaf = (int64_t(1) << LN) >> l0;
    const int rows = n0 * 2 * R, K = 2 * n0, cq = n0 * R;
    const int nch = rows / S0X_NC, kch = K / S0X_KC;
    const int64_t total = nleaf * cq;
    for (int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < total; g += int64_t(gridDim.x) * blockDim.x) {
        const int64_t b = g / cq;
        const int q = int(g - b * cq);                 // complex output row q = a R + t: real rows 2q, 2q + 1
        const int a = q / R, t = q - a * R;
        const float2* w = V0 + (int64_t(a) * nleaf + b) * (n0 * R) + t;   // w[j R]
        float mx = 0.f;
        for (int j = 0; j < n0; j++) mx = fmaxf(mx, fmaxf(fabsf(w[j * R].x), fabsf(w[j * R].y)));
        int e = 0;
        frexpf(mx, &e);                                // mx 2^-e in [0.5, 1)
        e = max(-126, min(126, e));
        S[b * cq + q] = uint8_t(e + 127);              // biased: the epilogue multiplies by 2^e
        for (int cp = 0; cp < 2; cp++) {
            const int n = 2 * q + cp, nc = n / S0X_NC;
            for (int k = 0; k < K; k++) {
                const float x = ldexpf(embed(w[(k >> 1) * R], cp, k & 1), -e);
                float hi, lo;
                tc::split_h(x, hi, lo);
                const int kc = k / S0X_KC;
                __half* tile = X + ((b * nch + nc) * kch + kc) * 2 * int64_t(S0X_NC * S0X_KC);
                const uint32_t off = tc::kmaj_off16(n % S0X_NC, k % S0X_KC, S0X_NC) / 2;
                tile[off] = __float2half_rn(hi);
                tile[S0X_NC * S0X_KC + off] = __float2half_rn(lo);
            }
        }
    }
}

template <int R, int N0>
struct S0H {
    static constexpr int K = 2 * N0;
    static constexpr int KS = K / S0X_KC;
    static constexpr int NCH = N0 * 2 * R / S0X_NC;
    static constexpr int NSTAGE = 2 * KS;                  // weight ring depth (16 KB stages)
    static constexpr uint32_t STAGE = 2 * S0H_TILE;        // hi + lo
    static constexpr int FS = N0 + 2;                      // padded staging rows (16-byte aligned, bank spread)
    static constexpr uint32_t FBYTES = 128u * FS * 8;
    static constexpr uint32_t OFF_F = NSTAGE * STAGE, OFF_BK = OFF_F + FBYTES, OFF_E = OFF_BK + 4 * N0 * 8;
    static constexpr size_t SMEM = size_t(OFF_E) + 4 * 128 * 4;
    static constexpr int A_COLS = K / 2;                   // packed FP16 pairs: hi at +0, lo at +A_COLS
    static constexpr int A_BUF = 2 * A_COLS;               // two A buffers (the split fills job j + 1 while
    static constexpr int D_OFF = 2 * A_BUF;                //   the tensor pipe runs job j)
    static constexpr int TMEM_COLS = tmem_cols_pow2<D_OFF + 2 * S0X_NC>();
    static_assert((N0 * 2 * R) % S0X_NC == 0 && KS >= 2, "tiling");
    static_assert(SMEM <= 232448 - 1024 && D_OFF + 2 * S0X_NC <= 512, "budget");
};

template <int R, int N0>
__global__ void __launch_bounds__(448, 1)
    s0_h16_kernel(const float2* __restrict__ F, int64_t ldf, const float2* __restrict__ ampb,
                  const __half* __restrict__ V0h, const uint8_t* __restrict__ V0s, float2* __restrict__ out, int LN,
                  int n_amp, int nv, int nvt)
{
    using C = S0H<R, N0>;
    extern __shared__ __align__(128) uint8_t sm_s0h[];
    uint8_t* ring = sm_s0h;
    float2* Fs = reinterpret_cast<float2*>(sm_s0h + C::OFF_F);    // [column][FS]
    float2* Bk = reinterpret_cast<float2*>(sm_s0h + C::OFF_BK);   // [k][N0] b_k(x)
    float* Es = reinterpret_cast<float*>(sm_s0h + C::OFF_E);       // [job % 4][128] 2^{e_v}
    __shared__ uint64_t full[C::NSTAGE], empty[C::NSTAGE], dfull[2], dempty[2], f_full, f_empty, a_full[2], a_free[2];
    __shared__ uint64_t e_full[4], e_empty[4];
    __shared__ uint32_t tmem_base;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t N = int64_t(1) << LN;
    const int64_t nleaf = N / N0;
    const int64_t njobs_all = nleaf * nvt;
    const int64_t njobs = (njobs_all - blockIdx.x + gridDim.x - 1) / gridDim.x;

    if (warp == 0) tc::tmem_alloc<C::TMEM_COLS>(&tmem_base);
    if (tid == 0) {
        for (int i = 0; i < C::NSTAGE; i++) {
            tc::mbar_init(&full[i], 1);
            tc::mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; i++) {
            tc::mbar_init(&dfull[i], 1);
            tc::mbar_init(&dempty[i], 256);
        }
        for (int i = 0; i < 4; i++) {
            tc::mbar_init(&e_full[i], 128);
            tc::mbar_init(&e_empty[i], 256);
        }
        tc::mbar_init(&f_full, 1);
        tc::mbar_init(&f_empty, 128);
        for (int i = 0; i < 2; i++) {
            tc::mbar_init(&a_full[i], 128);
            tc::mbar_init(&a_free[i], 1);
        }
        tc::mbar_fence_init();
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tmem_base;

    if (warp == 4) {
        // ---- loader: per job the F staging tile, and the weight ring (all jobs, in order).  The next job's F
        //      tile is issued a few weight tiles into the current job (as soon as the split has released the
        //      staging tile), so its latency hides behind the current job's MMAs ----
        if (lane == 0) {
            auto issue_f = [&](int64_t jl) {
                const unsigned job = unsigned(blockIdx.x + jl * gridDim.x);
                const int64_t b = job / unsigned(nvt);
                const int v0 = int(job % unsigned(nvt)) * 128, vw = min(128, nv - v0);
                const int c0 = v0 / n_amp, cw = (vw + n_amp - 1) / n_amp;
                if (jl > 0) tc::mbar_wait(&f_empty, uint32_t(jl - 1) & 1);
                tc::mbar_arrive_expect_tx(&f_full, uint32_t(cw) * N0 * 8 + uint32_t(n_amp) * N0 * 8);
                for (int cl = 0; cl < cw; cl++)
                    tc::bulk_g2s(Fs + cl * C::FS, F + b * N0 + int64_t(c0 + cl) * ldf, N0 * 8, &f_full);
                for (int k = 0; k < n_amp; k++) tc::bulk_g2s(Bk + k * N0, ampb + k * N + b * N0, N0 * 8, &f_full);
            };
            constexpr int WPJ = C::NCH * C::KS;                       // weight tiles per job
            constexpr int F_AT = C::NSTAGE < WPJ - 1 ? C::NSTAGE : WPJ - 1;
            if (njobs > 0) issue_f(0);
            int64_t it = 0;
            for (int64_t jl = 0; jl < njobs; jl++) {
                const int64_t b = unsigned(blockIdx.x + jl * gridDim.x) / unsigned(nvt);
                for (int w = 0; w < WPJ; w++, it++) {
                    const int st = int(it % C::NSTAGE);
                    if (it >= C::NSTAGE) tc::mbar_wait(&empty[st], uint32_t(it / C::NSTAGE - 1) & 1);
                    tc::mbar_arrive_expect_tx(&full[st], C::STAGE);
                    tc::bulk_g2s(ring + st * C::STAGE, V0h + (b * WPJ + w) * 2 * (S0X_NC * S0X_KC), C::STAGE, &full[st]);
                    if (w == F_AT && jl + 1 < njobs) issue_f(jl + 1);
                }
            }
        }
    } else if (warp < 4) {
        // ---- A = Y^T scaled by 2^{-e_v}, FP16 hi / lo packed into TMEM; thread = vector ----
        const int v = tid;
        const uint32_t lb = uint32_t(warp * 32) << 16;
        for (int64_t jl = 0; jl < njobs; jl++) {
            const unsigned job = unsigned(blockIdx.x + jl * gridDim.x);
            const int v0 = int(job % unsigned(nvt)) * 128, vg = v0 + v;
            const int c0 = v0 / n_amp;
            const int eb = int(jl & 3), ab = int(jl & 1);
            tc::mbar_wait(&f_full, uint32_t(jl & 1));
            if (jl >= 2) tc::mbar_wait(&a_free[ab], uint32_t((jl >> 1) - 1) & 1);
            if (jl >= 4) tc::mbar_wait(&e_empty[eb], uint32_t((jl >> 2) - 1) & 1);
            tc::fence_after_sync();
            const bool ok = vg < nv;
            const int cl = ok ? vg / n_amp - c0 : 0, k = ok ? vg % n_amp : 0;
            const float2* fc = Fs + cl * C::FS;
            const float2* bk = Bk + k * N0;
            float mx = 0.f;
#pragma unroll 4
            for (int j = 0; j < N0; j += 2) {
                const float4 f = *reinterpret_cast<const float4*>(fc + j);
                const float4 a = *reinterpret_cast<const float4*>(bk + j);
                const float2 y0 = cmul_tc(make_float2(a.x, a.y), make_float2(f.x, f.y));
                const float2 y1 = cmul_tc(make_float2(a.z, a.w), make_float2(f.z, f.w));
                mx = fmaxf(mx, fmaxf(fmaxf(fabsf(y0.x), fabsf(y0.y)), fmaxf(fabsf(y1.x), fabsf(y1.y))));
            }
            int e = 0;
            frexpf(ok ? mx : 0.f, &e);
            e = max(-126, min(126, e));
            const float sc = ldexpf(1.f, -e);
            Es[eb * 128 + v] = ldexpf(1.f, e);
            tc::mbar_arrive(&e_full[eb]);
#pragma unroll 1
            for (int j0 = 0; j0 < N0; j0 += 8) {
                float hi[8], lo[8];
#pragma unroll
                for (int jj = 0; jj < 8; jj += 2) {
                    const float4 f = *reinterpret_cast<const float4*>(fc + j0 + jj);
                    const float4 a = *reinterpret_cast<const float4*>(bk + j0 + jj);
                    float2 y[2] = {cmul_tc(make_float2(a.x, a.y), make_float2(f.x, f.y)),
                                   cmul_tc(make_float2(a.z, a.w), make_float2(f.z, f.w))};
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        if (!ok) y[h] = make_float2(0.f, 0.f);
                        // column j = (re, im) of complex j: K index 2j, 2j + 1
                        tc::split_h2(y[h].x * sc, y[h].y * sc, hi[jj + h], lo[jj + h]);
                    }
                }
                tc::tmem_st8(tmem + lb + uint32_t(ab * C::A_BUF + j0), hi);
                tc::tmem_st8(tmem + lb + uint32_t(ab * C::A_BUF + C::A_COLS + j0), lo);
            }
            tc::fence_before_sync();
            tc::mbar_arrive(&f_empty);
            tc::tmem_wait_st();
            tc::fence_before_sync();
            tc::mbar_arrive(&a_full[ab]);
        }
    } else if (warp == 5) {
        // ---- MMA issuer: per 32-wide K tile 3 passes x 2 kind::f16 MMAs (K = 16) ----
        constexpr uint32_t idesc = tc::idesc_f16(128, S0X_NC);
        constexpr uint32_t LBO_B = (S0X_NC / 8) * 128;
        const uint64_t dB0 = tc::desc_kmajor(tc::smem_u32(ring), LBO_B);
        int64_t gc = 0;
        for (int64_t jl = 0; jl < njobs; jl++) {
            const int ab = int(jl & 1);
            tc::mbar_wait(&a_full[ab], uint32_t(jl >> 1) & 1);
            tc::fence_after_sync();
            for (int nc = 0; nc < C::NCH; nc++, gc++) {
                const int slot = int(gc & 1);
                if (gc >= 2) tc::mbar_wait(&dempty[slot], uint32_t((gc >> 1) - 1) & 1);
                const int64_t it0 = gc * C::KS;
                const uint32_t d = tmem + uint32_t(C::D_OFF + slot * S0X_NC);
                for (int ks = 0; ks < C::KS; ks++) {
                    const int st = int((it0 + ks) % C::NSTAGE);
                    tc::mbar_wait(&full[st], uint32_t((it0 + ks) / C::NSTAGE) & 1);
                    tc::fence_after_sync();
#pragma unroll
                    for (int q = 0; q < 3; q++) {
                        const int pass = kPassOrder[q];
                        const uint64_t b = tc::desc_add(dB0, st * C::STAGE + (pass == 2 ? S0H_TILE : 0));
                        const uint32_t a = tmem + uint32_t(ab * C::A_BUF + (pass == 1 ? C::A_COLS : 0) + ks * (S0X_KC / 2));
#pragma unroll
                        for (int kk = 0; kk < S0X_KC / 16; kk++)
                            tc::mma_f16_ts_warp(d, a + kk * 8, tc::desc_add(b, kk * 2 * LBO_B), idesc,
                                                (q | ks | kk) ? 1u : 0u);
                    }
                    tc::commit_warp(&empty[st]);
                }
                tc::commit_warp(&dfull[slot]);
                __syncwarp();
            }
            tc::commit_warp(&a_free[ab]);
            __syncwarp();
        }
    } else {
        // ---- epilogue (warps 6-13): lane quarter warp % 4 = vectors, column half (warp - 6) / 4.  Output rows
        //      advance incrementally (t, then pair a at stride nleaf R nv); 2^{e_v + e_q} per complex row ----
        const int q4 = warp & 3, cbase = ((warp - 6) >> 2) * 64;
        constexpr int CQ = N0 * R;                                // complex output rows per leaf
        const int64_t strideA = nleaf * R * int64_t(nv), jumpA = strideA - int64_t(R) * nv;
        int64_t gc = 0;
        for (int64_t jl = 0; jl < njobs; jl++) {
            const unsigned job = unsigned(blockIdx.x + jl * gridDim.x);
            const int64_t b = job / unsigned(nvt);
            const int vg = int(job % unsigned(nvt)) * 128 + q4 * 32 + lane;
            const int eb = int(jl & 3);
            tc::mbar_wait(&e_full[eb], uint32_t(jl >> 2) & 1);
            const float sv = Es[eb * 128 + q4 * 32 + lane];
            tc::mbar_arrive(&e_empty[eb]);
            const uint8_t* Sb = V0s + b * CQ + (cbase >> 1);
            float2* const obase = out + b * R * int64_t(nv) + vg;
            uint4 ex[2];   // the biased exponents of this thread's 32 complex rows of the chunk (one chunk ahead)
            ex[0] = __ldg(reinterpret_cast<const uint4*>(Sb));
            ex[1] = __ldg(reinterpret_cast<const uint4*>(Sb) + 1);
            for (int nc = 0; nc < C::NCH; nc++, gc++) {
                const int slot = int(gc & 1);
                uint4 exn[2] = {ex[0], ex[1]};
                if (nc + 1 < C::NCH) {
                    exn[0] = __ldg(reinterpret_cast<const uint4*>(Sb + (nc + 1) * (S0X_NC / 2)));
                    exn[1] = __ldg(reinterpret_cast<const uint4*>(Sb + (nc + 1) * (S0X_NC / 2)) + 1);
                }
                tc::mbar_wait(&dfull[slot], uint32_t(gc >> 1) & 1);
                tc::fence_after_sync();
                const uint32_t taddr = tmem + (uint32_t(q4 * 32) << 16) + uint32_t(C::D_OFF + slot * S0X_NC + cbase);
                const int q0 = (nc * S0X_NC + cbase) >> 1;
                int t = q0 % R;
                float2* o = obase + int64_t(q0 / R) * strideA + int64_t(t) * nv;
#pragma unroll
                for (int c0 = 0; c0 < 64; c0 += 32) {
                    float x[32];
                    tc::tmem_ld16(taddr + c0, x);
                    tc::tmem_ld16(taddr + c0 + 16, x + 16);
                    tc::tmem_wait_ld();
                    if (c0 == 32) {
                        tc::fence_before_sync();
                        tc::mbar_arrive(&dempty[slot]);
                    }
                    const uint32_t* ew = reinterpret_cast<const uint32_t*>(&ex[c0 >> 5]);
#pragma unroll
                    for (int i = 0; i < 16; i++) {
                        const uint32_t be = (ew[i >> 2] >> (8 * (i & 3))) & 0xffu;
                        const float s2 = sv * __uint_as_float(be << 23);
                        if (vg < nv) *o = make_float2(x[2 * i] * s2, x[2 * i + 1] * s2);
                        o += nv;
                        if (++t == R) {
                            t = 0;
                            o += jumpA;
                        }
                    }
                }
                ex[0] = exn[0];
                ex[1] = exn[1];
            }
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) {
        tc::fence_after_sync();
        tc::tmem_dealloc<C::TMEM_COLS>(tmem);
    }
}

template <int R, int N0>
static cudaError_t s0_h16_go(const Dims& d, const float2* F, int64_t ldf, const float2* ampb, const __half* V0h,
                             const uint8_t* V0s, float2* out, int nv, cudaStream_t s)
{
    using C = S0H<R, N0>;
    auto kern = s0_h16_kernel<R, N0>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
    if (e != cudaSuccess) return e;
    const int nvt = (nv + 127) / 128;
    const int64_t jobs = (d.N / N0) * nvt;
    const unsigned grid = unsigned(jobs < sm_count() ? jobs : sm_count());
    kern<<<grid, 448, C::SMEM, s>>>(F, ldf, ampb, V0h, V0s, out, d.LN, d.n_amp, nv, nvt);
    return cudaGetLastError();
}

cudaError_t expand_s0_h16(const Dims& d, const float2* V0, void* V0h, void* V0s, cudaStream_t s)
{
    if (!leaf_tc_shape(d)) return cudaErrorInvalidValue;
    expand_s0_h16_kernel<<<148 * 16, 128, 0, s>>>(V0, static_cast<__half*>(V0h), static_cast<uint8_t*>(V0s), d.LN,
                                                  d.l0, d.R);
    return cudaGetLastError();
}

cudaError_t launch_s0_h16(const Dims& d, const float2* F, int64_t ldf, const float2* ampb, const void* V0h,
                          const void* V0s, float2* out, int nv, cudaStream_t s)
{
    const int n0 = 1 << d.l0;
    const __half* X = static_cast<const __half*>(V0h);
    const uint8_t* E8 = static_cast<const uint8_t*>(V0s);
#define S0H_CASE(RR)                                                                                       \
    if (d.R == RR)                                                                                         \
        return n0 == 64 ? s0_h16_go<RR, 64>(d, F, ldf, ampb, X, E8, out, nv, s)                            \
                        : s0_h16_go<RR, 32>(d, F, ldf, ampb, X, E8, out, nv, s);
    S0H_CASE(6) S0H_CASE(8) S0H_CASE(10) S0H_CASE(12) S0H_CASE(16)
#undef S0H_CASE
    return cudaErrorInvalidValue;
}

// =============================================================================================
// SL (eqn:bf3 P:791-797, amplitude post-scale and sum over k eqn:tg P:24-28) on the tensor cores,
// persistent.  A job = one T_X leaf a x one tile of 128 vectors (vector tile fastest).
// D[v][2j + c'] = sum over K = (b, t, c) of A[v][(b, t, c)] B[(j, c')][(b, t, c)], A = delta_D[a n0 + b][t][v]
// split hi/lo, B = the expanded U tiles of the leaf.  K streams in chunks of KP pairs, continuously across
// the CTA's jobs:
//   warp 12 (one thread)  bulk-copies the raw delta rows and the B tile of a chunk (NR-deep rings),
//   warps 0-3             split a raw chunk into one of two A stages in TMEM (lane = vector; the
//                         MMAs read A from TMEM, so shared memory carries only B),
//   warp 13               issues the 3 KC/8 MMAs of a chunk (elected lane); every SEG chunks it switches
//                         between two TMEM accumulators (short chains),
//   warps 4-11            drain each finished segment into FP32 registers (lane quarter = vectors, half
//                         the columns each); at the end of a job apply a_k, sum over k by lane shuffles
//                         and write G through a dedicated shared-memory transpose buffer, while the
//                         other roles already stream the next job.
// =============================================================================================
template <int R, int N0, int NA, int KP>
struct SLTC {
    static constexpr int NB = 2 * N0;
    static constexpr int KC = KP * 2 * R;
    static constexpr int NCH = N0 / KP;
#ifdef BF_SL_SEG
    static constexpr int SEG = BF_SL_SEG;                        // chunks per accumulation segment
#else
    static constexpr int SEG = 2;                                // chunks per accumulation segment
#endif
    static constexpr int NSEG = (NCH + SEG - 1) / SEG;
    static constexpr uint32_t RAW = uint32_t(KP) * R * 128 * 8;
    static constexpr uint32_t BT = uint32_t(NB) * KC * 4;   // one of hi / lo
    static constexpr uint32_t GS_STRIDE = N0 + 1;
    static constexpr uint32_t GS_BYTES = uint32_t(128 / NA) * GS_STRIDE * 8;
    static constexpr uint32_t AS_BYTES = uint32_t(NA) * N0 * 8;
    // separate rings: the coefficient rows come from DRAM (deep ring), the Ux tiles mostly from L2 (2 deep)
    static constexpr int NB_R = 3;                                   // Ux ring depth
    static constexpr int NR_FIT = int((232448 - 1024 - GS_BYTES - AS_BYTES - NB_R * 2 * BT) / RAW);
    static constexpr int NR = NR_FIT > 8 ? 8 : NR_FIT;               // raw ring depth
    static constexpr uint32_t OFF_B = NR * RAW, OFF_GS = OFF_B + 2 * NB_R * BT, OFF_AS = OFF_GS + GS_BYTES;
    static constexpr size_t SMEM = size_t(OFF_AS) + AS_BYTES;
    // TMEM: two A stages (hi KC columns, then lo KC columns) and two accumulators of NB columns
    static constexpr int A_COLS = 2 * KC, D_OFF = 2 * A_COLS;
    static constexpr int TMEM_COLS = tmem_cols_pow2<D_OFF + 2 * NB>();
    static_assert(KC % 8 == 0, "K chunk must be whole MMA K steps");
    static_assert(D_OFF + 2 * NB <= 512, "TMEM budget");
    static_assert(SMEM <= 232448 - 1024 && NR >= 2, "shared memory budget");
};

// CL = 2: launched as clusters of two CTAs that work on the two halves of a leaf's vector tiles at the same
// time; each CTA bulk-copies half of every Ux stage and multicasts it to both (half the L2 -> SM traffic of
// the 1.3 MB-per-job Ux stream), and a stage is refilled only after both CTAs' MMAs released it.
template <int R, int N0, int NA, int KP, int CL>
__global__ void __launch_bounds__(448, 1)
    sl_tc_kernel(const __grid_constant__ CUtensorMap tin, const float* __restrict__ Ux, const float2* __restrict__ ampa,
                 float2* __restrict__ G, int64_t ldg, int LN, int nv, int nvt)
{
    using C = SLTC<R, N0, NA, KP>;
    extern __shared__ __align__(128) uint8_t sm_sltc[];
    auto raw = [&](int e) { return sm_sltc + e * C::RAW; };
    auto opB = [&](int e, int lo) { return sm_sltc + C::OFF_B + (2 * e + lo) * C::BT; };
    float2* Gs = reinterpret_cast<float2*>(sm_sltc + C::OFF_GS);   // [128/NA][GS_STRIDE]
    float2* As = reinterpret_cast<float2*>(sm_sltc + C::OFF_AS);   // [NA][N0] a_k(x) of the current job
    __shared__ uint64_t raw_full[C::NR], raw_empty[C::NR], b_full[C::NB_R], b_empty[C::NB_R], a_full[2], a_empty[2],
        dfull[2], dempty[2];
    __shared__ uint32_t tmem_base;
    constexpr int TMEM_COLS = C::TMEM_COLS;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t N = int64_t(1) << LN;
    // job jl of this CTA -> (leaf a, first vector v0)
    const int cr = CL == 2 ? int(blockIdx.x & 1) : 0;
    const int64_t cid = CL == 2 ? int64_t(blockIdx.x >> 1) : int64_t(blockIdx.x);
    const int64_t ncl = CL == 2 ? int64_t(gridDim.x >> 1) : int64_t(gridDim.x);
    const int per = CL == 2 ? nvt / 2 : nvt;                 // units per leaf: vector tiles or tile pairs
    const int64_t units = (N / N0) * per;
    const int njobs = int((units - cid + ncl - 1) / ncl);
    auto job_of = [&](int jl, int64_t& a, int& v0) {
        const int64_t u = cid + int64_t(jl) * ncl;
        a = u / per;
        v0 = (CL == 2 ? int(u % per) * 2 + cr : int(u % per)) * 128;
    };
    const int nch_all = njobs * C::NCH;

    if (warp == 0) tc::tmem_alloc<TMEM_COLS>(&tmem_base);
    if (tid == 0) {
        for (int i = 0; i < C::NR; i++) {
            tc::mbar_init(&raw_full[i], 1);
            tc::mbar_init(&raw_empty[i], 128);
        }
        for (int i = 0; i < C::NB_R; i++) {
            tc::mbar_init(&b_full[i], 1);
            tc::mbar_init(&b_empty[i], CL);   // released by the MMA commit of every CTA of the cluster
        }
        for (int i = 0; i < 2; i++) {
            tc::mbar_init(&a_full[i], 128);
            tc::mbar_init(&a_empty[i], 1);
            tc::mbar_init(&dfull[i], 1);
            tc::mbar_init(&dempty[i], 256);
        }
        tc::mbar_fence_init();
    }
    tc::fence_before_sync();
    __syncthreads();
    if constexpr (CL == 2) tc::cluster_sync();   // both CTAs' barriers exist before any multicast
    tc::fence_after_sync();
    const uint32_t tmem = tmem_base;

    if (warp == 12) {
        // ---- loaders: lane 0 streams the coefficient rows (2-D TMA, deep ring), lane 1 the Ux tiles (bulk
        //      copies, 2-deep ring); the two streams only meet in the MMA ----
        if (lane == 0) {
            for (int gch = 0; gch < nch_all; gch++) {
                const int jl = gch / C::NCH, ch = gch - jl * C::NCH;
                int64_t a;
                int v0;
                job_of(jl, a, v0);
                const int e = gch % C::NR, use = gch / C::NR;
                if (use > 0) tc::mbar_wait(&raw_empty[e], (use - 1) & 1);
                // the chunk's KP R coefficient rows of this vector tile: one 2-D tensor copy (whole box, a
                // ragged tile zero-filled); per-row 1-D copies measured ~85 clk each to issue
                tc::mbar_arrive_expect_tx(&raw_full[e], C::RAW);
                const int64_t p0 = a * N0 + int64_t(ch) * KP;
                tc::tma_load_2d(raw(e), &tin, 2 * v0, int(p0 * R), &raw_full[e]);
            }
        } else if (lane == 1) {
            for (int gch = 0; gch < nch_all; gch++) {
                const int jl = gch / C::NCH, ch = gch - jl * C::NCH;
                int64_t a;
                int v0;
                job_of(jl, a, v0);
                const int e = gch % C::NB_R, use = gch / C::NB_R;
                if (use > 0) tc::mbar_wait(&b_empty[e], (use - 1) & 1);
                tc::mbar_arrive_expect_tx(&b_full[e], 2 * C::BT);   // both halves land here
                const float* src = Ux + (a * C::NCH + ch) * 2 * (C::BT / 4);
                if constexpr (CL == 2)
                    tc::bulk_g2s_mc(opB(e, cr), src + cr * (C::BT / 4), C::BT, &b_full[e], uint16_t(3));
                else
                    tc::bulk_g2s(opB(e, 0), src, 2 * C::BT, &b_full[e]);
            }
        }
    } else if (warp == 13) {
        // ---- MMA issuer (whole warp, one elected lane issues) ----
        constexpr uint32_t idesc = tc::idesc_tf32(128, C::NB);
        constexpr uint32_t LBO_B = (C::NB / 8) * 128;
        const uint64_t dB0 = tc::desc_kmajor(tc::smem_u32(opB(0, 0)), LBO_B);
        int gseg = 0;   // accumulation segments issued (slots alternate across jobs)
        for (int gch = 0; gch < nch_all; gch++) {
            const int ch = gch % C::NCH;
            const int e = gch % C::NB_R, sa = gch & 1, slot = gseg & 1, first = (ch % C::SEG) == 0;
            const bool last = (ch % C::SEG) == C::SEG - 1 || ch == C::NCH - 1;
            if (first && gseg >= 2) tc::mbar_wait(&dempty[slot], uint32_t((gseg >> 1) - 1) & 1);
            tc::mbar_wait(&a_full[sa], uint32_t(gch >> 1) & 1);
            tc::mbar_wait(&b_full[e], uint32_t(gch / C::NB_R) & 1);
            tc::fence_after_sync();
            const uint32_t d = tmem + uint32_t(C::D_OFF + slot * C::NB);
#pragma unroll
            for (int q = 0; q < 3; q++) {
                const int pass = kPassOrder[q];
                const uint32_t aa = tmem + uint32_t(sa * C::A_COLS + (pass == 1 ? C::KC : 0));
                const uint64_t bb = tc::desc_add(dB0, (2 * e + (pass == 2)) * C::BT);
#pragma unroll
                for (int ks = 0; ks < C::KC / 8; ks++)
                    tc::mma_tf32_ts_warp(d, aa + ks * 8, tc::desc_add(bb, ks * 2 * LBO_B), idesc,
                                         (first && q == 0 && ks == 0) ? 0u : 1u);
            }
            tc::commit_warp(&a_empty[sa]);
            if constexpr (CL == 2)
                tc::commit_mc_warp(&b_empty[e], uint16_t(3));
            else
                tc::commit_warp(&b_empty[e]);
            if (last) {
                tc::commit_warp(&dfull[slot]);
                gseg++;
            }
            __syncwarp();
        }
    } else if (warp < 4) {
        // ---- split: raw delta rows -> A stage (hi / lo) in TMEM; thread = vector (its lane) ----
        const int v = tid;
        const uint32_t lb = uint32_t(warp * 32) << 16;
        for (int gch = 0; gch < nch_all; gch++) {
            const int e = gch % C::NR, sa = gch & 1;
            tc::mbar_wait(&raw_full[e], uint32_t(gch / C::NR) & 1);
            if (gch >= 2) tc::mbar_wait(&a_empty[sa], uint32_t((gch >> 1) - 1) & 1);
            tc::fence_after_sync();
            const float2* rd = reinterpret_cast<const float2*>(raw(e));   // [KP R][128]
            float hi[C::KC], lo[C::KC];   // column (pl, t, c) = pl 2R + 2t + c
#pragma unroll
            for (int row = 0; row < KP * R; row++) {
                const float2 x = rd[row * 128 + v];
                tc::split(x.x, hi[2 * row], lo[2 * row]);
                tc::split(x.y, hi[2 * row + 1], lo[2 * row + 1]);
            }
            tc::fence_before_sync();
            tc::mbar_arrive(&raw_empty[e]);   // the raw rows are in registers now
            const uint32_t ta = tmem + lb + uint32_t(sa * C::A_COLS);
            tc::tmem_st_cols<C::KC>(ta, hi);
            tc::tmem_st_cols<C::KC>(ta + C::KC, lo);
            tc::tmem_wait_st();
            tc::fence_before_sync();
            tc::mbar_arrive(&a_full[sa]);
        }
    } else {
        // ---- drain + epilogue (warps 4-11): lane quarter warp % 4 = vectors, column half (warp - 4) / 4 ----
        constexpr int HC = C::NB / 2;   // columns per drain thread (j in a half of the leaf)
        const int q4 = warp & 3, half = (warp - 4) >> 2, vl = q4 * 32 + lane, dt = (warp - 4) * 32 + lane;
        const int k = vl % NA, cl = vl / NA;
        int gseg = 0;
        for (int jl = 0; jl < njobs; jl++) {
            int64_t a;
            int v0;
            job_of(jl, a, v0);
            const int vw = min(128, nv - v0);
            float sum[HC];
#pragma unroll
            for (int i = 0; i < HC; i++) sum[i] = 0.f;
            for (int seg = 0; seg < C::NSEG; seg++, gseg++) {
                const int slot = gseg & 1;
                tc::mbar_wait(&dfull[slot], uint32_t(gseg >> 1) & 1);
                tc::fence_after_sync();
                const uint32_t taddr =
                    tmem + (uint32_t(q4 * 32) << 16) + uint32_t(C::D_OFF + slot * C::NB + half * HC);
#pragma unroll
                for (int c0 = 0; c0 < HC; c0 += 32) {
                    float x[32];
                    tc::tmem_ld_cols<(HC < 32 ? HC : 32)>(taddr + c0, x);
                    tc::tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < (HC < 32 ? HC : 32); i++) sum[c0 + i] += x[i];
                }
                tc::fence_before_sync();
                tc::mbar_arrive(&dempty[slot]);
            }
            // epilogue of the job: a_k(x) (staged per job), sum over k, G transposed through Gs
            asm volatile("bar.sync 1, 256;" ::: "memory");   // the previous job's copy-out is done with Gs / As
            for (int i = dt; i < NA * N0; i += 256) As[i] = __ldg(ampa + (i / N0) * N + a * N0 + (i % N0));
            asm volatile("bar.sync 1, 256;" ::: "memory");
#pragma unroll
            for (int jj = 0; jj < HC / 2; jj++) {
                const int j = half * (HC / 2) + jj;
                float2 g = cmul_tc(As[k * N0 + j], make_float2(sum[2 * jj], sum[2 * jj + 1]));
#pragma unroll
                for (int m = 1; m < NA; m <<= 1) {
                    g.x += __shfl_xor_sync(0xffffffffu, g.x, m);
                    g.y += __shfl_xor_sync(0xffffffffu, g.y, m);
                }
                if ((j % NA) == k) Gs[cl * C::GS_STRIDE + j] = g;
            }
            asm volatile("bar.sync 1, 256;" ::: "memory");
            // copy out: RHS column c0 + cl, rows a n0 .. a n0 + n0 - 1 (contiguous)
            const int c0 = v0 / NA, cw = vw / NA;
            for (int idx = dt; idx < cw * N0; idx += 256) {
                const int cc = idx / N0, j = idx % N0;
                G[a * N0 + j + int64_t(c0 + cc) * ldg] = Gs[cc * C::GS_STRIDE + j];
            }
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if constexpr (CL == 2) tc::cluster_sync();   // no CTA leaves while its partner may still multicast into it
    if (warp == 0) {
        tc::fence_after_sync();
        tc::tmem_dealloc<TMEM_COLS>(tmem);
    }
}

template <int R, int N0, int NA, int KP>
static cudaError_t sl_tc_go(const Dims& d, const float2* in, const float* Ux, const float2* ampa, float2* G, int64_t ldg,
                            int nv, cudaStream_t s, bool multicast)
{
    using C = SLTC<R, N0, NA, KP>;
    const int nvt = (nv + 127) / 128;
    CUtensorMap tin;
    cudaError_t e = make_rows_tmap(&tin, in, d.N * R, nv, KP * R);
    if (e != cudaSuccess) return e;
    const int64_t leaves = d.N / N0;
    if (multicast && nvt % 2 == 0 && sm_count() >= 2) {
        auto kern = sl_tc_kernel<R, N0, NA, KP, 2>;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
        if (e != cudaSuccess) return e;
        const int64_t pairs = leaves * (nvt / 2);
        const int64_t ncl = std::min<int64_t>(pairs, sm_count() / 2);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(unsigned(2 * ncl));
        cfg.blockDim = dim3(448);
        cfg.dynamicSmemBytes = C::SMEM;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kern, tin, Ux, ampa, G, ldg, d.LN, nv, nvt);
    }
    auto kern = sl_tc_kernel<R, N0, NA, KP, 1>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
    if (e != cudaSuccess) return e;
    const int64_t jobs = leaves * nvt;
    const unsigned grid = unsigned(jobs < sm_count() ? jobs : sm_count());
    kern<<<grid, 448, C::SMEM, s>>>(tin, Ux, ampa, G, ldg, d.LN, nv, nvt);
    return cudaGetLastError();
}

bool sl_tc_supported(const Dims& d, int nv) { return leaf_tc_shape(d) && nv >= 64 && nv % 2 == 0; }

cudaError_t launch_sl_tc(const Dims& d, const float2* in, const float* Ux, const float2* ampa, float2* G, int64_t ldg,
                         int nv, cudaStream_t s, bool multicast)
{
    const int n0 = 1 << d.l0;
#define SLTC_NA(RR, N0_, KP_)                                                                 \
    if (d.R == RR && n0 == N0_) {                                                             \
        if (d.n_amp == 1) return sl_tc_go<RR, N0_, 1, KP_>(d, in, Ux, ampa, G, ldg, nv, s, multicast);  \
        if (d.n_amp == 2) return sl_tc_go<RR, N0_, 2, KP_>(d, in, Ux, ampa, G, ldg, nv, s, multicast);  \
        if (d.n_amp == 4) return sl_tc_go<RR, N0_, 4, KP_>(d, in, Ux, ampa, G, ldg, nv, s, multicast);  \
    }
    SLTC_NA(6, 64, 2) SLTC_NA(8, 64, 2) SLTC_NA(10, 64, 2) SLTC_NA(12, 64, 1) SLTC_NA(16, 64, 1)
    SLTC_NA(6, 32, 2) SLTC_NA(8, 32, 2) SLTC_NA(10, 32, 2) SLTC_NA(12, 32, 1) SLTC_NA(16, 32, 1)
#undef SLTC_NA
    return cudaErrorInvalidValue;
}

// =============================================================================================
// SL in FP16 split passes (BF_OPT_LEAF_F16 = 1, the default): the structure of sl_tc_kernel with
// kind::f16 MMAs (K = 16).  Every K chunk (KP pairs of the leaf, KC = KP 2r, a multiple of 16) is its own
// accumulation segment: the split scales each vector's chunk by 2^{-e_vc} (max |x| in [0.5, 1)) before
// the FP16 hi / lo split, and the drain adds 2^{e_vc} D_c into the FP32 register sums; the image rows
// (output point j, re / im) are scaled to max |x| in [0.5, 1) with the exponent applied with a_k at the
// end of the job.  Half the Ux image bytes, half the tensor time of the 3xTF32 SL.
// =============================================================================================
static int sl_kp_h(int R) { return (R == 12) ? 2 : (R == 16 ? 2 : 4); }   // KC = KP 2r multiple of 16

int64_t leafu_rows(const Dims& d) { return d.N; }   // biased exponents of the SL image: one per output point

__global__ void expand_sl_h16_kernel(const float2* __restrict__ U, __half* __restrict__ X, uint8_t* __restrict__ S,
                                     int LN, int l0, int R, int KP)
{
    const int n0 = 1 << l0;
    const int64_t nleaf = (int64_t(1) << LN) >> l0;
    const int rows = 2 * n0, K = n0 * 2 * R, KC = KP * 2 * R;
    const int nch = n0 / KP;
    const int64_t tile = int64_t(rows) * KC;
    const int64_t total = nleaf * n0;
    for (int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < total; g += int64_t(gridDim.x) * blockDim.x) {
        const int64_t a = g / n0;
        const int j = int(g - a * n0);
        const float2* w = U + (a * n0) * (n0 * R) + j;   // element (b, t): w[b n0 R + t n0]
        float mx = 0.f;
        for (int b = 0; b < n0; b++)
            for (int t = 0; t < R; t++) {
                const float2 x = w[(int64_t(b) * R + t) * n0];
                mx = fmaxf(mx, fmaxf(fabsf(x.x), fabsf(x.y)));
            }
        int e = 0;
        frexpf(mx, &e);
        e = max(-126, min(126, e));
        S[a * n0 + j] = uint8_t(e + 127);
        for (int cp = 0; cp < 2; cp++) {
            const int n = 2 * j + cp;
            for (int k = 0; k < K; k++) {
                const int b = k / (2 * R), t = (k / 2) % R, c = k & 1;
                const float x = ldexpf(embed(w[(int64_t(b) * R + t) * n0], cp, c), -e);
                float hi, lo;
                tc::split_h(x, hi, lo);
                const int ch = b / KP, kk = k - ch * KC;
                __half* tl = X + ((a * nch + ch) * 2) * tile;
                const uint32_t off = tc::kmaj_off16(n, kk, rows) / 2;
                tl[off] = __float2half_rn(hi);
                tl[tile + off] = __float2half_rn(lo);
            }
        }
    }
}

template <int R, int N0, int NA, int KP>
struct SLH {
    static constexpr int NB = 2 * N0;
    static constexpr int KC = KP * 2 * R;
    static constexpr int NCH = N0 / KP;
    static constexpr uint32_t RAW = uint32_t(KP) * R * 128 * 8;
    static constexpr uint32_t BT = uint32_t(NB) * KC * 2;          // one of hi / lo (FP16)
    static constexpr uint32_t GS_STRIDE = N0 + 1;
    static constexpr uint32_t GS_BYTES = uint32_t(128 / NA) * GS_STRIDE * 8;
    static constexpr uint32_t AS_BYTES = uint32_t(NA) * N0 * 8;
    static constexpr uint32_t ES_BYTES = 4 * 128 * 4;
    static constexpr size_t LIM = 232448 - 1024;
    static constexpr int NR_FIT = int((LIM - GS_BYTES - AS_BYTES - ES_BYTES) / (RAW + 2 * BT));
    static constexpr int NR = NR_FIT > 4 ? 4 : (NR_FIT < 2 ? 2 : NR_FIT);   // ring depth
    static constexpr uint32_t OFF_B = NR * RAW, OFF_GS = OFF_B + 2 * NR * BT, OFF_AS = OFF_GS + GS_BYTES;
    static constexpr uint32_t OFF_ES = OFF_AS + AS_BYTES;
    static constexpr size_t SMEM = size_t(OFF_ES) + ES_BYTES;
    static constexpr int A_COLS = KC;                                   // hi KC/2 packed columns, then lo
    static constexpr int D_OFF = 2 * A_COLS;
    static constexpr int TMEM_COLS = tmem_cols_pow2<D_OFF + 2 * NB>();
    // shapes that fit (otherwise the plan keeps the 3xTF32 SL): whole kind::f16 K steps, a ring of >= 2
    static constexpr bool OK = KC % 16 == 0 && NR_FIT >= 2 && D_OFF + 2 * NB <= 512 && SMEM <= LIM;
};

template <int R, int N0, int NA, int KP>
__global__ void __launch_bounds__(448, 1)
    sl_h16_kernel(const __grid_constant__ CUtensorMap tin, const __half* __restrict__ Uh,
                  const uint8_t* __restrict__ Ue, const float2* __restrict__ ampa, float2* __restrict__ G, int64_t ldg,
                  int LN, int nv, int nvt)
{
    using C = SLH<R, N0, NA, KP>;
    extern __shared__ __align__(128) uint8_t sm_slh[];
    auto raw = [&](int e) { return sm_slh + e * C::RAW; };
    auto opB = [&](int e, int lo) { return sm_slh + C::OFF_B + (2 * e + lo) * C::BT; };
    float2* Gs = reinterpret_cast<float2*>(sm_slh + C::OFF_GS);   // [128/NA][GS_STRIDE]
    float2* As = reinterpret_cast<float2*>(sm_slh + C::OFF_AS);   // [NA][N0] a_k(x) of the current job
    float* Es = reinterpret_cast<float*>(sm_slh + C::OFF_ES);      // [chunk % 4][128] 2^{e_vc}
    __shared__ uint64_t raw_full[C::NR], raw_empty[C::NR], b_full[C::NR], b_empty[C::NR], a_full[2], a_empty[2],
        dfull[2], dempty[2], e_full[4], e_empty[4];
    __shared__ uint32_t tmem_base;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t N = int64_t(1) << LN;
    const int64_t njobs_all = (N / N0) * nvt;
    const int njobs = int((njobs_all - blockIdx.x + gridDim.x - 1) / gridDim.x);
    const int nch_all = njobs * C::NCH;

    if (warp == 0) tc::tmem_alloc<C::TMEM_COLS>(&tmem_base);
    if (tid == 0) {
        for (int i = 0; i < C::NR; i++) {
            tc::mbar_init(&raw_full[i], 1);
            tc::mbar_init(&raw_empty[i], 128);
            tc::mbar_init(&b_full[i], 1);
            tc::mbar_init(&b_empty[i], 1);
        }
        for (int i = 0; i < 2; i++) {
            tc::mbar_init(&a_full[i], 128);
            tc::mbar_init(&a_empty[i], 1);
            tc::mbar_init(&dfull[i], 1);
            tc::mbar_init(&dempty[i], 256);
        }
        for (int i = 0; i < 4; i++) {
            tc::mbar_init(&e_full[i], 128);
            tc::mbar_init(&e_empty[i], 256);
        }
        tc::mbar_fence_init();
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tmem_base;

    if (warp == 12) {
        // ---- loader: the chunk stream of all this CTA's jobs (Ux tiles: bulk copy; delta rows: 2-D TMA) ----
        if (lane == 0) {
            for (int gch = 0; gch < nch_all; gch++) {
                const int jl = gch / C::NCH, ch = gch - jl * C::NCH;
                const unsigned job = unsigned(blockIdx.x + int64_t(jl) * gridDim.x);
                const int64_t a = job / unsigned(nvt);
                const int v0 = int(job % unsigned(nvt)) * 128;
                const int e = gch % C::NR, use = gch / C::NR;
                if (use > 0) tc::mbar_wait(&raw_empty[e], (use - 1) & 1);
                tc::mbar_arrive_expect_tx(&raw_full[e], C::RAW);
                const int64_t p0 = a * N0 + int64_t(ch) * KP;
                tc::tma_load_2d(raw(e), &tin, 2 * v0, int(p0 * R), &raw_full[e]);
                if (use > 0) tc::mbar_wait(&b_empty[e], (use - 1) & 1);
                tc::mbar_arrive_expect_tx(&b_full[e], 2 * C::BT);
                tc::bulk_g2s(opB(e, 0), Uh + (a * C::NCH + ch) * 2 * (C::BT / 2), 2 * C::BT, &b_full[e]);
            }
        }
    } else if (warp == 13) {
        // ---- MMA issuer: one accumulation segment per chunk, 3 passes x KC/16 kind::f16 MMAs ----
        constexpr uint32_t idesc = tc::idesc_f16(128, C::NB);
        constexpr uint32_t LBO_B = (C::NB / 8) * 128;
        const uint64_t dB0 = tc::desc_kmajor(tc::smem_u32(opB(0, 0)), LBO_B);
        for (int gch = 0; gch < nch_all; gch++) {
            const int e = gch % C::NR, sa = gch & 1, slot = gch & 1;
            if (gch >= 2) tc::mbar_wait(&dempty[slot], uint32_t((gch >> 1) - 1) & 1);
            tc::mbar_wait(&a_full[sa], uint32_t(gch >> 1) & 1);
            tc::mbar_wait(&b_full[e], uint32_t(gch / C::NR) & 1);
            tc::fence_after_sync();
            const uint32_t d = tmem + uint32_t(C::D_OFF + slot * C::NB);
#pragma unroll
            for (int q = 0; q < 3; q++) {
                const int pass = kPassOrder[q];
                const uint32_t aa = tmem + uint32_t(sa * C::A_COLS + (pass == 1 ? C::KC / 2 : 0));
                const uint64_t bb = tc::desc_add(dB0, (2 * e + (pass == 2)) * C::BT);
#pragma unroll
                for (int ks = 0; ks < C::KC / 16; ks++)
                    tc::mma_f16_ts_warp(d, aa + ks * 8, tc::desc_add(bb, ks * 2 * LBO_B), idesc, (q | ks) ? 1u : 0u);
            }
            tc::commit_warp(&a_empty[sa]);
            tc::commit_warp(&b_empty[e]);
            tc::commit_warp(&dfull[slot]);
            __syncwarp();
        }
    } else if (warp < 4) {
        // ---- split: raw delta rows of a chunk, scaled by 2^{-e_vc}, FP16 hi / lo packed into TMEM ----
        const int v = tid;
        const uint32_t lb = uint32_t(warp * 32) << 16;
        for (int gch = 0; gch < nch_all; gch++) {
            const int e = gch % C::NR, sa = gch & 1, eb = gch & 3;
            tc::mbar_wait(&raw_full[e], uint32_t(gch / C::NR) & 1);
            if (gch >= 2) tc::mbar_wait(&a_empty[sa], uint32_t((gch >> 1) - 1) & 1);
            if (gch >= 4) tc::mbar_wait(&e_empty[eb], uint32_t((gch >> 2) - 1) & 1);
            tc::fence_after_sync();
            const float2* rd = reinterpret_cast<const float2*>(raw(e));   // [KP R][128]
            float mx = 0.f;
#pragma unroll
            for (int row = 0; row < KP * R; row++) {
                const float2 x = rd[row * 128 + v];
                mx = fmaxf(mx, fmaxf(fabsf(x.x), fabsf(x.y)));
            }
            int ex = 0;
            frexpf(mx, &ex);
            ex = max(-126, min(126, ex));
            const float sc = ldexpf(1.f, -ex);
            Es[eb * 128 + v] = ldexpf(1.f, ex);
            tc::mbar_arrive(&e_full[eb]);
            float hi[C::KC / 2], lo[C::KC / 2];   // packed column (pl, t) = pl R + t: (re, im)
#pragma unroll
            for (int row = 0; row < KP * R; row++) {
                const float2 x = rd[row * 128 + v];
                tc::split_h2(x.x * sc, x.y * sc, hi[row], lo[row]);
            }
            tc::fence_before_sync();
            tc::mbar_arrive(&raw_empty[e]);
            const uint32_t ta = tmem + lb + uint32_t(sa * C::A_COLS);
            tc::tmem_st_cols<C::KC / 2>(ta, hi);
            tc::tmem_st_cols<C::KC / 2>(ta + C::KC / 2, lo);
            tc::tmem_wait_st();
            tc::fence_before_sync();
            tc::mbar_arrive(&a_full[sa]);
        }
    } else {
        // ---- drain + epilogue (warps 4-11): lane quarter warp % 4 = vectors, column half (warp - 4) / 4 ----
        constexpr int HC = C::NB / 2;   // columns per drain thread (j in a half of the leaf)
        const int q4 = warp & 3, half = (warp - 4) >> 2, vl = q4 * 32 + lane, dt = (warp - 4) * 32 + lane;
        const int k = vl % NA, cl = vl / NA;
        int gch = 0;
        for (int jl = 0; jl < njobs; jl++) {
            const unsigned job = unsigned(blockIdx.x + int64_t(jl) * gridDim.x);
            const int64_t a = job / unsigned(nvt);
            const int v0 = int(job % unsigned(nvt)) * 128, vw = min(128, nv - v0);
            // this thread's output points j = half HC/2 .. + HC/2: their image row exponents (read now, used at
            // the end of the job)
            uint32_t rexp[HC / 8];
#pragma unroll
            for (int u = 0; u < HC / 8; u++)
                rexp[u] = __ldg(reinterpret_cast<const uint32_t*>(Ue + a * N0 + half * (HC / 2)) + u);
            float sum[HC];
#pragma unroll
            for (int i = 0; i < HC; i++) sum[i] = 0.f;
            for (int ch = 0; ch < C::NCH; ch++, gch++) {
                const int slot = gch & 1, eb = gch & 3;
                tc::mbar_wait(&e_full[eb], uint32_t(gch >> 2) & 1);
                const float sv = Es[eb * 128 + vl];
                tc::mbar_arrive(&e_empty[eb]);
                tc::mbar_wait(&dfull[slot], uint32_t(gch >> 1) & 1);
                tc::fence_after_sync();
                const uint32_t taddr =
                    tmem + (uint32_t(q4 * 32) << 16) + uint32_t(C::D_OFF + slot * C::NB + half * HC);
#pragma unroll
                for (int c0 = 0; c0 < HC; c0 += 32) {
                    float x[32];
                    tc::tmem_ld_cols<(HC < 32 ? HC : 32)>(taddr + c0, x);
                    tc::tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < (HC < 32 ? HC : 32); i++) sum[c0 + i] = fmaf(x[i], sv, sum[c0 + i]);
                }
                tc::fence_before_sync();
                tc::mbar_arrive(&dempty[slot]);
            }
            // epilogue of the job: 2^{e_j} a_k(x) (staged per job), sum over k, G transposed through Gs
            asm volatile("bar.sync 1, 256;" ::: "memory");   // the previous job's copy-out is done with Gs / As
            for (int i = dt; i < NA * N0; i += 256) As[i] = __ldg(ampa + (i / N0) * N + a * N0 + (i % N0));
            asm volatile("bar.sync 1, 256;" ::: "memory");
#pragma unroll
            for (int jj = 0; jj < HC / 2; jj++) {
                const int j = half * (HC / 2) + jj;
                const uint32_t be = (rexp[jj >> 2] >> (8 * (jj & 3))) & 0xffu;
                const float sj = __uint_as_float(be << 23);
                float2 g = cmul_tc(As[k * N0 + j], make_float2(sum[2 * jj] * sj, sum[2 * jj + 1] * sj));
#pragma unroll
                for (int m = 1; m < NA; m <<= 1) {
                    g.x += __shfl_xor_sync(0xffffffffu, g.x, m);
                    g.y += __shfl_xor_sync(0xffffffffu, g.y, m);
                }
                if ((j % NA) == k) Gs[cl * C::GS_STRIDE + j] = g;
            }
            asm volatile("bar.sync 1, 256;" ::: "memory");
            const int c0 = v0 / NA, cw = vw / NA;
            for (int idx = dt; idx < cw * N0; idx += 256) {
                const int cc = idx / N0, j = idx % N0;
                G[a * N0 + j + int64_t(c0 + cc) * ldg] = Gs[cc * C::GS_STRIDE + j];
            }
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) {
        tc::fence_after_sync();
        tc::tmem_dealloc<C::TMEM_COLS>(tmem);
    }
}

template <int R, int N0, int NA, int KP>
static cudaError_t sl_h16_go(const Dims& d, const float2* in, const __half* Uh, const uint8_t* Ue, const float2* ampa,
                             float2* G, int64_t ldg, int nv, cudaStream_t s)
{
    using C = SLH<R, N0, NA, KP>;
    if constexpr (!C::OK) {
        return cudaErrorInvalidValue;
    } else {
    auto kern = sl_h16_kernel<R, N0, NA, KP>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
    if (e != cudaSuccess) return e;
    const int nvt = (nv + 127) / 128;
    const int64_t jobs = (d.N / N0) * nvt;
    const unsigned grid = unsigned(jobs < sm_count() ? jobs : sm_count());
    CUtensorMap tin;
    e = make_rows_tmap(&tin, in, d.N * R, nv, KP * R);
    if (e != cudaSuccess) return e;
    kern<<<grid, 448, C::SMEM, s>>>(tin, Uh, Ue, ampa, G, ldg, d.LN, nv, nvt);
    return cudaGetLastError();
    }
}

bool sl_h16_shape(const Dims& d)
{
    const int n0 = 1 << d.l0;
#define SLH_OK(RR, N0_, KP_)                                                                     \
    if (d.R == RR && n0 == N0_)                                                                  \
        return d.n_amp == 1 ? SLH<RR, N0_, 1, KP_>::OK                                           \
                            : (d.n_amp == 2 ? SLH<RR, N0_, 2, KP_>::OK : (d.n_amp == 4 && SLH<RR, N0_, 4, KP_>::OK));
    SLH_OK(6, 64, 4) SLH_OK(8, 64, 4) SLH_OK(10, 64, 4) SLH_OK(12, 64, 2) SLH_OK(16, 64, 2)
    SLH_OK(6, 32, 4) SLH_OK(8, 32, 4) SLH_OK(10, 32, 4) SLH_OK(12, 32, 2) SLH_OK(16, 32, 2)
#undef SLH_OK
    return false;
}

cudaError_t expand_sl_h16(const Dims& d, const float2* U, void* Uh, void* Ue, cudaStream_t s)
{
    if (!leaf_tc_shape(d)) return cudaErrorInvalidValue;
    expand_sl_h16_kernel<<<148 * 16, 128, 0, s>>>(U, static_cast<__half*>(Uh), static_cast<uint8_t*>(Ue), d.LN, d.l0,
                                                  d.R, sl_kp_h(d.R));
    return cudaGetLastError();
}

cudaError_t launch_sl_h16(const Dims& d, const float2* in, const void* Uh, const void* Ue, const float2* ampa,
                          float2* G, int64_t ldg, int nv, cudaStream_t s)
{
    const int n0 = 1 << d.l0;
    const __half* X = static_cast<const __half*>(Uh);
    const uint8_t* E8 = static_cast<const uint8_t*>(Ue);
#define SLH_NA(RR, N0_, KP_)                                                                        \
    if (d.R == RR && n0 == N0_) {                                                                   \
        if (d.n_amp == 1) return sl_h16_go<RR, N0_, 1, KP_>(d, in, X, E8, ampa, G, ldg, nv, s);    \
        if (d.n_amp == 2) return sl_h16_go<RR, N0_, 2, KP_>(d, in, X, E8, ampa, G, ldg, nv, s);    \
        if (d.n_amp == 4) return sl_h16_go<RR, N0_, 4, KP_>(d, in, X, E8, ampa, G, ldg, nv, s);    \
    }
    SLH_NA(6, 64, 4) SLH_NA(8, 64, 4) SLH_NA(10, 64, 4) SLH_NA(12, 64, 2) SLH_NA(16, 64, 2)
    SLH_NA(6, 32, 4) SLH_NA(8, 32, 4) SLH_NA(10, 32, 4) SLH_NA(12, 32, 2) SLH_NA(16, 32, 2)
#undef SLH_NA
    return cudaErrorInvalidValue;
}

// Band variant switch (BF_OPT_BAND_PIPELINES): 1 = single TMEM pipeline (default), 0 = two pipelines where
// they fit.  Measured at cfg4 (tools/band_trace.py, profiles/r1_band_variants.txt): the two-pipeline kernel
// halves the per-job cycle count on some SMs, but its concurrent tcgen05.st/ld traffic (two epilogues plus
// the split) slows the tensor pipe on others, and the launch is 1.4x slower overall.



// ---- timeline trace of the band kernel (diagnostic; CTA 0, first BT_JOBS jobs, SM clock) ----
constexpr int BT_JOBS = 64, BT_EV = 12;
__device__ long long g_band_trace[BT_JOBS * BT_EV];
// (constant bank: the check costs no memory round trip; tracing is off until BF_OPT_BAND_TRACE_J0 is set)
__constant__ int g_band_trace_j0 = 0;     // first traced job (BF_OPT_BAND_TRACE_J0: job + 65536 * cta)
__constant__ int g_band_trace_cta = -1;   // traced CTA (-1: off)
__device__ __forceinline__ void btrace(int64_t J, int ev)
{
    const int64_t j = J - g_band_trace_j0;
    if (int(blockIdx.x) == g_band_trace_cta && j >= 0 && j < BT_JOBS) g_band_trace[j * BT_EV + ev] = clock64();
}
void band_trace_window(int v)
{
    const int j0 = v & 65535, cta = v >> 16;
    cudaMemcpyToSymbol(g_band_trace_j0, &j0, sizeof(int));
    cudaMemcpyToSymbol(g_band_trace_cta, &cta, sizeof(int));
}

// =============================================================================================
// Transfer band of two levels (eqn:2 P:748-752 for l <= h, eqn:3 P:780-785 for l > h; the switch
// P:755-766 is folded into the level-h blocks) on the tensor cores, persistent (one CTA per SM).
// A group = 4 pairs at the input level closed under the two levels (fixed a0, 4 consecutive b),
// as in the SIMT band.  Per group and vector tile of 128:
//   warp 8 (one thread)   bulk-copies the 4 r raw coefficient rows (2-deep ring),
//   warps 0-3             split them hi/lo into an A buffer in TMEM (lane = vector, one slot of
//                         2r columns per pair; double-buffered when TMEM allows),
//   warp 9 (one thread)   level 1: per unit u (slots 2u, 2u+1 = K of 4r), D1_u = A B1_u with both
//                         outputs of the unit as N (4r, padded to 16); level 2 likewise from D2,
//   warps 4-7             drain D1, split it back into the A buffer at the level-2 slot order
//                         (output e of unit u -> slot 2e + u, so every level-2 unit again reads
//                         two adjacent slots), and finally store D2 to HBM (coalesced over v),
//   warps 10-11           expand the group's compact weight blocks into real-embedded hi/lo B
//                         tiles in shared memory, one group ahead (double-buffered when it fits).
// Each accumulator chain is 3 (4r/8) MMAs (15 at r = 10): short, FP32-accurate.
// =============================================================================================
template <int R>
struct BandTC {
    static constexpr int P = 4, U = 2;                 // pairs per group, units per level
    static constexpr int SC = 2 * R;                   // TMEM columns of one slot (r complex)
    static constexpr int KU = 4 * R;                   // MMA K of a unit (two slots)
    static constexpr int NU = 4 * R;                   // useful N of a unit (two outputs)
    static constexpr int NB = (NU + 15) / 16 * 16;     // MMA N
    static constexpr int ACOLS = 2 * P * SC;           // hi + lo of one A buffer
    static constexpr int DCOLS = U * NB;               // accumulators of one level
    static constexpr int NABUF = (2 * ACOLS + 2 * DCOLS <= 512) ? 2 : 1;
    static constexpr int D1_OFF = NABUF * ACOLS, D2_OFF = D1_OFF + DCOLS;
    static constexpr int TMEM_COLS = tmem_cols_pow2<D2_OFF + DCOLS>();
    static constexpr uint32_t RAW = uint32_t(P) * R * 128 * 8;   // raw rows of one vector tile
    static constexpr uint32_t WT = uint32_t(NB) * KU * 4;        // one B tile (hi or lo)
    static constexpr uint32_t WSET = 2 * U * 2 * WT;             // 2 levels x U units x (hi, lo)
    static constexpr uint32_t OFF_W = 2 * RAW;
    static constexpr int NWBUF = (size_t(OFF_W) + 2 * size_t(WSET) <= 232448 - 1024) ? 2 : 1;
    static constexpr size_t SMEM = size_t(OFF_W) + NWBUF * size_t(WSET);
    static constexpr int WTASKS = 2 * U * 2 * 2 * R * R;         // complex weight entries per group
    static constexpr int WPT = (WTASKS + 63) / 64;               // per weight thread
    static_assert(KU % 8 == 0 && D2_OFF + DCOLS <= 512 && SMEM <= 232448 - 1024, "band shape");
};

template <int R>
__global__ void __launch_bounds__(384, 1)
    band_tc_kernel(const float2* __restrict__ in, float2* __restrict__ out, const float2* __restrict__ W1,
                   const float2* __restrict__ W2, int LN, int l_first, int nv, int rh, int rhg, const bfs::PeerOut po)
{
    using C = BandTC<R>;
    extern __shared__ __align__(128) uint8_t sm_band[];
    auto raw = [&](int e) { return sm_band + e * C::RAW; };
    auto wtile = [&](int wb, int m, int u, int lo) {
        return sm_band + C::OFF_W + wb * C::WSET + ((m * C::U + u) * 2 + lo) * C::WT;
    };
    __shared__ uint64_t raw_full[2], raw_empty[2], a1_ready[2], a2_ready[2], a_free[2], w_full[2], w_free[2];
    __shared__ uint64_t d1_full, d1_free, d2_full, d2_free;
    __shared__ uint32_t tmem_base;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t N = int64_t(1) << LN;
    const int lin = l_first - 1, shg = LN - lin - 2;
    const int64_t ngroups = N >> 2;
    const int nvt = (nv + 127) / 128;
    const int64_t nit = (ngroups - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int64_t njobs = nit * nvt;

    if (warp == 0) tc::tmem_alloc<C::TMEM_COLS>(&tmem_base);
    if (tid == 0) {
        for (int i = 0; i < 2; i++) {
            tc::mbar_init(&raw_full[i], 1);
            tc::mbar_init(&raw_empty[i], 128);
            tc::mbar_init(&a1_ready[i], 128);
            tc::mbar_init(&a2_ready[i], 128);
            tc::mbar_init(&a_free[i], 1);
            tc::mbar_init(&w_full[i], 64);
            tc::mbar_init(&w_free[i], 1);
        }
        tc::mbar_init(&d1_full, 1);
        tc::mbar_init(&d1_free, 128);
        tc::mbar_init(&d2_full, 1);
        tc::mbar_init(&d2_free, 128);
        tc::mbar_fence_init();
    }
    if constexpr (C::NB > C::NU) {   // zero the pad rows of every B tile (never written afterwards)
        constexpr int PADQ = (C::NB - C::NU) * C::KU / 4;
        for (int idx = tid; idx < C::NWBUF * 2 * C::U * 2 * PADQ; idx += blockDim.x) {
            const int tile = idx / PADQ, o = idx % PADQ;
            const int row = C::NU + o % (C::NB - C::NU), k = 4 * (o / (C::NB - C::NU));
            st_f4(sm_band + C::OFF_W + tile * C::WT, tc::kmaj_off(row, k, C::NB), make_float4(0, 0, 0, 0));
        }
    }
    tc::fence_proxy_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tmem_base;

    if (warp < 4) {
        // ---- split: raw rows -> A buffer (TMEM), lane = vector ----
        const int v = tid;
        const uint32_t lb = uint32_t(warp * 32) << 16;
        for (int J = 0; J < int(njobs); J++) {
            const int e = int(J & 1);
            tc::mbar_wait(&raw_full[e], uint32_t(J >> 1) & 1);
            const int slot = int(J % C::NABUF);
            const int use = J / C::NABUF;
            if (use > 0) tc::mbar_wait(&a_free[slot], uint32_t(use - 1) & 1);
            tc::fence_after_sync();
            if (tid == 0) btrace(J, 0);
            const float2* rd = reinterpret_cast<const float2*>(raw(e));
#pragma unroll 1
            for (int s = 0; s < C::P; s++) {
                float hi[C::SC], lo[C::SC];
#pragma unroll
                for (int t = 0; t < R; t++) {
                    const float2 x = rd[(s * R + t) * 128 + v];
                    tc::split(x.x, hi[2 * t], lo[2 * t]);
                    tc::split(x.y, hi[2 * t + 1], lo[2 * t + 1]);
                }
                const uint32_t ta = tmem + lb + uint32_t(slot * C::ACOLS + s * C::SC);
                tc::tmem_st_cols<C::SC>(ta, hi);
                tc::tmem_st_cols<C::SC>(ta + C::P * C::SC, lo);
            }
            tc::tmem_wait_st();
            tc::fence_before_sync();
            if (tid == 0) btrace(J, 1);
            tc::mbar_arrive(&raw_empty[e]);
            tc::mbar_arrive(&a1_ready[slot]);
        }
    } else if (warp < 8) {
        // ---- epilogue: level-1 drain + re-split, level-2 drain + store ----
        const int v = tid - 128;
        const uint32_t lb = uint32_t((warp - 4) * 32) << 16;
        for (int J = 0; J < int(njobs); J++) {
            const int it = int(unsigned(J) / unsigned(nvt));
            const int vt = J - it * nvt;
            const int64_t g = blockIdx.x + int64_t(it) * gridDim.x;
            const int slot = int(J % C::NABUF);
            const uint32_t ph = uint32_t(J & 1);
            // every level-1 MMA must be complete before the in-place re-split (an output slot of unit 0 is an
            // input slot of unit 1)
            tc::mbar_wait(&d1_full, ph);
            tc::fence_after_sync();
            if (v == 0) btrace(J, 3);
#pragma unroll 1
            for (int u = 0; u < C::U; u++) {
                float d[C::NU];
                tc::tmem_ld_cols<C::NU>(tmem + lb + uint32_t(C::D1_OFF + u * C::NB), d);
                tc::tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 2; e++) {
                    float hi[C::SC], lo[C::SC];
#pragma unroll
                    for (int i = 0; i < C::SC; i++) tc::split(d[e * C::SC + i], hi[i], lo[i]);
                    const uint32_t ta = tmem + lb + uint32_t(slot * C::ACOLS + (2 * e + u) * C::SC);
                    tc::tmem_st_cols<C::SC>(ta, hi);
                    tc::tmem_st_cols<C::SC>(ta + C::P * C::SC, lo);
                }
            }
            tc::tmem_wait_st();
            tc::fence_before_sync();
            if (v == 0) btrace(J, 4);
            tc::mbar_arrive(&d1_free);
            tc::mbar_arrive(&a2_ready[slot]);

            tc::mbar_wait(&d2_full, ph);
            tc::fence_after_sync();
            if (v == 0) btrace(J, 6);
            float d[C::U][C::NU];
#pragma unroll
            for (int u = 0; u < C::U; u++) tc::tmem_ld_cols<C::NU>(tmem + lb + uint32_t(C::D2_OFF + u * C::NB), d[u]);
            tc::tmem_wait_ld();
            tc::fence_before_sync();
            tc::mbar_arrive(&d2_free);
            const int vg = vt * 128 + v;
            if (vg < nv) {
                const int64_t a0 = g >> shg, bq = g & ((int64_t(1) << shg) - 1);
#pragma unroll
                for (int u = 0; u < C::U; u++)
#pragma unroll
                    for (int e = 0; e < 2; e++) {
                        const int64_t p = (((a0 << 2) + 2 * u + e) << shg) + bq;
                        float2* o = bfs::pair_out(out, po, p, R, nv) + vg;
#pragma unroll
                        for (int t = 0; t < R; t++)
                            o[int64_t(t) * nv] = make_float2(d[u][e * C::SC + 2 * t], d[u][e * C::SC + 2 * t + 1]);
                    }
            }
        }
    } else if (warp == 8) {
        // ---- loader ----
        if (lane == 0) {
            for (int J = 0; J < int(njobs); J++) {
                const int it = int(unsigned(J) / unsigned(nvt));
                const int vt = J - it * nvt;
                const int64_t g = blockIdx.x + int64_t(it) * gridDim.x;
                const int e = int(J & 1);
                if (J >= 2) tc::mbar_wait(&raw_empty[e], uint32_t((J >> 1) - 1) & 1);
                btrace(J, 8);
                const int v0 = vt * 128, vw = min(128, nv - v0);
                const uint32_t row_bytes = uint32_t(vw) * 8;
                tc::mbar_arrive_expect_tx(&raw_full[e], C::P * R * row_bytes);
                const int64_t pin = rh ? bfs::recv_index(g * C::P, rh, rhg) : g * C::P;   // P pairs contiguous
                for (int row = 0; row < C::P * R; row++)
                    tc::bulk_g2s(raw(e) + row * 128 * 8, in + (pin * R + row) * int64_t(nv) + v0, row_bytes,
                                 &raw_full[e]);
            }
        }
    } else if (warp == 9) {
        // ---- MMA issuer (whole warp, one elected lane issues) ----
        constexpr uint32_t idesc = tc::idesc_tf32(128, C::NB);
        constexpr uint32_t LBO_B = (C::NB / 8) * 128;
        const uint64_t dW = tc::desc_kmajor(tc::smem_u32(sm_band + C::OFF_W), LBO_B);
        for (int J = 0; J < int(njobs); J++) {
            const int it = int(unsigned(J) / unsigned(nvt));
            const int vt = J - it * nvt;
            const int wb = int(it % C::NWBUF), slot = int(J % C::NABUF);
            if (vt == 0) tc::mbar_wait(&w_full[wb], uint32_t(it / C::NWBUF) & 1);
#pragma unroll 1
            for (int m = 0; m < 2; m++) {
                if (lane == 0) btrace(J, m == 0 ? 9 : 10);
                tc::mbar_wait(m == 0 ? &a1_ready[slot] : &a2_ready[slot], uint32_t(J / C::NABUF) & 1);
                if (J >= 1) tc::mbar_wait(m == 0 ? &d1_free : &d2_free, uint32_t(J - 1) & 1);
                tc::fence_after_sync();
#pragma unroll
                for (int u = 0; u < C::U; u++) {
                    const uint32_t d = tmem + uint32_t((m == 0 ? C::D1_OFF : C::D2_OFF) + u * C::NB);
                    const uint32_t ahi = tmem + uint32_t(slot * C::ACOLS + 2 * u * C::SC);
                    const uint64_t bhi = tc::desc_add(dW, wb * C::WSET + ((m * C::U + u) * 2) * C::WT);
#pragma unroll
                    for (int q = 0; q < 3; q++) {
                        const int pass = kPassOrder[q];
                        const uint32_t a = ahi + (pass == 1 ? C::P * C::SC : 0);
                        const uint64_t b = pass == 2 ? tc::desc_add(bhi, C::WT) : bhi;
#pragma unroll
                        for (int ks = 0; ks < C::KU / 8; ks++)
                            tc::mma_tf32_ts_warp(d, a + ks * 8, tc::desc_add(b, ks * 2 * LBO_B), idesc,
                                                 (q | ks) ? 1u : 0u);
                    }
                }
                if (lane == 0) btrace(J, m == 0 ? 2 : 5);
                tc::commit_warp(m == 0 ? &d1_full : &d2_full);
            }
            tc::commit_warp(&a_free[slot]);
            if (vt == nvt - 1) tc::commit_warp(&w_free[wb]);
            __syncwarp();
            if (lane == 0) btrace(J, 11);
        }
    } else {
        // ---- weights (warps 10-11): compact r x 2r blocks -> embedded hi/lo B tiles, one group ahead ----
        const int wt = tid - 320;
        for (int it = 0; it < int(nit); it++) {
            const int64_t g = blockIdx.x + int64_t(it) * gridDim.x;
            const int wb = int(it % C::NWBUF);
            if (it >= C::NWBUF) tc::mbar_wait(&w_free[wb], uint32_t(it / C::NWBUF - 1) & 1);
            const int64_t a0 = g >> shg, bq = g & ((int64_t(1) << shg) - 1);
            float2 w[C::WPT];
#pragma unroll
            for (int q = 0; q < C::WPT; q++) {
                const int idx = wt + 64 * q;
                w[q] = make_float2(0.f, 0.f);
                if (idx < C::WTASKS) {
                    // idx = (((m U + u) 2 + e) 2R + kcol) R + t
                    const int t = idx % R, kcol = (idx / R) % (2 * R), e = (idx / (2 * R * R)) & 1;
                    const int mu = idx / (4 * R * R), m = mu / C::U, u = mu % C::U;
                    const int lv = m + 1, ep = u >> (2 - lv), i = u & ((1 << (2 - lv)) - 1);
                    const int64_t p = (((a0 << lv) + 2 * ep + e) << (LN - lin - lv)) + (bq << (2 - lv)) + i;
                    w[q] = __ldg((lv == 1 ? W1 : W2) + p * (2 * R * R) + kcol * R + t);
                }
            }
#pragma unroll
            for (int q = 0; q < C::WPT; q++) {
                const int idx = wt + 64 * q;
                if (idx < C::WTASKS) {
                    const int t = idx % R, kcol = (idx / R) % (2 * R), e = (idx / (2 * R * R)) & 1;
                    const int mu = idx / (4 * R * R), m = mu / C::U, u = mu % C::U;
                    float hr, lr, hi_, li;
                    tc::split(w[q].x, hr, lr);
                    tc::split(w[q].y, hi_, li);
                    const int n = e * C::SC + 2 * t, k = 2 * kcol;
                    uint8_t* th = wtile(wb, m, u, 0);
                    uint8_t* tl = wtile(wb, m, u, 1);
                    const uint32_t o0 = tc::kmaj_off(n, k, C::NB), o1 = tc::kmaj_off(n + 1, k, C::NB);
                    *reinterpret_cast<float2*>(th + o0) = make_float2(hr, -hi_);
                    *reinterpret_cast<float2*>(tl + o0) = make_float2(lr, -li);
                    *reinterpret_cast<float2*>(th + o1) = make_float2(hi_, hr);
                    *reinterpret_cast<float2*>(tl + o1) = make_float2(li, lr);
                }
            }
            tc::fence_proxy_async();
            tc::mbar_arrive(&w_full[wb]);
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) {
        tc::fence_after_sync();
        tc::tmem_dealloc<C::TMEM_COLS>(tmem);
    }
}

// ---------------------------------------------------------------------------------------------
// Two-pipeline variant of the band (r <= 10; selectable with BF_OPT_BAND_PIPELINES = 2, not the default): jobs alternate between two TMEM pipelines (A buffer +
// one accumulator region shared by both levels), so while one job's level-1 accumulator is drained and
// re-split (E1) the tensor pipe runs the other job's MMAs.  Warp roles: 0-3 split (all jobs, in order),
// 4-7 / 8-11 epilogue of pipeline 0 / 1 (E1 and E2 of its jobs), 12 loader, 13 MMA, 14-15 weights.
// MMA order: L1(J), L1(J+1), L2(J), L2(J+1), L1(J+2), ...
// ---------------------------------------------------------------------------------------------
template <int R>
struct Band2P {
    using B = BandTC<R>;
    static constexpr int PCOLS = B::ACOLS + B::DCOLS;   // one pipeline: A (hi, lo) + accumulators
    static constexpr bool FITS = 2 * PCOLS <= 512;
    static constexpr int TMEM_COLS = 512;
};

template <int R>
__global__ void __launch_bounds__(512, 1)
    band_tc2p_kernel(const float2* __restrict__ in, float2* __restrict__ out, const float2* __restrict__ W1,
                     const float2* __restrict__ W2, int LN, int l_first, int nv, int rh, int rhg, const bfs::PeerOut po)
{
    using C = BandTC<R>;
    using Q = Band2P<R>;
    extern __shared__ __align__(128) uint8_t sm_band[];
    auto raw = [&](int e) { return sm_band + e * C::RAW; };
    auto wtile = [&](int wb, int m, int u, int lo) {
        return sm_band + C::OFF_W + wb * C::WSET + ((m * C::U + u) * 2 + lo) * C::WT;
    };
    __shared__ uint64_t raw_full[2], raw_empty[2], w_full[2], w_free[2];
    __shared__ uint64_t a1_ready[2], a2_ready[2], a_free[2], d1_full[2], d2_full[2], d2_free[2];   // per pipeline
    __shared__ uint32_t tmem_base;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t N = int64_t(1) << LN;
    const int lin = l_first - 1, shg = LN - lin - 2;
    const int64_t ngroups = N >> 2;
    const int nvt = (nv + 127) / 128;
    const int nit = int((ngroups - blockIdx.x + gridDim.x - 1) / gridDim.x);
    const int njobs = nit * nvt;

    if (warp == 0) tc::tmem_alloc<Q::TMEM_COLS>(&tmem_base);
    if (tid == 0) {
        for (int i = 0; i < 2; i++) {
            tc::mbar_init(&raw_full[i], 1);
            tc::mbar_init(&raw_empty[i], 128);
            tc::mbar_init(&w_full[i], 64);
            tc::mbar_init(&w_free[i], 1);
            tc::mbar_init(&a1_ready[i], 128);
            tc::mbar_init(&a2_ready[i], 128);
            tc::mbar_init(&a_free[i], 1);
            tc::mbar_init(&d1_full[i], 1);
            tc::mbar_init(&d2_full[i], 1);
            tc::mbar_init(&d2_free[i], 128);
        }
        tc::mbar_fence_init();
    }
    if constexpr (C::NB > C::NU) {   // zero the pad rows of every B tile (never written afterwards)
        constexpr int PADQ = (C::NB - C::NU) * C::KU / 4;
        for (int idx = tid; idx < C::NWBUF * 2 * C::U * 2 * PADQ; idx += blockDim.x) {
            const int tile = idx / PADQ, o = idx % PADQ;
            const int row = C::NU + o % (C::NB - C::NU), k = 4 * (o / (C::NB - C::NU));
            st_f4(sm_band + C::OFF_W + tile * C::WT, tc::kmaj_off(row, k, C::NB), make_float4(0, 0, 0, 0));
        }
    }
    tc::fence_proxy_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tmem_base;
    auto abuf = [&](int p) { return tmem + uint32_t(p * Q::PCOLS); };               // hi at +0, lo at +P SC
    auto dbuf = [&](int p) { return tmem + uint32_t(p * Q::PCOLS + C::ACOLS); };    // unit u at +u NB

    if (warp < 4) {
        // ---- split: raw rows -> the job's pipeline A buffer (TMEM), lane = vector ----
        const int v = tid;
        const uint32_t lb = uint32_t(warp * 32) << 16;
        for (int J = 0; J < njobs; J++) {
            const int e = J & 1, p = J & 1, use = J >> 1;
            tc::mbar_wait(&raw_full[e], uint32_t(use & 1));
            if (use > 0) tc::mbar_wait(&a_free[p], uint32_t(use - 1) & 1);
            tc::fence_after_sync();
            if (tid == 0) btrace(J, 0);
            const float2* rd = reinterpret_cast<const float2*>(raw(e));
#pragma unroll 1
            for (int s = 0; s < C::P; s++) {
                float hi[C::SC], lo[C::SC];
#pragma unroll
                for (int t = 0; t < R; t++) {
                    const float2 x = rd[(s * R + t) * 128 + v];
                    tc::split(x.x, hi[2 * t], lo[2 * t]);
                    tc::split(x.y, hi[2 * t + 1], lo[2 * t + 1]);
                }
                const uint32_t ta = abuf(p) + lb + uint32_t(s * C::SC);
                tc::tmem_st_cols<C::SC>(ta, hi);
                tc::tmem_st_cols<C::SC>(ta + C::P * C::SC, lo);
            }
            tc::tmem_wait_st();
            tc::fence_before_sync();
            if (tid == 0) btrace(J, 1);
            tc::mbar_arrive(&raw_empty[e]);
            tc::mbar_arrive(&a1_ready[p]);
        }
    } else if (warp < 12) {
        // ---- epilogue of pipeline p: level-1 drain + re-split, level-2 drain + store ----
        const int p = (warp - 4) >> 2;
        const int v = ((warp - 4) & 3) * 32 + lane;
        const uint32_t lb = uint32_t(((warp - 4) & 3) * 32) << 16;
        for (int J = p; J < njobs; J += 2) {
            const int use = J >> 1;
            const int it = int(unsigned(J) / unsigned(nvt));
            const int vt = J - it * nvt;
            const int64_t g = blockIdx.x + int64_t(it) * gridDim.x;
            const uint32_t ph = uint32_t(use & 1);
            tc::mbar_wait(&d1_full[p], ph);
            tc::fence_after_sync();
            if (v == 0) btrace(J, 3);
#pragma unroll 1
            for (int u = 0; u < C::U; u++) {
                float d[C::NU];
                tc::tmem_ld_cols<C::NU>(dbuf(p) + lb + uint32_t(u * C::NB), d);
                tc::tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 2; e++) {
                    float hi[C::SC], lo[C::SC];
#pragma unroll
                    for (int i = 0; i < C::SC; i++) tc::split(d[e * C::SC + i], hi[i], lo[i]);
                    const uint32_t ta = abuf(p) + lb + uint32_t((2 * e + u) * C::SC);
                    tc::tmem_st_cols<C::SC>(ta, hi);
                    tc::tmem_st_cols<C::SC>(ta + C::P * C::SC, lo);
                }
            }
            tc::tmem_wait_st();
            tc::fence_before_sync();
            if (v == 0) btrace(J, 4);
            tc::mbar_arrive(&a2_ready[p]);   // A is ready for level 2 and the accumulator is drained

            tc::mbar_wait(&d2_full[p], ph);
            tc::fence_after_sync();
            if (v == 0) btrace(J, 6);
            float d[C::U][C::NU];
#pragma unroll
            for (int u = 0; u < C::U; u++) tc::tmem_ld_cols<C::NU>(dbuf(p) + lb + uint32_t(u * C::NB), d[u]);
            tc::tmem_wait_ld();
            tc::fence_before_sync();
            tc::mbar_arrive(&d2_free[p]);
            const int vg = vt * 128 + v;
            if (vg < nv) {
                const int64_t a0 = g >> shg, bq = g & ((int64_t(1) << shg) - 1);
#pragma unroll
                for (int u = 0; u < C::U; u++)
#pragma unroll
                    for (int e = 0; e < 2; e++) {
                        const int64_t q = (((a0 << 2) + 2 * u + e) << shg) + bq;
                        float2* o = out + q * R * int64_t(nv) + vg;
#pragma unroll
                        for (int t = 0; t < R; t++)
                            o[int64_t(t) * nv] = make_float2(d[u][e * C::SC + 2 * t], d[u][e * C::SC + 2 * t + 1]);
                    }
            }
        }
    } else if (warp == 12) {
        // ---- loader ----
        if (lane == 0) {
            for (int J = 0; J < njobs; J++) {
                const int it = int(unsigned(J) / unsigned(nvt));
                const int vt = J - it * nvt;
                const int64_t g = blockIdx.x + int64_t(it) * gridDim.x;
                const int e = J & 1;
                if (J >= 2) tc::mbar_wait(&raw_empty[e], uint32_t((J >> 1) - 1) & 1);
                btrace(J, 8);
                const int v0 = vt * 128, vw = min(128, nv - v0);
                const uint32_t row_bytes = uint32_t(vw) * 8;
                tc::mbar_arrive_expect_tx(&raw_full[e], C::P * R * row_bytes);
                const int64_t pin = rh ? bfs::recv_index(g * C::P, rh, rhg) : g * C::P;   // P pairs contiguous
                for (int row = 0; row < C::P * R; row++)
                    tc::bulk_g2s(raw(e) + row * 128 * 8, in + (pin * R + row) * int64_t(nv) + v0, row_bytes,
                                 &raw_full[e]);
            }
        }
    } else if (warp == 13) {
        // ---- MMA issuer (whole warp, one elected lane issues) ----
        constexpr uint32_t idesc = tc::idesc_tf32(128, C::NB);
        constexpr uint32_t LBO_B = (C::NB / 8) * 128;
        const uint64_t dW = tc::desc_kmajor(tc::smem_u32(sm_band + C::OFF_W), LBO_B);
        auto level = [&](int J, int m) {
            const int it = int(unsigned(J) / unsigned(nvt));
            const int vt = J - it * nvt;
            const int wb = it % C::NWBUF, p = J & 1, use = J >> 1;
            if (lane == 0) btrace(J, m == 0 ? 9 : 10);
            if (m == 0) {
                if (vt == 0) tc::mbar_wait(&w_full[wb], uint32_t(it / C::NWBUF) & 1);
                tc::mbar_wait(&a1_ready[p], uint32_t(use & 1));
                if (use > 0) tc::mbar_wait(&d2_free[p], uint32_t(use - 1) & 1);
            } else {
                tc::mbar_wait(&a2_ready[p], uint32_t(use & 1));
            }
            tc::fence_after_sync();
#pragma unroll
            for (int u = 0; u < C::U; u++) {
                const uint32_t d = dbuf(p) + uint32_t(u * C::NB);
                const uint32_t ahi = abuf(p) + uint32_t(2 * u * C::SC);
                const uint64_t bhi = tc::desc_add(dW, wb * C::WSET + ((m * C::U + u) * 2) * C::WT);
#pragma unroll
                for (int q = 0; q < 3; q++) {
                    const int pass = kPassOrder[q];
                    const uint32_t a = ahi + (pass == 1 ? C::P * C::SC : 0);
                    const uint64_t b = pass == 2 ? tc::desc_add(bhi, C::WT) : bhi;
#pragma unroll
                    for (int ks = 0; ks < C::KU / 8; ks++)
                        tc::mma_tf32_ts_warp(d, a + ks * 8, tc::desc_add(b, ks * 2 * LBO_B), idesc, (q | ks) ? 1u : 0u);
                }
            }
            if (lane == 0) btrace(J, m == 0 ? 2 : 5);
            if (m == 0) {
                tc::commit_warp(&d1_full[p]);
            } else {
                tc::commit_warp(&d2_full[p]);
                tc::commit_warp(&a_free[p]);
                if (vt == nvt - 1) tc::commit_warp(&w_free[wb]);
            }
            __syncwarp();
        };
        for (int J0 = 0; J0 < njobs; J0 += 2) {
            level(J0, 0);
            if (J0 + 1 < njobs) level(J0 + 1, 0);
            level(J0, 1);
            if (J0 + 1 < njobs) level(J0 + 1, 1);
        }
    } else {
        // ---- weights (warps 14-15): compact r x 2r blocks -> embedded hi/lo B tiles, one group ahead ----
        const int wt = tid - 448;
        for (int it = 0; it < nit; it++) {
            const int64_t g = blockIdx.x + int64_t(it) * gridDim.x;
            const int wb = it % C::NWBUF;
            if (it >= C::NWBUF) tc::mbar_wait(&w_free[wb], uint32_t(it / C::NWBUF - 1) & 1);
            const int64_t a0 = g >> shg, bq = g & ((int64_t(1) << shg) - 1);
            constexpr int BATCH = 13;   // loads in flight per thread (bounded registers)
#pragma unroll 1
            for (int q0 = 0; q0 < C::WPT; q0 += BATCH) {
                float2 w[BATCH];
#pragma unroll
                for (int q = 0; q < BATCH; q++) {
                    const int idx = wt + 64 * (q0 + q);
                    w[q] = make_float2(0.f, 0.f);
                    if (q0 + q < C::WPT && idx < C::WTASKS) {
                        const int t = idx % R, kcol = (idx / R) % (2 * R), e = (idx / (2 * R * R)) & 1;
                        const int mu = idx / (4 * R * R), m = mu / C::U, u = mu % C::U;
                        const int lv = m + 1, ep = u >> (2 - lv), i = u & ((1 << (2 - lv)) - 1);
                        const int64_t pr = (((a0 << lv) + 2 * ep + e) << (LN - lin - lv)) + (bq << (2 - lv)) + i;
                        w[q] = __ldg((lv == 1 ? W1 : W2) + pr * (2 * R * R) + kcol * R + t);
                    }
                }
#pragma unroll
                for (int q = 0; q < BATCH; q++) {
                    const int idx = wt + 64 * (q0 + q);
                    if (q0 + q < C::WPT && idx < C::WTASKS) {
                        const int t = idx % R, kcol = (idx / R) % (2 * R), e = (idx / (2 * R * R)) & 1;
                        const int mu = idx / (4 * R * R), m = mu / C::U, u = mu % C::U;
                        float hr, lr, hi_, li;
                        tc::split(w[q].x, hr, lr);
                        tc::split(w[q].y, hi_, li);
                        const int n = e * C::SC + 2 * t, k = 2 * kcol;
                        uint8_t* th = wtile(wb, m, u, 0);
                        uint8_t* tl = wtile(wb, m, u, 1);
                        const uint32_t o0 = tc::kmaj_off(n, k, C::NB), o1 = tc::kmaj_off(n + 1, k, C::NB);
                        *reinterpret_cast<float2*>(th + o0) = make_float2(hr, -hi_);
                        *reinterpret_cast<float2*>(tl + o0) = make_float2(lr, -li);
                        *reinterpret_cast<float2*>(th + o1) = make_float2(hi_, hr);
                        *reinterpret_cast<float2*>(tl + o1) = make_float2(li, lr);
                    }
                }
            }
            tc::fence_proxy_async();
            tc::mbar_arrive(&w_full[wb]);
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) {
        tc::fence_after_sync();
        tc::tmem_dealloc<Q::TMEM_COLS>(tmem);
    }
}

// =============================================================================================
// Composed two-level band (the default tensor-core band).  The two transfer levels of a band map a
// group of 4 input pairs to 4 output pairs, and each output pair reaches each input pair through
// exactly one pair of the middle level (eqn:2 P:748-752 / eqn:3 P:780-785 applied twice), so the band
// is ONE dense 4 x 4 block operator per group,
//     C[o][i] = W2[o][.., s'] W1[(s', u')][.., s]       (o = 2u' + e', i = 2s' + s, r x r complex blocks)
// with the same 16 r^2 complex MACs per vector and group as the two levels applied one after the other.
// The weight warps form C per group from the two levels' compact blocks (FP32; 16 r^3 complex MACs per
// group, reused by every vector tile of the group) and write it real-embedded and split hi/lo as one
// K = N = 8r B tile; per job the tensor pipe then runs a single accumulation chain (3 passes x r K-steps,
// N = 8r) and the level-1 drain / re-split of band_tc_kernel disappears.
// Warps: 0-3 split the raw rows into A (TMEM), 4-11 epilogue (lane quadrant warp % 4, output half
// (warp - 4) / 4), 12 loader, 13 MMA issuer, 14-15 weights (compose one group ahead).
// =============================================================================================
template <int R>
struct BandCmp {
    static constexpr int P = 4;
    static constexpr int SC = 2 * R;                                  // real columns of one pair slot
    static constexpr int KB = P * SC;                                 // MMA K = N = 8r
    static constexpr int NB = KB;
    static constexpr int ACOLS = 2 * KB;                              // A buffer: hi at +0, lo at +KB
    static constexpr int NABUF = (2 * ACOLS + 2 * NB <= 512) ? 2 : 1;
    static constexpr int NDBUF = (NABUF * ACOLS + 2 * NB <= 512) ? 2 : 1;
    static constexpr int D_OFF = NABUF * ACOLS;
    static constexpr int TMEM_COLS = tmem_cols_pow2<D_OFF + NDBUF * NB>();
    static constexpr uint32_t SLOT = uint32_t(R) * 128 * 8;          // raw rows of one pair, one vector tile
    static constexpr uint32_t BLK = 2 * R * R;                        // complex entries of one compact block
    static constexpr uint32_t WST = 2 * P * BLK * 8;                  // staged compact blocks, both levels
    static constexpr uint32_t WT = uint32_t(NB) * KB * 4;             // one B tile (hi or lo)
    static constexpr uint32_t WSET = 2 * WT;
    static constexpr size_t LIM = 232448 - 1024;
    static constexpr int NWBUF = (8 * size_t(SLOT) + 2 * size_t(WST) + 2 * size_t(WSET) <= LIM) ? 2 : 1;
    // raw ring of single-pair slots (freed one pair at a time, so more bytes stay in flight)
    static constexpr int NQ_FIT = int((LIM - 2 * size_t(WST) - NWBUF * size_t(WSET)) / SLOT);
#ifdef BF_BAND_NQ
    static constexpr int NQ = NQ_FIT > BF_BAND_NQ ? BF_BAND_NQ : NQ_FIT;
#else
    static constexpr int NQ = NQ_FIT > 16 ? 16 : NQ_FIT;
#endif
    static constexpr uint32_t OFF_WST = uint32_t(NQ) * SLOT;          // two staging buffers (prefetch)
    static constexpr uint32_t OFF_W = OFF_WST + 2 * WST;
    static constexpr size_t SMEM = size_t(OFF_W) + NWBUF * size_t(WSET);
    static constexpr int ITEMS = P * P * R * 2;                       // (o, i, t', j half) compose items
#ifdef BF_BAND_SPLIT4
    static constexpr int NSPLIT = 4;                                  // split warps (the rest of 0-11: epilogue)
#else
    static constexpr int NSPLIT = 8;
#endif
    static_assert(KB % 16 == 0 && D_OFF + NDBUF * NB <= 512 && OFF_W % 128 == 0 && WT % 128 == 0 && NQ >= 8 &&
                      SMEM <= LIM, "composed band shape");
};

template <int R>
__global__ void __launch_bounds__(512, 1)
    band_cmp_kernel(const __grid_constant__ CUtensorMap tin, float2* __restrict__ out, const float2* __restrict__ W1,
                    const float2* __restrict__ W2, int LN, int l_first, int nv, int rh, int rhg, const bfs::PeerOut po)
{
    using C = BandCmp<R>;
    extern __shared__ __align__(128) uint8_t sm_cmp[];
    __shared__ uint64_t slot_full[16], slot_empty[16];
    __shared__ uint64_t a_ready[2], a_free[2], d_full[2], d_free[2], w_full[2], w_free[2];
    __shared__ uint64_t wst_full[2];
    __shared__ uint32_t tmem_base;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t N = int64_t(1) << LN;
    const int lin = l_first - 1, shg = LN - lin - 2;
    const int64_t ngroups = N >> 2;
    const int nvt = (nv + 127) / 128;
    const int nit = int((ngroups - blockIdx.x + gridDim.x - 1) / gridDim.x);
    const int njobs = nit * nvt;

    if (warp == 0) tc::tmem_alloc<C::TMEM_COLS>(&tmem_base);
    if (tid == 0) {
        for (int i = 0; i < C::NQ; i++) {
            tc::mbar_init(&slot_full[i], 1);
            tc::mbar_init(&slot_empty[i], 128);
        }
        for (int i = 0; i < 2; i++) {
            tc::mbar_init(&a_ready[i], 32 * C::NSPLIT);
            tc::mbar_init(&a_free[i], 1);
            tc::mbar_init(&d_full[i], 1);
            tc::mbar_init(&d_free[i], 32 * (12 - C::NSPLIT));
            tc::mbar_init(&w_full[i], 64);
            tc::mbar_init(&w_free[i], 1);
            tc::mbar_init(&wst_full[i], 1);
        }
        tc::mbar_fence_init();
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tmem_base;

    if (warp < C::NSPLIT) {
        // ---- split: raw rows -> A buffer (TMEM), lane = vector; with 8 split warps each lane quadrant has two
        //      warps, one per half of the group's 4 pair slots ----
        const int qd = warp & 3, hs = warp >> 2;
        const int v = qd * 32 + lane;
        constexpr int SPW = C::P * 4 / C::NSPLIT;   // pair slots per split warp
        const uint32_t lb = uint32_t(qd * 32) << 16;
        for (int J = 0; J < njobs; J++) {
            const int ab = J % C::NABUF, use = J / C::NABUF;
            if (use > 0) tc::mbar_wait(&a_free[ab], uint32_t(use - 1) & 1);
            tc::fence_after_sync();
            if (tid == 0) btrace(J, 1);
#pragma unroll 1
            for (int s = hs * SPW; s < (hs + 1) * SPW; s++) {
                const int k = J * C::P + s, q = k % C::NQ;
                tc::mbar_wait(&slot_full[q], uint32_t(k / C::NQ) & 1);
                if (tid == 0 && s == 0) btrace(J, 0);
                const float2* rd = reinterpret_cast<const float2*>(sm_cmp + q * C::SLOT);
                float hi[C::SC], lo[C::SC];
#pragma unroll
                for (int t = 0; t < R; t++) {
                    const float2 x = rd[t * 128 + v];
#ifdef BF_EXP_NO_SPLIT
                    hi[2 * t] = x.x; lo[2 * t] = 0.f; hi[2 * t + 1] = x.y; lo[2 * t + 1] = 0.f;
#else
                    tc::split(x.x, hi[2 * t], lo[2 * t]);
                    tc::split(x.y, hi[2 * t + 1], lo[2 * t + 1]);
#endif
                }
                tc::mbar_arrive(&slot_empty[q]);   // the slot's values are in registers
                const uint32_t ta = tmem + lb + uint32_t(ab * C::ACOLS + s * C::SC);
#ifndef BF_EXP_NO_TMEM_ST
                tc::tmem_st_cols<C::SC>(ta, hi);
                tc::tmem_st_cols<C::SC>(ta + C::KB, lo);
#endif
            }
            tc::tmem_wait_st();
            tc::fence_before_sync();
            if (tid == 0) btrace(J, 2);
            tc::mbar_arrive(&a_ready[ab]);
        }
    } else if (warp < 12) {
        // ---- epilogue: drain the accumulator row in halves of 2 output pairs and store them (8 epilogue warps:
        //      one half each; 4 warps: both halves) ----
        constexpr int HPW = 8 / (12 - C::NSPLIT);
        const int q = warp & 3, hf0 = ((warp - C::NSPLIT) >> 2) * HPW;
        const int v = q * 32 + lane;
        const uint32_t lb = uint32_t(q * 32) << 16;
        for (int J = 0; J < njobs; J++) {
            const int it = int(unsigned(J) / unsigned(nvt));
            const int vt = J - it * nvt;
            const int64_t g = blockIdx.x + int64_t(it) * gridDim.x;
            const int db = J % C::NDBUF;
            tc::mbar_wait(&d_full[db], uint32_t(J / C::NDBUF) & 1);
            tc::fence_after_sync();
            if (warp == C::NSPLIT && lane == 0) btrace(J, 5);
            const int vg = vt * 128 + v;
            const int64_t a0 = g >> shg, bq = g & ((int64_t(1) << shg) - 1);
#pragma unroll 1
            for (int h = 0; h < HPW; h++) {
                const int hf = hf0 + h;
                float d[2 * C::SC];
                tc::tmem_ld_cols<2 * C::SC>(tmem + lb + uint32_t(C::D_OFF + db * C::NB + hf * 2 * C::SC), d);
                tc::tmem_wait_ld();
                if (h == HPW - 1) {
                    tc::fence_before_sync();
                    tc::mbar_arrive(&d_free[db]);
                }
#ifdef BF_EXP_NO_STORE
                if (vg < 0) {
#else
                if (vg < nv) {
#endif
                    if (!po.on) {
                        // output pairs 2 hf, 2 hf + 1 are 2^shg pairs apart; rows t are nv apart (pointer walk)
                        const int64_t p = (((a0 << 2) + 2 * hf) << shg) + bq;
                        float2* o = out + p * R * int64_t(nv) + vg;
                        const int64_t pstep = (int64_t(1) << shg) * R * int64_t(nv) - int64_t(R) * nv;
#pragma unroll
                        for (int oo = 0; oo < 2; oo++) {
#pragma unroll
                            for (int t = 0; t < R; t++) {
                                *o = make_float2(d[oo * C::SC + 2 * t], d[oo * C::SC + 2 * t + 1]);
                                o += nv;
                            }
                            o += pstep;
                        }
                    } else {
#pragma unroll
                        for (int oo = 0; oo < 2; oo++) {
                            const int64_t p = (((a0 << 2) + 2 * hf + oo) << shg) + bq;
                            float2* o = bfs::pair_out(out, po, p, R, nv) + vg;
#pragma unroll
                            for (int t = 0; t < R; t++)
                                o[int64_t(t) * nv] = make_float2(d[oo * C::SC + 2 * t], d[oo * C::SC + 2 * t + 1]);
                        }
                    }
                }
            }
            if (warp == C::NSPLIT && lane == 0) btrace(J, 6);
        }
    } else if (warp == 12) {
        // ---- loader: the group's 4 r raw coefficient rows of one vector tile, one 2-D tensor copy per pair
        //      (40 separate 1-KB bulk copies measured ~85 clk each to issue: the loader was the bottleneck) ----
        for (int J = 0; J < njobs; J++) {
            const int it = int(unsigned(J) / unsigned(nvt));
            const int vt = J - it * nvt;
            const int64_t g = blockIdx.x + int64_t(it) * gridDim.x;
            const int64_t pin = rh ? bfs::recv_index(g * C::P, rh, rhg) : g * C::P;   // P pairs contiguous
            for (int s = 0; s < C::P; s++) {
                const int k = J * C::P + s, q = k % C::NQ;
                if (k >= C::NQ) tc::mbar_wait(&slot_empty[q], uint32_t(k / C::NQ - 1) & 1);
                if (lane == 0) {
                    if (s == 0) btrace(J, 7);
                    tc::mbar_arrive_expect_tx(&slot_full[q], C::SLOT);   // whole box (ragged tile: zero fill)
                    tc::tma_load_2d(sm_cmp + q * C::SLOT, &tin, 2 * vt * 128, int((pin + s) * R), &slot_full[q]);
                }
                __syncwarp();
            }
            if (lane == 0) btrace(J, 8);
        }
    } else if (warp == 13) {
        // ---- MMA issuer (whole warp, one elected lane issues): one chain of 3 x (8r / 8) MMAs per job ----
        constexpr uint32_t idesc = tc::idesc_tf32(128, C::NB);
        constexpr uint32_t LBO_B = (C::NB / 8) * 128;
        const uint64_t dW = tc::desc_kmajor(tc::smem_u32(sm_cmp + C::OFF_W), LBO_B);
        for (int J = 0; J < njobs; J++) {
            const int it = int(unsigned(J) / unsigned(nvt));
            const int vt = J - it * nvt;
            const int wb = it % C::NWBUF, ab = J % C::NABUF, db = J % C::NDBUF;
            if (vt == 0) tc::mbar_wait(&w_full[wb], uint32_t(it / C::NWBUF) & 1);
            if (lane == 0) btrace(J, 11);
            tc::mbar_wait(&a_ready[ab], uint32_t(J / C::NABUF) & 1);
            if (J >= C::NDBUF) tc::mbar_wait(&d_free[db], uint32_t(J / C::NDBUF - 1) & 1);
            tc::fence_after_sync();
            if (lane == 0) btrace(J, 3);
            const uint32_t d = tmem + uint32_t(C::D_OFF + db * C::NB);
            const uint32_t ahi = tmem + uint32_t(ab * C::ACOLS);
            const uint64_t bhi = tc::desc_add(dW, wb * C::WSET);
#pragma unroll
            for (int qq = 0; qq < 3; qq++) {
                const int pass = kPassOrder[qq];
                const uint32_t a = ahi + (pass == 1 ? C::KB : 0);
                const uint64_t b = pass == 2 ? tc::desc_add(bhi, C::WT) : bhi;
#pragma unroll
                for (int ks = 0; ks < C::KB / 8; ks++)
                    tc::mma_tf32_ts_warp(d, a + ks * 8, tc::desc_add(b, ks * 2 * LBO_B), idesc, (qq | ks) ? 1u : 0u);
            }
            tc::commit_warp(&d_full[db]);
            tc::commit_warp(&a_free[ab]);
            if (vt == nvt - 1) tc::commit_warp(&w_free[wb]);
            __syncwarp();
            if (lane == 0) btrace(J, 4);
        }
    } else {
        // ---- weights (warps 14-15): stage both levels' compact blocks (bulk copies, one group ahead),
        //      compose, embed + split into the B tile ----
        const int wt = tid - 448;
        // block (m, u, e) of group g: level 1 (m = 0) pair p1(u, e), level 2 (m = 1) pair p2(u, e)
        auto stage_group = [&](int it, int sb) {
            const int64_t g = blockIdx.x + int64_t(it) * gridDim.x;
            const int64_t a0 = g >> shg, bq = g & ((int64_t(1) << shg) - 1);
            uint8_t* dst = sm_cmp + C::OFF_WST + sb * C::WST;
            tc::mbar_arrive_expect_tx(&wst_full[sb], C::WST);
            for (int b = 0; b < 8; b++) {
                const int m = b >> 2, u = (b >> 1) & 1, e = b & 1;
                const int64_t p = m == 0 ? ((((a0 << 1) + e) << (LN - lin - 1)) + (bq << 1) + u)
                                         : ((((a0 << 2) + 2 * u + e) << shg) + bq);
                tc::bulk_g2s(dst + b * C::BLK * 8, (m == 0 ? W1 : W2) + p * C::BLK, C::BLK * 8, &wst_full[sb]);
            }
        };
        if (wt == 0 && nit > 0) stage_group(0, 0);
        for (int it = 0; it < nit; it++) {
            const int wb = it % C::NWBUF, sb = it & 1;
            if (wt == 0 && it + 1 < nit) stage_group(it + 1, sb ^ 1);   // its buffer was released by the bar.sync
            tc::mbar_wait(&wst_full[sb], uint32_t(it >> 1) & 1);
            const float2* st = reinterpret_cast<const float2*>(sm_cmp + C::OFF_WST + sb * C::WST);
            if (it >= C::NWBUF) tc::mbar_wait(&w_free[wb], uint32_t(it / C::NWBUF - 1) & 1);
            if (wt == 0) btrace(int64_t(it) * nvt, 9);
            uint8_t* th = sm_cmp + C::OFF_W + wb * C::WSET;
            uint8_t* tl = th + C::WT;
            // item = (o, i, t', half of j): R / 2 independent complex accumulators per thread (ILP), the
            // L1 row pairs (j, j'), (j, j' + 1) as one 16-byte load
            constexpr int H = R / 2;
#pragma unroll 1
#ifdef BF_EXP_NO_COMPOSE
            for (int item = wt; item < 0; item += 64) {
#else
            for (int item = wt; item < C::ITEMS; item += 64) {
#endif
                const int jh = item & 1, r2 = item >> 1;
                const int tp = r2 % R, oi = r2 / R, o = oi >> 2, i = oi & 3;
                const int up = o >> 1, sp = i >> 1, s = i & 1;
                const float2* L2 = st + (4 + o) * C::BLK + sp * R * R + tp;              // W2[p2(o)][(s' R + j') R + t']
                const float2* L1 = st + (sp * 2 + up) * C::BLK + s * R * R + jh * H * R;   // W1[p1(s', u')][(s R + j) R + j']
                float2 c[H];
#pragma unroll
                for (int jj = 0; jj < H; jj++) c[jj] = make_float2(0.f, 0.f);
#pragma unroll
                for (int jp = 0; jp < R; jp += 2) {
                    const float2 wa = L2[jp * R], wb = L2[(jp + 1) * R];
#pragma unroll
                    for (int jj = 0; jj < H; jj++) {
                        const float4 w1 = *reinterpret_cast<const float4*>(L1 + jj * R + jp);
                        c[jj].x = fmaf(wa.x, w1.x, c[jj].x);
                        c[jj].y = fmaf(wa.x, w1.y, c[jj].y);
                        c[jj].x = fmaf(-wa.y, w1.y, c[jj].x);
                        c[jj].y = fmaf(wa.y, w1.x, c[jj].y);
                        c[jj].x = fmaf(wb.x, w1.z, c[jj].x);
                        c[jj].y = fmaf(wb.x, w1.w, c[jj].y);
                        c[jj].x = fmaf(-wb.y, w1.w, c[jj].x);
                        c[jj].y = fmaf(wb.y, w1.z, c[jj].y);
                    }
                }
#pragma unroll
                for (int jj = 0; jj < H; jj++) {
                    const int j = jh * H + jj;
                    float hr, lr, hi_, li;
                    tc::split(c[jj].x, hr, lr);
                    tc::split(c[jj].y, hi_, li);
                    const int n = o * C::SC + 2 * tp, k = i * C::SC + 2 * j;
                    const uint32_t o0 = tc::kmaj_off(n, k, C::NB), o1 = tc::kmaj_off(n + 1, k, C::NB);
                    *reinterpret_cast<float2*>(th + o0) = make_float2(hr, -hi_);
                    *reinterpret_cast<float2*>(tl + o0) = make_float2(lr, -li);
                    *reinterpret_cast<float2*>(th + o1) = make_float2(hi_, hr);
                    *reinterpret_cast<float2*>(tl + o1) = make_float2(li, lr);
                }
            }
            tc::fence_proxy_async();
            if (wt == 0) btrace(int64_t(it) * nvt, 10);
            tc::mbar_arrive(&w_full[wb]);
            asm volatile("bar.sync 1, 64;" ::: "memory");   // staging buffer sb free for group it + 2
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) {
        tc::fence_after_sync();
        tc::tmem_dealloc<C::TMEM_COLS>(tmem);
    }
}

// =============================================================================================
// Composed band in FP16 split passes (BF_OPT_BAND_F16 = 1).  Same job structure as band_cmp_kernel; the
// A operand of a job (4 pairs x r coefficients of one vector) is scaled by 2^{-e_v} with e_v from its max
// (the two split warps of a lane quadrant exchange their halves' maxima through shared memory), the
// composed block operator C of a group by 2^{-e_g} (its max), both split into FP16 hi + lo and multiplied
// with kind::f16 MMAs (K = 16): half the MMAs, half the TMEM stores and half the B bytes of the 3xTF32
// band.  The epilogue multiplies by 2^{e_v + e_g}.
// =============================================================================================
template <int R>
struct BandH {
    using B = BandCmp<R>;
    static constexpr int P = 4, SC = 2 * R, KB = P * SC, NB = KB;
    static constexpr int ACOLS = KB;                                  // hi KB/2 packed columns, then lo
    static constexpr int NABUF = 2, NDBUF = 2;
    static constexpr int D_OFF = NABUF * ACOLS;
    static constexpr int TMEM_COLS = tmem_cols_pow2<D_OFF + NDBUF * NB>();
    static constexpr uint32_t SLOT = B::SLOT, BLK = B::BLK, WST = B::WST;
    static constexpr uint32_t WT = uint32_t(NB) * KB * 2;             // one FP16 B tile (hi or lo)
    static constexpr uint32_t WSET = 2 * WT;
    static constexpr uint32_t CST = uint32_t(P) * P * R * R * 8;      // the composed C (FP32 complex)
    static constexpr uint32_t XCH = 2 * 2 * 128 * 4 + 4 * 128 * 4 + 4 * 4;   // maxima exchange, e_v ring, e_g ring
    static constexpr size_t LIM = 232448 - 1024;
    static constexpr int NQ_FIT = int((LIM - 2 * size_t(WST) - CST - 2 * size_t(WSET) - XCH) / SLOT);
    static constexpr int NQ = NQ_FIT > 16 ? 16 : NQ_FIT;
    static constexpr uint32_t OFF_WST = uint32_t(NQ) * SLOT;
    static constexpr uint32_t OFF_CST = OFF_WST + 2 * WST;
    static constexpr uint32_t OFF_W = OFF_CST + CST;
    static constexpr uint32_t OFF_X = OFF_W + 2 * WSET;
    static constexpr size_t SMEM = size_t(OFF_X) + XCH;
    static constexpr int ITEMS = P * P * R * 2;
    static_assert(KB % 16 == 0 && D_OFF + NDBUF * NB <= 512 && OFF_W % 128 == 0 && WT % 128 == 0 && NQ >= 6 &&
                      SMEM <= LIM, "FP16 band shape");
};

template <int R>
__global__ void __launch_bounds__(512, 1)
    band_h16_kernel(const __grid_constant__ CUtensorMap tin, float2* __restrict__ out, const float2* __restrict__ W1,
                    const float2* __restrict__ W2, int LN, int l_first, int nv, int rh, int rhg, const bfs::PeerOut po)
{
    using C = BandH<R>;
    extern __shared__ __align__(128) uint8_t sm_bh[];
    __shared__ uint64_t slot_full[16], slot_empty[16];
    __shared__ uint64_t a_ready[2], a_free[2], d_full[2], d_free[2], w_full[2], w_free[2], wst_full[2];
    __shared__ uint64_t e_full[4], e_empty[4], g_full[4], g_empty[4];
    __shared__ float red[2];
    __shared__ uint32_t tmem_base;
    float* Mx = reinterpret_cast<float*>(sm_bh + C::OFF_X);           // [J & 1][half][128] split maxima
    float* Ev = Mx + 2 * 2 * 128;                                      // [J & 3][128] 2^{e_v}
    float* Eg = Ev + 4 * 128;                                          // [group & 3] 2^{e_g}

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t N = int64_t(1) << LN;
    const int lin = l_first - 1, shg = LN - lin - 2;
    const int64_t ngroups = N >> 2;
    const int nvt = (nv + 127) / 128;
    const int nit = int((ngroups - blockIdx.x + gridDim.x - 1) / gridDim.x);
    const int njobs = nit * nvt;

    if (warp == 0) tc::tmem_alloc<C::TMEM_COLS>(&tmem_base);
    if (tid == 0) {
        for (int i = 0; i < C::NQ; i++) {
            tc::mbar_init(&slot_full[i], 1);
            tc::mbar_init(&slot_empty[i], 128);
        }
        for (int i = 0; i < 2; i++) {
            tc::mbar_init(&a_ready[i], 256);
            tc::mbar_init(&a_free[i], 1);
            tc::mbar_init(&d_full[i], 1);
            tc::mbar_init(&d_free[i], 128);
            tc::mbar_init(&w_full[i], 64);
            tc::mbar_init(&w_free[i], 1);
            tc::mbar_init(&wst_full[i], 1);
        }
        for (int i = 0; i < 4; i++) {
            tc::mbar_init(&e_full[i], 128);
            tc::mbar_init(&e_empty[i], 128);
            tc::mbar_init(&g_full[i], 64);
            tc::mbar_init(&g_empty[i], 128);
        }
        tc::mbar_fence_init();
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tmem_base;

    if (warp < 8) {
        // ---- split (two warps per lane quadrant, one per half of the group's 4 pair slots) ----
        const int qd = warp & 3, hs = warp >> 2;
        const int v = qd * 32 + lane;
        const uint32_t lb = uint32_t(qd * 32) << 16;
        for (int J = 0; J < njobs; J++) {
            const int ab = J & 1, use = J >> 1, eb = J & 3;
            if (use > 0) tc::mbar_wait(&a_free[ab], uint32_t(use - 1) & 1);
            if (hs == 0 && J >= 4) tc::mbar_wait(&e_empty[eb], uint32_t((J >> 2) - 1) & 1);
            tc::fence_after_sync();
            float mx = 0.f;
#pragma unroll 1
            for (int s = 2 * hs; s < 2 * hs + 2; s++) {
                const int k = J * C::P + s, q = k % C::NQ;
                tc::mbar_wait(&slot_full[q], uint32_t(k / C::NQ) & 1);
                const float2* rd = reinterpret_cast<const float2*>(sm_bh + q * C::SLOT);
#pragma unroll
                for (int t = 0; t < R; t++) {
                    const float2 x = rd[t * 128 + v];
                    mx = fmaxf(mx, fmaxf(fabsf(x.x), fabsf(x.y)));
                }
            }
            Mx[(ab * 2 + hs) * 128 + v] = mx;
            asm volatile("bar.sync %0, 64;" ::"r"(2 + qd) : "memory");   // the two warps of this quadrant
            mx = fmaxf(mx, Mx[(ab * 2 + (hs ^ 1)) * 128 + v]);
            int e = 0;
            frexpf(mx, &e);
            e = max(-126, min(126, e));
            const float sc = ldexpf(1.f, -e);
            if (hs == 0) {
                Ev[eb * 128 + v] = ldexpf(1.f, e);
                tc::mbar_arrive(&e_full[eb]);
            }
            float hi[2 * R], lo[2 * R];   // this half's two pair slots, packed (re, im) columns
#pragma unroll
            for (int s2 = 0; s2 < 2; s2++) {
                const int k = J * C::P + 2 * hs + s2, q = k % C::NQ;
                const float2* rd = reinterpret_cast<const float2*>(sm_bh + q * C::SLOT);
#pragma unroll
                for (int t = 0; t < R; t++) {
                    const float2 x = rd[t * 128 + v];
                    tc::split_h2(x.x * sc, x.y * sc, hi[s2 * R + t], lo[s2 * R + t]);
                }
                tc::mbar_arrive(&slot_empty[q]);
            }
            const uint32_t ta = tmem + lb + uint32_t(ab * C::ACOLS + 2 * hs * R);
            tc::tmem_st_cols<2 * R>(ta, hi);
            tc::tmem_st_cols<2 * R>(ta + C::KB / 2, lo);
            tc::tmem_wait_st();
            tc::fence_before_sync();
            tc::mbar_arrive(&a_ready[ab]);
        }
    } else if (warp < 12) {
        // ---- epilogue (4 warps): drain the accumulator row in halves, scale by 2^{e_v + e_g}, store ----
        const int q = warp & 3;
        const int v = q * 32 + lane;
        const uint32_t lb = uint32_t(q * 32) << 16;
        float sg = 1.f;
        for (int J = 0; J < njobs; J++) {
            const int it = int(unsigned(J) / unsigned(nvt));
            const int vt = J - it * nvt;
            const int64_t g = blockIdx.x + int64_t(it) * gridDim.x;
            const int db = J & 1, eb = J & 3;
            if (vt == 0) {
                tc::mbar_wait(&g_full[it & 3], uint32_t(it >> 2) & 1);
                sg = Eg[it & 3];
                tc::mbar_arrive(&g_empty[it & 3]);
            }
            tc::mbar_wait(&e_full[eb], uint32_t(J >> 2) & 1);
            const float s2 = Ev[eb * 128 + v] * sg;
            tc::mbar_arrive(&e_empty[eb]);
            tc::mbar_wait(&d_full[db], uint32_t(J >> 1) & 1);
            tc::fence_after_sync();
            const int vg = vt * 128 + v;
            const int64_t a0 = g >> shg, bq = g & ((int64_t(1) << shg) - 1);
#pragma unroll 1
            for (int hf = 0; hf < 2; hf++) {
                float d[2 * C::SC];
                tc::tmem_ld_cols<2 * C::SC>(tmem + lb + uint32_t(C::D_OFF + db * C::NB + hf * 2 * C::SC), d);
                tc::tmem_wait_ld();
                if (hf == 1) {
                    tc::fence_before_sync();
                    tc::mbar_arrive(&d_free[db]);
                }
                if (vg < nv) {
                    if (!po.on) {
                        const int64_t p = (((a0 << 2) + 2 * hf) << shg) + bq;
                        float2* o = out + p * R * int64_t(nv) + vg;
                        const int64_t pstep = (int64_t(1) << shg) * R * int64_t(nv) - int64_t(R) * nv;
#pragma unroll
                        for (int oo = 0; oo < 2; oo++) {
#pragma unroll
                            for (int t = 0; t < R; t++) {
                                *o = make_float2(d[oo * C::SC + 2 * t] * s2, d[oo * C::SC + 2 * t + 1] * s2);
                                o += nv;
                            }
                            o += pstep;
                        }
                    } else {
#pragma unroll
                        for (int oo = 0; oo < 2; oo++) {
                            const int64_t p = (((a0 << 2) + 2 * hf + oo) << shg) + bq;
                            float2* o = bfs::pair_out(out, po, p, R, nv) + vg;
#pragma unroll
                            for (int t = 0; t < R; t++)
                                o[int64_t(t) * nv] =
                                    make_float2(d[oo * C::SC + 2 * t] * s2, d[oo * C::SC + 2 * t + 1] * s2);
                        }
                    }
                }
            }
        }
    } else if (warp == 12) {
        // ---- loader: one 2-D tensor copy per pair slot ----
        for (int J = 0; J < njobs; J++) {
            const int it = int(unsigned(J) / unsigned(nvt));
            const int vt = J - it * nvt;
            const int64_t g = blockIdx.x + int64_t(it) * gridDim.x;
            const int64_t pin = rh ? bfs::recv_index(g * C::P, rh, rhg) : g * C::P;
            for (int s = 0; s < C::P; s++) {
                const int k = J * C::P + s, q = k % C::NQ;
                if (k >= C::NQ) tc::mbar_wait(&slot_empty[q], uint32_t(k / C::NQ - 1) & 1);
                if (lane == 0) {
                    tc::mbar_arrive_expect_tx(&slot_full[q], C::SLOT);
                    tc::tma_load_2d(sm_bh + q * C::SLOT, &tin, 2 * vt * 128, int((pin + s) * R), &slot_full[q]);
                }
                __syncwarp();
            }
        }
    } else if (warp == 13) {
        // ---- MMA issuer: one chain of 3 x (8r / 16) kind::f16 MMAs per job ----
        constexpr uint32_t idesc = tc::idesc_f16(128, C::NB);
        constexpr uint32_t LBO_B = (C::NB / 8) * 128;
        const uint64_t dW = tc::desc_kmajor(tc::smem_u32(sm_bh + C::OFF_W), LBO_B);
        for (int J = 0; J < njobs; J++) {
            const int it = int(unsigned(J) / unsigned(nvt));
            const int vt = J - it * nvt;
            const int wb = it & 1, ab = J & 1, db = J & 1;
            if (vt == 0) tc::mbar_wait(&w_full[wb], uint32_t(it >> 1) & 1);
            tc::mbar_wait(&a_ready[ab], uint32_t(J >> 1) & 1);
            if (J >= 2) tc::mbar_wait(&d_free[db], uint32_t((J >> 1) - 1) & 1);
            tc::fence_after_sync();
            const uint32_t d = tmem + uint32_t(C::D_OFF + db * C::NB);
            const uint32_t ahi = tmem + uint32_t(ab * C::ACOLS);
            const uint64_t bhi = tc::desc_add(dW, wb * C::WSET);
#pragma unroll
            for (int qq = 0; qq < 3; qq++) {
                const int pass = kPassOrder[qq];
                const uint32_t a = ahi + (pass == 1 ? C::KB / 2 : 0);
                const uint64_t b = pass == 2 ? tc::desc_add(bhi, C::WT) : bhi;
#pragma unroll
                for (int ks = 0; ks < C::KB / 16; ks++)
                    tc::mma_f16_ts_warp(d, a + ks * 8, tc::desc_add(b, ks * 2 * LBO_B), idesc, (qq | ks) ? 1u : 0u);
            }
            tc::commit_warp(&d_full[db]);
            tc::commit_warp(&a_free[ab]);
            if (vt == nvt - 1) tc::commit_warp(&w_free[wb]);
            __syncwarp();
        }
    } else {
        // ---- weights (warps 14-15): stage compact blocks (bulk, one group ahead), compose C in FP32 into
        //      shared memory, take the group max, write the scaled FP16 hi / lo B tile ----
        const int wt = tid - 448;
        auto stage_group = [&](int it, int sb) {
            const int64_t g = blockIdx.x + int64_t(it) * gridDim.x;
            const int64_t a0 = g >> shg, bq = g & ((int64_t(1) << shg) - 1);
            uint8_t* dst = sm_bh + C::OFF_WST + sb * C::WST;
            tc::mbar_arrive_expect_tx(&wst_full[sb], C::WST);
            for (int b = 0; b < 8; b++) {
                const int m = b >> 2, u = (b >> 1) & 1, e = b & 1;
                const int64_t p = m == 0 ? ((((a0 << 1) + e) << (LN - lin - 1)) + (bq << 1) + u)
                                         : ((((a0 << 2) + 2 * u + e) << shg) + bq);
                tc::bulk_g2s(dst + b * C::BLK * 8, (m == 0 ? W1 : W2) + p * C::BLK, C::BLK * 8, &wst_full[sb]);
            }
        };
        float2* Cs = reinterpret_cast<float2*>(sm_bh + C::OFF_CST);   // [o][t'][i][j]
        if (wt == 0 && nit > 0) stage_group(0, 0);
        for (int it = 0; it < nit; it++) {
            const int wb = it & 1, sb = it & 1, gb = it & 3;
            if (wt == 0 && it + 1 < nit) stage_group(it + 1, sb ^ 1);
            tc::mbar_wait(&wst_full[sb], uint32_t(it >> 1) & 1);
            const float2* st = reinterpret_cast<const float2*>(sm_bh + C::OFF_WST + sb * C::WST);
            constexpr int H = R / 2;
            float mx = 0.f;
#pragma unroll 1
            for (int item = wt; item < C::ITEMS; item += 64) {
                const int jh = item & 1, r2 = item >> 1;
                const int tp = r2 % R, oi = r2 / R, o = oi >> 2, i = oi & 3;
                const int up = o >> 1, sp = i >> 1, s = i & 1;
                const float2* L2 = st + (4 + o) * C::BLK + sp * R * R + tp;
                const float2* L1 = st + (sp * 2 + up) * C::BLK + s * R * R + jh * H * R;
                float2 c[H];
#pragma unroll
                for (int jj = 0; jj < H; jj++) c[jj] = make_float2(0.f, 0.f);
#pragma unroll
                for (int jp = 0; jp < R; jp += 2) {
                    const float2 wa = L2[jp * R], wb2 = L2[(jp + 1) * R];
#pragma unroll
                    for (int jj = 0; jj < H; jj++) {
                        const float4 w1 = *reinterpret_cast<const float4*>(L1 + jj * R + jp);
                        c[jj].x = fmaf(wa.x, w1.x, c[jj].x);
                        c[jj].y = fmaf(wa.x, w1.y, c[jj].y);
                        c[jj].x = fmaf(-wa.y, w1.y, c[jj].x);
                        c[jj].y = fmaf(wa.y, w1.x, c[jj].y);
                        c[jj].x = fmaf(wb2.x, w1.z, c[jj].x);
                        c[jj].y = fmaf(wb2.x, w1.w, c[jj].y);
                        c[jj].x = fmaf(-wb2.y, w1.w, c[jj].x);
                        c[jj].y = fmaf(wb2.y, w1.z, c[jj].y);
                    }
                }
#pragma unroll
                for (int jj = 0; jj < H; jj++) {
                    Cs[((o * R + tp) * 4 + i) * R + jh * H + jj] = c[jj];
                    mx = fmaxf(mx, fmaxf(fabsf(c[jj].x), fabsf(c[jj].y)));
                }
            }
            // group max over the 64 weight threads
#pragma unroll
            for (int m = 16; m > 0; m >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, m));
            if (lane == 0) red[wt >> 5] = mx;
            asm volatile("bar.sync 1, 64;" ::: "memory");   // C and the two warp maxima are in shared memory
            mx = fmaxf(red[0], red[1]);
            int e = 0;
            frexpf(mx, &e);
            e = max(-126, min(126, e));
            const float sc = ldexpf(1.f, -e);
            if (it >= 2) tc::mbar_wait(&w_free[wb], uint32_t((it >> 1) - 1) & 1);
            uint8_t* th = sm_bh + C::OFF_W + wb * C::WSET;
            uint8_t* tl = th + C::WT;
            // real embedding of C[o][t'][i][j] at rows n = o 2r + 2t' (+1), K columns k = i 2r + 2j (+1)
            for (int idx = wt; idx < C::P * R * C::P * R; idx += 64) {
                const int orow = idx / (C::P * R), icol = idx - orow * (C::P * R);   // (o, t'), (i, j)
                const int o = orow / R, tp = orow - o * R, i = icol / R, j = icol - i * R;
                const float2 cv = Cs[((o * R + tp) * 4 + i) * R + j];
                float hr, hm, lr, lm;   // packed halves: (re, -im) for row n, (im, re) for row n + 1
                tc::split_h2(cv.x * sc, -cv.y * sc, hr, lr);
                tc::split_h2(cv.y * sc, cv.x * sc, hm, lm);
                const int n = o * C::SC + 2 * tp, k = i * C::SC + 2 * j;
                const uint32_t o0 = tc::kmaj_off16(n, k, C::NB), o1 = tc::kmaj_off16(n + 1, k, C::NB);
                *reinterpret_cast<float*>(th + o0) = hr;
                *reinterpret_cast<float*>(tl + o0) = lr;
                *reinterpret_cast<float*>(th + o1) = hm;
                *reinterpret_cast<float*>(tl + o1) = lm;
            }
            tc::fence_proxy_async();
            tc::mbar_arrive(&w_full[wb]);
            if (it >= 4) tc::mbar_wait(&g_empty[gb], uint32_t((it >> 2) - 1) & 1);
            if (wt == 0) Eg[gb] = ldexpf(1.f, e);
            tc::mbar_arrive(&g_full[gb]);
            asm volatile("bar.sync 1, 64;" ::: "memory");   // staging buffer sb and Cs free for the next group
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) {
        tc::fence_after_sync();
        tc::tmem_dealloc<C::TMEM_COLS>(tmem);
    }
}

template <int R>
static cudaError_t band_tc_go(const Dims& d, int l_first, const float2* in, float2* out, const float2* const* W, int nv,
                              cudaStream_t s, int rh, int rhg, const bfs::PeerOut& po, const BandVariant& bv)
{
    const bool compose = bv.compose;
    using C = BandTC<R>;
    const int64_t groups = d.N >> 2;
    const unsigned grid = unsigned(groups < sm_count() ? groups : sm_count());
    if (compose && bv.f16) {
        using CH = BandH<R>;
        auto kern = band_h16_kernel<R>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(CH::SMEM));
        if (e != cudaSuccess) return e;
        CUtensorMap tin;
        e = make_rows_tmap(&tin, in, d.N * R, nv, R);
        if (e != cudaSuccess) return e;
        kern<<<grid, 512, CH::SMEM, s>>>(tin, out, W[0], W[1], d.LN, l_first, nv, rh, rhg, po);
        return cudaGetLastError();
    }
    if (compose) {
        using CC = BandCmp<R>;
        auto kern = band_cmp_kernel<R>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(CC::SMEM));
        if (e != cudaSuccess) return e;
        CUtensorMap tin;
        e = make_rows_tmap(&tin, in, d.N * R, nv, R);
        if (e != cudaSuccess) return e;
        kern<<<grid, 512, CC::SMEM, s>>>(tin, out, W[0], W[1], d.LN, l_first, nv, rh, rhg, po);
        return cudaGetLastError();
    }
    if constexpr (Band2P<R>::FITS) {
        if (bv.two_pipelines) {
            auto kern = band_tc2p_kernel<R>;
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
            if (e != cudaSuccess) return e;
            kern<<<grid, 512, C::SMEM, s>>>(in, out, W[0], W[1], d.LN, l_first, nv, rh, rhg, po);
            return cudaGetLastError();
        }
    }
    auto kern = band_tc_kernel<R>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
    if (e != cudaSuccess) return e;
    kern<<<grid, 384, C::SMEM, s>>>(in, out, W[0], W[1], d.LN, l_first, nv, rh, rhg, po);
    return cudaGetLastError();
}

cudaError_t band_trace(long long* out, int n)
{
    if (n > BT_JOBS * BT_EV) n = BT_JOBS * BT_EV;
    return cudaMemcpyFromSymbol(out, g_band_trace, size_t(n) * sizeof(long long));
}

bool band_tc_supported(const Dims& d, int nv)
{
    return (d.R == 6 || d.R == 8 || d.R == 10 || d.R == 12) && nv >= 64 && nv % 2 == 0;
}

cudaError_t launch_band_tc(const Dims& d, int l_first, const float2* in, float2* out, const float2* const* W, int nv,
                           cudaStream_t s, int rh, int rhg, const bfs::PeerOut* po, const BandVariant& bv)
{
    const bfs::PeerOut pz = po ? *po : bfs::PeerOut{};
    switch (d.R) {
    case 6: return band_tc_go<6>(d, l_first, in, out, W, nv, s, rh, rhg, pz, bv);
    case 8: return band_tc_go<8>(d, l_first, in, out, W, nv, s, rh, rhg, pz, bv);
    case 10: return band_tc_go<10>(d, l_first, in, out, W, nv, s, rh, rhg, pz, bv);
    case 12: return band_tc_go<12>(d, l_first, in, out, W, nv, s, rh, rhg, pz, bv);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace bfk
