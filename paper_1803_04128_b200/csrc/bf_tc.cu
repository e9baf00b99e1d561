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

// The 2x S0 image (S0TC I2): any leaf shape whose N chunks hold whole (a, t) halves (n0 r a multiple of 64);
// BF_S0_IMAGE4 builds keep the 4x image.
constexpr bool s0_i2(int R, int N0)
{
#ifdef BF_S0_IMAGE4
    return false && R && N0;
#else
    return (N0 * R) % 64 == 0;
#endif
}

int64_t leafx_floats(const Dims& d) { return d.N * int64_t(2 * d.R) * int64_t(2 << d.l0) * 2; }

// i2: the 2x image (section 5.1): per N chunk of 128 rows, rows c' 64 + m hold V0r / V0i of output m of the chunk's
// 64 (a, t); K = j in tiles of 16 (8 KB hi + 8 KB lo per tile), no real embedding
__global__ void expand_s0_kernel(const float2* __restrict__ V0, float* __restrict__ X, int LN, int l0, int R, int i2)
{
    const int n0 = 1 << l0;
    const int64_t nleaf = (int64_t(1) << LN) >> l0;
    const int rows = n0 * 2 * R, K = i2 ? n0 : 2 * n0;
    const int KT = i2 ? S0X_KC / 2 : S0X_KC;
    const int64_t TF = int64_t(S0X_NC) * KT;   // floats of one tile (hi or lo)
    const int nch = rows / S0X_NC, kch = K / KT;
    const int64_t total = nleaf * rows * int64_t(K);
    for (int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < total; g += int64_t(gridDim.x) * blockDim.x) {
        const int64_t b = g / (int64_t(rows) * K);
        const int rem = int(g - b * rows * K);
        const int n = rem / K, k = rem - n * K;
        float hi, lo;
        if (i2) {
            const int nc = n / S0X_NC, m = n % S0X_NC, cp = m / 64, q = nc * 64 + (m % 64), a = q / R, t = q % R;
            const float2 w = V0[(int64_t(a) * nleaf + b) * (n0 * R) + int64_t(k) * R + t];
            tc::split(cp ? w.y : w.x, hi, lo);
        } else {
            const int a = n / (2 * R), t = (n / 2) % R, cp = n & 1, j = k >> 1, c = k & 1;
            const float2 w = V0[(int64_t(a) * nleaf + b) * (n0 * R) + int64_t(j) * R + t];
            tc::split(embed(w, cp, c), hi, lo);
        }
        const int nc = n / S0X_NC, kc = k / KT;
        float* tile = X + ((b * nch + nc) * kch + kc) * 2 * TF;
        const uint32_t off = tc::kmaj_off(n % S0X_NC, k % KT, S0X_NC) / 4;
        tile[off] = hi;
        tile[TF + off] = lo;
    }
}

// SL: per T_X leaf a the B matrix has rows n = (j, c') (2 n0) and K = (b, t, c) (n0 2r), stored as
// [leaf][K chunk of KP pairs][hi | lo][canonical K-major 2 n0 x KP 2r tile].
static int sl_kp(int R) { return R >= 12 ? 1 : 2; }

// The 2x SL image (rows n = c' n0 + j holding Ur / Ui, K = (b, t); SLTC I2) where the chunk's K (KP r) is a whole
// number of MMA K steps: r = 8 (KP 2) and r = 16 (KP 1).  BF_SL_IMAGE4 builds keep the 4x image everywhere.
constexpr bool sl_i2(int R)
{
#ifdef BF_SL_IMAGE4
    return false && R;
#else
    return R == 8 || R == 16;
#endif
}

__global__ void expand_sl_kernel(const float2* __restrict__ U, float* __restrict__ X, int LN, int l0, int R, int KP,
                                 int i2)
{
    const int n0 = 1 << l0;
    const int64_t nleaf = (int64_t(1) << LN) >> l0;
    const int rows = 2 * n0, K = i2 ? n0 * R : n0 * 2 * R, KC = i2 ? KP * R : KP * 2 * R;
    const int nch = n0 / KP;
    const int64_t tile = int64_t(rows) * KC;
    const int64_t total = nleaf * rows * int64_t(K);
    for (int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < total; g += int64_t(gridDim.x) * blockDim.x) {
        const int64_t a = g / (int64_t(rows) * K);
        const int rem = int(g - a * rows * K);
        const int n = rem / K, k = rem - n * K;
        float hi, lo;
        int b;
        if (i2) {   // n = c' n0 + j, k = b r + t: Ur (c' = 0) / Ui (c' = 1), no embedding
            const int cp = n / n0, j = n - cp * n0, t = k % R;
            b = k / R;
            const float2 w = U[(a * n0 + b) * (n0 * R) + int64_t(t) * n0 + j];
            tc::split(cp ? w.y : w.x, hi, lo);
        } else {
            const int j = n >> 1, cp = n & 1, t = (k / 2) % R, c = k & 1;
            b = k / (2 * R);
            const float2 w = U[(a * n0 + b) * (n0 * R) + int64_t(t) * n0 + j];
            tc::split(embed(w, cp, c), hi, lo);
        }
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
        expand_s0_kernel<<<grid, 256, 0, s>>>(V0, V0x, d.LN, d.l0, d.R, s0_i2(d.R, 1 << d.l0) ? 1 : 0);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    if (Ux) expand_sl_kernel<<<grid, 256, 0, s>>>(U, Ux, d.LN, d.l0, d.R, sl_kp(d.R), sl_i2(d.R) ? 1 : 0);
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

template <int R, int N0, bool I2 = false>
struct S0TC {
    static constexpr int K = 2 * N0;
    static constexpr int KS = K / S0X_KC;                 // K tiles per chunk (2 or 4): 16 complex j each
    static constexpr int KT = I2 ? S0X_KC / 2 : S0X_KC;   // B tile K (real columns)
    static constexpr int NCH = N0 * 2 * R / S0X_NC;       // 128-row N chunks per job
    static constexpr int NSTAGE = I2 ? 2 * KS + 1 : KS + 1;   // weight ring depth (32 KB stages, 16 KB for I2)
    static constexpr int64_t TILE_FLOATS = int64_t(S0X_NC) * KT;
    static constexpr uint32_t TILE = uint32_t(TILE_FLOATS) * 4;   // 16 KB (8 KB for I2)
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
template <int R, int N0, int CL, bool I2>
__global__ void __launch_bounds__(448, 1)
    s0_tc_kernel(const float2* __restrict__ F, int64_t ldf, const float2* __restrict__ ampb,
                 const float* __restrict__ V0x, float2* __restrict__ out, int LN, int n_amp, int nv, int nvt)
{
    using C = S0TC<R, N0, I2>;
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
                    const float* src = V0x + (b * WPJ + w) * 2 * C::TILE_FLOATS;
                    if constexpr (CL == 2)
                        tc::bulk_g2s_mc(ring + st * C::STAGE + cr * C::TILE, src + cr * C::TILE_FLOATS, C::TILE,
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
                    if constexpr (I2) {   // [re of the tile's 16 j | im of them]: hi[0..8) re, hi[8..16) im
                        tc::split(y0.x, hi[jj], lo[jj]);
                        tc::split(y1.x, hi[jj + 1], lo[jj + 1]);
                        tc::split(y0.y, hi[8 + jj], lo[8 + jj]);
                        tc::split(y1.y, hi[8 + jj + 1], lo[8 + jj + 1]);
                    } else {
                        tc::split(y0.x, hi[2 * jj], lo[2 * jj]);
                        tc::split(y0.y, hi[2 * jj + 1], lo[2 * jj + 1]);
                        tc::split(y1.x, hi[2 * jj + 2], lo[2 * jj + 2]);
                        tc::split(y1.y, hi[2 * jj + 3], lo[2 * jj + 3]);
                    }
                }
                if constexpr (I2) {
                    const uint32_t cb = uint32_t(kt * S0X_KC + (j0 % (S0X_KC / 2)));
                    tc::tmem_st8(tmem + lb + cb, hi);
                    tc::tmem_st8(tmem + lb + cb + S0X_KC / 2, hi + 8);
                    tc::tmem_st8(tmem + lb + uint32_t(C::A_COLS) + cb, lo);
                    tc::tmem_st8(tmem + lb + uint32_t(C::A_COLS) + cb + S0X_KC / 2, lo + 8);
                } else {
                    tc::tmem_st16(tmem + lb + uint32_t(2 * j0), hi);
                    tc::tmem_st16(tmem + lb + uint32_t(C::A_COLS + 2 * j0), lo);
                }
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
                        if constexpr (I2) {
                            // D[:, 0:128] += A_R [V0r; V0i]^T, D[:, 0:64] += A_I (-V0i)^T, D[:, 64:128] += A_I V0r^T
                            constexpr uint32_t idh = tc::idesc_tf32(128, S0X_NC / 2);
                            constexpr uint32_t HALF = (S0X_NC / 2 / 8) * 128;
#pragma unroll
                            for (int kk = 0; kk < C::KT / 8; kk++) {
                                const uint64_t bk = tc::desc_add(b, kk * 2 * LBO_B);
                                tc::mma_tf32_ts_warp(d, a + kk * 8, bk, idesc, (q | ks | kk) ? 1u : 0u);
                                tc::mma_tf32_ts_warp(d, a + S0X_KC / 2 + kk * 8, tc::desc_add(bk, HALF), idh | (1u << 14),
                                                     1u);
                                tc::mma_tf32_ts_warp(d + S0X_NC / 2, a + S0X_KC / 2 + kk * 8, bk, idh, 1u);
                            }
                        } else {
#pragma unroll
                        for (int kk = 0; kk < S0X_KC / 8; kk++)
                            tc::mma_tf32_ts_warp(d, a + kk * 8, tc::desc_add(b, kk * 2 * LBO_B), idesc,
                                                 (q | ks | kk) ? 1u : 0u);
                        }
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
                // I2: output m of the chunk has its re part in column m, its im part in column 64 + m; this thread
                // takes m in [half 32, half 32 + 32) -- the same outputs (a, t) as the interleaved layout
                const uint32_t taddr = tmem + (uint32_t(q4 * 32) << 16) +
                                       uint32_t(C::D_OFF + slot * S0X_NC + (I2 ? cbase / 2 : cbase));
                const int q0 = (nc * S0X_NC + cbase) >> 1;
                int t = q0 % R;
                float2* o = obase + int64_t(q0 / R) * strideA + int64_t(t) * nv;
#pragma unroll
                for (int c0 = 0; c0 < 64; c0 += 32) {
                    float x[32];
                    if constexpr (I2) {   // x[2i] = re, x[2i + 1] = im of output c0/2 + i
                        float xr[16], xi[16];
                        tc::tmem_ld16(taddr + c0 / 2, xr);
                        tc::tmem_ld16(taddr + S0X_NC / 2 + c0 / 2, xi);
                        tc::tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 16; i++) {
                            x[2 * i] = xr[i];
                            x[2 * i + 1] = xi[i];
                        }
                    } else {
                        tc::tmem_ld16(taddr + c0, x);
                        tc::tmem_ld16(taddr + c0 + 16, x + 16);
                        tc::tmem_wait_ld();
                    }
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
    constexpr bool I2 = s0_i2(R, N0);
    using C = S0TC<R, N0, I2>;
    const int nvt = (nv + 127) / 128;
    const int64_t leaves = d.N / N0;
    cudaError_t e;
    if (multicast && nvt % 2 == 0 && sm_count() >= 2) {
        auto kern = s0_tc_kernel<R, N0, 2, I2>;
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
    auto kern = s0_tc_kernel<R, N0, 1, I2>;
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
// I2: the "2x" Ux image (hi/lo of the compact blocks stacked [Ur; Ui], rows n = c' n0 + j, K = (pl, t)) instead of
// the real-embedded 4x image; the MMA schedule forms the complex product (section 5.1): per K step of 8
//   D[:, 0:NB]      += A_R [Ur; Ui]^T          (N = NB)
//   D[:, 0:NB/2]    += A_I (-Ui)^T             (N = NB/2, negate-B bit)
//   D[:, NB/2:NB]   += A_I Ur^T                (N = NB/2)
// with A = [A_R | A_I] (re / im parts of the chunk's coefficients as separate K blocks).
template <int R, int N0, int NA, int KP, bool I2 = false>
struct SLTC {
    static constexpr int NB = 2 * N0;
    static constexpr int KC = I2 ? KP * R : KP * 2 * R;      // B tile K (real columns) per chunk
    static constexpr int AH = I2 ? 2 * KC : KC;              // A columns of one split part (hi or lo)
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
    static constexpr uint32_t AS_BYTES = 2 * uint32_t(NA) * N0 * 8;   // a_k(x) of two jobs (double-buffered)
    // separate rings: the coefficient rows come from DRAM (deep ring), the Ux tiles mostly from L2 (2 deep)
    static constexpr int NB_R = 3;                                   // Ux ring depth (2 / 4 measured: 0.95x / 1.0x)
    static constexpr int NR_FIT = int((232448 - 1024 - GS_BYTES - AS_BYTES - NB_R * 2 * BT) / RAW);
    static constexpr int NR = NR_FIT > 8 ? 8 : NR_FIT;               // raw ring depth
    static constexpr uint32_t OFF_B = NR * RAW, OFF_GS = OFF_B + 2 * NB_R * BT, OFF_AS = OFF_GS + GS_BYTES;
    static constexpr size_t SMEM = size_t(OFF_AS) + AS_BYTES;
    // TMEM: two A stages (hi KC columns, then lo KC columns) and two accumulators of NB columns
    // A stages: as many as TMEM holds beside the two accumulators (up to 4): the split of chunk g + NAS overlaps
    // the MMAs of the chunks before it instead of waiting for chunk g's MMAs to finish (2 stages left the tensor
    // pipe idle across every split + mbarrier round trip)
    static constexpr int A_COLS = 2 * AH;
    static constexpr int NAS = (512 - 2 * NB) / A_COLS >= 4 ? 4 : (512 - 2 * NB) / A_COLS;
    static constexpr int D_OFF = NAS * A_COLS;
    static constexpr int TMEM_COLS = tmem_cols_pow2<D_OFF + 2 * NB>();
    static_assert(KC % 8 == 0, "K chunk must be whole MMA K steps");
    static_assert(NAS >= 2 && D_OFF + 2 * NB <= 512, "TMEM budget");
    static_assert(SMEM <= 232448 - 1024 && NR >= 2, "shared memory budget");
};

// CL = 2: launched as clusters of two CTAs that work on the two halves of a leaf's vector tiles at the same
// time; each CTA bulk-copies half of every Ux stage and multicasts it to both (half the L2 -> SM traffic of
// the 1.3 MB-per-job Ux stream), and a stage is refilled only after both CTAs' MMAs released it.
template <int R, int N0, int NA, int KP, int CL, bool I2>
__global__ void __launch_bounds__(448, 1)
    sl_tc_kernel(const __grid_constant__ CUtensorMap tin, const float* __restrict__ Ux, const float2* __restrict__ ampa,
                 float2* __restrict__ G, int64_t ldg, int LN, int nv, int nvt)
{
    using C = SLTC<R, N0, NA, KP, I2>;
    extern __shared__ __align__(128) uint8_t sm_sltc[];
    auto raw = [&](int e) { return sm_sltc + e * C::RAW; };
    auto opB = [&](int e, int lo) { return sm_sltc + C::OFF_B + (2 * e + lo) * C::BT; };
    float2* Gs = reinterpret_cast<float2*>(sm_sltc + C::OFF_GS);   // [128/NA][GS_STRIDE]
    float2* As = reinterpret_cast<float2*>(sm_sltc + C::OFF_AS);   // [2][NA][N0] a_k(x) of the current / next job
    __shared__ uint64_t raw_full[C::NR], raw_empty[C::NR], b_full[C::NB_R], b_empty[C::NB_R], a_full[4], a_empty[4],
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
            tc::mbar_init(&dfull[i], 1);
            tc::mbar_init(&dempty[i], 256);
        }
        for (int i = 0; i < C::NAS; i++) {
            tc::mbar_init(&a_full[i], 128);
            tc::mbar_init(&a_empty[i], 1);
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
            const int e = gch % C::NB_R, sa = gch % C::NAS, slot = gseg & 1, first = (ch % C::SEG) == 0;
            const bool last = (ch % C::SEG) == C::SEG - 1 || ch == C::NCH - 1;
            if (first && gseg >= 2) tc::mbar_wait(&dempty[slot], uint32_t((gseg >> 1) - 1) & 1);
            tc::mbar_wait(&a_full[sa], uint32_t(gch / C::NAS) & 1);
            tc::mbar_wait(&b_full[e], uint32_t(gch / C::NB_R) & 1);
            tc::fence_after_sync();
            const uint32_t d = tmem + uint32_t(C::D_OFF + slot * C::NB);
#pragma unroll
            for (int q = 0; q < 3; q++) {
                const int pass = kPassOrder[q];
                const uint32_t aa = tmem + uint32_t(sa * C::A_COLS + (pass == 1 ? C::AH : 0));
                const uint64_t bb = tc::desc_add(dB0, (2 * e + (pass == 2)) * C::BT);
#pragma unroll
                for (int ks = 0; ks < C::KC / 8; ks++) {
#ifdef BF_SL_EXP_NO_MMA   // diagnostics: the kernel without its MMAs (data movement, split, drain only)
                    if (q < 0)
#endif
                    {
                        const uint64_t bk = tc::desc_add(bb, ks * 2 * LBO_B);
                        tc::mma_tf32_ts_warp(d, aa + ks * 8, bk, idesc, (first && q == 0 && ks == 0) ? 0u : 1u);
                        if constexpr (I2) {
                            constexpr uint32_t idh = tc::idesc_tf32(128, C::NB / 2);
                            constexpr uint32_t HALF = (C::NB / 2 / 8) * 128;   // bytes to the Ui rows
                            tc::mma_tf32_ts_warp(d, aa + C::KC + ks * 8, tc::desc_add(bk, HALF), idh | (1u << 14), 1u);
                            tc::mma_tf32_ts_warp(d + C::NB / 2, aa + C::KC + ks * 8, bk, idh, 1u);
                        }
                    }
                }
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
            const int e = gch % C::NR, sa = gch % C::NAS;
            tc::mbar_wait(&raw_full[e], uint32_t(gch / C::NR) & 1);
            if (gch >= C::NAS) tc::mbar_wait(&a_empty[sa], uint32_t(gch / C::NAS - 1) & 1);
            tc::fence_after_sync();
            const float2* rd = reinterpret_cast<const float2*>(raw(e));   // [KP R][128]
            float hi[C::AH], lo[C::AH];   // column (pl, t, c) = pl 2R + 2t + c; I2: c KC + pl R + t
#pragma unroll
            for (int row = 0; row < KP * R; row++) {
                const float2 x = rd[row * 128 + v];
                if constexpr (I2) {
                    tc::split(x.x, hi[row], lo[row]);
                    tc::split(x.y, hi[C::KC + row], lo[C::KC + row]);
                } else {
                    tc::split(x.x, hi[2 * row], lo[2 * row]);
                    tc::split(x.y, hi[2 * row + 1], lo[2 * row + 1]);
                }
            }
            tc::fence_before_sync();
            tc::mbar_arrive(&raw_empty[e]);   // the raw rows are in registers now
            const uint32_t ta = tmem + lb + uint32_t(sa * C::A_COLS);
#ifndef BF_SL_EXP_NO_TMEM_ST   // diagnostics: the split without its TMEM stores
            tc::tmem_st_cols<C::AH>(ta, hi);
            tc::tmem_st_cols<C::AH>(ta + C::AH, lo);
#else
            if (hi[0] == 1234.5f && lo[1] == 0.5f) tc::tmem_st_cols<4>(ta, hi);
#endif
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
            // a_k(x) of this job's leaf: cp.async into the job's half of the double-buffered As now, so the
            // global-load latency hides behind the segment drains (it sat on the epilogue's critical path, while
            // the MMA can run only two segments ahead)
            float2* Asj = As + (jl & 1) * (NA * N0);
            for (int i = dt; i < NA * N0; i += 256)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(tc::smem_u32(Asj + i)),
                             "l"(ampa + (i / N0) * N + a * N0 + (i % N0))
                             : "memory");
            asm volatile("cp.async.commit_group;" ::: "memory");
            float sum[HC];
#pragma unroll
            for (int i = 0; i < HC; i++) sum[i] = 0.f;
            for (int seg = 0; seg < C::NSEG; seg++, gseg++) {
                const int slot = gseg & 1;
                tc::mbar_wait(&dfull[slot], uint32_t(gseg >> 1) & 1);
                tc::fence_after_sync();
                // I2: a thread's half of the leaf (j in [half HC/2, (half + 1) HC/2)) has its re parts at columns
                // half HC/2 .. and its im parts NB/2 further; sum[0, HC/2) = re, sum[HC/2, HC) = im
                const uint32_t taddr = tmem + (uint32_t(q4 * 32) << 16) +
                                       uint32_t(C::D_OFF + slot * C::NB + (I2 ? half * (HC / 2) : half * HC));
#pragma unroll
                if constexpr (I2) {
#pragma unroll
                    for (int hpart = 0; hpart < 2; hpart++) {
                        float x[HC / 2];
#ifndef BF_SL_EXP_NO_DRAIN
                        tc::tmem_ld_cols<HC / 2>(taddr + hpart * (C::NB / 2), x);
                        tc::tmem_wait_ld();
#else
#pragma unroll
                        for (int i = 0; i < HC / 2; i++) x[i] = 0.f;
#endif
#pragma unroll
                        for (int i = 0; i < HC / 2; i++) sum[hpart * (HC / 2) + i] += x[i];
                    }
                } else {
#pragma unroll
                for (int c0 = 0; c0 < HC; c0 += 32) {
                    float x[32];
#ifndef BF_SL_EXP_NO_DRAIN   // diagnostics: segments released without reading the accumulators
                    tc::tmem_ld_cols<(HC < 32 ? HC : 32)>(taddr + c0, x);
                    tc::tmem_wait_ld();
#else
#pragma unroll
                    for (int i = 0; i < 32; i++) x[i] = 0.f;
#endif
#pragma unroll
                    for (int i = 0; i < (HC < 32 ? HC : 32); i++) sum[c0 + i] += x[i];
                }
                }
                tc::fence_before_sync();
                tc::mbar_arrive(&dempty[slot]);
            }
            // epilogue of the job: a_k(x) (staged per job), sum over k, G transposed through Gs
            asm volatile("cp.async.wait_all;" ::: "memory");
            asm volatile("bar.sync 1, 256;" ::: "memory");   // Asj complete; the previous job is done with Gs
#pragma unroll
            for (int jj = 0; jj < HC / 2; jj++) {
                const int j = half * (HC / 2) + jj;
                float2 g = cmul_tc(Asj[k * N0 + j], I2 ? make_float2(sum[jj], sum[HC / 2 + jj])
                                                       : make_float2(sum[2 * jj], sum[2 * jj + 1]));
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
    constexpr bool I2 = sl_i2(R);
    using C = SLTC<R, N0, NA, KP, I2>;
    const int nvt = (nv + 127) / 128;
    CUtensorMap tin;
    cudaError_t e = make_rows_tmap(&tin, in, d.N * R, nv, KP * R);
    if (e != cudaSuccess) return e;
    const int64_t leaves = d.N / N0;
    if (multicast && nvt % 2 == 0 && sm_count() >= 2) {
        auto kern = sl_tc_kernel<R, N0, NA, KP, 2, I2>;
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
    auto kern = sl_tc_kernel<R, N0, NA, KP, 1, I2>;
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
            tc::mbar_arrive(&d1_free);
            tc::mbar_arrive(&a2_ready[slot]);

            tc::mbar_wait(&d2_full, ph);
            tc::fence_after_sync();
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
                tc::commit_warp(m == 0 ? &d1_full : &d2_full);
            }
            tc::commit_warp(&a_free[slot]);
            if (vt == nvt - 1) tc::commit_warp(&w_free[wb]);
            __syncwarp();
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
// NS = weight staging depth (groups in flight).  4 instead of 2 for one-tile chunks (nv <= 128) was measured
// slower (nv = 64: 5.6 vs 4.7 ms per band at cfg4; the raw ring it displaces matters more), so 2 is used.
template <int R, int NS = 2>
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
    static constexpr int NWBUF = (8 * size_t(SLOT) + NS * size_t(WST) + 2 * size_t(WSET) <= LIM) ? 2 : 1;
    // raw ring of single-pair slots (freed one pair at a time, so more bytes stay in flight)
    static constexpr int NQ_FIT = int((LIM - NS * size_t(WST) - NWBUF * size_t(WSET)) / SLOT);
#ifdef BF_BAND_NQ
    static constexpr int NQ = NQ_FIT > BF_BAND_NQ ? BF_BAND_NQ : NQ_FIT;
#else
    static constexpr int NQ = NQ_FIT > 16 ? 16 : NQ_FIT;
#endif
    static constexpr uint32_t OFF_WST = uint32_t(NQ) * SLOT;          // NS staging buffers (prefetch)
    static constexpr uint32_t OFF_W = OFF_WST + NS * WST;
    static constexpr size_t SMEM = size_t(OFF_W) + NWBUF * size_t(WSET);
    static constexpr int ITEMS = P * P * R * 2;                       // (o, i, t', j half) compose items
#ifdef BF_BAND_SPLIT4
    static constexpr int NSPLIT = 4;                                  // split warps (the rest of 0-11: epilogue)
#else
    static constexpr int NSPLIT = 8;
#endif
    static_assert(KB % 16 == 0 && D_OFF + NDBUF * NB <= 512 && OFF_W % 128 == 0 && WT % 128 == 0 &&
                      NQ >= (NS > 2 ? 6 : 8) && SMEM <= LIM, "composed band shape");
};

template <int R, int NS>
__global__ void __launch_bounds__(512, 1)
    band_cmp_kernel(const __grid_constant__ CUtensorMap tin, float2* __restrict__ out, const float2* __restrict__ W1,
                    const float2* __restrict__ W2, const float2* __restrict__ Cpre, int LN, int l_first, int nv, int rh,
                    int rhg, const bfs::PeerOut po)
{
    using C = BandCmp<R, NS>;
    extern __shared__ __align__(128) uint8_t sm_cmp[];
    __shared__ uint64_t slot_full[16], slot_empty[16];
    __shared__ uint64_t a_ready[2], a_free[2], d_full[2], d_free[2], w_full[2], w_free[2];
    __shared__ uint64_t wst_full[NS];
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
        }
        for (int i = 0; i < NS; i++) tc::mbar_init(&wst_full[i], 1);
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
#pragma unroll 1
            for (int s = hs * SPW; s < (hs + 1) * SPW; s++) {
                const int k = J * C::P + s, q = k % C::NQ;
                tc::mbar_wait(&slot_full[q], uint32_t(k / C::NQ) & 1);
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
                    tc::mbar_arrive_expect_tx(&slot_full[q], C::SLOT);   // whole box (ragged tile: zero fill)
                    tc::tma_load_2d(sm_cmp + q * C::SLOT, &tin, 2 * vt * 128, int((pin + s) * R), &slot_full[q]);
                }
                __syncwarp();
            }
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
            tc::mbar_wait(&a_ready[ab], uint32_t(J / C::NABUF) & 1);
            if (J >= C::NDBUF) tc::mbar_wait(&d_free[db], uint32_t(J / C::NDBUF - 1) & 1);
            tc::fence_after_sync();
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
            if (Cpre) {   // the group's precomposed operator (16 r^2 complex = the bytes of its 8 compact blocks)
                tc::bulk_g2s(dst, Cpre + g * (C::WST / 8), C::WST, &wst_full[sb]);
                return;
            }
            for (int b = 0; b < 8; b++) {
                const int m = b >> 2, u = (b >> 1) & 1, e = b & 1;
                const int64_t p = m == 0 ? ((((a0 << 1) + e) << (LN - lin - 1)) + (bq << 1) + u)
                                         : ((((a0 << 2) + 2 * u + e) << shg) + bq);
                tc::bulk_g2s(dst + b * C::BLK * 8, (m == 0 ? W1 : W2) + p * C::BLK, C::BLK * 8, &wst_full[sb]);
            }
        };
        if (wt == 0)
            for (int q = 0; q < NS - 1 && q < nit; q++) stage_group(q, q);
        for (int it = 0; it < nit; it++) {
            const int wb = it % C::NWBUF, sb = it % NS;
            // group it + NS - 1 into the buffer of group it - 1 (released by the bar.sync that ended it - 1)
            if (wt == 0 && it + NS - 1 < nit) stage_group(it + NS - 1, (it + NS - 1) % NS);
            tc::mbar_wait(&wst_full[sb], uint32_t(it / NS) & 1);
            const float2* st = reinterpret_cast<const float2*>(sm_cmp + C::OFF_WST + sb * C::WST);
            if (it >= C::NWBUF) tc::mbar_wait(&w_free[wb], uint32_t(it / C::NWBUF - 1) & 1);
            uint8_t* th = sm_cmp + C::OFF_W + wb * C::WSET;
            uint8_t* tl = th + C::WT;
            if (Cpre) {
                // precomposed C[o][i](t', j) (layout [o][i][t'][j], bf_plan finalize): embed + split only.  A thread
                // takes whole rows (o, i, t') -- r contiguous complex, 16-byte loads -- and writes the 2 x 2 real
                // blocks [[re, -im], [im, re]] of its row at offsets that are compile-time steps from one base
                // (rows n = o 2r + 2t', n + 1; columns k = i 2r + 2j, k + 1; i 2r = 0 mod 4 for even r).  Item
                // order (one complex per thread, as in the compose loop) spent ~3x the instructions on index math;
                // store orders with fewer bank conflicts cost selects or a second split per complex and measured
                // slower (the fill is issue-bound on the two weight warps, not bound by shared-memory wavefronts).
                constexpr uint32_t KSTEP = (C::NB / 8) * 128;   // bytes between K-adjacent core matrices
#pragma unroll 1
                for (int row = wt; row < 16 * R; row += 64) {
                    const int tp = row % R, oi = row / R, o = oi >> 2, i = oi & 3;
                    const int n = o * C::SC + 2 * tp;
                    const uint32_t base = tc::kmaj_off(n, i * C::SC, C::NB);
                    const float2* src = st + row * R;
#pragma unroll
                    for (int j2 = 0; j2 < R; j2 += 2) {
                        const float4 cc = *reinterpret_cast<const float4*>(src + j2);
#pragma unroll
                        for (int h = 0; h < 2; h++) {
                            const float re = h ? cc.z : cc.x, im = h ? cc.w : cc.y;
                            float hr, lr, hi_, li;
                            tc::split(re, hr, lr);
                            tc::split(im, hi_, li);
                            const uint32_t off = base + uint32_t(j2 >> 1) * KSTEP + uint32_t(h) * 8;
                            *reinterpret_cast<float2*>(th + off) = make_float2(hr, -hi_);
                            *reinterpret_cast<float2*>(tl + off) = make_float2(lr, -li);
                            *reinterpret_cast<float2*>(th + off + 16) = make_float2(hi_, hr);
                            *reinterpret_cast<float2*>(tl + off + 16) = make_float2(li, lr);
                        }
                    }
                }
            } else {
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
            }
            tc::fence_proxy_async();
            tc::mbar_arrive(&w_full[wb]);
            asm volatile("bar.sync 1, 64;" ::: "memory");   // staging buffer sb free for group it + NS
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
                              cudaStream_t s, int rh, int rhg, const bfs::PeerOut& po, const BandVariant& bv,
                              const float2* Cpre)
{
    const bool compose = bv.compose;
    using C = BandTC<R>;
    const int64_t groups = d.N >> 2;
    const unsigned grid = unsigned(groups < sm_count() ? groups : sm_count());
    if (compose) {
        using CC = BandCmp<R, 2>;
        auto kern = band_cmp_kernel<R, 2>;
        const size_t smem = CC::SMEM;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
        CUtensorMap tin;
        e = make_rows_tmap(&tin, in, d.N * R, nv, R);
        if (e != cudaSuccess) return e;
        kern<<<grid, 512, smem, s>>>(tin, out, W[0], W[1], Cpre, d.LN, l_first, nv, rh, rhg, po);
        return cudaGetLastError();
    }
    auto kern = band_tc_kernel<R>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
    if (e != cudaSuccess) return e;
    kern<<<grid, 384, C::SMEM, s>>>(in, out, W[0], W[1], d.LN, l_first, nv, rh, rhg, po);
    return cudaGetLastError();
}

bool band_tc_supported(const Dims& d, int nv)
{
    return (d.R == 6 || d.R == 8 || d.R == 10 || d.R == 12) && nv >= 64 && nv % 2 == 0;
}

cudaError_t launch_band_tc(const Dims& d, int l_first, const float2* in, float2* out, const float2* const* W, int nv,
                           cudaStream_t s, int rh, int rhg, const bfs::PeerOut* po, const BandVariant& bv,
                           const float2* Cpre)
{
    const bfs::PeerOut pz = po ? *po : bfs::PeerOut{};
    switch (d.R) {
    case 6: return band_tc_go<6>(d, l_first, in, out, W, nv, s, rh, rhg, pz, bv, Cpre);
    case 8: return band_tc_go<8>(d, l_first, in, out, W, nv, s, rh, rhg, pz, bv, Cpre);
    case 10: return band_tc_go<10>(d, l_first, in, out, W, nv, s, rh, rhg, pz, bv, Cpre);
    case 12: return band_tc_go<12>(d, l_first, in, out, W, nv, s, rh, rhg, pz, bv, Cpre);
    default: return cudaErrorInvalidValue;
    }
}

// ---------------------------------------------------------------------------------------------
// Plan finalization for small vector batches: the composed operator of a two-level band, per group g
// (fixed a0 at the input level l_first - 1, 4 consecutive b) and block path (o, i):
//     C_g[o][i](t', j) = sum_{j'} W2[p2(o)](t', (i >> 1) r + j') W1[p1(i >> 1, o >> 1)](j', (i & 1) r + j)
// with p1(u, e) = (((2 a0 + e) << (LN - l_first)) + 2 bq + u, p2(o) = ((4 a0 + o) << shg) + bq -- the algebra
// the band kernel otherwise forms on chip per group (band_cmp_kernel), here once in FP64 and rounded to
// complex64.  Layout [g][o][i][t'][j]: 16 r^2 complex per group, the bytes of the group's 8 compact blocks.
// ---------------------------------------------------------------------------------------------
__global__ void compose_band_kernel(const float2* __restrict__ W1, const float2* __restrict__ W2, float2* __restrict__ Cg,
                                    int LN, int l_first, int R)
{
    const int64_t N = int64_t(1) << LN;
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t per = int64_t(16) * R * R;
    if (idx >= (N >> 2) * per) return;
    const int64_t g = idx / per;
    const int r = int(idx % per), j = r % R, tp = (r / R) % R, oi = r / (R * R), o = oi >> 2, i = oi & 3;
    const int lin = l_first - 1, shg = LN - lin - 2;
    const int64_t a0 = g >> shg, bq = g & ((int64_t(1) << shg) - 1);
    const int sp = i >> 1, sv = i & 1, up = o >> 1;
    const int64_t p1 = ((((a0 << 1) + up) << (LN - lin - 1)) + (bq << 1) + sp);
    const int64_t p2 = ((((a0 << 2) + o) << shg) + bq);
    const float2* w2 = W2 + p2 * 2 * R * R;   // column-major r x 2r
    const float2* w1 = W1 + p1 * 2 * R * R;
    double cr = 0, ci = 0;
    for (int jp = 0; jp < R; jp++) {
        const float2 a = w2[(sp * R + jp) * R + tp], b = w1[(sv * R + j) * R + jp];
        cr += double(a.x) * b.x - double(a.y) * b.y;
        ci += double(a.x) * b.y + double(a.y) * b.x;
    }
    Cg[idx] = make_float2(float(cr), float(ci));
}

cudaError_t launch_compose_band(const Dims& d, int l_first, const float2* W1, const float2* W2, float2* Cg,
                                cudaStream_t s)
{
    const int64_t n = (d.N >> 2) * 16 * d.R * d.R;
    compose_band_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(W1, W2, Cg, d.LN, l_first, d.R);
    return cudaGetLastError();
}

// shared with bf_band3.cu
cudaError_t rows_tmap(CUtensorMap* m, const float2* base, int64_t rows, int nv, int box_rows)
{
    return make_rows_tmap(m, base, rows, nv, box_rows);
}
int tc_sm_count() { return sm_count(); }

int64_t ux_floats(const Dims& d) { return sl_i2(d.R) ? leafx_floats(d) / 2 : leafx_floats(d); }
int64_t v0x_floats(const Dims& d) { return s0_i2(d.R, 1 << d.l0) ? leafx_floats(d) / 2 : leafx_floats(d); }

}  // namespace bfk
