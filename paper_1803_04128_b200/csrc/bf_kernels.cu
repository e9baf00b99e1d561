// bf_kernels.cu -- sm_100a kernels of the IBF-MAT apply (arXiv:1803.04128).
//
// Every stage of eqn:BFM is a batch of small dense complex block
// products that share nothing but the coefficient arrays, so each is written
// as an FP32 register-blocked "outer product" loop: a thread owns TN
// consecutive vectors of one unit (leaf / butterfly / T_X leaf) and R (or JT)
// output rows; the block entries of one unit are warp-uniform loads (L1
// broadcast), the vector operands are coalesced 16-byte loads.  4 FFMA per
// complex MAC, FP32 accumulation (north_star).
//
// Coefficient layout (workspace): delta[pair][t][v], v < nv fastest,
// v = c * n_amp + k (RHS column c, amplitude term k).  See DESIGN.md section 4.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>

#include "bf_internal.h"
#include "bf_shard.h"

namespace bfk {

__device__ __forceinline__ void cmac(float2& acc, const float2 w, const float2 v)
{
    acc.x = fmaf(w.x, v.x, acc.x);
    acc.x = fmaf(-w.y, v.y, acc.x);
    acc.y = fmaf(w.x, v.y, acc.y);
    acc.y = fmaf(w.y, v.x, acc.y);
}

// explicit FMAs: every kernel variant rounds a product the same way (bitwise batch consistency)
__device__ __forceinline__ float2 cmul(const float2 a, const float2 b)
{
    return make_float2(fmaf(a.x, b.x, -(a.y * b.y)), fmaf(a.x, b.y, a.y * b.x));
}

// Load / store K consecutive complex values (16-byte vectors where possible).
template <int K>
__device__ __forceinline__ void ldc(float2 (&v)[K], const float2* p)
{
    if constexpr (K % 2 == 0) {
#pragma unroll
        for (int i = 0; i < K / 2; i++) {
            float4 q = reinterpret_cast<const float4*>(p)[i];
            v[2 * i] = make_float2(q.x, q.y);
            v[2 * i + 1] = make_float2(q.z, q.w);
        }
    } else {
#pragma unroll
        for (int i = 0; i < K; i++) v[i] = p[i];
    }
}

template <int K>
__device__ __forceinline__ void ldc_ro(float2 (&v)[K], const float2* __restrict__ p)
{
    if constexpr (K % 2 == 0) {
#pragma unroll
        for (int i = 0; i < K / 2; i++) {
            float4 q = __ldg(reinterpret_cast<const float4*>(p) + i);
            v[2 * i] = make_float2(q.x, q.y);
            v[2 * i + 1] = make_float2(q.z, q.w);
        }
    } else {
#pragma unroll
        for (int i = 0; i < K; i++) v[i] = __ldg(p + i);
    }
}

template <int K>
__device__ __forceinline__ void stc(float2* p, const float2 (&v)[K])
{
    if constexpr (K % 2 == 0) {
#pragma unroll
        for (int i = 0; i < K / 2; i++)
            reinterpret_cast<float4*>(p)[i] = make_float4(v[2 * i].x, v[2 * i].y, v[2 * i + 1].x, v[2 * i + 1].y);
    } else {
#pragma unroll
        for (int i = 0; i < K; i++) p[i] = v[i];
    }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem)
{
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }


// A lane's 4 vectors as two 2-vector chunks, HALF apart: every LDS.128/STG.128 instruction of a warp
// then covers 32 x 16 contiguous bytes (conflict-free, fully coalesced).  pos(i) is the vector offset
// (within the tile) of the lane's i-th vector.
template <int HALF>
__device__ __forceinline__ int qpos(int col, int i) { return (i < 2 ? 0 : HALF) + 2 * col + (i & 1); }

template <int HALF>
__device__ __forceinline__ void ldq(float2 (&v)[4], const float2* base, int col)
{
    float4 a = *reinterpret_cast<const float4*>(base + 2 * col);
    float4 b = *reinterpret_cast<const float4*>(base + HALF + 2 * col);
    v[0] = make_float2(a.x, a.y);
    v[1] = make_float2(a.z, a.w);
    v[2] = make_float2(b.x, b.y);
    v[3] = make_float2(b.z, b.w);
}

template <int HALF>
__device__ __forceinline__ void stq(float2* base, int col, const float2 (&v)[4], bool lo_ok, bool hi_ok)
{
    if (lo_ok) *reinterpret_cast<float4*>(base + 2 * col) = make_float4(v[0].x, v[0].y, v[1].x, v[1].y);
    if (hi_ok) *reinterpret_cast<float4*>(base + HALF + 2 * col) = make_float4(v[2].x, v[2].y, v[3].x, v[3].y);
}

// ---------------------------------------------------------------------------
// S0: amplitude pre-scale + leaf interpolation (eqn:1; eqn:tg P:24-28).
// CTA = 32 columns (lanes) x 8 warps.  A column is (leaf b, vector group vg).
// The scaled leaf inputs y[j][v] = b_k(x) F[x, c] are staged once in shared
// memory; warp w computes the pairs (a, b) for a = w, w+8, ...
// ---------------------------------------------------------------------------
template <int R, int TN>
__global__ void __launch_bounds__(256) s0_kernel(const float2* __restrict__ F, int64_t ldf,
                                                 const float2* __restrict__ ampb, const float2* __restrict__ V0,
                                                 float2* __restrict__ out, int LN, int l0, int n_amp, int nv)
{
    extern __shared__ float4 smem_s0[];
    float2* Ys = reinterpret_cast<float2*>(smem_s0);   // [n0][32 * TN]
    const int64_t N = int64_t(1) << LN;
    const int n0 = 1 << l0;
    const int64_t nleaf = N >> l0;
    const int cpu = nv / TN;   // columns per leaf
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int64_t col0 = int64_t(blockIdx.x) * 32;
    constexpr int W = 32 * TN;

    for (int e = threadIdx.x; e < n0 * W; e += blockDim.x) {
        const int j = e % n0, ci = e / n0, col = ci / TN, i = ci % TN;
        const int64_t gcol = col0 + col, b = gcol / cpu;
        float2 val = make_float2(0.f, 0.f);
        if (b < nleaf) {
            const int v = int(gcol % cpu) * TN + i, c = v / n_amp, k = v % n_amp;
            const int64_t x = b * n0 + j;
            val = cmul(__ldg(ampb + k * N + x), __ldg(F + x + c * ldf));
        }
        Ys[j * W + col * TN + i] = val;
    }
    __syncthreads();

    const int64_t gc = col0 + lane, b = gc / cpu;
    if (b >= nleaf) return;
    const int vg = int(gc % cpu);
    for (int a = warp; a < n0; a += nwarps) {
        const int64_t p = int64_t(a) * nleaf + b;
        const float2* Vb = V0 + p * n0 * R;   // column-major r x n0: column j at j*R
        float2 acc[R][TN];
#pragma unroll
        for (int t = 0; t < R; t++)
#pragma unroll
            for (int i = 0; i < TN; i++) acc[t][i] = make_float2(0.f, 0.f);
#pragma unroll 2
        for (int j = 0; j < n0; j++) {
            float2 y[TN], w[R];
            ldc<TN>(y, Ys + j * W + lane * TN);
            ldc_ro<R>(w, Vb + j * R);
#pragma unroll
            for (int t = 0; t < R; t++)
#pragma unroll
                for (int i = 0; i < TN; i++) cmac(acc[t][i], w[t], y[i]);
        }
        float2* o = out + p * R * nv + vg * TN;
#pragma unroll
        for (int t = 0; t < R; t++) stc<TN>(o + int64_t(t) * nv, acc[t]);
    }
}

// ---------------------------------------------------------------------------
// Transfer level (eqn:2 P:748-752 for l <= h, eqn:3 P:780-785 for l > h).
// A butterfly unit u = P 2^(LN-l) + b reads the two pairs 2u, 2u+1 of level
// l-1 (contiguous: [2 R][nv]) and writes the pairs (2P+e) 2^(LN-l) + b, e=0,1.
// One thread: both outputs (2 R rows) x TN vectors.  (The switch, is folded into the
// level-h blocks at plan finalization.)
// ---------------------------------------------------------------------------
template <int R, int TN>
__global__ void __launch_bounds__(128) xfer_kernel(const float2* __restrict__ in, float2* __restrict__ out,
                                                   const float2* __restrict__ Wl,
                                                   int LN, int l, int nv, int rh, int rhg, const bfs::PeerOut po)
{
    const int64_t N = int64_t(1) << LN;
    const int cpu = nv / TN;
    const int64_t gc = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t u = gc / cpu;
    if (u >= N / 2) return;
    const int vg = int(gc % cpu);
    const int sh = LN - l;
    const int64_t P = u >> sh, b = u & ((int64_t(1) << sh) - 1);
    const int64_t p0 = (2 * P << sh) + b, p1 = p0 + (int64_t(1) << sh);
    // inputs: pairs 2u, 2u+1 of level l-1 (in a receive buffer of the index-sharded exchange when rh > 0)
    const int64_t pin = rh ? bfs::recv_index(2 * u, rh, rhg) : 2 * u;
    const float2* x = in + pin * R * nv + vg * TN;
    const float2* W0 = Wl + p0 * 2 * R * R;   // column-major r x 2r: column k at k*R
    const float2* W1 = Wl + p1 * 2 * R * R;

    float2 acc0[R][TN], acc1[R][TN];
#pragma unroll
    for (int t = 0; t < R; t++)
#pragma unroll
        for (int i = 0; i < TN; i++) acc0[t][i] = acc1[t][i] = make_float2(0.f, 0.f);

#pragma unroll 2
    for (int k = 0; k < 2 * R; k++) {
        float2 xv[TN], w[R];
        ldc_ro<TN>(xv, x + int64_t(k) * nv);
        ldc_ro<R>(w, W0 + k * R);
#pragma unroll
        for (int t = 0; t < R; t++)
#pragma unroll
            for (int i = 0; i < TN; i++) cmac(acc0[t][i], w[t], xv[i]);
        ldc_ro<R>(w, W1 + k * R);
#pragma unroll
        for (int t = 0; t < R; t++)
#pragma unroll
            for (int i = 0; i < TN; i++) cmac(acc1[t][i], w[t], xv[i]);
    }

#pragma unroll
    for (int e = 0; e < 2; e++) {
        float2 (&acc)[R][TN] = e ? acc1 : acc0;
        const int64_t p = e ? p1 : p0;
        float2* o = bfs::pair_out(out, po, p, R, nv) + vg * TN;
#pragma unroll
        for (int t = 0; t < R; t++) stc<TN>(o + int64_t(t) * nv, acc[t]);
    }
}

// ---------------------------------------------------------------------------
constexpr int S0T_VT = 128;   // vectors per tile
constexpr int S0T_AG = 8;     // values of a per chunk (= warps)
constexpr int S0T_PAD = 2;    // Y row padding (complex) against bank conflicts of the fill

template <int R>
__host__ __device__ constexpr size_t s0t_smem_bytes(int n0)
{
    return (size_t(n0) * (S0T_VT + S0T_PAD) + size_t(S0T_AG) * n0 * R) * sizeof(float2);
}

// ---------------------------------------------------------------------------
// S0, tiled (large nv): CTA = one leaf b x 128 vectors, looping over all n0 values of a in chunks of 8.
// Y = b_k o F (n0 x 128) is staged in shared memory once; the V0 blocks of each chunk of 8 pairs are
// loaded with cp.async (single buffer: two CTAs per SM cover each other's loads).  Warp w computes
// pair (a, b), a = 8 chunk + w, for its 128 vectors (lane: 4 consecutive vectors x all R rows), every
// operand from shared memory (weights: warp-uniform broadcast LDS.128).
template <int R>
__global__ void __launch_bounds__(256, 2) s0_tile_kernel(const float2* __restrict__ F, int64_t ldf,
                                                         const float2* __restrict__ ampb,
                                                         const float2* __restrict__ V0, float2* __restrict__ out,
                                                         int LN, int l0, int n_amp, int nv)
{
    constexpr int TN = 4, VT = S0T_VT, YS = S0T_VT + S0T_PAD;
    extern __shared__ float4 smem_s0t[];
    const int n0 = 1 << l0;
    float2* Ys = reinterpret_cast<float2*>(smem_s0t);   // [n0][YS]
    float2* Vs = Ys + n0 * YS;                          // [8][n0 (j)][R (t)]
    const int64_t N = int64_t(1) << LN;
    const int64_t nleaf = N >> l0;
    const int64_t b = blockIdx.x;
    const int v0 = blockIdx.y * VT;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nchunk = n0 / S0T_AG;
    const int blk = n0 * R;   // complex per V0 block

    auto load_v0 = [&](int ch) {
        float2* dst = Vs;
        for (int idx = tid; idx < S0T_AG * blk / 2; idx += 256) {
            const int w = idx / (blk / 2), o = idx % (blk / 2);
            const int64_t p = int64_t(ch * S0T_AG + w) * nleaf + b;
            cp_async16(dst + w * blk + 2 * o, V0 + p * blk + 2 * o);
        }
        cp_async_commit();
    };
    load_v0(0);
    // Y[j][v] = b_k(x) F[x, c],  x = b n0 + j, v = c n_amp + k  (zero beyond nv); 8 loads in flight per thread
    for (int base = tid; base < n0 * VT; base += 256 * 8) {
        float2 fv[8], bv[8];
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const int idx = base + q * 256;
            fv[q] = bv[q] = make_float2(0.f, 0.f);
            const int j = idx % n0, v = v0 + idx / n0;
            if (idx < n0 * VT && v < nv) {
                const int c = v / n_amp, k = v - c * n_amp;
                const int64_t x = b * n0 + j;
                fv[q] = __ldg(F + x + c * ldf);
                bv[q] = __ldg(ampb + k * N + x);
            }
        }
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const int idx = base + q * 256;
            if (idx < n0 * VT) Ys[(idx % n0) * YS + idx / n0] = cmul(bv[q], fv[q]);
        }
    }

    const int v_lo = v0 + 2 * lane, v_hi = v0 + VT / 2 + 2 * lane;   // nv % 4 == 0: chunks all-or-nothing
    for (int ch = 0; ch < nchunk; ch++) {
        if (ch > 0) load_v0(ch);
        cp_async_wait_all();
        __syncthreads();
        const float2* Vb = Vs + warp * blk;
        float2 acc[R][TN];
#pragma unroll
        for (int t = 0; t < R; t++)
#pragma unroll
            for (int i = 0; i < TN; i++) acc[t][i] = make_float2(0.f, 0.f);
#pragma unroll 2
        for (int j = 0; j < n0; j++) {
            float2 y[TN], w[R];
            ldq<VT / 2>(y, Ys + j * YS, lane);
            ldc<R>(w, Vb + j * R);
#pragma unroll
            for (int t = 0; t < R; t++)
#pragma unroll
                for (int i = 0; i < TN; i++) cmac(acc[t][i], w[t], y[i]);
        }
        __syncthreads();   // the V0 chunk is consumed: the next iteration refills it
        {
            const int64_t p = int64_t(ch * S0T_AG + warp) * nleaf + b;
            float2* o = out + p * R * nv + v0;
#pragma unroll
            for (int t = 0; t < R; t++) stq<VT / 2>(o + int64_t(t) * nv, lane, acc[t], v_lo < nv, v_hi < nv);
        }
    }
}

// ---------------------------------------------------------------------------
// SL, tiled (large nv): CTA = one T_X leaf a x 128 vectors, n0/8 warps; warp w
// owns output rows j in [8w, 8w+8), lane 4 consecutive vectors.  The K = n0 R
// reduction (b, t) streams through shared memory in chunks of 2 pairs
// (coefficients [2R][128] and U blocks [2][R][n0]), double-buffered with
// cp.async.  Epilogue: a_k(x) scaling and the sum over k in registers, then the
// G tile is transposed through shared memory so each RHS column is written as
// n0 contiguous complex values.
// ---------------------------------------------------------------------------
constexpr int SLT_VT = 128;
constexpr int SLT_BC = 2;   // pairs per K chunk

template <int R>
__host__ __device__ constexpr size_t slt_smem_bytes(int n0)
{
    return size_t(2) * (size_t(SLT_BC) * R * SLT_VT + size_t(SLT_BC) * R * n0) * sizeof(float2);
}

template <int R, int NA>
__global__ void __launch_bounds__(256, 2) sl_tile_kernel(const float2* __restrict__ in, const float2* __restrict__ U,
                                                         const float2* __restrict__ ampa, float2* __restrict__ G,
                                                         int64_t ldg, int LN, int l0, int nv)
{
    constexpr int TN = 4, JT = 8, VT = SLT_VT, BC = SLT_BC;
    static_assert(TN % NA == 0, "a thread owns whole RHS columns");
    extern __shared__ float4 smem_slt[];
    const int n0 = 1 << l0;
    float2* Ds = reinterpret_cast<float2*>(smem_slt);   // [2][BC R][VT]
    float2* Us = Ds + 2 * BC * R * VT;                   // [2][BC][R][n0]
    const int64_t N = int64_t(1) << LN;
    const int64_t a = blockIdx.x;
    const int v0 = blockIdx.y * VT;
    const int vw = min(VT, nv - v0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = blockDim.x;
    const int j0 = warp * JT;

    auto load_chunk = [&](int ch, int buf) {
        const int64_t p0 = a * n0 + int64_t(ch) * BC;   // first pair of the chunk (level D)
        float2* D = Ds + buf * BC * R * VT;
        for (int idx = tid; idx < BC * R * (VT / 2); idx += nthr) {
            const int row = idx / (VT / 2), vv = (idx % (VT / 2)) * 2;
            if (vv < vw) cp_async16(D + row * VT + vv, in + (p0 * R + row) * int64_t(nv) + v0 + vv);
        }
        float2* Ub = Us + buf * BC * R * n0;
        for (int idx = tid; idx < BC * R * n0 / 2; idx += nthr) cp_async16(Ub + 2 * idx, U + p0 * R * n0 + 2 * idx);
        cp_async_commit();
    };

    float2 acc[JT][TN];
#pragma unroll
    for (int jj = 0; jj < JT; jj++)
#pragma unroll
        for (int i = 0; i < TN; i++) acc[jj][i] = make_float2(0.f, 0.f);

    const int nch = n0 / BC;
    load_chunk(0, 0);
    for (int ch = 0; ch < nch; ch++) {
        const int buf = ch & 1;
        if (ch + 1 < nch) {
            load_chunk(ch + 1, buf ^ 1);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            cp_async_wait_all();
        }
        __syncthreads();
        const float2* D = Ds + buf * BC * R * VT;
        const float2* Ub = Us + buf * BC * R * n0 + j0;
#pragma unroll 2
        for (int k = 0; k < BC * R; k++) {
            float2 xv[TN], w[JT];
            if constexpr (NA <= 2) ldq<VT / 2>(xv, D + k * VT, lane);
            else ldc<TN>(xv, D + k * VT + lane * TN);
            ldc<JT>(w, Ub + k * n0);
#pragma unroll
            for (int jj = 0; jj < JT; jj++)
#pragma unroll
                for (int i = 0; i < TN; i++) cmac(acc[jj][i], w[jj], xv[i]);
        }
        __syncthreads();   // buffer `buf` is reloaded two chunks later
    }

    // epilogue: g(x, c) = sum_k a_k(x) u_k(x), staged as Gs[j][c_local] (reuses the chunk buffers) so that
    // each RHS column leaves as n0 contiguous complex values
    constexpr int CPT = TN / NA;                 // RHS columns per thread
    constexpr int CT = VT / NA;                  // RHS columns per tile
    float2* Gs = Ds;                             // [n0][CT + 1]
#pragma unroll
    for (int jj = 0; jj < JT; jj++) {
        const int64_t x = a * n0 + j0 + jj;
        float2 ak[NA];
#pragma unroll
        for (int k = 0; k < NA; k++) ak[k] = __ldg(ampa + k * N + x);
#pragma unroll
        for (int cc = 0; cc < CPT; cc++) {
            float2 g = make_float2(0.f, 0.f);
#pragma unroll
            for (int k = 0; k < NA; k++) cmac(g, ak[k], acc[jj][cc * NA + k]);
            const int cl = (NA <= 2 ? qpos<VT / 2>(lane, cc * NA) : lane * TN + cc * NA) / NA;
            Gs[(j0 + jj) * (CT + 1) + cl] = g;
        }
    }
    __syncthreads();
    const int c0 = v0 / NA, cw = vw / NA;
    for (int idx = tid; idx < CT * n0; idx += nthr) {
        const int j = idx % n0, cl = idx / n0;
        if (cl < cw) G[a * n0 + j + int64_t(c0 + cl) * ldg] = Gs[j * (CT + 1) + cl];
    }
}

// ---------------------------------------------------------------------------
// Band: K consecutive transfer levels fused in one CTA (SURVEY 8(a) "fusion
// geometry").  A group of 2^K pairs closed under K levels -- fixed a0 at the
// input level l_first-1 and 2^K consecutive b's -- is loaded once per vector
// tile into shared memory (cp.async), carried through the K levels in place,
// and only the last level is written to HBM: the coefficient traffic of the
// band is one read + one write instead of K of each.  The weights of all K
// levels stay resident
// in shared memory while the CTA sweeps the vector tiles.
//
// In place: at band level m the unit (e', i) reads the physical slots
// phi_{m-1}(e', 2i+c) = (2i+c) 2^(m-1) + bitrev_{m-1}(e') and writes its two
// outputs back into the same two slots (phi_m(E, i) = i 2^m + bitrev_m(E)), so
// a thread only ever touches its own (slot, vector) cells within a level and
// one barrier per level suffices.
// ---------------------------------------------------------------------------
struct BandArgs {
    const float2* W[4];   // weights of band levels 1..K (bf.h XFER layout; level h has the switch folded in)
    bfs::PeerOut po;      // fused exchange: peer stores of the last level (po.on)
    int rh, rhg;          // > 0: the input is a receive buffer of the index-sharded exchange (bf_shard.h)
};


template <int K>
__host__ __device__ constexpr int band_vt() { return 1024 >> K; }   // 256 threads = U units x 2 outputs x VT/4

template <int R, int K>
__host__ __device__ constexpr size_t band_smem_bytes()
{
    return (size_t((1 << K) * R * band_vt<K>()) + size_t(K * (1 << (K - 1)) * 4 * R * R)) * sizeof(float2);
}

// One thread owns ONE output pair (e) of a unit x 4 vectors (R x 4 accumulators: each weight is reused
// across 4 vectors, each vector element across R rows).  Both threads of a unit read the same two
// input slots, so the in-place write-back waits for a barrier after the reads.
template <int R, int K>
__global__ void __launch_bounds__(256, (R <= 10 ? 2 : 1))
    band_kernel(const float2* __restrict__ in, float2* __restrict__ out, const BandArgs args, int LN, int l_first, int nv)
{
    constexpr int TN = 4;
    constexpr int U = 1 << (K - 1);   // butterfly units per level
    constexpr int P = 1 << K;         // pairs per group
    constexpr int VT = band_vt<K>();  // vectors per tile
    constexpr int COLS = VT / TN;     // thread columns per (unit, output)
    extern __shared__ float4 smem_band[];
    float2* X = reinterpret_cast<float2*>(smem_band);   // [P][R][VT]
    float2* Ws = X + P * R * VT;                         // [K][U][2R (k)][2R (e R + t)]

    const int lin = l_first - 1;   // input level
    const int shg = LN - lin - K;
    const int64_t g = blockIdx.x;
    const int64_t a0 = g >> shg, bq = g & ((int64_t(1) << shg) - 1);
    const int tid = threadIdx.x;
    const int col = tid % COLS, e = (tid / COLS) & 1, u = tid / (2 * COLS);

#pragma unroll
    for (int m = 1; m <= K; m++) {
        const int sh = LN - lin - m;   // log2 of the b-range at level lin + m
        for (int idx = tid; idx < U * 4 * R * R; idx += 256) {
            const int t = idx % R, k = (idx / R) % (2 * R), ee = (idx / (2 * R * R)) & 1, uu = idx / (4 * R * R);
            const int ep = uu >> (K - m), i = uu & ((1 << (K - m)) - 1);
            const int64_t p = (((a0 << m) + 2 * ep + ee) << sh) + (bq << (K - m)) + i;
            Ws[(((m - 1) * U + uu) * 2 * R + k) * 2 * R + ee * R + t] = __ldg(args.W[m - 1] + p * 2 * R * R + k * R + t);
        }
    }
    const int nvt = (nv + VT - 1) / VT;
    for (int vt = 0; vt < nvt; vt++) {
        const int v0 = vt * VT;
        const int vw = min(VT, nv - v0);
        __syncthreads();   // the previous tile is consumed; weights are in place
        const int64_t pin = args.rh ? bfs::recv_index(g * P, args.rh, args.rhg) : g * P;   // P pairs contiguous
        const float2* src = in + pin * R * int64_t(nv) + v0;
        for (int idx = tid; idx < P * R * (VT / 2); idx += 256) {
            const int vv = (idx % (VT / 2)) * 2, row = idx / (VT / 2);
            if (vv < vw) cp_async16(X + row * VT + vv, src + int64_t(row) * nv + vv);
        }
        cp_async_commit();
        cp_async_wait_all();
        __syncthreads();

        // vectors {2 col, 2 col + 1} and {VT/2 + 2 col, ...}: each 2-vector chunk is valid or not as a whole
        const bool lo_ok = 2 * col < vw, hi_ok = VT / 2 + 2 * col < vw, active = lo_ok;
#pragma unroll 1
        for (int m = 1; m <= K; m++) {
            const int ep = u >> (K - m), i = u & ((1 << (K - m)) - 1);
            const int br = (m > 1) ? int(__brev(unsigned(ep)) >> (33 - m)) : 0;
            const int s0 = (2 * i) * (1 << (m - 1)) + br, s1 = s0 + (1 << (m - 1));
            float2 acc[R][TN];
#pragma unroll
            for (int t = 0; t < R; t++)
#pragma unroll
                for (int q = 0; q < TN; q++) acc[t][q] = make_float2(0.f, 0.f);
            if (active) {
                const float2* W = Ws + ((m - 1) * U + u) * 4 * R * R + e * R;
#pragma unroll 1
                for (int c = 0; c < 2; c++) {
                    const float2* xs = X + (c ? s1 : s0) * R * VT;
                    const float2* wc = W + c * R * 2 * R;
#pragma unroll 1
                    for (int k = 0; k < R; k++) {
                        float2 x[TN], w[R];
                        ldq<VT / 2>(x, xs + k * VT, col);
                        ldc<R>(w, wc + k * 2 * R);
#pragma unroll
                        for (int t = 0; t < R; t++)
#pragma unroll
                            for (int q = 0; q < TN; q++) cmac(acc[t][q], w[t], x[q]);
                    }
                }
            }
            if (m < K) __syncthreads();   // both outputs of every unit have read the input slots
            if (active) {
                // destination of output row t: the thread's own slot (in place) or, at the last level, HBM
                float2* dst;
                int64_t rstride;
                if (m < K) {
                    dst = X + ((e ? s1 : s0) * R) * VT;
                    rstride = VT;
                } else {
                    const int64_t p = (((a0 << K) + 2 * ep + e) << (LN - lin - K)) + bq;
                    dst = bfs::pair_out(out, args.po, p, R, nv) + v0;
                    rstride = nv;
                }
#pragma unroll
                for (int t = 0; t < R; t++) stq<VT / 2>(dst + t * rstride, col, acc[t], lo_ok, hi_ok);
            }
            if (m < K) __syncthreads();
        }
    }
}

// ---------------------------------------------------------------------------
// SL: leaf evaluation (eqn:bf3) + amplitude post-scale and sum over
// k (eqn:tg).  CTA = 32 columns (T_X leaf a, vector group) x n0/JT
// warps; warp w owns the JT output rows j in [w JT, w JT + JT).
// ---------------------------------------------------------------------------
template <int R, int TN, int JT, int NA>
__global__ void __launch_bounds__(256) sl_kernel(const float2* __restrict__ in, const float2* __restrict__ U,
                                                 const float2* __restrict__ ampa, float2* __restrict__ G, int64_t ldg,
                                                 int LN, int l0, int nv)
{
    static_assert(TN % NA == 0, "a thread owns whole RHS columns");
    const int64_t N = int64_t(1) << LN;
    const int n0 = 1 << l0;
    const int64_t nleaf = N >> l0;
    const int cpu = nv / TN;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t gc = int64_t(blockIdx.x) * 32 + lane, a = gc / cpu;
    if (a >= nleaf) return;
    const int vg = int(gc % cpu);
    const int j0 = warp * JT;

    float2 acc[JT][TN];
#pragma unroll
    for (int jj = 0; jj < JT; jj++)
#pragma unroll
        for (int i = 0; i < TN; i++) acc[jj][i] = make_float2(0.f, 0.f);

    for (int b = 0; b < n0; b++) {
        const int64_t p = a * n0 + b;
        const float2* x = in + p * R * nv + vg * TN;
        const float2* Ub = U + p * R * n0 + j0;   // column-major n0 x r: column t at t*n0
#pragma unroll 2
        for (int t = 0; t < R; t++) {
            float2 xv[TN], w[JT];
            ldc_ro<TN>(xv, x + int64_t(t) * nv);
            ldc_ro<JT>(w, Ub + t * n0);
#pragma unroll
            for (int jj = 0; jj < JT; jj++)
#pragma unroll
                for (int i = 0; i < TN; i++) cmac(acc[jj][i], w[jj], xv[i]);
        }
    }
    // epilogue: G[x, c] = sum_k a_k(x) u_k(x)
    const int c0 = vg * (TN / NA);
#pragma unroll
    for (int jj = 0; jj < JT; jj++) {
        const int64_t xrow = a * n0 + j0 + jj;
        float2 ak[NA];
#pragma unroll
        for (int k = 0; k < NA; k++) ak[k] = __ldg(ampa + k * N + xrow);
#pragma unroll
        for (int cc = 0; cc < TN / NA; cc++) {
            float2 g = make_float2(0.f, 0.f);
#pragma unroll
            for (int k = 0; k < NA; k++) cmac(g, ak[k], acc[jj][cc * NA + k]);
            G[xrow + int64_t(c0 + cc) * ldg] = g;
        }
    }
}

// a global load ptxas keeps in program order (volatile asm): the tiny kernels issue a whole block of operand
// loads before their first MAC -- with plain loads the scheduler interleaved one load per MAC pair, one memory
// round trip each
__device__ __forceinline__ float2 ldg_early(const float2* p)
{
    float2 v;
    asm volatile("ld.global.nc.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
    return v;
}

// ---------------------------------------------------------------------------
// Tiny vector batches (nv <= 4: cfg1 has nv = 2): one thread per output row and all nv vectors in registers,
// reduction loops fully unrolled so each thread keeps a dozen independent loads in flight.  The per-column
// kernels above give such batches a few hundred threads that each walk ~200 dependent load rounds (30-66 us per
// stage at N = 2^10); these have N r threads.  Every output is accumulated in the same order with the same
// cmac/cmul as s0_kernel / xfer_kernel / sl_kernel (bitwise equal results).
// ---------------------------------------------------------------------------
template <int R, int NV>
__global__ void __launch_bounds__(256, 1) s0_tiny_kernel(const float2* __restrict__ F, int64_t ldf,
                                                      const float2* __restrict__ ampb, const float2* __restrict__ V0,
                                                      float2* __restrict__ out, int LN, int l0, int n_amp)
{
    const int64_t N = int64_t(1) << LN;
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= N * R) return;
    const int64_t p = idx / R;
    const int t = int(idx % R), n0 = 1 << l0;
    const int64_t nleaf = N >> l0, b = p % nleaf;
    float2 acc[NV];
#pragma unroll
    for (int v = 0; v < NV; v++) acc[v] = make_float2(0.f, 0.f);
    const float2* Vb = V0 + p * n0 * R + t;   // column-major r x n0: element (t, j) at j R + t
    for (int j0 = 0; j0 < n0; j0 += 8) {      // n0 >= 8: stage 8 columns' operands, then their MACs
        float2 w[8], fa[8][NV], fb[8][NV];
#pragma unroll
        for (int jj = 0; jj < 8; jj++) {
            const int64_t x = b * n0 + j0 + jj;
            w[jj] = ldg_early(Vb + (j0 + jj) * R);
#pragma unroll
            for (int v = 0; v < NV; v++) {
                const int c = v / n_amp, k = v - c * n_amp;
                fa[jj][v] = ldg_early(ampb + k * N + x);
                fb[jj][v] = ldg_early(F + x + c * ldf);
            }
        }
        #pragma unroll
        for (int jj = 0; jj < 8; jj++)
#pragma unroll
            for (int v = 0; v < NV; v++) cmac(acc[v], w[jj], cmul(fa[jj][v], fb[jj][v]));
    }
#pragma unroll
    for (int v = 0; v < NV; v++) out[(p * R + t) * NV + v] = acc[v];
}

template <int R, int NV>
__global__ void __launch_bounds__(256, 1) xfer_tiny_kernel(const float2* __restrict__ in, float2* __restrict__ out,
                                                        const float2* __restrict__ Wl, int LN, int l, int rh, int rhg,
                                                        const bfs::PeerOut po)
{
    const int64_t N = int64_t(1) << LN;
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= N * R) return;
    const int64_t p = idx / R;
    const int t = int(idx % R), sh = LN - l;
    const int64_t a = p >> sh, b = p & ((int64_t(1) << sh) - 1);
    const int64_t u = ((a >> 1) << sh) + b;   // the butterfly unit: inputs 2u, 2u+1 of level l-1
    const int64_t pin = rh ? bfs::recv_index(2 * u, rh, rhg) : 2 * u;
    const float2* x = in + pin * R * NV;
    const float2* W = Wl + p * 2 * R * R + t;   // column-major r x 2r: element (t, k) at k R + t
    float2 acc[NV];
#pragma unroll
    for (int v = 0; v < NV; v++) acc[v] = make_float2(0.f, 0.f);
    float2 w[2 * R], xv[2 * R][NV];   // all operands first (one memory round trip), then the 2r MACs
#pragma unroll
    for (int k = 0; k < 2 * R; k++) {
        w[k] = ldg_early(W + k * R);
#pragma unroll
        for (int v = 0; v < NV; v++) xv[k][v] = ldg_early(x + k * NV + v);
    }
#pragma unroll
    for (int k = 0; k < 2 * R; k++)
#pragma unroll
        for (int v = 0; v < NV; v++) cmac(acc[v], w[k], xv[k][v]);
    float2* o = bfs::pair_out(out, po, p, R, NV) + t * NV;
#pragma unroll
    for (int v = 0; v < NV; v++) o[v] = acc[v];
}

// SL: a CTA takes LPB whole T_X leaves: their U blocks and coefficient rows (contiguous in HBM) are staged in
// shared memory with 16-byte loads from all threads at once (one memory round trip), then thread (leaf, x, v)
// -- v fastest, so the n_amp vectors of a column sit in adjacent lanes -- runs the (b, t) reduction in
// sl_kernel's order and lane k = 0 forms sum_k a_k(x) u_k(x) from its neighbours (warp shuffles).
template <int R, int NV, int NA>
__global__ void __launch_bounds__(256, 1) sl_tiny_kernel(const float2* __restrict__ in, const float2* __restrict__ U,
                                                         const float2* __restrict__ ampa, float2* __restrict__ G,
                                                         int64_t ldg, int LN, int l0, int LPB)
{
    extern __shared__ float4 smem_sltiny[];
    const int64_t N = int64_t(1) << LN;
    const int n0 = 1 << l0;
    const int64_t nleaf = N >> l0, a0 = int64_t(blockIdx.x) * LPB;
    const int nl = int(nleaf - a0 < LPB ? nleaf - a0 : LPB);
    const int ue = n0 * R * n0, xe = n0 * R * NV;   // complex per leaf
    float2* Us = reinterpret_cast<float2*>(smem_sltiny);
    float2* Xs = Us + LPB * ue;
    {   // cp.async: every 16-byte copy in flight at once (a load-then-store loop waited one round trip each)
        const float2* su = U + a0 * ue;
        for (int i = threadIdx.x; i < nl * ue / 2; i += blockDim.x) cp_async16(Us + 2 * i, su + 2 * i);
        const float2* sx = in + a0 * xe;
        for (int i = threadIdx.x; i < nl * xe / 2; i += blockDim.x) cp_async16(Xs + 2 * i, sx + 2 * i);
        cp_async_commit();
        cp_async_wait_all();
    }
    __syncthreads();
    const int li = threadIdx.x / (n0 * NV), rem = threadIdx.x % (n0 * NV), j = rem / NV, v = rem % NV;
    const bool live = li < nl;
    float2 acc = make_float2(0.f, 0.f);
    if (live) {
        const float2* Ub = Us + li * ue + j;   // column-major n0 x r per pair: element (j, t) at t n0 + j
        const float2* xb = Xs + li * xe + v;
        for (int b = 0; b < n0; b++) {
#pragma unroll
            for (int t = 0; t < R; t++) cmac(acc, Ub[(b * R + t) * n0], xb[(b * R + t) * NV]);
        }
    }
    float2 uk[NA];
#pragma unroll
    for (int k = 0; k < NA; k++) {
        uk[k].x = __shfl_sync(0xffffffffu, acc.x, (threadIdx.x & 31) + k, 32);
        uk[k].y = __shfl_sync(0xffffffffu, acc.y, (threadIdx.x & 31) + k, 32);
    }
    if (!live || v % NA) return;
    const int64_t x = (a0 + li) * n0 + j;
    float2 g = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < NA; k++) cmac(g, __ldg(ampa + k * N + x), uk[k]);
    G[x + int64_t(v / NA) * ldg] = g;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
bool rank_supported(int R) { return R == 6 || R == 8 || R == 10 || R == 12 || R == 14 || R == 16; }

static inline int pick_tn(int nv, int maxtn)
{
    if (maxtn >= 4 && nv % 4 == 0) return 4;
    if (maxtn >= 2 && nv % 2 == 0) return 2;
    return 1;
}

template <int R, int TN>
static cudaError_t s0_go(const Dims& d, const float2* F, int64_t ldf, const float2* ampb, const float2* V0, float2* out,
                         int nv, cudaStream_t s)
{
    const int64_t cols = (d.N >> d.l0) * (nv / TN);
    const size_t shm = size_t(1 << d.l0) * 32 * TN * sizeof(float2);
    auto kern = s0_kernel<R, TN>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm));
    if (e != cudaSuccess) return e;
    kern<<<unsigned((cols + 31) / 32), 256, shm, s>>>(F, ldf, ampb, V0, out, d.LN, d.l0, d.n_amp, nv);
    return cudaGetLastError();
}

template <int R, int TN>
static cudaError_t xfer_go(const Dims& d, int l, const float2* in, float2* out, const float2* W, int nv, int rh, int rhg,
                           const bfs::PeerOut& po, cudaStream_t s)
{
    const int64_t threads = (d.N / 2) * (nv / TN);
    xfer_kernel<R, TN><<<unsigned((threads + 127) / 128), 128, 0, s>>>(in, out, W, d.LN, l, nv, rh, rhg, po);
    return cudaGetLastError();
}

template <int R, int TN, int NA>
static cudaError_t sl_go(const Dims& d, const float2* in, const float2* U, const float2* ampa, float2* G, int64_t ldg,
                         int nv, cudaStream_t s)
{
    constexpr int JT = 8;
    const int n0 = 1 << d.l0;
    const int64_t cols = (d.N >> d.l0) * (nv / TN);
    sl_kernel<R, TN, JT, NA><<<unsigned((cols + 31) / 32), 32 * (n0 / JT), 0, s>>>(in, U, ampa, G, ldg, d.LN, d.l0, nv);
    return cudaGetLastError();
}

#define BF_DISPATCH_R(R, CALL)                                                                                         \
    switch (R) {                                                                                                       \
    case 6: { constexpr int RR = 6; return CALL; }                                                                     \
    case 8: { constexpr int RR = 8; return CALL; }                                                                     \
    case 10: { constexpr int RR = 10; return CALL; }                                                                   \
    case 12: { constexpr int RR = 12; return CALL; }                                                                   \
    case 14: { constexpr int RR = 14; return CALL; }                                                                   \
    case 16: { constexpr int RR = 16; return CALL; }                                                                   \
    default: return cudaErrorInvalidValue;                                                                             \
    }

template <int R>
static cudaError_t s0t_go(const Dims& d, const float2* F, int64_t ldf, const float2* ampb, const float2* V0,
                          float2* out, int nv, cudaStream_t s)
{
    const int n0 = 1 << d.l0;
    const size_t shm = s0t_smem_bytes<R>(n0);
    auto kern = s0_tile_kernel<R>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm));
    if (e != cudaSuccess) return e;
    dim3 grid(unsigned(d.N >> d.l0), unsigned((nv + S0T_VT - 1) / S0T_VT));
    kern<<<grid, 256, shm, s>>>(F, ldf, ampb, V0, out, d.LN, d.l0, d.n_amp, nv);
    return cudaGetLastError();
}

static bool tiled_ok(const Dims& d, int nv) { return nv >= 64 && nv % 4 == 0 && d.l0 <= 6; }

template <int R, int NV>
static cudaError_t s0_tiny_go(const Dims& d, const float2* F, int64_t ldf, const float2* ampb, const float2* V0,
                              float2* out, cudaStream_t s)
{
    const int64_t n = d.N * R;
    s0_tiny_kernel<R, NV><<<unsigned((n + 255) / 256), 256, 0, s>>>(F, ldf, ampb, V0, out, d.LN, d.l0, d.n_amp);
    return cudaGetLastError();
}

template <int R, int NV>
static cudaError_t xfer_tiny_go(const Dims& d, int l, const float2* in, float2* out, const float2* W, int rh, int rhg,
                                const bfs::PeerOut& po, cudaStream_t s)
{
    const int64_t n = d.N * R;
    xfer_tiny_kernel<R, NV><<<unsigned((n + 255) / 256), 256, 0, s>>>(in, out, W, d.LN, l, rh, rhg, po);
    return cudaGetLastError();
}

// leaves per CTA of sl_tiny_kernel (0: the leaf does not fit shared memory / 256 threads)
static int sl_tiny_lpb(const Dims& d, int nv)
{
    const int n0 = 1 << d.l0;
    const size_t leaf = size_t(n0) * d.R * (n0 + nv) * sizeof(float2);
    int lpb = int((96 * 1024) / leaf);
    if (lpb * n0 * nv > 256) lpb = 256 / (n0 * nv);
    return lpb;
}

template <int R, int NV, int NA>
static cudaError_t sl_tiny_go(const Dims& d, const float2* in, const float2* U, const float2* ampa, float2* G,
                              int64_t ldg, cudaStream_t s)
{
    const int n0 = 1 << d.l0, lpb = sl_tiny_lpb(d, NV);
    const size_t shm = size_t(lpb) * n0 * R * (n0 + NV) * sizeof(float2);
    auto kern = sl_tiny_kernel<R, NV, NA>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm));
    if (e != cudaSuccess) return e;
    const int64_t nleaf = d.N >> d.l0;
    const int threads = (lpb * n0 * NV + 31) / 32 * 32;
    kern<<<unsigned((nleaf + lpb - 1) / lpb), threads, shm, s>>>(in, U, ampa, G, ldg, d.LN, d.l0, lpb);
    return cudaGetLastError();
}

#define BF_TINY_NV(NVV, CALL)                                                                                  \
    switch (NVV) {                                                                                             \
    case 1: { constexpr int NN = 1; BF_DISPATCH_R(d.R, CALL) }                                                 \
    case 2: { constexpr int NN = 2; BF_DISPATCH_R(d.R, CALL) }                                                 \
    case 3: { constexpr int NN = 3; BF_DISPATCH_R(d.R, CALL) }                                                 \
    default: { constexpr int NN = 4; BF_DISPATCH_R(d.R, CALL) }                                                \
    }

cudaError_t launch_s0(const Dims& d, const float2* F, int64_t ldf, const float2* ampb, const float2* V0, float2* out,
                      int nv, cudaStream_t s)
{
    if (nv <= 4) BF_TINY_NV(nv, (s0_tiny_go<RR, NN>(d, F, ldf, ampb, V0, out, s)))
    if (tiled_ok(d, nv)) BF_DISPATCH_R(d.R, (s0t_go<RR>(d, F, ldf, ampb, V0, out, nv, s)))
    const int tn = pick_tn(nv, 4);
    if (tn == 4) BF_DISPATCH_R(d.R, (s0_go<RR, 4>(d, F, ldf, ampb, V0, out, nv, s)))
    if (tn == 2) BF_DISPATCH_R(d.R, (s0_go<RR, 2>(d, F, ldf, ampb, V0, out, nv, s)))
    BF_DISPATCH_R(d.R, (s0_go<RR, 1>(d, F, ldf, ampb, V0, out, nv, s)))
}

cudaError_t launch_xfer(const Dims& d, int l, const float2* in, float2* out, const float2* W, int nv, cudaStream_t s,
                        int rh, int rhg, const bfs::PeerOut* po)
{
    const bfs::PeerOut pz = po ? *po : bfs::PeerOut{};
    if (nv <= 4) BF_TINY_NV(nv, (xfer_tiny_go<RR, NN>(d, l, in, out, W, rh, rhg, pz, s)))
    const int tn = pick_tn(nv, 2);
    if (tn == 2) BF_DISPATCH_R(d.R, (xfer_go<RR, 2>(d, l, in, out, W, nv, rh, rhg, pz, s)))
    BF_DISPATCH_R(d.R, (xfer_go<RR, 1>(d, l, in, out, W, nv, rh, rhg, pz, s)))
}

template <int R, int NA>
static cudaError_t slt_go(const Dims& d, const float2* in, const float2* U, const float2* ampa, float2* G, int64_t ldg,
                          int nv, cudaStream_t s)
{
    const int n0 = 1 << d.l0;
    size_t shm = slt_smem_bytes<R>(n0);
    const size_t gsb = size_t(SLT_VT / NA + 1) * n0 * sizeof(float2);   // epilogue staging reuses the buffers
    if (gsb > shm) shm = gsb;
    auto kern = sl_tile_kernel<R, NA>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm));
    if (e != cudaSuccess) return e;
    dim3 grid(unsigned(d.N >> d.l0), unsigned((nv + SLT_VT - 1) / SLT_VT));
    kern<<<grid, 32 * (n0 / 8), shm, s>>>(in, U, ampa, G, ldg, d.LN, d.l0, nv);
    return cudaGetLastError();
}

cudaError_t launch_sl(const Dims& d, const float2* in, const float2* U, const float2* ampa, float2* G, int64_t ldg,
                      int nv, cudaStream_t s)
{
    if (nv <= 4 && sl_tiny_lpb(d, nv) >= 1) {
        if (d.n_amp == 1) BF_TINY_NV(nv, (sl_tiny_go<RR, NN, 1>(d, in, U, ampa, G, ldg, s)))
        if (d.n_amp == 2 && nv % 2 == 0) {
            if (nv == 2) BF_DISPATCH_R(d.R, (sl_tiny_go<RR, 2, 2>(d, in, U, ampa, G, ldg, s)))
            BF_DISPATCH_R(d.R, (sl_tiny_go<RR, 4, 2>(d, in, U, ampa, G, ldg, s)))
        }
        if (d.n_amp == 4 && nv == 4) BF_DISPATCH_R(d.R, (sl_tiny_go<RR, 4, 4>(d, in, U, ampa, G, ldg, s)))
    }
    if (tiled_ok(d, nv)) {
        if (d.n_amp == 4) BF_DISPATCH_R(d.R, (slt_go<RR, 4>(d, in, U, ampa, G, ldg, nv, s)))
        if (d.n_amp == 2) BF_DISPATCH_R(d.R, (slt_go<RR, 2>(d, in, U, ampa, G, ldg, nv, s)))
        BF_DISPATCH_R(d.R, (slt_go<RR, 1>(d, in, U, ampa, G, ldg, nv, s)))
    }
    // a thread must own whole RHS columns (all n_amp terms of a column): TN % n_amp == 0
    int tn = pick_tn(nv, 4);
    if (tn % d.n_amp != 0) tn = d.n_amp;
    if (d.n_amp == 4) BF_DISPATCH_R(d.R, (sl_go<RR, 4, 4>(d, in, U, ampa, G, ldg, nv, s)))
    if (d.n_amp == 2) {
        if (tn == 4) BF_DISPATCH_R(d.R, (sl_go<RR, 4, 2>(d, in, U, ampa, G, ldg, nv, s)))
        BF_DISPATCH_R(d.R, (sl_go<RR, 2, 2>(d, in, U, ampa, G, ldg, nv, s)))
    }
    if (tn == 4) BF_DISPATCH_R(d.R, (sl_go<RR, 4, 1>(d, in, U, ampa, G, ldg, nv, s)))
    if (tn == 2) BF_DISPATCH_R(d.R, (sl_go<RR, 2, 1>(d, in, U, ampa, G, ldg, nv, s)))
    BF_DISPATCH_R(d.R, (sl_go<RR, 1, 1>(d, in, U, ampa, G, ldg, nv, s)))
}

bool band_supported(int R, int nv) { return (R == 6 || R == 8 || R == 10 || R == 12) && nv % 4 == 0 && nv >= 128; }

template <int R, int K>
static cudaError_t band_go(const Dims& d, int l_first, const float2* in, float2* out, const float2* const* W, int nv,
                           cudaStream_t s, int rh, int rhg, const bfs::PeerOut* po)
{
    BandArgs a{};
    for (int m = 0; m < K; m++) a.W[m] = W[m];
    if (po) a.po = *po;
    a.rh = rh;
    a.rhg = rhg;
    const size_t shm = band_smem_bytes<R, K>();
    auto kern = band_kernel<R, K>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm));
    if (e != cudaSuccess) return e;
    const int64_t groups = d.N >> K;
    kern<<<unsigned(groups), 256, shm, s>>>(in, out, a, d.LN, l_first, nv);
    return cudaGetLastError();
}

cudaError_t launch_band(const Dims& d, int l_first, int K, const float2* in, float2* out, const float2* const* W, int nv,
                        cudaStream_t s, int rh, int rhg, const bfs::PeerOut* po)
{
#define BF_BAND_CASE(RR, KK) \
    case RR: return band_go<RR, KK>(d, l_first, in, out, W, nv, s, rh, rhg, po);
    if (K == 2) {
        switch (d.R) {
            BF_BAND_CASE(6, 2) BF_BAND_CASE(8, 2) BF_BAND_CASE(10, 2) BF_BAND_CASE(12, 2)
        default: return cudaErrorInvalidValue;
        }
    }
    if (K == 1) {
        switch (d.R) {
            BF_BAND_CASE(6, 1) BF_BAND_CASE(8, 1) BF_BAND_CASE(10, 1) BF_BAND_CASE(12, 1)
        default: return cudaErrorInvalidValue;
        }
    }
#undef BF_BAND_CASE
    return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------------------
// Plan finalization: fold the switch into the factor that produces level h.
// The BF is the product U G^{L-1}..G^{h+1} M^h G^h..G^{l0+1} V (eqn:BFM); M^h is
// block diagonal over the level-h pairs with the r x r blocks Sw[p], and the factor producing
// level h has the same pairs as its block rows, so M^h G^h is again block diagonal with blocks
// Sw[p] W[p] (r x cols).  One thread per (pair, column); FP64 accumulation, complex64 result,
// written in place over W.
// ---------------------------------------------------------------------------
__global__ void fold_switch_kernel(const float2* __restrict__ Sw, float2* __restrict__ W, int64_t npairs, int R,
                                   int cols)
{
    const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g >= npairs * cols) return;
    const int64_t p = g / cols;
    const int k = int(g % cols);
    float2* w = W + (p * cols + k) * R;   // column k of W[p] (column-major r x cols)
    const float2* S = Sw + p * R * R;     // column-major r x r
    double xr[16], xi[16];
    for (int s = 0; s < R; s++) {
        xr[s] = w[s].x;
        xi[s] = w[s].y;
    }
    for (int t = 0; t < R; t++) {
        double yr = 0, yi = 0;
        for (int s = 0; s < R; s++) {
            const float2 a = S[s * R + t];
            yr += double(a.x) * xr[s] - double(a.y) * xi[s];
            yi += double(a.x) * xi[s] + double(a.y) * xr[s];
        }
        w[t] = make_float2(float(yr), float(yi));
    }
}

cudaError_t launch_fold_switch(const float2* Sw, float2* W, int64_t npairs, int R, int cols, cudaStream_t s)
{
    if (R > 16) return cudaErrorInvalidValue;
    const int64_t n = npairs * cols;
    fold_switch_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(Sw, W, npairs, R, cols);
    return cudaGetLastError();
}


// ---------------------------------------------------------------------------
// Adjoint plan (bf_plan_create_adjoint): K* = sum_k conj(b_k) o BF*(conj(a_k) o .), and BF* is the factor
// product of eqn:BFM conjugate-transposed in reverse order.  With the roles of the two trees
// swapped (the adjoint's level-m pair (a~, b~) is the forward's level-(LN - m) pair (b~, a~)) BF* is a
// butterfly of the same shape, so the adjoint runs the forward kernels on re-assembled blocks.  Pure data
// movement plus conjugation: exact.
// ---------------------------------------------------------------------------
namespace {

// out block q = x K2 + y (cols_in x rows_in, column-major) = conj(in block p = y K1 + x)^T (rows_in x cols_in)
__global__ void adj_leaf_kernel(const float2* __restrict__ in, float2* __restrict__ out, int rows_in, int cols_in,
                                int64_t K1, int64_t K2, int64_t total)
{
    const int64_t per = int64_t(rows_in) * cols_in;
    for (int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < total; g += int64_t(gridDim.x) * blockDim.x) {
        const int64_t q = g / per;
        const int e = int(g % per);
        const int i = e % cols_in, j = e / cols_in;   // out(i, j): i < cols_in, j < rows_in
        const int64_t p = (q % K2) * K1 + q / K2;
        const float2 v = in[p * per + int64_t(i) * rows_in + j];
        out[g] = make_float2(v.x, -v.y);
    }
}

// adjoint transfer level m (output pairs (a~, b~), b~ < 2^lnb, lnb = LN - m) from the forward factor of level
// LN - m + 1, whose pairs are (a, b) with b < 2^(m-1):
//   W~[(a~,b~)](t, c r + s) = conj(W[(2 b~ + c) 2^(m-1) + (a~ >> 1)](s, (a~ & 1) r + t))
__global__ void adj_xfer_kernel(const float2* __restrict__ W, float2* __restrict__ out, int R, int lnb, int lfb,
                                int64_t total)
{
    const int64_t per = 2 * int64_t(R) * R;
    for (int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < total; g += int64_t(gridDim.x) * blockDim.x) {
        const int64_t q = g / per;
        const int e = int(g % per);
        const int t = e % R, col = e / R, c = col / R, s = col % R;
        const int64_t a = q >> lnb, b = q & ((int64_t(1) << lnb) - 1);
        const int64_t qf = ((2 * b + c) << lfb) + (a >> 1);
        const float2 v = W[qf * per + (int64_t(a & 1) * R + t) * R + s];
        out[g] = make_float2(v.x, -v.y);
    }
}

__global__ void conj_copy_kernel(const float2* __restrict__ in, float2* __restrict__ out, int64_t n)
{
    for (int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < n; g += int64_t(gridDim.x) * blockDim.x) {
        const float2 v = in[g];
        out[g] = make_float2(v.x, -v.y);
    }
}

unsigned grid_for(int64_t n) { return unsigned(std::min<int64_t>((n + 255) / 256, int64_t(148) * 16)); }

}  // namespace

cudaError_t launch_adjoint_factors(const Dims& d, const float2* amp_a, const float2* amp_b, const float2* v0,
                                   const float2* u, const float2* const* xfer, float2* adj_amp_a, float2* adj_amp_b,
                                   float2* adj_v0, float2* adj_u, float2* const* adj_xfer, cudaStream_t s)
{
    const int64_t N = d.N, n0 = int64_t(1) << d.l0, R = d.R, na = int64_t(d.n_amp) * N;
    conj_copy_kernel<<<grid_for(na), 256, 0, s>>>(amp_b, adj_amp_a, na);   // pre-scale conj(a_k) ...
    conj_copy_kernel<<<grid_for(na), 256, 0, s>>>(amp_a, adj_amp_b, na);   // ... post-scale conj(b_k)
    // S0~ pair a~ (N/n0) + b~ = U[b~ n0 + a~]^*;  SL~ pair a~ n0 + b~ = V0[b~ (N/n0) + a~]^*
    adj_leaf_kernel<<<grid_for(N * n0 * R), 256, 0, s>>>(u, adj_v0, int(n0), int(R), n0, N / n0, N * n0 * R);
    adj_leaf_kernel<<<grid_for(N * n0 * R), 256, 0, s>>>(v0, adj_u, int(R), int(n0), N / n0, n0, N * n0 * R);
    const int nx = d.D - d.l0;
    for (int i = 0; i < nx; i++) {   // adjoint level m = l0 + 1 + i from forward level LN - m + 1 (index nx - 1 - i)
        const int m = d.l0 + 1 + i;
        adj_xfer_kernel<<<grid_for(N * 2 * R * R), 256, 0, s>>>(xfer[nx - 1 - i], adj_xfer[i], int(R), d.LN - m, m - 1,
                                                               N * 2 * R * R);
    }
    return cudaGetLastError();
}

}  // namespace bfk
