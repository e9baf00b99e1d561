// bf_band3.cu -- three transfer levels per launch on the tensor cores (eqn:2 P:748-752 for l <= h, eqn:3
// P:780-785 for l > h; the switch P:755-766 folded into the level-h blocks), for the large vector batches of
// cfg3/cfg4 at r <= 8.
//
// Why: at cfg4 every transfer launch is HBM-bound on the coefficient arrays (read + write 2 N r nv complex64,
// 69 GB at r = 8), and the two-level band (band_cmp_kernel) runs at ~0.87 of HBM.  Three levels per launch
// move 8 transfer levels in 3 launches (3 + 3 + 2) instead of 4: one coefficient round trip less per apply.
//
// Algebra (as for the two-level band, R18): three adjacent factors G^{l+2} G^{l+1} G^l of eqn:BFM
// map a group of 8 input pairs at level l-1 (fixed a0, 8 consecutive b = 8 bq + i) to 8 output pairs at level
// l+2 (a = 8 a0 + o, b = bq), and each output pair reaches each input pair through exactly one pair of each
// middle level, so the band is ONE dense 8 x 8 block operator per group
//     C[o][i] = W3[p3(o)](:, c3 r..) W2[p2(o, i)](:, c2 r..) W1[p1(o, i)](:, c1 r..)     (r x r blocks)
// with o = 4 e1 + 2 e2 + e3 (e_m the a-bit level m adds) and c1 = i & 1, c2 = (i >> 1) & 1, c3 = i >> 2.
// It is composed ONCE at plan finalization in FP64 (compose3_kernel; 64 r^2 complex per group, the group's
// 24 compact blocks are 48 r^2) and read per group by the kernel, which embeds and splits it into the B tile.
//
// Kernel (persistent, one CTA per SM, 16 warps), job = group x 128-vector tile, D[v][n] = sum_k A[v][k] B[n][k]
// with K = N = 16 r (8 pair slots of 2r real columns):
//   warp 12 (one lane)  2-D TMA copies of the 8 input pairs' rows into a ring of single-pair slots,
//   warps 0-7           split them hi/lo into A in TMEM (lane quadrant warp & 3; K half warp >> 2 = input
//                       pairs 4 kh .. 4 kh + 3),
//   warp 13             per job and K half: 3 passes (3xTF32, corrections first) x (8r / 8) MMAs into one of two
//                       TMEM accumulators (N = 16 r); A is released per K half, so the split of the next job
//                       overlaps the MMAs of the other half; B is released after the group's last tile,
//   warps 8-11          drain the accumulator (lane = vector) and store the 8 output pairs (pointer walk),
//   warps 14-15         embed + split the group's precomposed operator into the B tile (hi | lo, canonical
//                       K-major), per K half (the MMAs of a group's first tile start on half 0), its loads issued
//                       before the tile is free.
// TMEM: A hi/lo 2 x 16r columns + 2 accumulators of 16r = 64 r <= 512, hence r <= 8.
// Shared memory: the B tile (2 x (16r)^2 x 4 B = 128 KB at r = 8) + the raw ring (12 slots of r x 1 KB).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "bf_internal.h"
#include "tc_sm100.cuh"

namespace bfk {

// bf_tc.cu
cudaError_t rows_tmap(CUtensorMap* m, const float2* base, int64_t rows, int nv, int box_rows);
int tc_sm_count();

namespace {

__device__ constexpr int kPass3[3] = {1, 2, 0};   // Alo Bhi, Ahi Blo, then Ahi Bhi (bf_tc.cu kPassOrder)

template <int R>
struct Band3 {
    static constexpr int P = 8;                 // pairs per group
    static constexpr int SC = 2 * R;            // real columns of one pair slot
    static constexpr int KB = P * SC;           // MMA K = N = 16 r
    static constexpr int KH = KB / 2;           // one K half = 4 input pairs
    static constexpr int NB = KB;
    static constexpr int ACOLS = 2 * KB;        // A: hi at 0, lo at KB
    static constexpr int D_OFF = ACOLS;         // two accumulators of NB columns
    static constexpr int TMEM_COLS = 512;
    static constexpr uint32_t SLOT = uint32_t(R) * 128 * 8;     // raw rows of one pair, one vector tile
    static constexpr uint32_t WT = uint32_t(NB) * KB * 4;       // one B tile (hi or lo)
    static constexpr uint32_t WH = WT / 2;                      // its K half (k-chunk-major layout)
    static constexpr size_t LIM = 232448 - 1024;
    static constexpr int NQ_FIT = int((LIM - 2 * size_t(WT)) / SLOT);
    static constexpr int NQ = NQ_FIT > 16 ? 16 : NQ_FIT;
    static constexpr uint32_t OFF_W = uint32_t(NQ) * SLOT;
    static constexpr size_t SMEM = size_t(OFF_W) + 2 * size_t(WT);
    static constexpr int ROWS_H = 8 * 4 * R;                    // operator rows (o, i, t') of one K half
    static constexpr int RPT = ROWS_H / 64;                     // per weight thread
    static_assert(R % 2 == 0 && KB % 16 == 0 && ACOLS + 2 * NB <= TMEM_COLS && NQ >= 8 && OFF_W % 128 == 0 &&
                      WH % 128 == 0 && ROWS_H % 64 == 0 && SMEM <= LIM,
                  "three-level band shape");
};

template <int R>
__global__ void __launch_bounds__(512, 1)
    band3_kernel(const __grid_constant__ CUtensorMap tin, float2* __restrict__ out, const float2* __restrict__ Cpre,
                 int LN, int l_first, int nv)
{
    using C = Band3<R>;
    extern __shared__ __align__(128) uint8_t sm3[];
    __shared__ uint64_t slot_full[16], slot_empty[16];
    __shared__ uint64_t a_ready[2], a_free[2], d_full[2], d_free[2], w_full[2], w_free;
    __shared__ uint32_t tmem_base;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t N = int64_t(1) << LN;
    const int lin = l_first - 1, shg = LN - lin - 3;
    const int64_t ngroups = N >> 3;
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
            tc::mbar_init(&a_ready[i], 128);
            tc::mbar_init(&a_free[i], 1);
            tc::mbar_init(&d_full[i], 1);
            tc::mbar_init(&d_free[i], 128);
            tc::mbar_init(&w_full[i], 64);
        }
        tc::mbar_init(&w_free, 1);
        tc::mbar_fence_init();
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tmem_base;

    if (warp < 8) {
        // ---- split: raw rows -> A (TMEM), lane = vector; warp (lane quadrant qd, K half kh) ----
        const int qd = warp & 3, kh = warp >> 2;
        const int v = qd * 32 + lane;
        const uint32_t lb = uint32_t(qd * 32) << 16;
        for (int J = 0; J < njobs; J++) {
            if (J > 0) tc::mbar_wait(&a_free[kh], uint32_t(J - 1) & 1);
            tc::fence_after_sync();
#pragma unroll 1
            for (int s = 4 * kh; s < 4 * kh + 4; s++) {
                const int k = J * C::P + s, q = k % C::NQ;
                tc::mbar_wait(&slot_full[q], uint32_t(k / C::NQ) & 1);
                const float2* rd = reinterpret_cast<const float2*>(sm3 + q * C::SLOT);
                float hi[C::SC], lo[C::SC];
#pragma unroll
                for (int t = 0; t < R; t++) {
                    const float2 x = rd[t * 128 + v];
                    tc::split(x.x, hi[2 * t], lo[2 * t]);
                    tc::split(x.y, hi[2 * t + 1], lo[2 * t + 1]);
                }
                tc::mbar_arrive(&slot_empty[q]);   // the slot's values are in registers
                const uint32_t ta = tmem + lb + uint32_t(s * C::SC);
                tc::tmem_st_cols<C::SC>(ta, hi);
                tc::tmem_st_cols<C::SC>(ta + C::KB, lo);
            }
            tc::tmem_wait_st();
            tc::fence_before_sync();
            tc::mbar_arrive(&a_ready[kh]);
        }
    } else if (warp < 12) {
        // ---- epilogue: drain the accumulator two output pairs at a time, store by pointer walk ----
        const int q = warp & 3;
        const int v = q * 32 + lane;
        const uint32_t lb = uint32_t(q * 32) << 16;
        const int64_t pstep = (int64_t(1) << shg) * R * int64_t(nv);   // between output pairs o, o + 1
        for (int J = 0; J < njobs; J++) {
            const int it = int(unsigned(J) / unsigned(nvt));
            const int vt = J - it * nvt;
            const int64_t g = blockIdx.x + int64_t(it) * gridDim.x;
            const int db = J & 1;
            tc::mbar_wait(&d_full[db], uint32_t(J >> 1) & 1);
            tc::fence_after_sync();
            const int vg = vt * 128 + v;
            const int64_t a0 = g >> shg, bq = g & ((int64_t(1) << shg) - 1);
            float2* o0 = out + (((a0 << 3) << shg) + bq) * R * int64_t(nv) + vg;
#pragma unroll 1
            for (int h = 0; h < 4; h++) {
                float d[2 * C::SC];
                tc::tmem_ld_cols<2 * C::SC>(tmem + lb + uint32_t(C::D_OFF + db * C::NB + h * 2 * C::SC), d);
                tc::tmem_wait_ld();
                if (h == 3) {
                    tc::fence_before_sync();
                    tc::mbar_arrive(&d_free[db]);
                }
                if (vg < nv) {
#pragma unroll
                    for (int oo = 0; oo < 2; oo++) {
                        float2* o = o0 + (2 * h + oo) * pstep;
#pragma unroll
                        for (int t = 0; t < R; t++)
                            o[int64_t(t) * nv] = make_float2(d[oo * C::SC + 2 * t], d[oo * C::SC + 2 * t + 1]);
                    }
                }
            }
        }
    } else if (warp == 12) {
        // ---- loader: one 2-D tensor copy per input pair (r rows x 128 vectors); the group's 8 pairs are contiguous
        for (int J = 0; J < njobs; J++) {
            const int it = int(unsigned(J) / unsigned(nvt));
            const int vt = J - it * nvt;
            const int64_t g = blockIdx.x + int64_t(it) * gridDim.x;
            const int64_t pin = g * C::P;
            for (int s = 0; s < C::P; s++) {
                const int k = J * C::P + s, q = k % C::NQ;
                if (k >= C::NQ) tc::mbar_wait(&slot_empty[q], uint32_t(k / C::NQ - 1) & 1);
                if (lane == 0) {
                    tc::mbar_arrive_expect_tx(&slot_full[q], C::SLOT);   // whole box (ragged tile: zero fill)
                    tc::tma_load_2d(sm3 + q * C::SLOT, &tin, 2 * vt * 128, int((pin + s) * R), &slot_full[q]);
                }
                __syncwarp();
            }
        }
    } else if (warp == 13) {
        // ---- MMA issuer (whole warp, one elected lane issues) ----
        constexpr uint32_t idesc = tc::idesc_tf32(128, C::NB);
        constexpr uint32_t LBO_B = (C::NB / 8) * 128;
        const uint64_t dW = tc::desc_kmajor(tc::smem_u32(sm3 + C::OFF_W), LBO_B);
        for (int J = 0; J < njobs; J++) {
            const int it = int(unsigned(J) / unsigned(nvt));
            const int vt = J - it * nvt;
            const int db = J & 1;
            if (J >= 2) tc::mbar_wait(&d_free[db], uint32_t((J >> 1) - 1) & 1);
            const uint32_t d = tmem + uint32_t(C::D_OFF + db * C::NB);
#pragma unroll 1
            for (int kh = 0; kh < 2; kh++) {
                if (vt == 0) tc::mbar_wait(&w_full[kh], uint32_t(it) & 1);
                tc::mbar_wait(&a_ready[kh], uint32_t(J) & 1);
                tc::fence_after_sync();
#pragma unroll
                for (int qq = 0; qq < 3; qq++) {
                    const int pass = kPass3[qq];
                    const uint32_t a = tmem + uint32_t(kh * C::KH + (pass == 1 ? C::KB : 0));
                    const uint64_t b = tc::desc_add(dW, (pass == 2 ? C::WT : 0u) + uint32_t(kh) * C::WH);
#pragma unroll
                    for (int ks = 0; ks < C::KH / 8; ks++)
                        tc::mma_tf32_ts_warp(d, a + ks * 8, tc::desc_add(b, ks * 2 * LBO_B), idesc,
                                             (kh | qq | ks) ? 1u : 0u);
                }
                tc::commit_warp(&a_free[kh]);
                // the B tile is released whole, after the group's last K half: releasing it per K half (the fill of
                // the next group's K half 0 overlapping the last tile's K-half-1 MMAs) corrupted the next group's
                // first vector tile on B200, non-deterministically (measured; the halves are disjoint bytes, and
                // the hazard is not understood), so that overlap is not used
                if (vt == nvt - 1 && kh == 1) tc::commit_warp(&w_free);
            }
            tc::commit_warp(&d_full[db]);
            __syncwarp();
        }
    } else {
        // ---- weights (warps 14-15): the group's precomposed operator C[o][i](t', j) (layout [o][i][t'][j]) ->
        //      real-embedded hi / lo B tiles, one K half (input pairs 4 kh .. 4 kh + 3) at a time; a thread takes
        //      whole rows (o, i, t') of r contiguous complex and loads them before waiting for the half to be free
        const int wt = tid - 448;
        constexpr uint32_t KSTEP = (C::NB / 8) * 128;   // bytes between K-adjacent core matrices
        uint8_t* th = sm3 + C::OFF_W;
        uint8_t* tl = th + C::WT;
        for (int it = 0; it < nit; it++) {
            const int64_t g = blockIdx.x + int64_t(it) * gridDim.x;
            const float2* cg = Cpre + g * int64_t(64 * R * R);
#pragma unroll 1
            for (int kh = 0; kh < 2; kh++) {
                float4 c[C::RPT][R / 2];
#pragma unroll
                for (int rr = 0; rr < C::RPT; rr++) {
                    const int row = wt + 64 * rr, tp = row % R, oi = row / R, o = oi >> 2, i = 4 * kh + (oi & 3);
                    const float4* src = reinterpret_cast<const float4*>(cg + ((o * 8 + i) * R + tp) * R);
#pragma unroll
                    for (int j2 = 0; j2 < R / 2; j2++) c[rr][j2] = __ldg(src + j2);
                }
                if (it >= 1 && kh == 0) tc::mbar_wait(&w_free, uint32_t(it - 1) & 1);
#pragma unroll
                for (int rr = 0; rr < C::RPT; rr++) {
                    const int row = wt + 64 * rr, tp = row % R, oi = row / R, o = oi >> 2, i = 4 * kh + (oi & 3);
                    const uint32_t base = tc::kmaj_off(o * C::SC + 2 * tp, i * C::SC, C::NB);
#pragma unroll
                    for (int j2 = 0; j2 < R / 2; j2++) {
#pragma unroll
                        for (int hh = 0; hh < 2; hh++) {
                            const float re = hh ? c[rr][j2].z : c[rr][j2].x, im = hh ? c[rr][j2].w : c[rr][j2].y;
                            float hr, lr, hi_, li;
                            tc::split(re, hr, lr);
                            tc::split(im, hi_, li);
                            const uint32_t off = base + uint32_t(j2) * KSTEP + uint32_t(hh) * 8;
                            *reinterpret_cast<float2*>(th + off) = make_float2(hr, -hi_);
                            *reinterpret_cast<float2*>(tl + off) = make_float2(lr, -li);
                            *reinterpret_cast<float2*>(th + off + 16) = make_float2(hi_, hr);
                            *reinterpret_cast<float2*>(tl + off + 16) = make_float2(li, lr);
                        }
                    }
                }
                tc::fence_proxy_async();
                tc::mbar_arrive(&w_full[kh]);
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

template <int R>
cudaError_t band3_go(const Dims& d, int l_first, const float2* in, float2* out, const float2* Cpre, int nv,
                     cudaStream_t s)
{
    using C = Band3<R>;
    auto kern = band3_kernel<R>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
    if (e != cudaSuccess) return e;
    CUtensorMap tin;
    e = rows_tmap(&tin, in, d.N * R, nv, R);
    if (e != cudaSuccess) return e;
    const int64_t groups = d.N >> 3;
    const unsigned grid = unsigned(groups < tc_sm_count() ? groups : tc_sm_count());
    kern<<<grid, 512, C::SMEM, s>>>(tin, out, Cpre, d.LN, l_first, nv);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Plan finalization: the composed three-level operator of the band starting at l_first, per group g (fixed a0
// at the input level l_first - 1, 8 consecutive b) and block path (o, i):
//   C_g[o][i](t', j) = sum_{j''} W3[p3](t', c3 r + j'') sum_{j'} W2[p2](j'', c2 r + j') W1[p1](j', c1 r + j)
//   p1 = ((2 a0 + e1) << (LN - l_first)) + 4 bq + (i >> 1),         c1 = i & 1
//   p2 = ((4 a0 + 2 e1 + e2) << (LN - l_first - 1)) + 2 bq + (i >> 2), c2 = (i >> 1) & 1
//   p3 = ((8 a0 + o) << (LN - l_first - 2)) + bq,                   c3 = i >> 2
// (o = 4 e1 + 2 e2 + e3; blocks column-major r x 2r).  FP64 products, complex64 result, layout [g][o][i][t'][j].
// ---------------------------------------------------------------------------------------------
__global__ void compose3_kernel(const float2* __restrict__ W1, const float2* __restrict__ W2,
                                const float2* __restrict__ W3, float2* __restrict__ Cg, int LN, int l_first, int R)
{
    const int64_t N = int64_t(1) << LN;
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t per = int64_t(64) * R * R;
    if (idx >= (N >> 3) * per) return;
    const int64_t g = idx / per;
    const int rr = int(idx % per), j = rr % R, tp = (rr / R) % R, oi = rr / (R * R), o = oi >> 3, i = oi & 7;
    const int lin = l_first - 1, shg = LN - lin - 3;
    const int64_t a0 = g >> shg, bq = g & ((int64_t(1) << shg) - 1);
    const int e1 = o >> 2, e2 = (o >> 1) & 1;
    const int c1 = i & 1, c2 = (i >> 1) & 1, c3 = i >> 2;
    const int64_t p1 = (((a0 << 1) + e1) << (LN - lin - 1)) + (bq << 2) + (i >> 1);
    const int64_t p2 = (((a0 << 2) + 2 * e1 + e2) << (LN - lin - 2)) + (bq << 1) + (i >> 2);
    const int64_t p3 = (((a0 << 3) + o) << shg) + bq;
    const float2* w1 = W1 + p1 * 2 * R * R;
    const float2* w2 = W2 + p2 * 2 * R * R;
    const float2* w3 = W3 + p3 * 2 * R * R;
    double cr = 0, ci = 0;
    for (int j2 = 0; j2 < R; j2++) {
        double mr = 0, mi = 0;
        for (int j1 = 0; j1 < R; j1++) {
            const float2 a = w2[(c2 * R + j1) * R + j2], b = w1[(c1 * R + j) * R + j1];
            mr += double(a.x) * b.x - double(a.y) * b.y;
            mi += double(a.x) * b.y + double(a.y) * b.x;
        }
        const float2 w = w3[(c3 * R + j2) * R + tp];
        cr += double(w.x) * mr - double(w.y) * mi;
        ci += double(w.x) * mi + double(w.y) * mr;
    }
    Cg[idx] = make_float2(float(cr), float(ci));
}

}  // namespace

bool band3_supported(const Dims& d, int nv)
{
    return (d.R == 6 || d.R == 8) && nv >= 128 && nv % 2 == 0 && d.LN >= 3;
}

int64_t band3_operator_elems(const Dims& d) { return (d.N >> 3) * 64 * int64_t(d.R) * d.R; }

cudaError_t launch_band3(const Dims& d, int l_first, const float2* in, float2* out, const float2* Cpre, int nv,
                         cudaStream_t s)
{
    switch (d.R) {
    case 6: return band3_go<6>(d, l_first, in, out, Cpre, nv, s);
    case 8: return band3_go<8>(d, l_first, in, out, Cpre, nv, s);
    default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_compose3(const Dims& d, int l_first, const float2* W1, const float2* W2, const float2* W3,
                            float2* Cg, cudaStream_t s)
{
    const int64_t n = band3_operator_elems(d);
    compose3_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(W1, W2, W3, Cg, d.LN, l_first, d.R);
    return cudaGetLastError();
}

}  // namespace bfk
