// bf_recompress.cu -- recompression of the interpolative butterfly to a smaller rank r' (SURVEY 8(f) NEXT-3:
// "structure-preserving sweeping matrix compression", deferred there to [IBF]; R21).
//
// Plan-finalization work on the device in FP64 (like the switch fold and the band precomposition), one thread
// per pair.  Every coefficient space delta_l[p] in C^r of the factor product eqn:BFM carries the block
// K(A,B) = S_p R_p (R_p: input -> delta_l[p], S_p: delta_l[p] -> output).  Balanced truncation keeps its r'
// dominant directions:
//   Gamma_out[p] = S_p^H S_p   top-down:  U^H U at level D,  sum_e W_c^H Gamma_out[parent_e] W_c below
//   Gamma_in[p]  = R_p R_p^H   bottom-up over the already truncated lower levels
//   Gamma_out = Lo Lo^H, Gamma_in = Li Li^H (Cholesky),  C = Lo^H Li = X Sigma Y^H (one-sided Jacobi SVD),
//   P = Sigma_r'^{-1/2} X_r'^H Lo^H (r' x r),  Q = Li Y_r' Sigma_r'^{-1/2} (r x r'),
// so S_p Q P R_p is the best rank-r' approximation of the block.  New factors: V0' = P V0,
// W'_l = P_l W_l blockdiag(Q_{l-1}(q_0), Q_{l-1}(q_1)), U' = U Q_D.  The oracle (oracle/recompress.py) does the
// same with numpy's eigh square roots and SVD; the truncated operator does not depend on the square roots chosen.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>

#include "bf_internal.h"

namespace bfk {

namespace {

constexpr int RMAX = 12;   // source rank

struct zc {
    double x, y;
};
__device__ __forceinline__ zc mk(double a, double b) { return zc{a, b}; }
__device__ __forceinline__ zc zf(float2 v) { return zc{v.x, v.y}; }
__device__ __forceinline__ zc add(zc a, zc b) { return zc{a.x + b.x, a.y + b.y}; }
__device__ __forceinline__ zc sub(zc a, zc b) { return zc{a.x - b.x, a.y - b.y}; }
__device__ __forceinline__ zc mul(zc a, zc b) { return zc{a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x}; }
__device__ __forceinline__ zc cj(zc a) { return zc{a.x, -a.y}; }
__device__ __forceinline__ zc scl(zc a, double s) { return zc{a.x * s, a.y * s}; }
__device__ __forceinline__ double nrm2(zc a) { return a.x * a.x + a.y * a.y; }

// lower Cholesky of a Hermitian PSD r x r matrix (row-major), regularized by tiny * max diagonal
__device__ void chol(zc* A, int r)
{
    double md = 0;
    for (int i = 0; i < r; i++) md = fmax(md, A[i * r + i].x);
    const double reg = 1e-14 * (md > 0 ? md : 1.0);
    for (int j = 0; j < r; j++) {
        double d = A[j * r + j].x + reg;
        for (int k = 0; k < j; k++) d -= nrm2(A[j * r + k]);
        d = sqrt(fmax(d, reg));
        A[j * r + j] = mk(d, 0);
        for (int i = j + 1; i < r; i++) {
            zc s = add(A[i * r + j], mk(0, 0));
            for (int k = 0; k < j; k++) s = sub(s, mul(A[i * r + k], cj(A[j * r + k])));
            A[i * r + j] = scl(s, 1.0 / d);
        }
        for (int i = 0; i < j; i++) A[i * r + j] = mk(0, 0);
    }
}

// Balanced truncation of one pair: Gin, Gout (r x r, Hermitian, row-major; overwritten) -> P (rp x r) and
// Q (r x rp), row-major.
__device__ void truncate(zc* Gin, zc* Gout, int r, int rp, zc* P, zc* Q)
{
    chol(Gout, r);   // Lo
    chol(Gin, r);    // Li
    zc C[RMAX * RMAX], V[RMAX * RMAX];
    for (int i = 0; i < r; i++)
        for (int j = 0; j < r; j++) {
            zc s = mk(0, 0);
            for (int k = 0; k < r; k++) s = add(s, mul(cj(Gout[k * r + i]), Gin[k * r + j]));   // (Lo^H Li)(i, j)
            C[i * r + j] = s;
            V[i * r + j] = mk(i == j ? 1.0 : 0.0, 0);
        }
    // one-sided Jacobi (Hestenes): rotate column pairs of C (and V) until every pair is orthogonal
    for (int sweep = 0; sweep < 40; sweep++) {
        double off = 0;
        for (int i = 0; i < r - 1; i++)
            for (int j = i + 1; j < r; j++) {
                double a = 0, b = 0;
                zc g = mk(0, 0);
                for (int k = 0; k < r; k++) {
                    a += nrm2(C[k * r + i]);
                    b += nrm2(C[k * r + j]);
                    g = add(g, mul(cj(C[k * r + i]), C[k * r + j]));
                }
                const double ag = sqrt(nrm2(g));
                if (ag <= 1e-15 * sqrt(a * b) || ag == 0) continue;
                off = fmax(off, ag / sqrt(a * b));
                const zc ph = scl(cj(g), 1.0 / ag);   // e^{-i phi}: column j times it makes c_i^H c_j real
                const double zeta = (b - a) / (2 * ag);
                const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1 + zeta * zeta));
                const double cs = 1 / sqrt(1 + t * t), sn = cs * t;
                for (int k = 0; k < r; k++) {
                    const zc ci = C[k * r + i], cjp = mul(C[k * r + j], ph);
                    C[k * r + i] = sub(scl(ci, cs), scl(cjp, sn));
                    C[k * r + j] = add(scl(ci, sn), scl(cjp, cs));
                    const zc vi = V[k * r + i], vjp = mul(V[k * r + j], ph);
                    V[k * r + i] = sub(scl(vi, cs), scl(vjp, sn));
                    V[k * r + j] = add(scl(vi, sn), scl(vjp, cs));
                }
            }
        if (off < 1e-15) break;
    }
    double sig[RMAX];
    bool used[RMAX];
    for (int k = 0; k < r; k++) {
        double s = 0;
        for (int i = 0; i < r; i++) s += nrm2(C[i * r + k]);
        sig[k] = sqrt(s);
        used[k] = false;
    }
    for (int m = 0; m < rp; m++) {   // the rp largest singular values, in decreasing order
        int best = -1;
        for (int k = 0; k < r; k++)
            if (!used[k] && (best < 0 || sig[k] > sig[best])) best = k;
        used[best] = true;
        const double s = sig[best] > 0 ? sig[best] : 1e-300;
        const double w = 1 / sqrt(s);
        // P row m = w conj(Lo x_m)^T with x_m = C(:, best) / s;  Q column m = w Li y_m
        for (int i = 0; i < r; i++) {
            zc lo = mk(0, 0), li = mk(0, 0);
            for (int k = 0; k <= i; k++) {
                lo = add(lo, mul(Gout[i * r + k], C[k * r + best]));
                li = add(li, mul(Gin[i * r + k], V[k * r + best]));
            }
            P[m * r + i] = scl(cj(lo), w / s);
            Q[i * rp + m] = scl(li, w);
        }
    }
}

// Gamma_out at level D: U^H U (U column-major n0 x r)
__global__ void gout_leaf_kernel(const float2* __restrict__ U, zc* __restrict__ G, int r, int n0, int64_t N)
{
    const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= N) return;
    const float2* u = U + p * r * n0;
    zc* g = G + p * r * r;
    for (int t = 0; t < r; t++)
        for (int s = t; s < r; s++) {
            zc acc = mk(0, 0);
            for (int j = 0; j < n0; j++) acc = add(acc, mul(cj(zf(u[t * n0 + j])), zf(u[s * n0 + j])));
            g[t * r + s] = acc;
            g[s * r + t] = cj(acc);
        }
}

// Gamma_out at level l from level l + 1: parents (2a + e, b >> 1), column block c = b & 1 of W_{l+1}
__global__ void gout_level_kernel(const float2* __restrict__ W, const zc* __restrict__ Gup, zc* __restrict__ G, int r,
                                  int LN, int l, int64_t N)
{
    const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= N) return;
    const int sh = LN - l;
    const int64_t a = p >> sh, b = p & ((int64_t(1) << sh) - 1);
    const int c = int(b & 1);
    zc acc[RMAX * RMAX];
    for (int i = 0; i < r * r; i++) acc[i] = mk(0, 0);
    for (int e = 0; e < 2; e++) {
        const int64_t pp = ((2 * a + e) << (sh - 1)) + (b >> 1);
        const float2* w = W + pp * 2 * r * r + int64_t(c) * r * r;   // Wc(t, s) = w[s r + t]
        const zc* gu = Gup + pp * r * r;
        zc M[RMAX * RMAX];   // M = Gup Wc
        for (int t = 0; t < r; t++)
            for (int s = 0; s < r; s++) {
                zc m = mk(0, 0);
                for (int k = 0; k < r; k++) m = add(m, mul(gu[t * r + k], zf(w[s * r + k])));
                M[t * r + s] = m;
            }
        for (int s = 0; s < r; s++)
            for (int s2 = 0; s2 < r; s2++) {
                zc m = mk(0, 0);
                for (int t = 0; t < r; t++) m = add(m, mul(cj(zf(w[s * r + t])), M[t * r + s2]));
                acc[s * r + s2] = add(acc[s * r + s2], m);
            }
    }
    for (int i = 0; i < r * r; i++) G[p * r * r + i] = acc[i];
}

// One level of the bottom-up sweep.  l == l0: the source factor is V0 (r x n0); else W_l (r x 2r) whose inputs are
// re-expressed in the truncated coordinates of level l - 1 (Qprev, r x rp) with Grams Ginp (rp x rp).
__global__ void sweep_kernel(const float2* __restrict__ Wsrc, const zc* __restrict__ Gout, const zc* __restrict__ Qprev,
                             const zc* __restrict__ Ginp, zc* __restrict__ Qout, zc* __restrict__ Ginp_out,
                             float2* __restrict__ Wnew, int r, int rp, int n0, int LN, int l, int leaf, int64_t N)
{
    const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= N) return;
    zc Gin[RMAX * RMAX], Go[RMAX * RMAX], P[RMAX * RMAX], Q[RMAX * RMAX];
    zc Wt[RMAX * 2 * RMAX];   // r x 2rp (transfer levels), row-major
    for (int i = 0; i < r * r; i++) {
        Go[i] = Gout[p * r * r + i];
        Gin[i] = mk(0, 0);
    }
    if (leaf) {
        const float2* v = Wsrc + p * r * n0;   // column-major r x n0
        for (int t = 0; t < r; t++)
            for (int s = t; s < r; s++) {
                zc acc = mk(0, 0);
                for (int j = 0; j < n0; j++) acc = add(acc, mul(zf(v[j * r + t]), cj(zf(v[j * r + s]))));
                Gin[t * r + s] = acc;
                Gin[s * r + t] = cj(acc);
            }
    } else {
        const int sh = LN - l;
        const int64_t a = p >> sh, b = p & ((int64_t(1) << sh) - 1);
        const int64_t q0 = ((a >> 1) << (sh + 1)) + 2 * b;
        const float2* w = Wsrc + p * 2 * r * r;   // column-major r x 2r
        for (int c = 0; c < 2; c++) {
            const zc* qc = Qprev + (q0 + c) * r * rp;   // r x rp row-major
            for (int t = 0; t < r; t++)
                for (int m = 0; m < rp; m++) {
                    zc acc = mk(0, 0);
                    for (int s = 0; s < r; s++) acc = add(acc, mul(zf(w[(c * r + s) * r + t]), qc[s * rp + m]));
                    Wt[t * 2 * rp + c * rp + m] = acc;
                }
            const zc* gp = Ginp + (q0 + c) * rp * rp;
            for (int t = 0; t < r; t++) {   // Gin += Wt_c Ginp_c Wt_c^H
                zc row[RMAX];
                for (int m = 0; m < rp; m++) {
                    zc acc = mk(0, 0);
                    for (int k = 0; k < rp; k++) acc = add(acc, mul(Wt[t * 2 * rp + c * rp + k], gp[k * rp + m]));
                    row[m] = acc;
                }
                for (int t2 = 0; t2 < r; t2++) {
                    zc acc = mk(0, 0);
                    for (int m = 0; m < rp; m++) acc = add(acc, mul(row[m], cj(Wt[t2 * 2 * rp + c * rp + m])));
                    Gin[t * r + t2] = add(Gin[t * r + t2], acc);
                }
            }
        }
    }
    zc Gkeep[RMAX * RMAX];
    for (int i = 0; i < r * r; i++) Gkeep[i] = Gin[i];
    truncate(Gin, Go, r, rp, P, Q);
    // new block = P . (V0 or Wt), complex64 column-major
    if (leaf) {
        const float2* v = Wsrc + p * r * n0;
        for (int j = 0; j < n0; j++)
            for (int m = 0; m < rp; m++) {
                zc acc = mk(0, 0);
                for (int t = 0; t < r; t++) acc = add(acc, mul(P[m * r + t], zf(v[j * r + t])));
                Wnew[p * rp * n0 + j * rp + m] = make_float2(float(acc.x), float(acc.y));
            }
    } else {
        for (int k = 0; k < 2 * rp; k++)
            for (int m = 0; m < rp; m++) {
                zc acc = mk(0, 0);
                for (int t = 0; t < r; t++) acc = add(acc, mul(P[m * r + t], Wt[t * 2 * rp + k]));
                Wnew[p * 2 * rp * rp + k * rp + m] = make_float2(float(acc.x), float(acc.y));
            }
    }
    // Gram of the truncated coefficients: P Gin P^H
    for (int m = 0; m < rp; m++) {
        zc row[RMAX];
        for (int t = 0; t < r; t++) {
            zc acc = mk(0, 0);
            for (int k = 0; k < r; k++) acc = add(acc, mul(P[m * r + k], Gkeep[k * r + t]));
            row[t] = acc;
        }
        for (int m2 = 0; m2 < rp; m2++) {
            zc acc = mk(0, 0);
            for (int t = 0; t < r; t++) acc = add(acc, mul(row[t], cj(P[m2 * r + t])));
            Ginp_out[p * rp * rp + m * rp + m2] = acc;
        }
    }
    for (int i = 0; i < r * rp; i++) Qout[p * r * rp + i] = Q[i];
}

// U' = U Q_D  (U column-major n0 x r, result column-major n0 x rp)
__global__ void u_final_kernel(const float2* __restrict__ U, const zc* __restrict__ Q, float2* __restrict__ Un, int r,
                               int rp, int n0, int64_t N)
{
    const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g >= N * n0) return;
    const int64_t p = g / n0;
    const int j = int(g % n0);
    for (int m = 0; m < rp; m++) {
        zc acc = mk(0, 0);
        for (int t = 0; t < r; t++) acc = add(acc, mul(zf(U[p * r * n0 + t * n0 + j]), Q[p * r * rp + t * rp + m]));
        Un[p * rp * n0 + m * n0 + j] = make_float2(float(acc.x), float(acc.y));
    }
}

}  // namespace

size_t recompress_gram_bytes(int r) { return size_t(r) * r * sizeof(zc); }

// out_v0 (N x rp x n0), out_x[i] (N x rp x 2rp), out_u (N x n0 x rp): the new factors; scratch: see bf_plan.cu
cudaError_t launch_recompress(const Dims& d, int rp, const float2* v0, const float2* const* xfer, const float2* u,
                              float2* out_v0, float2* const* out_x, float2* out_u, void* gout, void* q2, void* gin2,
                              cudaStream_t s)
{
    const int r = d.R, n0 = 1 << d.l0, nl = d.D - d.l0 + 1;
    if (r > RMAX || rp > r || rp < 1) return cudaErrorInvalidValue;
    const int64_t N = d.N;
    const unsigned blocks = unsigned((N + 63) / 64);
    zc* G = static_cast<zc*>(gout);                     // [nl][N][r][r]: level l at (l - l0)
    zc* Q[2] = {static_cast<zc*>(q2), static_cast<zc*>(q2) + N * r * rp};
    zc* Gi[2] = {static_cast<zc*>(gin2), static_cast<zc*>(gin2) + N * rp * rp};
    auto Gl = [&](int l) { return G + int64_t(l - d.l0) * N * r * r; };
    gout_leaf_kernel<<<blocks, 64, 0, s>>>(u, Gl(d.D), r, n0, N);
    for (int l = d.D - 1; l >= d.l0; l--)
        gout_level_kernel<<<blocks, 64, 0, s>>>(xfer[l + 1 - d.l0 - 1], Gl(l + 1), Gl(l), r, d.LN, l, N);
    sweep_kernel<<<blocks, 64, 0, s>>>(v0, Gl(d.l0), nullptr, nullptr, Q[0], Gi[0], out_v0, r, rp, n0, d.LN, d.l0, 1, N);
    int cur = 0;
    for (int l = d.l0 + 1; l <= d.D; l++) {
        sweep_kernel<<<blocks, 64, 0, s>>>(xfer[l - d.l0 - 1], Gl(l), Q[cur], Gi[cur], Q[1 - cur], Gi[1 - cur],
                                           out_x[l - d.l0 - 1], r, rp, n0, d.LN, l, 0, N);
        cur = 1 - cur;
    }
    u_final_kernel<<<unsigned((N * n0 + 255) / 256), 256, 0, s>>>(u, Q[cur], out_u, r, rp, n0, N);
    (void)nl;
    return cudaGetLastError();
}

}  // namespace bfk
