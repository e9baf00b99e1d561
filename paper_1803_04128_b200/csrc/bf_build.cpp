// bf_build.cpp -- host-side (untimed) FP64 construction of the IBF-MAT factors
// (include/bf_build.h).  Independent of the oracle: every block is assembled in
// the factored form of Algorithm 2 (eqn:ab1/eqn:ab2),
//     block = diag(row phases) . (Lagrange matrix shared by the level) . diag(column phases),
// because the Mock-Chebyshev grids of one level are translates of each other
// (eqn:gdA/gdB: "we can simply shift the grid points").
#include <cuda_runtime.h>
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <vector>

#include "../../include/bf.h"
#include "../../include/bf_build.h"
#include "../../include/bf_nufft.h"
#include "bf_plan_internal.h"

namespace {

using cd = std::complex<double>;

struct Shape {
    int kernel, amp, LN, l0, r, D, h;
    int64_t N, n0;
};

bool make_shape(const bf_fio_t* k, Shape* s)
{
    if (!k || k->abi_version != BF_ABI_VERSION) return false;
    if (k->kernel < 0 || k->kernel > 3 || bf_build_n_amp(k->amp) < 1) return false;
    if (k->log2n < 2 || k->log2n > 30 || k->log2n % 2 || k->log2leaf < 1 || 2 * k->log2leaf > k->log2n) return false;
    if (k->rank < 2 || k->rank > 64 || k->rank > (1 << k->log2leaf)) return false;
    s->kernel = k->kernel;
    s->amp = k->amp;
    s->LN = k->log2n;
    s->l0 = k->log2leaf;
    s->r = k->rank;
    s->N = int64_t(1) << s->LN;
    s->n0 = int64_t(1) << s->l0;
    s->D = s->LN - s->l0;
    s->h = s->LN / 2;
    return true;
}

// c(x) of Phi(x, xi) = x xi + c(x)|xi|  (BASELINE configs); cfg3 builds the BF on this smooth part.
inline double cfun(int kernel, double x)
{
    if (kernel == BF_KERNEL_DFT) return 0.0;
    const double amp = (kernel == BF_KERNEL_FIO_PAPER) ? 0.2 : 1.0;
    return (2.0 + amp * std::sin(2.0 * M_PI * x)) / 16.0;
}

// e^{sgn 2 pi i Phi(x_i, xi_j)}, Phi reduced mod 1 first: the x xi = i (j - N/2)/N part exactly in integers.
inline cd expphi(const Shape& S, int64_t i, int64_t j, double sgn)
{
    const int64_t xi = j - S.N / 2;
    const int64_t m = (i * xi) & (S.N - 1);   // two's complement: i xi mod N in [0, N)
    double f = std::ldexp(double(m), -S.LN);
    const double t = cfun(S.kernel, std::ldexp(double(i), -S.LN)) * double(xi < 0 ? -xi : xi);
    f += t - std::floor(t);
    f -= std::floor(f);
    double sn, cs;
    sincos(2.0 * M_PI * f, &sn, &cs);
    return cd(cs, sgn * sn);
}

// Mock-Chebyshev nodes of a block of n indices, relative to its first index: eqn:gdA with z_t ascending
// (DESIGN R2) and Round half away from zero (R3).  The expression is evaluated exactly as written so
// that exact .5 ties are decided by the same IEEE arithmetic everywhere.
std::vector<int64_t> nodes(int64_t n, int r)
{
    std::vector<int64_t> g(r);
    for (int t = 1; t <= r; t++) g[t - 1] = int64_t(std::llround(t + (n - r) * (0.5 - 0.5 * std::cos((t - 1) * M_PI / (r - 1))))) - 1;
    return g;
}

// Lagrange basis M_t(q) on nodes g.
inline double lag(const std::vector<int64_t>& g, int t, double q)
{
    double v = 1.0;
    for (size_t j = 0; j < g.size(); j++)
        if (int(j) != t) v *= (q - double(g[j])) / double(g[t] - g[j]);
    return v;
}

inline int64_t mid(int64_t lo, int64_t n) { return lo + (n - 1) / 2; }   // center, ties low (R4)

inline bf_c64 c64(cd z) { return bf_c64{float(z.real()), float(z.imag())}; }

int64_t block_elems(const Shape& S, int stage)
{
    switch (stage) {
    case BF_STAGE_V0: return S.r * S.n0;
    case BF_STAGE_SW: return int64_t(S.r) * S.r;
    case BF_STAGE_U: return S.n0 * S.r;
    default:
        if (stage >= BF_STAGE_XFER0 && stage < BF_STAGE_XFER0 + (S.D - S.l0)) return 2 * int64_t(S.r) * S.r;
        return 0;
    }
}

// V0 (initialization eqn:1): A = A(l0,a), B = B(l0,b) a leaf of n0 columns.
// block r x n0 column-major: [j][t] = e^{-i..Phi(c_A, xi_t^B)} M_t^B(xi_j) e^{i..Phi(c_A, xi_j)}
void build_v0(const Shape& S, int64_t p0, int64_t cnt, bf_c64* out)
{
    const int r = S.r;
    const int64_t n0 = S.n0, nleaf = S.N >> S.l0, nA = S.N >> S.l0;
    const auto g = nodes(n0, r);
    std::vector<double> L(r * n0);
    for (int t = 0; t < r; t++)
        for (int64_t j = 0; j < n0; j++) L[t * n0 + j] = lag(g, t, double(j));
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < cnt; q++) {
        const int64_t p = p0 + q, a = p / nleaf, b = p % nleaf;
        const int64_t cA = mid(a * nA, nA), loB = b * n0;
        cd rowp[64], colp[128];
        for (int t = 0; t < r; t++) rowp[t] = expphi(S, cA, loB + g[t], -1.0);
        for (int64_t j = 0; j < n0; j++) colp[j] = expphi(S, cA, loB + j, +1.0);
        bf_c64* o = out + q * r * n0;
        for (int64_t j = 0; j < n0; j++)
            for (int t = 0; t < r; t++) o[j * r + t] = c64(rowp[t] * L[t * n0 + j] * colp[j]);
    }
}

// Transfer level l, first half (eqn:2): A = A(l,a), B = B(l,b), C_c = B(l-1, 2b+c).
// block r x 2r column-major: [(c r + s)][t] = e^{-..Phi(c_A, xi_t^B)} M_t^B(xi_s^{C_c}) e^{..Phi(c_A, xi_s^{C_c})}
// Second half (eqn:3): P = A(l-1, a>>1):
// [(c r + s)][t] = e^{..Phi(x_t^A, c_{C_c})} M_s^P(x_t^A) e^{-..Phi(x_s^P, c_{C_c})}
void build_xfer(const Shape& S, int l, int64_t p0, int64_t cnt, bf_c64* out)
{
    const int r = S.r;
    const int sh = S.LN - l;
    const int64_t nB = int64_t(1) << l, nC = nB / 2;   // |B(l,.)|, |B(l-1,.)|
    const int64_t nA = S.N >> l, nP = nA * 2;          // |A(l,.)|, |A(l-1,.)|
    if (l <= S.h) {
        const auto gB = nodes(nB, r), gC = nodes(nC, r);
        std::vector<double> L(r * 2 * r);   // [t][c r + s], relative to B's first index
        for (int t = 0; t < r; t++)
            for (int c = 0; c < 2; c++)
                for (int s = 0; s < r; s++) L[t * 2 * r + c * r + s] = lag(gB, t, double(c * nC + gC[s]));
#pragma omp parallel for schedule(static)
        for (int64_t q = 0; q < cnt; q++) {
            const int64_t p = p0 + q, a = p >> sh, b = p & ((int64_t(1) << sh) - 1);
            const int64_t cA = mid(a * nA, nA), loB = b * nB;
            cd rowp[64], colp[128];
            for (int t = 0; t < r; t++) rowp[t] = expphi(S, cA, loB + gB[t], -1.0);
            for (int c = 0; c < 2; c++)
                for (int s = 0; s < r; s++) colp[c * r + s] = expphi(S, cA, loB + c * nC + gC[s], +1.0);
            bf_c64* o = out + q * 2 * r * r;
            for (int k = 0; k < 2 * r; k++)
                for (int t = 0; t < r; t++) o[k * r + t] = c64(rowp[t] * L[t * 2 * r + k] * colp[k]);
        }
    } else {
        const auto gA = nodes(nA, r), gP = nodes(nP, r);
        std::vector<double> L(2 * r * r);   // [e][t][s] = M_s^P(x_t^A), A the e-th child of P
        for (int e = 0; e < 2; e++)
            for (int t = 0; t < r; t++)
                for (int s = 0; s < r; s++) L[(e * r + t) * r + s] = lag(gP, s, double(e * nA + gA[t]));
#pragma omp parallel for schedule(static)
        for (int64_t q = 0; q < cnt; q++) {
            const int64_t p = p0 + q, a = p >> sh, b = p & ((int64_t(1) << sh) - 1);
            const int64_t loA = a * nA, loP = (a >> 1) * nP;
            const int e = int(a & 1);
            bf_c64* o = out + q * 2 * r * r;
            for (int c = 0; c < 2; c++) {
                const int64_t cC = mid((2 * b + c) * nC, nC);
                cd rowp[64], colp[64];
                for (int t = 0; t < r; t++) rowp[t] = expphi(S, loA + gA[t], cC, +1.0);
                for (int s = 0; s < r; s++) colp[s] = expphi(S, loP + gP[s], cC, -1.0);
                for (int s = 0; s < r; s++)
                    for (int t = 0; t < r; t++)
                        o[(c * r + s) * r + t] = c64(rowp[t] * L[(e * r + t) * r + s] * colp[s]);
            }
        }
    }
}

// Switch: A = A(h,a), B = B(h,b); block r x r column-major: [s][t] = e^{..Phi(x_t^A, xi_s^B)}
void build_sw(const Shape& S, int64_t p0, int64_t cnt, bf_c64* out)
{
    const int r = S.r, sh = S.LN - S.h;
    const int64_t nA = S.N >> S.h, nB = int64_t(1) << S.h;
    const auto gA = nodes(nA, r), gB = nodes(nB, r);
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < cnt; q++) {
        const int64_t p = p0 + q, a = p >> sh, b = p & ((int64_t(1) << sh) - 1);
        bf_c64* o = out + q * r * r;
        for (int s = 0; s < r; s++)
            for (int t = 0; t < r; t++) o[s * r + t] = c64(expphi(S, a * nA + gA[t], b * nB + gB[s], +1.0));
    }
}

// U (termination eqn:bf3): A = A(D,a) a leaf of n0 rows, B = B(D,b), b < n0.
// block n0 x r column-major: [t][j] = e^{..Phi(x_j, c_B)} M_t^A(x_j) e^{-..Phi(x_t^A, c_B)}
void build_u(const Shape& S, int64_t p0, int64_t cnt, bf_c64* out)
{
    const int r = S.r;
    const int64_t n0 = S.n0, nB = S.N >> S.l0;
    const auto g = nodes(n0, r);
    std::vector<double> L(n0 * r);
    for (int64_t j = 0; j < n0; j++)
        for (int t = 0; t < r; t++) L[j * r + t] = lag(g, t, double(j));
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < cnt; q++) {
        const int64_t p = p0 + q, a = p / n0, b = p % n0;
        const int64_t loA = a * n0, cB = mid(b * nB, nB);
        cd rowp[128], colp[64];
        for (int64_t j = 0; j < n0; j++) rowp[j] = expphi(S, loA + j, cB, +1.0);
        for (int t = 0; t < r; t++) colp[t] = expphi(S, loA + g[t], cB, -1.0);
        bf_c64* o = out + q * n0 * r;
        for (int t = 0; t < r; t++)
            for (int64_t j = 0; j < n0; j++) o[t * n0 + j] = c64(rowp[j] * L[j * r + t] * colp[t]);
    }
}


// ---------------------------------------------------------------------------------------------------------
// Structured (interpolative) factors (include/bf.h "structured plans").  Every block of
// Algorithm 4.1 is diag(row phases) . L . diag(column phases) with L the Lagrange matrix the whole level shares
// (the grids of one level are translates).  The row phases of one level and the column phases of the
// next act on the same coefficients, so they are merged: the plan carries eta_l = rowp_l^-1 o delta_l on the
// first half and zeta_l = colp_{l+1} o delta_l on the second half, and stores per pair only
//   S0:     omega[p][j]   = e(+Phi(c_A, xi_j))                                   (n0 per pair; L0 = M^B_t(xi_j))
//   first:  psi[p][c r+s] = e(+Phi(c_A, xi_s^C)) e(-Phi(c_P, xi_s^C))            (2r;  L1 = M^B_t(xi_s^{C_c}))
//   second: chi[p][c r+t] = e(+Phi(x_t^A, c_{C_c})) e(-Phi(x_t^A, c_B))          (2r;  L2_e = M^P_s(x_t^A))
//   SL:     Omega[p][j]   = e(+Phi(x_j, c_B))                                    (n0;  L_SL = M^A_t(x_j))
// with C = C_c = B(l-1, 2b+c), P = A(l-1, a>>1), e = a & 1.  Level h carries the switch with both
// neighbouring phases as ONE dense r x 2r block (or a dense V0 when h == l0):
//   W_h[p] = diag(e(-Phi(x_t^A, c_B))) Sw[p] diag(e(-Phi(c_A, xi_t^B))) L1 diag(psi_h[p]).
// ---------------------------------------------------------------------------------------------------------
inline cd rowp_first(const Shape& S, int l, int64_t a, int64_t b, const std::vector<int64_t>& gB, int t)
{   // e(-Phi(c_A, xi_t^B)) for the level-l pair (a, b); gB = nodes(2^l, r)
    const int64_t nA = S.N >> l, nB = int64_t(1) << l;
    return expphi(S, mid(a * nA, nA), b * nB + gB[t], -1.0);
}

inline cd colp_second(const Shape& S, int l, int64_t a, int64_t b, const std::vector<int64_t>& gA, int t)
{   // e(-Phi(x_t^A, c_B)) for the level-l pair (a, b); gA = nodes(N / 2^l, r)
    const int64_t nA = S.N >> l, nB = int64_t(1) << l;
    return expphi(S, a * nA + gA[t], mid(b * nB, nB), -1.0);
}

void st_lag_s0(const Shape& S, float* L)   // r x n0 column-major
{
    const auto g = nodes(S.n0, S.r);
    for (int64_t j = 0; j < S.n0; j++)
        for (int t = 0; t < S.r; t++) L[j * S.r + t] = float(lag(g, t, double(j)));
}

void st_lag_sl(const Shape& S, float* L)   // n0 x r column-major
{
    const auto g = nodes(S.n0, S.r);
    for (int t = 0; t < S.r; t++)
        for (int64_t j = 0; j < S.n0; j++) L[t * S.n0 + j] = float(lag(g, t, double(j)));
}

void st_lag_xfer(const Shape& S, int l, float* L)
{
    const int r = S.r;
    const int64_t nB = int64_t(1) << l, nC = nB / 2, nA = S.N >> l;
    if (l <= S.h) {   // r x 2r column-major: (t, c r + s) = M^B_t(xi_s^{C_c})
        const auto gB = nodes(nB, r), gC = nodes(nC, r);
        for (int c = 0; c < 2; c++)
            for (int sidx = 0; sidx < r; sidx++)
                for (int t = 0; t < r; t++) L[(c * r + sidx) * r + t] = float(lag(gB, t, double(c * nC + gC[sidx])));
    } else {          // 2 x (r x r column-major): (e; t, s) = M^P_s(x_t^A), A the e-th child of P
        const auto gA = nodes(nA, r), gP = nodes(2 * nA, r);
        for (int e = 0; e < 2; e++)
            for (int sidx = 0; sidx < r; sidx++)
                for (int t = 0; t < r; t++) L[(e * r + sidx) * r + t] = float(lag(gP, sidx, double(e * nA + gA[t])));
    }
}

// per-pair data of one structured stage: S0 omega, transfer psi / chi, SL Omega
void st_phase(const Shape& S, int stage, int64_t p0, int64_t cnt, bf_c64* out)
{
    const int r = S.r;
    const int64_t n0 = S.n0;
    if (stage == BF_STAGE_V0) {
        const int64_t nleaf = S.N >> S.l0, nA = S.N >> S.l0;
#pragma omp parallel for schedule(static)
        for (int64_t q = 0; q < cnt; q++) {
            const int64_t p = p0 + q, a = p / nleaf, b = p % nleaf;
            for (int64_t j = 0; j < n0; j++) out[q * n0 + j] = c64(expphi(S, mid(a * nA, nA), b * n0 + j, +1.0));
        }
    } else if (stage == BF_STAGE_U) {
        const int64_t nB = S.N >> S.l0;
#pragma omp parallel for schedule(static)
        for (int64_t q = 0; q < cnt; q++) {
            const int64_t p = p0 + q, a = p / n0, b = p % n0;
            for (int64_t j = 0; j < n0; j++) out[q * n0 + j] = c64(expphi(S, a * n0 + j, mid(b * nB, nB), +1.0));
        }
    } else {
        const int l = S.l0 + 1 + (stage - BF_STAGE_XFER0);
        const int sh = S.LN - l;
        const int64_t nB = int64_t(1) << l, nC = nB / 2, nA = S.N >> l;
        if (l <= S.h) {
            const auto gC = nodes(nC, r);
#pragma omp parallel for schedule(static)
            for (int64_t q = 0; q < cnt; q++) {
                const int64_t p = p0 + q, a = p >> sh, b = p & ((int64_t(1) << sh) - 1);
                const int64_t cA = mid(a * nA, nA), cP = mid((a >> 1) * 2 * nA, 2 * nA);
                for (int c = 0; c < 2; c++)
                    for (int sidx = 0; sidx < r; sidx++) {
                        const int64_t xi = (2 * b + c) * nC + gC[sidx];
                        out[q * 2 * r + c * r + sidx] = c64(expphi(S, cA, xi, +1.0) * expphi(S, cP, xi, -1.0));
                    }
            }
        } else {
            const auto gA = nodes(nA, r);
#pragma omp parallel for schedule(static)
            for (int64_t q = 0; q < cnt; q++) {
                const int64_t p = p0 + q, a = p >> sh, b = p & ((int64_t(1) << sh) - 1);
                const int64_t cB = mid(b * nB, nB);
                for (int c = 0; c < 2; c++) {
                    const int64_t cC = mid((2 * b + c) * nC, nC);
                    for (int t = 0; t < r; t++) {
                        const int64_t x = a * nA + gA[t];
                        out[q * 2 * r + c * r + t] = c64(expphi(S, x, cC, +1.0) * expphi(S, x, cB, -1.0));
                    }
                }
            }
        }
    }
}

// The dense level-h factor of a structured plan (switch and both neighbouring phase diagonals folded in):
// XFER_h blocks (r x 2r) when h > l0, else V0 blocks (r x n0).
void st_dense_h(const Shape& S, int64_t p0, int64_t cnt, bf_c64* out)
{
    const int r = S.r, h = S.h, sh = S.LN - h;
    const int64_t nA = S.N >> h, nB = int64_t(1) << h, nC = nB / 2;
    const bool at_leaf = (h == S.l0);
    const int64_t cols = at_leaf ? S.n0 : 2 * r;
    const auto gA = nodes(nA, r), gB = nodes(nB, r);
    std::vector<float> L(r * cols);
    if (at_leaf) st_lag_s0(S, L.data()); else st_lag_xfer(S, h, L.data());
    std::vector<bf_c64> ph(cols);
#pragma omp parallel for schedule(static) firstprivate(ph)
    for (int64_t q = 0; q < cnt; q++) {
        const int64_t p = p0 + q, a = p >> sh, b = p & ((int64_t(1) << sh) - 1);
        // M = diag(rowp) L diag(colphase)   (r x cols), FP64
        std::vector<cd> M(r * cols), Y(r * cols);
        if (at_leaf) {
            st_phase(S, BF_STAGE_V0, p, 1, ph.data());
        } else {
            // psi_h of this pair (same formula as the first-half levels)
            const auto gC = nodes(nC, r);
            const int64_t cA = mid(a * nA, nA), cP = mid((a >> 1) * 2 * nA, 2 * nA);
            for (int c = 0; c < 2; c++)
                for (int sidx = 0; sidx < r; sidx++) {
                    const int64_t xi = (2 * b + c) * nC + gC[sidx];
                    ph[c * r + sidx] = c64(expphi(S, cA, xi, +1.0) * expphi(S, cP, xi, -1.0));
                }
        }
        cd rp[64], cp[64], Sw[64 * 64];
        for (int t = 0; t < r; t++) {
            rp[t] = rowp_first(S, h, a, b, gB, t);
            cp[t] = colp_second(S, h, a, b, gA, t);
            for (int sidx = 0; sidx < r; sidx++) Sw[t * r + sidx] = expphi(S, a * nA + gA[t], b * nB + gB[sidx], +1.0);
        }
        for (int64_t k = 0; k < cols; k++) {
            const cd pk(ph[k].re, ph[k].im);
            for (int t = 0; t < r; t++) M[k * r + t] = rp[t] * double(L[k * r + t]) * pk;
        }
        // Y = diag(colp) Sw M, Sw(t, s) = e(+Phi(x_t^A, xi_s^B))
        for (int t = 0; t < r; t++)
            for (int64_t k = 0; k < cols; k++) {
                cd acc = 0;
                for (int sidx = 0; sidx < r; sidx++) acc += Sw[t * r + sidx] * M[k * r + sidx];
                Y[k * r + t] = cp[t] * acc;
            }
        bf_c64* o = out + q * r * cols;
        for (int64_t k = 0; k < r * cols; k++) o[k] = c64(Y[k]);
    }
}

// The level-h factor of a structured plan as kind BF_LEVEL_FIRST_SWITCH: per pair [psi_h (2r) | Sw' (r x r,
// column-major)], Sw'(t, s) = e(-Phi(x_t^A, c_B)) e(+Phi(x_t^A, xi_s^B)) e(-Phi(c_A, xi_s^B)) -- the switch
// with the row phases of level h and the column phases of level h+1; the level computes
// Sw' L1 (psi o x).  2r + r^2 complex per pair instead of the 2r^2 of the dense block.
void st_switch_h(const Shape& S, int64_t p0, int64_t cnt, bf_c64* out)
{
    const int r = S.r, h = S.h, sh = S.LN - h;
    const int64_t nA = S.N >> h, nB = int64_t(1) << h, nC = nB / 2;
    const auto gA = nodes(nA, r), gB = nodes(nB, r), gC = nodes(nC, r);
    const int per = 2 * r + r * r;
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < cnt; q++) {
        const int64_t p = p0 + q, a = p >> sh, b = p & ((int64_t(1) << sh) - 1);
        bf_c64* o = out + q * per;
        const int64_t cA = mid(a * nA, nA), cP = mid((a >> 1) * 2 * nA, 2 * nA);
        for (int c = 0; c < 2; c++)
            for (int sidx = 0; sidx < r; sidx++) {
                const int64_t xi = (2 * b + c) * nC + gC[sidx];
                o[c * r + sidx] = c64(expphi(S, cA, xi, +1.0) * expphi(S, cP, xi, -1.0));
            }
        for (int sidx = 0; sidx < r; sidx++) {
            const cd rp = rowp_first(S, h, a, b, gB, sidx);
            for (int t = 0; t < r; t++)
                o[2 * r + sidx * r + t] =
                    c64(colp_second(S, h, a, b, gA, t) * expphi(S, a * nA + gA[t], b * nB + gB[sidx], +1.0) * rp);
        }
    }
}
}  // namespace

extern "C" {

int32_t bf_build_n_amp(int32_t amp)
{
    switch (amp) {
    case BF_AMP_ONE: return 1;
    case BF_AMP_CFG1:
    case BF_AMP_CFG2: return 2;
    case BF_AMP_CFG3: return 4;
    default: return -1;
    }
}

int64_t bf_build_block_elems(const bf_fio_t* k, int32_t stage)
{
    Shape S;
    if (!make_shape(k, &S)) return 0;
    return block_elems(S, stage);
}

// Amplitude split of DESIGN R11 (jump of cfg3 folded into b_k, R8).
bf_status_t bf_build_amp(const bf_fio_t* k, bf_c64* amp_a, bf_c64* amp_b)
{
    Shape S;
    if (!make_shape(k, &S) || !amp_a || !amp_b) return bfp_fail(BF_ERR_INVALID_ARG, "bf_build_amp: bad arguments");
    const int64_t N = S.N;
    const double Nd = double(N);
    const int na = bf_build_n_amp(S.amp);
#pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < N; n++) {
        const double x = std::ldexp(double(n), -S.LN), xi = double(n - N / 2);
        for (int kk = 0; kk < na; kk++) {
            cd av(1.0, 0.0), bv(1.0, 0.0);
            switch (S.amp) {
            case BF_AMP_CFG1:   // alpha = 1 + 0.5 cos(2 pi x) cos(pi xi/N)
                if (kk == 1) {
                    av = 0.5 * std::cos(2.0 * M_PI * x);
                    bv = std::cos(M_PI * xi / Nd);
                }
                break;
            case BF_AMP_CFG2:   // alpha = (1 + 0.3 sin 2 pi x)(1 + 0.3 cos(2 pi xi/N)), held as two terms
                av = 1.0 + 0.3 * std::sin(2.0 * M_PI * x);
                if (kk == 1) bv = 0.3 * std::cos(2.0 * M_PI * xi / Nd);
                break;
            case BF_AMP_CFG3: {   // alpha = exp(-(x-1/2)^2)(1 + 0.2 sin(4 pi xi/N)) e^{2 pi i 0.25 sign(x-1/3) xi}
                const double s = (kk < 2) ? 1.0 : -1.0;
                const double sx = (3 * n > N) ? 1.0 : -1.0;
                av = (sx == s) ? std::exp(-(x - 0.5) * (x - 0.5)) : 0.0;
                double jp = 0.25 * s * xi;
                jp -= std::floor(jp);
                bv = cd(std::cos(2.0 * M_PI * jp), std::sin(2.0 * M_PI * jp));
                if (kk % 2 == 1) bv *= 0.2 * std::sin(4.0 * M_PI * xi / Nd);
                break;
            }
            default: break;
            }
            amp_a[kk * N + n] = c64(av);
            amp_b[kk * N + n] = c64(bv);
        }
    }
    return BF_OK;
}

bf_status_t bf_build_blocks(const bf_fio_t* k, int32_t stage, int64_t block_begin, int64_t block_count, bf_c64* out)
{
    Shape S;
    if (!make_shape(k, &S)) return bfp_fail(BF_ERR_INVALID_ARG, "bf_build_blocks: bad kernel descriptor");
    if (S.n0 > 64 || S.r > 64) return bfp_fail(BF_ERR_NOT_SUPPORTED, "bf_build_blocks: leaf > 64 or rank > 64");
    if (block_elems(S, stage) == 0) return bfp_fail(BF_ERR_INVALID_ARG, "bf_build_blocks: bad stage");
    if (block_begin < 0 || block_count < 0 || block_begin + block_count > S.N || (!out && block_count))
        return bfp_fail(BF_ERR_INVALID_ARG, "bf_build_blocks: bad block range");
    switch (stage) {
    case BF_STAGE_V0: build_v0(S, block_begin, block_count, out); break;
    case BF_STAGE_SW: build_sw(S, block_begin, block_count, out); break;
    case BF_STAGE_U: build_u(S, block_begin, block_count, out); break;
    default: build_xfer(S, S.l0 + 1 + (stage - BF_STAGE_XFER0), block_begin, block_count, out); break;
    }
    return BF_OK;
}

}  // extern "C"

namespace {

// Build shard slot `si` (representing rank q of 2^g) of plan p: every stage's local blocks, in slices of
// at most staging_bytes through two pinned buffers (build of slice i+1 overlaps the upload of slice i).
// Local -> global block map (include/bf.h "index-sharded plans"): first-half stages (V0, SW, XFER of
// levels <= h) hold runs of 2^(LN-l-g) consecutive global blocks per a; second-half stages (XFER of
// levels > h, U) the contiguous range [q N/G, (q+1) N/G).
bf_status_t stream_build(bf_plan_t plan, const bf_fio_t* k, const Shape& S, int si, int q, int g,
                         int64_t staging_bytes)
{
    const int na = bf_build_n_amp(S.amp);
    const int64_t nloc = S.N >> g;
    bf_status_t st = BF_OK;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(bfp_device(plan));
    bf_c64* buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    cudaStream_t cs = nullptr;
    auto cleanup = [&]() {
        if (cs) cudaStreamSynchronize(cs);
        for (int i = 0; i < 2; i++) {
            if (buf[i]) cudaFreeHost(buf[i]);
            if (ev[i]) cudaEventDestroy(ev[i]);
        }
        if (cs) cudaStreamDestroy(cs);
        if (prev >= 0) cudaSetDevice(prev);
    };
    if (cudaMallocHost(reinterpret_cast<void**>(&buf[0]), size_t(staging_bytes)) != cudaSuccess ||
        cudaMallocHost(reinterpret_cast<void**>(&buf[1]), size_t(staging_bytes)) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming) != cudaSuccess ||
        cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        cleanup();
        return bfp_fail(BF_ERR_OOM, "factor upload: pinned staging allocation failed");
    }
    // amplitudes: a_k on this shard's x-rows, b_k on its xi-rows (both [q N/G, (q+1) N/G))
    {
        std::vector<bf_c64> a(size_t(na) * S.N), b(size_t(na) * S.N);
        bf_build_amp(k, a.data(), b.data());
        for (int which = 0; which < 2 && st == BF_OK; which++) {
            const std::vector<bf_c64>& src = which ? b : a;
            void* dst = nullptr;
            if ((st = bfp_stage_dst(plan, si, which ? BF_STAGE_AMP_B : BF_STAGE_AMP_A, 0, na, &dst)) != BF_OK) break;
            for (int kk = 0; kk < na; kk++)
                if (cudaMemcpy(static_cast<bf_c64*>(dst) + kk * nloc, src.data() + kk * S.N + q * nloc,
                               size_t(nloc) * sizeof(bf_c64), cudaMemcpyHostToDevice) != cudaSuccess) {
                    cudaGetLastError();
                    st = bfp_fail(BF_ERR_CUDA, "factor upload: amplitude copy failed");
                    break;
                }
        }
        if (st != BF_OK) {
            cleanup();
            return st;
        }
    }
    std::vector<int> stages = {BF_STAGE_V0, BF_STAGE_SW, BF_STAGE_U};
    for (int i = 0; i < S.D - S.l0; i++) stages.push_back(BF_STAGE_XFER0 + i);
    int cur = 0;
    bool used[2] = {false, false};
    for (int stage : stages) {
        const int lvl = stage == BF_STAGE_V0 ? S.l0 : stage == BF_STAGE_SW ? S.h : stage == BF_STAGE_U ? S.D
                                                                                       : S.l0 + 1 + (stage - BF_STAGE_XFER0);
        const bool first = (stage == BF_STAGE_SW) || lvl <= S.h;
        const int sb = S.LN - lvl - g;   // first half: log2 of a local b-run
        const int64_t elems = block_elems(S, stage);
        const int64_t per = std::max<int64_t>(1, staging_bytes / (elems * int64_t(sizeof(bf_c64))));
        for (int64_t b0 = 0; b0 < nloc; b0 += per) {
            const int64_t cnt = std::min(per, nloc - b0);
            if (used[cur]) cudaEventSynchronize(ev[cur]);   // slice buffer free again
            for (int64_t pos = b0; pos < b0 + cnt;) {
                int64_t glob, run;
                if (first) {
                    const int64_t a = pos >> sb, bl = pos & ((int64_t(1) << sb) - 1);
                    run = std::min((int64_t(1) << sb) - bl, b0 + cnt - pos);
                    glob = (a << (S.LN - lvl)) + (int64_t(q) << sb) + bl;
                } else {
                    run = b0 + cnt - pos;
                    glob = int64_t(q) * nloc + pos;
                }
                bf_build_blocks(k, stage, glob, run, buf[cur] + (pos - b0) * elems);
                pos += run;
            }
            void* dst = nullptr;
            if ((st = bfp_stage_dst(plan, si, stage, b0, cnt, &dst)) != BF_OK) {
                cleanup();
                return st;
            }
            if (cudaMemcpyAsync(dst, buf[cur], size_t(cnt * elems) * sizeof(bf_c64), cudaMemcpyHostToDevice, cs) !=
                cudaSuccess) {
                cudaGetLastError();
                cleanup();
                return bfp_fail(BF_ERR_CUDA, "factor upload failed");
            }
            cudaEventRecord(ev[cur], cs);
            used[cur] = true;
            cur ^= 1;
        }
    }
    cleanup();
    return BF_OK;
}

bf_status_t build_plan(const bf_fio_t* k, int device, int world, int rank, int mode, const void* nccl_id,
                       int64_t max_nrhs_chunk, int64_t staging_bytes, bf_plan_t* out)
{
    Shape S;
    if (!out) return bfp_fail(BF_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (!make_shape(k, &S)) return bfp_fail(BF_ERR_INVALID_ARG, "bad kernel descriptor");
    bf_desc_t meta{};
    meta.abi_version = BF_ABI_VERSION;
    meta.log2n = S.LN;
    meta.log2leaf = S.l0;
    meta.rank = S.r;
    meta.n_amp = bf_build_n_amp(S.amp);
    meta.memory = BF_MEM_HOST;
    bf_plan_t plan = nullptr;
    bf_status_t st = bfp_plan_alloc_sharded(&meta, device, max_nrhs_chunk, world, rank, mode, nccl_id, &plan);
    if (st != BF_OK) return st;
    int g = 0;
    while ((1 << g) < world) g++;
    if (staging_bytes < (int64_t(1) << 20)) staging_bytes = int64_t(1) << 20;
    const int nsh = bfp_num_shards(plan);
    for (int si = 0; si < nsh && st == BF_OK; si++)
        st = stream_build(plan, k, S, si, mode == BF_SHARD_EMULATED ? si : rank, g, staging_bytes);
    if (st == BF_OK) st = bf_plan_finalize(plan);
    if (st != BF_OK) {
        bfp_plan_free(plan);
        return st;
    }
    *out = plan;
    return BF_OK;
}

}  // namespace

extern "C" {

bf_status_t bf_plan_build_fio(const bf_fio_t* k, int device, int64_t max_nrhs_chunk, int64_t staging_bytes,
                              bf_plan_t* out)
{
    return build_plan(k, device, 1, 0, BF_SHARD_NONE, nullptr, max_nrhs_chunk, staging_bytes, out);
}

bf_status_t bf_build_structured(const bf_fio_t* k, int32_t stage, int64_t block_begin, int64_t block_count,
                                bf_c64* out)
{
    Shape S;
    if (!make_shape(k, &S)) return bfp_fail(BF_ERR_INVALID_ARG, "bf_build_structured: bad kernel descriptor");
    if (S.n0 > 64 || S.r > 16) return bfp_fail(BF_ERR_NOT_SUPPORTED, "bf_build_structured: leaf > 64 or rank > 16");
    const bool xf = stage >= BF_STAGE_XFER0 && stage < BF_STAGE_XFER0 + (S.D - S.l0);
    if (!(stage == BF_STAGE_V0 || stage == BF_STAGE_U || xf))
        return bfp_fail(BF_ERR_INVALID_ARG, "bf_build_structured: bad stage");
    if (block_begin < 0 || block_count < 0 || block_begin + block_count > S.N || (!out && block_count))
        return bfp_fail(BF_ERR_INVALID_ARG, "bf_build_structured: bad block range");
    if (stage == BF_STAGE_V0 && S.h == S.l0) st_dense_h(S, block_begin, block_count, out);
    else if (xf && S.l0 + 1 + (stage - BF_STAGE_XFER0) == S.h) st_switch_h(S, block_begin, block_count, out);
    else st_phase(S, stage, block_begin, block_count, out);
    return BF_OK;
}

bf_status_t bf_build_structured_lag(const bf_fio_t* k, int32_t stage, float* out)
{
    Shape S;
    if (!make_shape(k, &S) || !out) return bfp_fail(BF_ERR_INVALID_ARG, "bf_build_structured_lag: bad arguments");
    if (stage == BF_STAGE_V0) st_lag_s0(S, out);
    else if (stage == BF_STAGE_U) st_lag_sl(S, out);
    else if (stage >= BF_STAGE_XFER0 && stage < BF_STAGE_XFER0 + (S.D - S.l0))
        st_lag_xfer(S, S.l0 + 1 + (stage - BF_STAGE_XFER0), out);
    else return bfp_fail(BF_ERR_INVALID_ARG, "bf_build_structured_lag: bad stage");
    return BF_OK;
}

bf_status_t bf_plan_build_fio_structured(const bf_fio_t* k, int device, int64_t max_nrhs_chunk, int64_t staging_bytes,
                                         bf_plan_t* out)
{
    Shape S;
    if (!out) return bfp_fail(BF_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (!make_shape(k, &S)) return bfp_fail(BF_ERR_INVALID_ARG, "bad kernel descriptor");
    if (S.n0 > 64 || S.r > 16) return bfp_fail(BF_ERR_NOT_SUPPORTED, "structured build: leaf > 64 or rank > 16");
    if (staging_bytes < (int64_t(1) << 20)) staging_bytes = int64_t(1) << 20;
    int prev = -1;
    cudaGetDevice(&prev);
    if (cudaSetDevice(device) != cudaSuccess) {
        cudaGetLastError();
        return bfp_fail(BF_ERR_INVALID_ARG, "bad device");
    }
    const int r = S.r, nx = S.D - S.l0, na = bf_build_n_amp(S.amp);
    const int64_t N = S.N, n0 = S.n0;
    // device staging of every stage (the plan deep-copies them; structured factors are small)
    std::vector<void*> dev;
    auto dalloc = [&](size_t bytes) -> void* {
        void* x = nullptr;
        if (cudaMalloc(&x, bytes) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        dev.push_back(x);
        return x;
    };
    bf_status_t st = BF_OK;
    std::vector<bf_c64> a(size_t(na) * N), b(size_t(na) * N);
    bf_build_amp(k, a.data(), b.data());
    std::vector<float> L0(r * n0), Lsl(n0 * r), Lx(size_t(nx) * 2 * r * r);
    st_lag_s0(S, L0.data());
    st_lag_sl(S, Lsl.data());
    std::vector<bf_slevel_t> lv(nx);
    bf_sdesc_t d{};
    d.abi_version = BF_ABI_VERSION;
    d.log2n = S.LN;
    d.log2leaf = S.l0;
    d.rank = r;
    d.n_amp = na;
    d.memory = BF_MEM_DEVICE;
    d.amp_a = a.data();
    d.amp_b = b.data();
    d.s0_kind = (S.h == S.l0) ? BF_LEVEL_DENSE : BF_LEVEL_FIRST;
    d.s0_lag = L0.data();
    d.sl_lag = Lsl.data();
    d.xfer = lv.data();
    // stage list: (what, elems per pair, device array); what: -1 S0, -2 SL, i >= 0 transfer level index
    std::vector<bf_c64> host(size_t(staging_bytes / sizeof(bf_c64)));
    auto fill = [&](int what, int64_t per, bf_c64* dst) -> bool {
        const int64_t chunk = std::max<int64_t>(1, int64_t(host.size()) / per);
        for (int64_t p0 = 0; p0 < N; p0 += chunk) {
            const int64_t cnt = std::min(chunk, N - p0);
            if (what == -1) {
                if (S.h == S.l0) st_dense_h(S, p0, cnt, host.data()); else st_phase(S, BF_STAGE_V0, p0, cnt, host.data());
            } else if (what == -2) {
                st_phase(S, BF_STAGE_U, p0, cnt, host.data());
            } else if (S.l0 + 1 + what == S.h) {
                st_switch_h(S, p0, cnt, host.data());
            } else {
                st_phase(S, BF_STAGE_XFER0 + what, p0, cnt, host.data());
            }
            if (cudaMemcpy(dst + p0 * per, host.data(), size_t(cnt * per) * sizeof(bf_c64), cudaMemcpyHostToDevice) !=
                cudaSuccess) {
                cudaGetLastError();
                return false;
            }
        }
        return true;
    };
    do {
        const int64_t s0per = (S.h == S.l0) ? n0 * r : n0;
        bf_c64* s0d = static_cast<bf_c64*>(dalloc(size_t(N * s0per) * sizeof(bf_c64)));
        bf_c64* sld = static_cast<bf_c64*>(dalloc(size_t(N * n0) * sizeof(bf_c64)));
        if (!s0d || !sld) {
            st = bfp_fail(BF_ERR_OOM, "structured build: staging allocation failed");
            break;
        }
        if (!fill(-1, s0per, s0d) || !fill(-2, n0, sld)) {
            st = bfp_fail(BF_ERR_CUDA, "structured build: upload failed");
            break;
        }
        d.s0_data = s0d;
        d.sl_phase = sld;
        for (int i = 0; i < nx && st == BF_OK; i++) {
            const int l = S.l0 + 1 + i;
            const bool at_h = (l == S.h);
            const int64_t per = at_h ? 2 * r + r * r : 2 * r;
            bf_c64* xd = static_cast<bf_c64*>(dalloc(size_t(N * per) * sizeof(bf_c64)));
            if (!xd) {
                st = bfp_fail(BF_ERR_OOM, "structured build: staging allocation failed");
                break;
            }
            if (!fill(i, per, xd)) {
                st = bfp_fail(BF_ERR_CUDA, "structured build: upload failed");
                break;
            }
            lv[i].kind = at_h ? BF_LEVEL_FIRST_SWITCH : (l < S.h ? BF_LEVEL_FIRST : BF_LEVEL_SECOND);
            lv[i].data = xd;
            st_lag_xfer(S, l, Lx.data() + size_t(i) * 2 * r * r);
            lv[i].lag = Lx.data() + size_t(i) * 2 * r * r;
        }
        if (st != BF_OK) break;
        st = bf_plan_create_structured(&d, device, max_nrhs_chunk, out);
    } while (false);
    for (void* x : dev) cudaFree(x);
    if (prev >= 0) cudaSetDevice(prev);
    return st;
}

bf_status_t bf_plan_build_fio_sharded(const bf_fio_t* k, int device, int32_t rank, int32_t world,
                                      const void* nccl_unique_id, int64_t max_nrhs_chunk, int64_t staging_bytes,
                                      bf_plan_t* out)
{
    return build_plan(k, device, world, rank, BF_SHARD_NCCL, nccl_unique_id, max_nrhs_chunk, staging_bytes, out);
}

bf_status_t bf_plan_build_fio_emulated(const bf_fio_t* k, int device, int32_t world, int64_t max_nrhs_chunk,
                                       int64_t staging_bytes, bf_plan_t* out)
{
    return build_plan(k, device, world, 0, BF_SHARD_EMULATED, nullptr, max_nrhs_chunk, staging_bytes, out);
}

// NUFFT path (include/bf_nufft.h): the configs' phases are exactly rank 1 on xi < 0 and xi >= 0,
// Phi(x, xi) = (x -+ c(x)) xi there (eqn:phlr P:1125-1131 for the wave-equation FIO; P:571 submatrices), so the
// targets are t_-(x) = x - c(x) and t_+(x) = x + c(x), in FP64; the amplitude split is bf_build_amp's.
bf_status_t bf_nufft_build_fio(const bf_fio_t* k, int device, int64_t max_nrhs_chunk, double eps, bf_nufft_t* out)
{
    if (!k || !out) return bfp_fail(BF_ERR_INVALID_ARG, "bf_nufft_build_fio: null");
    if (k->abi_version != BF_ABI_VERSION || k->kernel < 0 || k->kernel > 3 || bf_build_n_amp(k->amp) < 1 ||
        k->log2n < 4 || k->log2n > 26)
        return bfp_fail(BF_ERR_SHAPE, "bf_nufft_build_fio: kernel, amplitude or log2n");
    const int64_t N = int64_t(1) << k->log2n;
    const int na = bf_build_n_amp(k->amp);
    std::vector<double> t(size_t(2 * N));
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; i++) {
        const double x = std::ldexp(double(i), -k->log2n), c = cfun(k->kernel, x);
        t[size_t(i)] = x - c;
        t[size_t(N + i)] = x + c;
    }
    std::vector<bf_c64> a(size_t(na) * N), b(size_t(na) * N);
    bf_fio_t kk = *k;
    if (kk.log2leaf < 1 || 2 * kk.log2leaf > kk.log2n) kk.log2leaf = 1;   // bf_build_amp checks a BF shape
    if (kk.rank < 2 || kk.rank > (1 << kk.log2leaf)) kk.rank = 2;
    if (kk.log2n % 2) return bfp_fail(BF_ERR_SHAPE, "bf_nufft_build_fio: log2n must be even");
    bf_status_t st = bf_build_amp(&kk, a.data(), b.data());
    if (st != BF_OK) return st;
    bf_nufft_desc_t d{};
    d.abi_version = BF_ABI_VERSION;
    d.log2n = k->log2n;
    d.n_amp = na;
    d.n_sub = 2;
    d.targets = t.data();
    d.amp_a = a.data();
    d.amp_b = b.data();
    d.eps = eps;
    return bf_nufft_create(&d, device, max_nrhs_chunk, out);
}

}  // extern "C"
