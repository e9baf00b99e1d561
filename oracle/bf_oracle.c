/*
 * oracle/bf_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, double-precision CPU transcription of what the IBF-MAT apply
 * path computes (arXiv:1803.04128, H. Yang).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_1803_04128_b200/csrc); the two are independent implementations of the
 * same paper passages.  Citations "P:L" are lines of the paper's LaTeX
 * (PAPER.md); "DESIGN Rn" are the readings listed in DESIGN.md section 3.
 *
 * What it computes
 *   O0  direct sum    g_c(x_i) = sum_j alpha(x_i,xi_j) e^{2 pi i Phi(x_i,xi_j)} F[j,c]
 *                     (eqn:1D-FIO P:899-902; problem statement P:623-626)
 *   O1-O7  the butterfly application of Algorithm 4.1 with the
 *          amplitude split of eqn:tg:  g = sum_k a_k o BF(b_k o f),
 *          every block generated on the fly from its formula.
 *   O0*, O8  the adjoint: direct sum of conj(K) transposed, and the factors of
 *          O2-O6 conjugate-transposed in reverse order.
 *
 * Pins: tests/test_oracle_pins.py (closed forms, paper-printed eps^b values of
 * tab:1D-FIO, brute-force dense assembly, Lagrange/grid invariants).
 * Nothing on the hot path is "parity unpinned".
 *
 * Index conventions (0-based; DESIGN R1, R6):
 *   N = 2^LN, x_i = i/N, xi_j = j - N/2             (eqn:1D-xandxi P:905-907, shifted to 0-based)
 *   leaf n0 = 2^l0, D = LN - l0, h = LN/2
 *   A(l,a) = rows   [a N/2^l, (a+1) N/2^l)          (node a of T_X at level l)
 *   B(l,b) = cols   [b 2^l,   (b+1) 2^l)            (node b of T_Omega at level LN-l)
 *   pair index at level l:  p = a * 2^(LN-l) + b
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef double complex cplx;

#define ORC_VERSION 1

/* kernels (phase functions) */
enum { ORC_K_FIO = 0,        /* BASELINE cfg1/2/4/5: Phi = x xi + c(x)|xi|, c=(2+sin 2pi x)/16          */
       ORC_K_FIO_PAPER = 1,  /* eqn:1D-FIO-kernal P:893-895: c = (2+0.2 sin 2pi x)/16                    */
       ORC_K_DFT = 2,        /* Phi = x xi  (the sanity case of BASELINE cfg1)                          */
       ORC_K_FIO_JUMP = 3 }; /* BASELINE cfg3: Phi = x xi + c(x)|xi| + 0.25 sign(x-1/3) xi             */

/* amplitudes */
enum { ORC_A_ONE = 0,        /* alpha = 1 (tab:1D-FIO)                                           */
       ORC_A_CFG1 = 1,       /* alpha = 1 + 0.5 cos(2 pi x) cos(pi xi/N)         (cfg1, cfg4, cfg5)    */
       ORC_A_CFG2 = 2,       /* alpha = (1+0.3 sin 2 pi x)(1+0.3 cos(2 pi xi/N))  (cfg2)               */
       ORC_A_CFG3 = 3 };     /* alpha = exp(-(x-1/2)^2)(1+0.2 sin(4 pi xi/N))     (cfg3)               */

int orc_version(void) { return ORC_VERSION; }

/* ------------------------------------------------------------------------- */
/* Grid points x_i, xi_j (eqn:1D-xandxi, P:905-907, 0-based)                  */
/* ------------------------------------------------------------------------- */
static double x_of(int LN, int64_t i) { return ldexp((double)i, -LN); }
static int64_t xi_of(int LN, int64_t j) { return j - ((int64_t)1 << (LN - 1)); }

/* c(x) of the phase (P:894 for the paper kernel, BASELINE configs otherwise). */
static double c_of(int kernel, double x)
{
    switch (kernel) {
    case ORC_K_FIO:
    case ORC_K_FIO_JUMP: return (2.0 + sin(2.0 * M_PI * x)) / 16.0;
    case ORC_K_FIO_PAPER: return (2.0 + 0.2 * sin(2.0 * M_PI * x)) / 16.0;
    default: return 0.0;
    }
}

/* Fractional part of Phi(x_i, xi_j), i.e. Phi mod 1, in [0,1).
 * x xi = i (j - N/2) / N is reduced exactly in integers before the division;
 * c(x)|xi| and the jump are reduced separately (DESIGN R12).
 * full=1: the complete phase (the direct sum, O0);
 * full=0: the phase the butterfly is built on (cfg3's jump is folded into the
 *         amplitude terms, DESIGN R8). */
static double phase_frac(int kernel, int LN, int64_t i, int64_t j, int full)
{
    const int64_t N = (int64_t)1 << LN;
    const int64_t xi = xi_of(LN, j);
    int64_t m = (i * xi) % N;                  /* |i xi| < 2^(2 LN) <= 2^44: exact */
    if (m < 0) m += N;
    double f = ldexp((double)m, -LN);          /* frac(x xi), exact */
    double cx = c_of(kernel, x_of(LN, i)) * (double)(xi < 0 ? -xi : xi);
    f += cx - floor(cx);
    if (full && kernel == ORC_K_FIO_JUMP) {
        double s = (3 * i > N) ? 1.0 : -1.0;   /* sign(x - 1/3); x = i/N never equals 1/3 */
        double jmp = 0.25 * s * (double)xi;    /* exact: xi integer */
        f += jmp - floor(jmp);
    }
    return f - floor(f);
}

/* Phi(x_i, xi_j) in cycles, unreduced (exported for tests). */
double orc_phi(int kernel, int LN, int64_t i, int64_t j, int full)
{
    const double x = x_of(LN, i), xi = (double)xi_of(LN, j);
    double p = x * xi + c_of(kernel, x) * fabs(xi);
    if (full && kernel == ORC_K_FIO_JUMP) p += 0.25 * ((3 * i > ((int64_t)1 << LN)) ? 1.0 : -1.0) * xi;
    return p;
}

/* E(Phi) = e^{2 pi i Phi}; sgn = +1 or -1 (for e^{-2 pi i Phi}). */
static cplx E(int kernel, int LN, int64_t i, int64_t j, int sgn, int full)
{
    double f = phase_frac(kernel, LN, i, j, full);
    double th = 2.0 * M_PI * f;
    return cos(th) + (double)sgn * sin(th) * I;
}

/* ------------------------------------------------------------------------- */
/* Amplitude alpha and its exact split alpha ~ sum_k a_k(x) b_k(xi) (eqn:tg,  */
/* P:24-28; DESIGN R11).                                                       */
/* ------------------------------------------------------------------------- */
int orc_n_amp(int amp)
{
    switch (amp) {
    case ORC_A_ONE: return 1;
    case ORC_A_CFG1: return 2;
    case ORC_A_CFG2: return 2;
    case ORC_A_CFG3: return 4;
    default: return -1;
    }
}

/* The amplitude function alpha(x_i, xi_j) as BASELINE.json states it. */
cplx orc_alpha(int amp, int LN, int64_t i, int64_t j)
{
    const double N = ldexp(1.0, LN), x = x_of(LN, i), xi = (double)xi_of(LN, j);
    switch (amp) {
    case ORC_A_ONE: return 1.0;
    case ORC_A_CFG1: return 1.0 + 0.5 * cos(2.0 * M_PI * x) * cos(M_PI * xi / N);
    case ORC_A_CFG2: return (1.0 + 0.3 * sin(2.0 * M_PI * x)) * (1.0 + 0.3 * cos(2.0 * M_PI * xi / N));
    case ORC_A_CFG3: return exp(-(x - 0.5) * (x - 0.5)) * (1.0 + 0.2 * sin(4.0 * M_PI * xi / N));
    default: return NAN;
    }
}

/* a_k(x_i) for i < N (side 0) or b_k(xi_j) for j < N (side 1). DESIGN R11:
 *   CFG1: (1, 1), (0.5 cos 2 pi x, cos(pi xi/N))
 *   CFG2: (1+0.3 sin 2 pi x, 1), (1+0.3 sin 2 pi x, 0.3 cos(2 pi xi/N))
 *   CFG3: k = 2 q + m, s = +1 (q=0) / -1 (q=1), m in {0,1}:
 *         a_k = exp(-(x-1/2)^2) 1[sign(x-1/3) = s],
 *         b_k = e^{2 pi i 0.25 s xi} (1 or 0.2 sin(4 pi xi/N))        (jump folded, DESIGN R8) */
int orc_amp_term(int amp, int LN, int k, int side, cplx *out)
{
    const int64_t N = (int64_t)1 << LN;
    const double Nd = (double)N;
    if (k < 0 || k >= orc_n_amp(amp)) return -1;
    for (int64_t n = 0; n < N; n++) {
        const double x = x_of(LN, n), xi = (double)xi_of(LN, n);
        cplx v = 1.0;
        switch (amp) {
        case ORC_A_ONE: v = 1.0; break;
        case ORC_A_CFG1:
            if (k == 0) v = 1.0;
            else v = side == 0 ? 0.5 * cos(2.0 * M_PI * x) : cos(M_PI * xi / Nd);
            break;
        case ORC_A_CFG2:
            if (side == 0) v = 1.0 + 0.3 * sin(2.0 * M_PI * x);
            else v = (k == 0) ? 1.0 : 0.3 * cos(2.0 * M_PI * xi / Nd);
            break;
        case ORC_A_CFG3: {
            const double s = (k / 2 == 0) ? 1.0 : -1.0;
            if (side == 0) {
                const double sx = (3 * n > N) ? 1.0 : -1.0;
                v = (sx == s) ? exp(-(x - 0.5) * (x - 0.5)) : 0.0;
            } else {
                double jmp = 0.25 * s * xi;
                double th = 2.0 * M_PI * (jmp - floor(jmp));
                v = cos(th) + sin(th) * I;
                if (k % 2 == 1) v *= 0.2 * sin(4.0 * M_PI * xi / Nd);
            }
            break;
        }
        default: return -1;
        }
        out[n] = v;
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* O0: direct sum on a set of rows (the definition of g = K f).               */
/* F: N x nrhs column-major (ld = ldf); out: nrows x nrhs column-major.        */
/* ------------------------------------------------------------------------- */
void orc_direct_rows(int kernel, int amp, int LN, int64_t nrhs, const cplx *F, int64_t ldf,
                     const int64_t *rows, int64_t nrows, cplx *out)
{
    const int64_t N = (int64_t)1 << LN;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < nrows; q++) {
        const int64_t i = rows[q];
        cplx *acc = calloc((size_t)nrhs, sizeof(cplx));
        for (int64_t j = 0; j < N; j++) {
            cplx K = orc_alpha(amp, LN, i, j) * E(kernel, LN, i, j, +1, 1);
            for (int64_t c = 0; c < nrhs; c++) acc[c] += K * F[j + c * ldf];
        }
        for (int64_t c = 0; c < nrhs; c++) out[q + c * nrows] = acc[c];
        free(acc);
    }
}

/* Dense kernel matrix K(i,j) = alpha E(Phi) (row-major N x N), tiny N only. */
void orc_dense_kernel(int kernel, int amp, int LN, cplx *K)
{
    const int64_t N = (int64_t)1 << LN;
    for (int64_t i = 0; i < N; i++)
        for (int64_t j = 0; j < N; j++) K[i * N + j] = orc_alpha(amp, LN, i, j) * E(kernel, LN, i, j, +1, 1);
}

/* ------------------------------------------------------------------------- */
/* Interpolation machinery of Algorithm 2.                        */
/* ------------------------------------------------------------------------- */

/* Mock-Chebyshev grid adapted to the index block [lo, lo+n), eqn:gdA/gdB
 * (P:214-226), read with z_t ascending (DESIGN R2) and Round = round half away
 * from zero (DESIGN R3).  0-based indices are returned in g[0..r-1]. */
void orc_grid(int64_t lo, int64_t n, int r, int64_t *g)
{
    for (int t = 1; t <= r; t++) {
        double z = -0.5 * cos((t - 1) * M_PI / (r - 1));           /* DESIGN R2 */
        g[t - 1] = lo - 1 + (int64_t)llround(t + (n - r) * (z + 0.5));
    }
}

/* Center of the block [lo, lo+n): the index closest to the mean, ties to the
 * smaller one (DESIGN R4). */
int64_t orc_center(int64_t lo, int64_t n) { return lo + (n - 1) / 2; }

/* Lagrange basis polynomial M_t(q) = prod_{j != t} (q - g_j)/(g_t - g_j). */
double orc_lagrange(const int64_t *g, int r, int t, double q)
{
    double v = 1.0;
    for (int j = 0; j < r; j++)
        if (j != t) v *= (q - (double)g[j]) / (double)(g[t] - g[j]);
    return v;
}

/* ------------------------------------------------------------------------- */
/* The blocks of Algorithm 4.1, each from its own equation.        */
/* ------------------------------------------------------------------------- */
typedef struct {
    int kernel, LN, l0, r;
    int64_t N, n0;
    int D, h;
} bfctx;

static int ctx_init(bfctx *c, int kernel, int LN, int l0, int r)
{
    if (LN < 2 || LN % 2 != 0 || l0 < 1 || 2 * l0 > LN || r < 2 || r > (1 << l0) || LN > 30) return -1;
    c->kernel = kernel; c->LN = LN; c->l0 = l0; c->r = r;
    c->N = (int64_t)1 << LN; c->n0 = (int64_t)1 << l0;
    c->D = LN - l0; c->h = LN / 2;
    return 0;
}

/* A(l,a) and B(l,b) as [lo, lo+n) */
static void nodeA(const bfctx *c, int l, int64_t a, int64_t *lo, int64_t *n) { *n = c->N >> l; *lo = a * *n; }
static void nodeB(const bfctx *c, int l, int64_t b, int64_t *lo, int64_t *n) { (void)c; *n = (int64_t)1 << l; *lo = b * *n; }

#define EB(i, j, s) E(c->kernel, c->LN, (i), (j), (s), 0)

/* Initialization eqn:1 with A = A(l0,a) (DESIGN R1/R6); B = B(l0,b) a leaf of n0 columns:
 *   V[t][j] = e^{-2 pi i Phi(c_A, xi_t^B)} M_t^B(xi_j) e^{2 pi i Phi(c_A, xi_j)},  t < r, j < n0. */
static void blk_init(const bfctx *c, int64_t a, int64_t b, cplx *V)
{
    int64_t loA, nA, loB, nB, gB[64];
    nodeA(c, c->l0, a, &loA, &nA);
    nodeB(c, c->l0, b, &loB, &nB);
    const int64_t cA = orc_center(loA, nA);
    orc_grid(loB, nB, c->r, gB);
    cplx ecol[64];
    for (int64_t j = 0; j < nB; j++) ecol[j] = EB(cA, loB + j, +1);
    for (int t = 0; t < c->r; t++) {
        const cplx erow = EB(cA, gB[t], -1);
        for (int64_t j = 0; j < nB; j++)
            V[t * nB + j] = erow * orc_lagrange(gB, c->r, t, (double)(loB + j)) * ecol[j];
    }
}

/* Recursion, first half, eqn:2; A = A(l,a), B = B(l,b), C_c = B(l-1, 2b+c):
 *   W[t][c r + s] = e^{-2 pi i Phi(c_A, xi_t^B)} M_t^B(xi_s^{C_c}) e^{2 pi i Phi(c_A, xi_s^{C_c})}. */
static void blk_first(const bfctx *c, int l, int64_t a, int64_t b, cplx *W)
{
    const int r = c->r;
    int64_t loA, nA, loB, nB, gB[64], gC[64];
    nodeA(c, l, a, &loA, &nA);
    nodeB(c, l, b, &loB, &nB);
    const int64_t cA = orc_center(loA, nA);
    orc_grid(loB, nB, r, gB);
    for (int cc = 0; cc < 2; cc++) {
        int64_t loC, nC;
        nodeB(c, l - 1, 2 * b + cc, &loC, &nC);
        orc_grid(loC, nC, r, gC);
        cplx ecol[32];
        for (int s = 0; s < r; s++) ecol[s] = EB(cA, gC[s], +1);
        for (int t = 0; t < r; t++) {
            const cplx erow = EB(cA, gB[t], -1);
            for (int s = 0; s < r; s++)
                W[t * 2 * r + cc * r + s] = erow * orc_lagrange(gB, r, t, (double)gC[s]) * ecol[s];
        }
    }
}

/* Switch; A = A(h,a), B = B(h,b):  S[t][s] = e^{2 pi i Phi(x_t^A, xi_s^B)}. */
static void blk_switch(const bfctx *c, int64_t a, int64_t b, cplx *S)
{
    const int r = c->r;
    int64_t loA, nA, loB, nB, gA[64], gB[64];
    nodeA(c, c->h, a, &loA, &nA);
    nodeB(c, c->h, b, &loB, &nB);
    orc_grid(loA, nA, r, gA);
    orc_grid(loB, nB, r, gB);
    for (int t = 0; t < r; t++)
        for (int s = 0; s < r; s++) S[t * r + s] = EB(gA[t], gB[s], +1);
}

/* Recursion, second half, eqn:3; A = A(l,a), P = A(l-1, a>>1), C_c = B(l-1, 2b+c):
 *   W[t][c r + s] = e^{2 pi i Phi(x_t^A, c_{C_c})} M_s^P(x_t^A) e^{-2 pi i Phi(x_s^P, c_{C_c})}. */
static void blk_second(const bfctx *c, int l, int64_t a, int64_t b, cplx *W)
{
    const int r = c->r;
    int64_t loA, nA, loP, nP, gA[64], gP[64];
    nodeA(c, l, a, &loA, &nA);
    nodeA(c, l - 1, a >> 1, &loP, &nP);
    orc_grid(loA, nA, r, gA);
    orc_grid(loP, nP, r, gP);
    for (int cc = 0; cc < 2; cc++) {
        int64_t loC, nC;
        nodeB(c, l - 1, 2 * b + cc, &loC, &nC);
        const int64_t cC = orc_center(loC, nC);
        cplx ecol[32];
        for (int s = 0; s < r; s++) ecol[s] = EB(gP[s], cC, -1);
        for (int t = 0; t < r; t++) {
            const cplx erow = EB(gA[t], cC, +1);
            for (int s = 0; s < r; s++)
                W[t * 2 * r + cc * r + s] = erow * orc_lagrange(gP, r, s, (double)gA[t]) * ecol[s];
        }
    }
}

/* Termination eqn:bf3 with B = B(D,b) (DESIGN R6); A = A(D,a) a leaf of n0 rows:
 *   U[j][t] = e^{2 pi i Phi(x_j, c_B)} M_t^A(x_j) e^{-2 pi i Phi(x_t^A, c_B)},  j < n0, t < r. */
static void blk_term(const bfctx *c, int64_t a, int64_t b, cplx *U)
{
    const int r = c->r;
    int64_t loA, nA, loB, nB, gA[64];
    nodeA(c, c->D, a, &loA, &nA);
    nodeB(c, c->D, b, &loB, &nB);
    const int64_t cB = orc_center(loB, nB);
    orc_grid(loA, nA, r, gA);
    cplx ecol[32];
    for (int t = 0; t < r; t++) ecol[t] = EB(gA[t], cB, -1);
    for (int64_t j = 0; j < nA; j++) {
        const cplx erow = EB(loA + j, cB, +1);
        for (int t = 0; t < r; t++)
            U[j * r + t] = erow * orc_lagrange(gA, r, t, (double)(loA + j)) * ecol[t];
    }
}

/* Export one block for tests: stage 0 = init (r x n0), 1 = transfer at level l
 * (r x 2r; first half if l <= h else second half), 2 = switch (r x r), 3 = termination (n0 x r). */
int orc_bf_block(int kernel, int LN, int l0, int r, int stage, int l, int64_t a, int64_t b, cplx *out)
{
    bfctx c;
    if (ctx_init(&c, kernel, LN, l0, r) || r > 32 || l0 > 6) return -1;
    switch (stage) {
    case 0: blk_init(&c, a, b, out); return 0;
    case 1:
        if (l <= l0 || l > c.D) return -1;
        if (l <= c.h) blk_first(&c, l, a, b, out); else blk_second(&c, l, a, b, out);
        return 0;
    case 2: blk_switch(&c, a, b, out); return 0;
    case 3: blk_term(&c, a, b, out); return 0;
    default: return -1;
    }
}

/* Every block of one stage in pair order (the "bf-stored" input layout): stage 0 init (level l0),
 * 1 transfer at level l, 2 switch (level h), 3 termination (level D); pair p = a 2^(LN - level) + b. */
int orc_bf_blocks(int kernel, int LN, int l0, int r, int stage, int l, cplx *out)
{
    bfctx c;
    if (ctx_init(&c, kernel, LN, l0, r) || r > 32 || l0 > 6) return -1;
    const int level = stage == 0 ? l0 : stage == 1 ? l : stage == 2 ? c.h : c.D;
    if (stage == 1 && (l <= l0 || l > c.D)) return -1;
    if (stage < 0 || stage > 3) return -1;
    const int64_t nb = (int64_t)1 << (LN - level);
    const int64_t sz = stage == 0 ? r * c.n0 : stage == 1 ? 2 * r * r : stage == 2 ? r * r : c.n0 * r;
    int rc = 0;
#pragma omp parallel for schedule(static) reduction(| : rc)
    for (int64_t p = 0; p < c.N; p++) rc |= orc_bf_block(kernel, LN, l0, r, stage, l, p / nb, p % nb, out + p * sz);
    return rc;
}

/* ------------------------------------------------------------------------- */
/* O1-O7: Algorithm 4.1 applied to nv vectors Y (N x nv, column-major),        */
/* result U_out (N x nv, column-major).  delta arrays: [pair][t][v].           */
/* Blocks are generated on the fly from their formulas ("bf-otf")   */
/* or, when st != NULL, read from caller-supplied arrays ("bf-stored"): every  */
/* block in pair order, row-major as orc_bf_block returns it (init r x n0,     */
/* transfer r x 2r per level l0+1..D, switch r x r, termination n0 x r).       */
/* ------------------------------------------------------------------------- */
typedef struct {
    const cplx *v0, *sw, *u;
    const cplx *const *xfer;   /* [D - l0] */
} bfstore;

static int butterfly_apply(const bfctx *c, int64_t nv, const cplx *Y, cplx *Uout, const bfstore *st)
{
    const int r = c->r;
    const int64_t N = c->N, n0 = c->n0;
    cplx *d0 = malloc(sizeof(cplx) * (size_t)(N * r * nv));
    cplx *d1 = malloc(sizeof(cplx) * (size_t)(N * r * nv));
    if (!d0 || !d1) { free(d0); free(d1); return -2; }

    /* O2 Initialization (eqn:1): delta_{l0}[a,b] = V[a,b] y_B for a < n0, leaf b < N/n0. */
    {
        const int64_t nb = N >> c->l0;
#pragma omp parallel for schedule(static)
        for (int64_t p = 0; p < N; p++) {
            const int64_t a = p / nb, b = p % nb;
            cplx *V = malloc(sizeof(cplx) * (size_t)(r * n0));
            if (st) memcpy(V, st->v0 + p * r * n0, sizeof(cplx) * (size_t)(r * n0));
            else blk_init(c, a, b, V);
            for (int t = 0; t < r; t++)
                for (int64_t v = 0; v < nv; v++) {
                    cplx s = 0;
                    for (int64_t j = 0; j < n0; j++) s += V[t * n0 + j] * Y[(b * n0 + j) + v * N];
                    d0[(p * r + t) * nv + v] = s;
                }
            free(V);
        }
    }
    /* O3 / O5 Recursion (eqn:2 for l <= h, eqn:3 for l > h), with the switch O4 at l = h. */
    for (int l = c->l0; l <= c->D; l++) {
        if (l > c->l0) {
            const int64_t nbl = (int64_t)1 << (c->LN - l);   /* b-range at level l */
#pragma omp parallel for schedule(static)
            for (int64_t p = 0; p < N; p++) {
                const int64_t a = p / nbl, b = p % nbl;
                cplx W[32 * 64];
                if (st) memcpy(W, st->xfer[l - c->l0 - 1] + p * 2 * r * r, sizeof(cplx) * (size_t)(2 * r * r));
                else if (l <= c->h) blk_first(c, l, a, b, W);
                else blk_second(c, l, a, b, W);
                for (int t = 0; t < r; t++)
                    for (int64_t v = 0; v < nv; v++) {
                        cplx s = 0;
                        for (int cc = 0; cc < 2; cc++) {
                            const int64_t q = (a >> 1) * (2 * nbl) + 2 * b + cc;   /* pair (P, C_c) at l-1 */
                            for (int ss = 0; ss < r; ss++) s += W[t * 2 * r + cc * r + ss] * d0[(q * r + ss) * nv + v];
                        }
                        d1[(p * r + t) * nv + v] = s;
                    }
            }
            cplx *tmp = d0; d0 = d1; d1 = tmp;
        }
        if (l == c->h) {   /* O4 Switch */
            const int64_t nbh = (int64_t)1 << (c->LN - c->h);
#pragma omp parallel for schedule(static)
            for (int64_t p = 0; p < N; p++) {
                const int64_t a = p / nbh, b = p % nbh;
                cplx S[32 * 32];
                if (st) memcpy(S, st->sw + p * r * r, sizeof(cplx) * (size_t)(r * r));
                else blk_switch(c, a, b, S);
                for (int t = 0; t < r; t++)
                    for (int64_t v = 0; v < nv; v++) {
                        cplx s = 0;
                        for (int ss = 0; ss < r; ss++) s += S[t * r + ss] * d0[(p * r + ss) * nv + v];
                        d1[(p * r + t) * nv + v] = s;
                    }
            }
            cplx *tmp = d0; d0 = d1; d1 = tmp;
        }
    }
    /* O6 Termination (eqn:bf3): u(x) = sum_{b < n0} (U[a,b] delta_D[a,b])_x for each leaf a. */
    {
        const int64_t na = N >> c->l0;
#pragma omp parallel for schedule(static)
        for (int64_t a = 0; a < na; a++) {
            cplx *U = malloc(sizeof(cplx) * (size_t)(n0 * r));
            for (int64_t j = 0; j < n0; j++)
                for (int64_t v = 0; v < nv; v++) Uout[(a * n0 + j) + v * N] = 0;
            for (int64_t b = 0; b < n0; b++) {
                const int64_t p = a * n0 + b;   /* pair index at level D: a 2^(LN-D) + b */
                if (st) memcpy(U, st->u + p * n0 * r, sizeof(cplx) * (size_t)(n0 * r));
                else blk_term(c, a, b, U);
                for (int64_t j = 0; j < n0; j++)
                    for (int64_t v = 0; v < nv; v++) {
                        cplx s = 0;
                        for (int t = 0; t < r; t++) s += U[j * r + t] * d0[(p * r + t) * nv + v];
                        Uout[(a * n0 + j) + v * N] += s;
                    }
            }
            free(U);
        }
    }
    free(d0); free(d1);
    return 0;
}

/* Apply the IBF-MAT to F (N x nrhs, ld ldf) and write G (N x nrhs, ld ldg):
 *   g = sum_k a_k o BF(b_k o f)   (eqn:tg P:24-28; O7).
 * Vectors are processed in chunks of at most vchunk (memory bound only; the
 * vectors are independent).  Returns 0 on success. */
static int apply_all(const bfctx *cp, int namp, const cplx *a, const cplx *b, int64_t nrhs, const cplx *F,
                     int64_t ldf, cplx *G, int64_t ldg, int64_t vchunk, const bfstore *st);

int orc_bf_apply(int kernel, int amp, int LN, int l0, int r, int64_t nrhs, const cplx *F, int64_t ldf,
                 cplx *G, int64_t ldg, int64_t vchunk)
{
    bfctx c;
    if (ctx_init(&c, kernel, LN, l0, r) || r > 32 || l0 > 6) return -1;
    const int namp = orc_n_amp(amp);
    if (namp < 1) return -1;
    const int64_t N = c.N;
    cplx *a = malloc(sizeof(cplx) * (size_t)(N * namp)), *b = malloc(sizeof(cplx) * (size_t)(N * namp));
    for (int k = 0; k < namp; k++) {
        orc_amp_term(amp, LN, k, 0, a + k * N);
        orc_amp_term(amp, LN, k, 1, b + k * N);
    }
    const int rc = apply_all(&c, namp, a, b, nrhs, F, ldf, G, ldg, vchunk, NULL);
    free(a); free(b);
    return rc;
}

/* "bf-stored" (SURVEY 8(c) oracle modes): the same O1-O7 steps applied to caller-supplied blocks (complex128,
 * layouts of butterfly_apply above) and amplitude terms a, b ([namp][N]); kernel-independent.  With the
 * oracle's own blocks it reproduces orc_bf_apply; with blocks rounded to complex64 it measures what the
 * factors' storage precision alone contributes to the GPU path's error. */
int orc_bf_apply_stored(int LN, int l0, int r, int namp, const cplx *a, const cplx *b, const cplx *v0,
                        const cplx *const *xfer, const cplx *sw, const cplx *u, int64_t nrhs, const cplx *F,
                        int64_t ldf, cplx *G, int64_t ldg, int64_t vchunk)
{
    bfctx c;
    if (ctx_init(&c, ORC_K_FIO, LN, l0, r) || r > 32 || l0 > 6 || namp < 1) return -1;
    const bfstore st = {v0, sw, u, xfer};
    return apply_all(&c, namp, a, b, nrhs, F, ldf, G, ldg, vchunk, &st);
}

static int apply_all(const bfctx *cp, int namp, const cplx *a, const cplx *b, int64_t nrhs, const cplx *F,
                     int64_t ldf, cplx *G, int64_t ldg, int64_t vchunk, const bfstore *st)
{
    const bfctx c = *cp;
    const int64_t N = c.N;
    if (vchunk < 1) vchunk = 1;
    /* vectors v = (column cidx, term k) */
    const int64_t nvec = nrhs * namp;
    for (int64_t v0 = 0; v0 < nvec; v0 += vchunk) {
        const int64_t nv = (nvec - v0 < vchunk) ? nvec - v0 : vchunk;
        cplx *Y = malloc(sizeof(cplx) * (size_t)(N * nv)), *Uo = malloc(sizeof(cplx) * (size_t)(N * nv));
        for (int64_t v = 0; v < nv; v++) {
            const int64_t col = (v0 + v) / namp, k = (v0 + v) % namp;
            for (int64_t j = 0; j < N; j++) Y[j + v * N] = b[k * N + j] * F[j + col * ldf];   /* y = b_k o f */
        }
        int rc = butterfly_apply(&c, nv, Y, Uo, st);
        if (rc) { free(Y); free(Uo); return rc; }
        for (int64_t v = 0; v < nv; v++) {
            const int64_t col = (v0 + v) / namp, k = (v0 + v) % namp;
            for (int64_t i = 0; i < N; i++) {
                if (k == 0) G[i + col * ldg] = 0;
                G[i + col * ldg] += a[k * N + i] * Uo[i + v * N];                             /* sum_k a_k o u_k */
            }
        }
        free(Y); free(Uo);
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* O8: the adjoint apply K* (needed by Scenario 2 and FIO  */
/* composition).  K*(xi_j, x_i) = conj(K(x_i, xi_j)), so    */
/* with eqn:tg and eqn:BFM  K* ~ sum_k conj(b_k) o BF* (conj(a_k) o .)  and    */
/* BF* = V^* G_{l0+1}^* ... G_h^* Sw^* G_{h+1}^* ... G_D^* U^*: the factors of */
/* O2-O6 conjugate-transposed and applied in reverse order.  Written as        */
/* gathers (each output coefficient sums its own inputs), blocks generated on  */
/* the fly from the same equations as O1-O7.  Y: N x nv over x; Uout over xi.  */
/* ------------------------------------------------------------------------- */
static int butterfly_adjoint(const bfctx *c, int64_t nv, const cplx *Y, cplx *Uout)
{
    const int r = c->r;
    const int64_t N = c->N, n0 = c->n0;
    cplx *d0 = malloc(sizeof(cplx) * (size_t)(N * r * nv));
    cplx *d1 = malloc(sizeof(cplx) * (size_t)(N * r * nv));
    if (!d0 || !d1) { free(d0); free(d1); return -2; }

    /* O6*: gamma_D[a,b] = U[a,b]^* y_A for each T_X leaf a and b < n0 (pair a n0 + b at level D). */
    {
#pragma omp parallel for schedule(static)
        for (int64_t p = 0; p < N; p++) {
            const int64_t a = p / n0, b = p % n0;
            cplx *U = malloc(sizeof(cplx) * (size_t)(n0 * r));
            blk_term(c, a, b, U);
            for (int t = 0; t < r; t++)
                for (int64_t v = 0; v < nv; v++) {
                    cplx s = 0;
                    for (int64_t j = 0; j < n0; j++) s += conj(U[j * r + t]) * Y[(a * n0 + j) + v * N];
                    d0[(p * r + t) * nv + v] = s;
                }
            free(U);
        }
    }
    /* O5* / O4* / O3*: levels D .. l0+1 in reverse, the switch adjoint at l = h before G_h^*. */
    for (int l = c->D; l >= c->l0; l--) {
        if (l == c->h) {   /* O4*: gamma_h[p] = Sw[p]^* gamma_h[p] */
            const int64_t nbh = (int64_t)1 << (c->LN - c->h);
#pragma omp parallel for schedule(static)
            for (int64_t p = 0; p < N; p++) {
                cplx S[32 * 32];
                blk_switch(c, p / nbh, p % nbh, S);
                for (int s = 0; s < r; s++)
                    for (int64_t v = 0; v < nv; v++) {
                        cplx acc = 0;
                        for (int t = 0; t < r; t++) acc += conj(S[t * r + s]) * d0[(p * r + t) * nv + v];
                        d1[(p * r + s) * nv + v] = acc;
                    }
            }
            cplx *tmp = d0; d0 = d1; d1 = tmp;
        }
        if (l > c->l0) {   /* G_l^*: pair q = (a', b') at level l-1 gathers from its parents (2a'+e, b'>>1) at l */
            const int64_t nbl = (int64_t)1 << (c->LN - l);   /* b-range at level l   */
            const int64_t nbq = 2 * nbl;                     /* b-range at level l-1 */
#pragma omp parallel for schedule(static)
            for (int64_t q = 0; q < N; q++) {
                const int64_t a1 = q / nbq, b1 = q % nbq;
                const int cc = (int)(b1 & 1);   /* q's B is child cc of the parents' B */
                cplx W[2][32 * 64];
                int64_t par[2];
                for (int e = 0; e < 2; e++) {
                    const int64_t a = 2 * a1 + e, b = b1 >> 1;
                    par[e] = a * nbl + b;
                    if (l <= c->h) blk_first(c, l, a, b, W[e]); else blk_second(c, l, a, b, W[e]);
                }
                for (int s = 0; s < r; s++)
                    for (int64_t v = 0; v < nv; v++) {
                        cplx acc = 0;
                        for (int e = 0; e < 2; e++)
                            for (int t = 0; t < r; t++)
                                acc += conj(W[e][t * 2 * r + cc * r + s]) * d0[(par[e] * r + t) * nv + v];
                        d1[(q * r + s) * nv + v] = acc;
                    }
            }
            cplx *tmp = d0; d0 = d1; d1 = tmp;
        }
    }
    /* O2*: u(xi) = sum_{a < n0} (V[a,b]^* gamma_{l0}[a,b])_xi for each leaf b of T_Omega. */
    {
        const int64_t nb = N >> c->l0;
#pragma omp parallel for schedule(static)
        for (int64_t b = 0; b < nb; b++) {
            cplx *V = malloc(sizeof(cplx) * (size_t)(r * n0));
            for (int64_t j = 0; j < n0; j++)
                for (int64_t v = 0; v < nv; v++) Uout[(b * n0 + j) + v * N] = 0;
            for (int64_t a = 0; a < n0; a++) {
                const int64_t p = a * nb + b;
                blk_init(c, a, b, V);
                for (int64_t j = 0; j < n0; j++)
                    for (int64_t v = 0; v < nv; v++) {
                        cplx s = 0;
                        for (int t = 0; t < r; t++) s += conj(V[t * n0 + j]) * d0[(p * r + t) * nv + v];
                        Uout[(b * n0 + j) + v * N] += s;
                    }
            }
            free(V);
        }
    }
    free(d0); free(d1);
    return 0;
}

/* G = K* F = sum_k conj(b_k) o BF*(conj(a_k) o F): F indexed by x (N x nrhs), G by xi. */
int orc_bf_apply_adjoint(int kernel, int amp, int LN, int l0, int r, int64_t nrhs, const cplx *F, int64_t ldf,
                         cplx *G, int64_t ldg, int64_t vchunk)
{
    bfctx c;
    if (ctx_init(&c, kernel, LN, l0, r) || r > 32 || l0 > 6) return -1;
    const int namp = orc_n_amp(amp);
    if (namp < 1) return -1;
    const int64_t N = c.N;
    if (vchunk < 1) vchunk = 1;
    cplx *a = malloc(sizeof(cplx) * (size_t)(N * namp)), *b = malloc(sizeof(cplx) * (size_t)(N * namp));
    for (int k = 0; k < namp; k++) {
        orc_amp_term(amp, LN, k, 0, a + k * N);
        orc_amp_term(amp, LN, k, 1, b + k * N);
    }
    const int64_t nvec = nrhs * namp;
    int rc = 0;
    for (int64_t v0 = 0; v0 < nvec && !rc; v0 += vchunk) {
        const int64_t nv = (nvec - v0 < vchunk) ? nvec - v0 : vchunk;
        cplx *Y = malloc(sizeof(cplx) * (size_t)(N * nv)), *Uo = malloc(sizeof(cplx) * (size_t)(N * nv));
        for (int64_t v = 0; v < nv; v++) {
            const int64_t col = (v0 + v) / namp, k = (v0 + v) % namp;
            for (int64_t i = 0; i < N; i++) Y[i + v * N] = conj(a[k * N + i]) * F[i + col * ldf];   /* conj(a_k) o f */
        }
        rc = butterfly_adjoint(&c, nv, Y, Uo);
        for (int64_t v = 0; v < nv && !rc; v++) {
            const int64_t col = (v0 + v) / namp, k = (v0 + v) % namp;
            for (int64_t j = 0; j < N; j++) {
                if (k == 0) G[j + col * ldg] = 0;
                G[j + col * ldg] += conj(b[k * N + j]) * Uo[j + v * N];                       /* sum_k conj(b_k) o u_k */
            }
        }
        free(Y); free(Uo);
    }
    free(a); free(b);
    return rc;
}

/* O0*: the adjoint direct sum on a set of xi-rows:  out[q, c] = sum_i conj(alpha(x_i, xi_j) e^{2 pi i Phi(x_i, xi_j)})
 * F[i, c] with j = rows[q] -- the definition of K* applied to F. */
void orc_direct_adjoint_rows(int kernel, int amp, int LN, int64_t nrhs, const cplx *F, int64_t ldf,
                             const int64_t *rows, int64_t nrows, cplx *out)
{
    const int64_t N = (int64_t)1 << LN;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < nrows; q++) {
        const int64_t j = rows[q];
        cplx *acc = calloc((size_t)nrhs, sizeof(cplx));
        for (int64_t i = 0; i < N; i++) {
            cplx K = conj(orc_alpha(amp, LN, i, j) * E(kernel, LN, i, j, +1, 1));
            for (int64_t cidx = 0; cidx < nrhs; cidx++) acc[cidx] += K * F[i + cidx * ldf];
        }
        for (int64_t cidx = 0; cidx < nrhs; cidx++) out[q + cidx * nrows] = acc[cidx];
        free(acc);
    }
}

int orc_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
