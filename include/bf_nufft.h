/*
 * bf_nufft.h -- C ABI of the NUFFT path of the unified framework (arXiv:1803.04128 section 3, "NUFFT and
 * dimension lifting"; SURVEY 8(f) NEXT-4 second half).
 *
 * When the phase is (piecewise) of the form Phi(x, xi) = sum_j p_j(x) q_j(xi) -- Algorithm 6 decides
 * this in O(N) -- eqn:tg3 evaluates the oscillatory transform with r-dimensional NUFFTs instead of a
 * butterfly:
 *
 *      g(x_i) = sum_k a_k(x_i) sum_s sum_{xi in X_s} e^{2 pi i t_s(x_i) xi} b_k(xi) f(xi)            (r = 1)
 *
 * over n_sub submatrices X_s of the frequency grid ("the NUFFT approach ... can be applied to submatrices
 * of K"): the configs' kernels Phi = x xi + c(x)|xi| are exactly rank 1 on xi < 0 and xi >= 0, with
 * t_-(x) = x - c(x), t_+(x) = x + c(x) (eqn:phlr P:1125-1131 for the wave-equation FIO).  Each inner sum is a
 * one-dimensional type-2 NUFFT (uniform frequencies, non-uniform targets), computed on the device as
 *   1. pre-scale and place: h(kappa) = b_k(xi) f(xi) / phi^(kappa) on an oversampled grid of n_f = 2 M points
 *      (M = |X_s|, kappa = xi - xi_c centred), zero elsewhere;
 *   2. one batched inverse FFT of size n_f (cuFFT);
 *   3. interpolation at n_f t_s(x_i) with the w-point "exponential of semicircle" kernel
 *      phi(z) = e^{beta (sqrt(1 - z^2) - 1)}, times e^{2 pi i t_s(x_i) xi_c}, a_k(x_i), summed over k and s,
 * with phi^ the kernel's Fourier transform (FP64 quadrature at plan creation) and w, beta set by eps
 * (w = ceil(-log10 eps) + 2, beta = 2.30 w).  FP32 arithmetic on the device (cuFFT C2C single precision); the
 * targets, kernel weights and phases are computed in FP64 on the host and rounded once.
 *
 * Grid (eqn:1D-xandxi P:905-907, 0-based, as bf.h): x_i = i/N are the rows of G, xi_j = j - N/2 the rows of F.
 * Submatrix s covers the contiguous frequency rows [s N / n_sub, (s+1) N / n_sub).
 *
 * Errors as bf.h (bf_status_t, bf_last_error).  Ownership: the plan copies everything it is given.
 */
#ifndef BF_NUFFT_H_
#define BF_NUFFT_H_

#include "bf.h"
#include "bf_build.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bf_nufft_s *bf_nufft_t;

typedef struct {
    int32_t abi_version;     /* BF_ABI_VERSION */
    int32_t log2n;           /* N = 2^log2n, 4 <= log2n <= 26 */
    int32_t n_amp;           /* amplitude terms k (1..8) */
    int32_t n_sub;           /* frequency submatrices: 1 or 2 */
    const double *targets;   /* host [n_sub][N]: t_s(x_i), Phi(x_i, xi) = t_s(x_i) xi for xi in X_s (any real) */
    const bf_c64 *amp_a;     /* host [n_amp][N]: a_k(x_i) */
    const bf_c64 *amp_b;     /* host [n_amp][N]: b_k(xi_j) */
    double eps;              /* target accuracy of each NUFFT, 1e-12 <= eps <= 1e-2 */
} bf_nufft_desc_t;

/* Creates a plan on `device` for RHS chunks of up to max_nrhs_chunk columns (the placed grids and their
 * transforms are sized for it: 2 x n_sub n_amp max_nrhs_chunk n_f complex64, n_f = 2 N / n_sub).  BF_ERR_SHAPE / BF_ERR_INVALID_ARG on bad
 * arguments, BF_ERR_OOM, BF_ERR_CUDA (cuFFT plan failures included). */
bf_status_t bf_nufft_create(const bf_nufft_desc_t *desc, int device, int64_t max_nrhs_chunk, bf_nufft_t *out);

/* G = the NUFFT path applied to F (device, column-major N x nrhs, leading dimensions ldf, ldg >= N; F and G
 * must not alias; F 16-byte aligned with even ldf, G 8-byte aligned, else BF_ERR_ALIGNMENT).  Enqueues on `stream` (cudaStream_t; NULL = legacy default stream), chunks
 * of max_nrhs_chunk columns; nrhs = 0 is a no-op.  One apply in flight per plan (shared workspace). */
bf_status_t bf_nufft_apply(bf_nufft_t plan, const bf_c64 *F, int64_t ldf, bf_c64 *G, int64_t ldg, int64_t nrhs,
                           void *stream);

typedef struct {
    int64_t n;               /* N */
    int32_t width;           /* w: kernel points per target */
    double beta;             /* ES kernel shape */
    int64_t grid;            /* n_f: oversampled FFT size per submatrix */
    int64_t workspace_bytes; /* placed grids + their transforms for one chunk */
    int32_t launches_per_chunk; /* own kernels per chunk (the cuFFT launches not counted) */
} bf_nufft_info_t;
bf_status_t bf_nufft_get_info(bf_nufft_t plan, bf_nufft_info_t *info);

/* Waits for the plan's work and frees it. */
bf_status_t bf_nufft_destroy(bf_nufft_t plan);

/* Algorithm 6 with r = 1 on the host (plan construction, untimed, FP64): does the NUFFT apply to
 * K = (U2 V2^T) o e^{2 pi i U1 V1^T} (m rows x_i, n columns xi_j)?  Steps: the leading singular pair of the phase
 * U1 V1^T by a randomized range finder (r1 + 4 Gaussian test vectors, seeded), P q^T; rq = q sampled columns of
 * (U2 V2^T) o e^{2 pi i (U1 V1^T - P q^T)}; Householder QR with column pivoting; n_rank = the number of |R_kk| >
 * |R_11| eps; y = 1 iff n_rank <= rank_budget (reading R24).  If y = 1 and `targets` is not NULL, the
 * column factor must be a multiple of xi (q_j = alpha xi_j: uniform frequencies, the type-2 NUFFT of
 * bf_nufft_create) and targets[i] = alpha P_i, so that P q^T = t(x_i) xi_j -- else BF_ERR_NOT_SUPPORTED.
 * Layouts: u1 [r1][m], v1 [r1][n] real; u2 [r2][m], v2 [r2][n] complex as interleaved doubles; xi [n]. */
typedef struct {
    int64_t m, n;            /* rows, columns (>= 2) */
    int32_t r1, r2;          /* phase / amplitude factor ranks, 1..16 */
    const double *u1, *v1;   /* phase factors */
    const double *u2, *v2;   /* amplitude factors (complex, {re, im} pairs) */
    const double *xi;        /* [n] column frequencies (for the targets; may be NULL when targets is NULL) */
    int32_t rank_budget;     /* r_eps */
    int32_t q;               /* columns sampled (r q with r = 1) */
    double eps;              /* rank threshold relative to |R_11| */
    uint64_t seed;
} bf_nufft_decide_t;
bf_status_t bf_nufft_decide(const bf_nufft_decide_t *d, int32_t *y, int32_t *n_rank, double *targets);

/* The closed-form kernels of bf_build.h as an NUFFT plan: n_sub = 2 (xi < 0, xi >= 0) with
 * t_-(x) = x - c(x), t_+(x) = x + c(x) (the DFT kernel: t = x on both), and the amplitude split of bf_build_amp
 * (cfg3's jump folded into it, DESIGN R8).  k->log2leaf and k->rank are ignored. */
bf_status_t bf_nufft_build_fio(const bf_fio_t *k, int device, int64_t max_nrhs_chunk, double eps, bf_nufft_t *out);

#ifdef __cplusplus
}
#endif

#endif /* BF_NUFFT_H_ */
