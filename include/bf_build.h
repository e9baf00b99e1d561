/*
 * bf_build.h -- host-side (untimed) construction of the IBF-MAT factors for the
 * closed-form kernels of the BASELINE workloads (arXiv:1803.04128).
 *
 * Factor construction is host work done once per plan (north_star: "Factor
 * construction ... runs once on the host and is not timed").  The builder
 * evaluates, in FP64, the interpolative blocks of Algorithm 4.1
 * built from Algorithm 2: Mock-Chebyshev grids eqn:gdA/gdB
 * (DESIGN R2/R3), Lagrange bases, centers (R4),
 * and writes them as complex64 blocks in the layouts of bf.h.  The amplitude
 * split alpha ~ sum_k a_k b_k is the exact analytic split of DESIGN R11
 * (with cfg3's phase jump folded in, R8).
 *
 * All functions are host-only, thread-safe, and use OpenMP internally.
 */
#ifndef BF_BUILD_H_
#define BF_BUILD_H_

#include "bf.h"

#ifdef __cplusplus
extern "C" {
#endif

/* phase kernels */
#define BF_KERNEL_FIO 0        /* Phi = x xi + c(x)|xi|, c = (2 + sin 2 pi x)/16   (BASELINE cfg1,2,4,5) */
#define BF_KERNEL_FIO_PAPER 1  /* c = (2 + 0.2 sin 2 pi x)/16                      (eqn:1D-FIO-kernal P:894) */
#define BF_KERNEL_DFT 2        /* Phi = x xi                                        (cfg1 sanity case) */
#define BF_KERNEL_FIO_JUMP 3   /* cfg3: BF on the smooth part, jump 0.25 sign(x-1/3) xi in the amplitude */

/* amplitudes */
#define BF_AMP_ONE 0   /* alpha = 1                                             n_amp 1 */
#define BF_AMP_CFG1 1  /* alpha = 1 + 0.5 cos(2 pi x) cos(pi xi/N)               n_amp 2 */
#define BF_AMP_CFG2 2  /* alpha = (1 + 0.3 sin 2 pi x)(1 + 0.3 cos(2 pi xi/N))   n_amp 2 */
#define BF_AMP_CFG3 3  /* alpha = exp(-(x-1/2)^2)(1 + 0.2 sin(4 pi xi/N))        n_amp 4 */

typedef struct {
    int32_t abi_version;  /* BF_ABI_VERSION */
    int32_t kernel;       /* BF_KERNEL_* */
    int32_t amp;          /* BF_AMP_* */
    int32_t log2n;        /* LN (even) */
    int32_t log2leaf;     /* l0 */
    int32_t rank;         /* r */
} bf_fio_t;

/* Number of amplitude terms of `amp` (-1 if unknown). */
int32_t bf_build_n_amp(int32_t amp);

/* a_k (x_i) and b_k(xi_j) into host arrays [n_amp][N]. */
bf_status_t bf_build_amp(const bf_fio_t *k, bf_c64 *amp_a, bf_c64 *amp_b);

/* Blocks [block_begin, block_begin + block_count) of one stage (BF_STAGE_V0,
 * BF_STAGE_XFER0 + i, BF_STAGE_SW, BF_STAGE_U) into the host array `out`
 * (block_count * block_elems complex64, layouts of bf.h). */
bf_status_t bf_build_blocks(const bf_fio_t *k, int32_t stage, int64_t block_begin, int64_t block_count,
                            bf_c64 *out);

/* Complex64 elements of one block of `stage` (0 on a bad stage id). */
int64_t bf_build_block_elems(const bf_fio_t *k, int32_t stage);

/* Build every factor on the host in slices of at most staging_bytes and stream
 * them into a new plan on `device` (bf_plan_alloc + bf_plan_upload + finalize),
 * overlapping the build of slice i+1 with the upload of slice i. */
bf_status_t bf_plan_build_fio(const bf_fio_t *k, int device, int64_t max_nrhs_chunk, int64_t staging_bytes,
                              bf_plan_t *out);

/* The same operator as structured factors (bf.h "structured plans", NEXT-1): phases and shared Lagrange
 * matrices per level, the switch with its neighbouring phases as the dense level-h factor (V0 when h == l0).
 * Built on the host in FP64 (phases and the dense level rounded to complex64, Lagrange matrices to FP32) and
 * streamed into bf_plan_create_structured's layout in slices of at most staging_bytes. */
bf_status_t bf_plan_build_fio_structured(const bf_fio_t *k, int device, int64_t max_nrhs_chunk,
                                         int64_t staging_bytes, bf_plan_t *out);

/* Host-side pieces of the structured factors (tests, custom plans): the per-pair data of one stage for blocks
 * [block_begin, block_begin + block_count) -- BF_STAGE_V0: omega [n0] per pair (the dense r x n0 V0 with the
 * switch when h == l0); BF_STAGE_XFER0 + i: psi (first half) / chi (second half) [2r] per pair, the dense
 * r x 2r block at level h; BF_STAGE_U: Omega [n0] -- and the stage's Lagrange matrix (bf.h layouts: S0 r x n0,
 * first r x 2r, second 2 x r x r, SL n0 x r; unused for the dense level h). */
bf_status_t bf_build_structured(const bf_fio_t *k, int32_t stage, int64_t block_begin, int64_t block_count,
                                bf_c64 *out);
bf_status_t bf_build_structured_lag(const bf_fio_t *k, int32_t stage, float *out);

/* Index-sharded construction (bf.h, "index-sharded plans"): rank `rank` of `world` builds only
 * its own blocks (1/world of every stage) and joins the NCCL communicator of nccl_unique_id. */
bf_status_t bf_plan_build_fio_sharded(const bf_fio_t *k, int device, int32_t rank, int32_t world,
                                      const void *nccl_unique_id, int64_t max_nrhs_chunk, int64_t staging_bytes,
                                      bf_plan_t *out);

/* All `world` shards of the index-sharded plan on ONE device, the exchange done by device copies
 * (validation of the sharded path without a multi-GPU box).  bf_apply takes the full N-row F/G and
 * returns the same result as the unsharded plan. */
bf_status_t bf_plan_build_fio_emulated(const bf_fio_t *k, int device, int32_t world, int64_t max_nrhs_chunk,
                                       int64_t staging_bytes, bf_plan_t *out);

#ifdef __cplusplus
}
#endif
#endif /* BF_BUILD_H_ */
