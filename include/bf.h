/*
 * bf.h -- C ABI of the B200-native IBF-MAT apply (arXiv:1803.04128, H. Yang).
 *
 * The library applies a complementary-low-rank butterfly factorization (BF) of
 * the phase matrix e^{2 pi i Phi}, together with a low-rank amplitude split
 * alpha(x,xi) ~ sum_k a_k(x) b_k(xi), to a batch of right-hand sides:
 *
 *      G = sum_k a_k o BF(b_k o F)                       eqn:tg
 *
 * where BF is the factor form eqn:BFM  K ~ U^L G^{L-1}...G^h M^h (H^h)*...(H^1)*(V^0)*
 * whose blocks are produced by Algorithm 4.1.
 *
 * Notation (0-based; DESIGN.md sections 2-3):
 *   N = 2^LN (LN even), leaf n0 = 2^l0 (r <= n0, 2 l0 <= LN), D = LN - l0, h = LN/2.
 *   Level l in [l0, D]:  A(l,a) = rows [a N/2^l, (a+1) N/2^l),  a < 2^l
 *                        B(l,b) = cols [b 2^l, (b+1) 2^l),       b < 2^(LN-l)
 *   Pairs (A,B) at level l have l_A + l_B = LN (width product 1);
 *   there are N pairs per level, pair index p = a * 2^(LN-l) + b.
 *   r = block rank (number of interpolation points r_eps); n_amp = number of
 *   amplitude terms k.
 *
 * Complex values are interleaved {re, im} single precision (complex64), little
 * endian.  Every factor block is stored COLUMN-MAJOR: element (row, col) of an
 * m x k block sits at col*m + row.  Blocks of one stage are stored in pair order.
 *
 * Stages of one apply (all FP32 FFMA accumulation):
 *   V0   (S0)  per pair at level l0 an r x n0 block  (initialization eqn:1, P:698-702;
 *              A = A(l0,a), B = B(l0,b) is a leaf of n0 columns)
 *   XFER       per transfer level l = l0+1..D and pair an r x 2r block acting on
 *              [delta_{l-1}(a>>1, 2b); delta_{l-1}(a>>1, 2b+1)]
 *              (first half l <= h: eqn:2 P:748-752; second half l > h: eqn:3 P:780-785)
 *   SW         per pair at level h an r x r block (switch)
 *   U    (SL)  per pair at level D an n0 x r block; the n0 pairs (a, b<n0) of a
 *              T_X leaf a are summed (termination eqn:bf3)
 *
 * Errors: every call returns a bf_status_t; nothing throws or aborts across the
 * ABI.  Argument, shape and alignment errors are detected synchronously.  Kernel
 * launch errors are reported by the launching call; asynchronous device faults
 * surface at the next synchronizing call (bf_plan_destroy, bf_apply_host, or the
 * caller's own stream synchronization).  bf_last_error() returns a thread-local
 * message describing the last non-OK status of the calling thread.
 */
#ifndef BF_H_
#define BF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BF_ABI_VERSION 1

typedef struct { float re, im; } bf_c64;   /* complex64, layout-compatible with float2 */

typedef enum {
    BF_OK = 0,
    BF_ERR_INVALID_ARG = 1,   /* null pointer, negative count, bad stage id, ...            */
    BF_ERR_SHAPE = 2,         /* N / leaf / rank / n_amp combination not supported          */
    BF_ERR_ALIGNMENT = 3,     /* F/G/workspace not 16-byte aligned, ld too small            */
    BF_ERR_OOM = 4,           /* device or pinned-host allocation failed                    */
    BF_ERR_CUDA = 5,          /* CUDA runtime error (message in bf_last_error)              */
    BF_ERR_NCCL = 6,          /* reserved for the index-sharded plan                        */
    BF_ERR_NOT_SUPPORTED = 7, /* e.g. odd rank, rank > 16, n_amp not in {1,2,4}             */
    BF_ERR_STATE = 8          /* plan not finalized / stage not uploaded / already final    */
} bf_status_t;

/* stage ids for bf_plan_upload */
#define BF_STAGE_V0 0
#define BF_STAGE_SW 1
#define BF_STAGE_U 2
#define BF_STAGE_AMP_A 3   /* blocks = the n_amp rows of N values each */
#define BF_STAGE_AMP_B 4
#define BF_STAGE_XFER0 16  /* BF_STAGE_XFER0 + i is transfer level l = l0 + 1 + i, i < D - l0 */

#define BF_MEM_HOST 0
#define BF_MEM_DEVICE 1

typedef struct bf_plan_s *bf_plan_t;

/* Factor arrays of one BF (see the stage list above for shapes).
 *   amp_a  [n_amp][N]        a_k(x_i)
 *   amp_b  [n_amp][N]        b_k(xi_j)
 *   v0     [N][n0][r]        pair p = a (N/n0) + b at level l0; block r x n0 column-major
 *   xfer   D-l0 pointers; xfer[i] is [N][2r][r] for level l = l0+1+i, pair p = a 2^(LN-l) + b;
 *          column c r + s of a block multiplies delta_{l-1}(a>>1, 2b+c)[s]
 *   sw     [N][r][r]         pair p = a 2^h + b at level h
 *   u      [N][r][n0]        pair p = a n0 + b at level D (a < N/n0 a T_X leaf, b < n0);
 *                            block n0 x r column-major: row j is output x = a n0 + j
 * Any of the array pointers may be NULL in a descriptor passed to bf_plan_alloc. */
typedef struct {
    int32_t abi_version;       /* BF_ABI_VERSION */
    int32_t log2n;             /* LN, even, 2 <= LN <= 26 */
    int32_t log2leaf;          /* l0, 1 <= l0, 2 l0 <= LN */
    int32_t rank;              /* r, even, 2 <= r <= 16, r <= n0 */
    int32_t n_amp;             /* n_amp in {1, 2, 4} */
    int32_t memory;            /* BF_MEM_HOST or BF_MEM_DEVICE: where the arrays below live */
    const bf_c64 *amp_a;
    const bf_c64 *amp_b;
    const bf_c64 *v0;
    const bf_c64 *const *xfer;
    const bf_c64 *sw;
    const bf_c64 *u;
} bf_desc_t;

typedef struct {
    int32_t log2n, log2leaf, rank, n_amp, switch_level, n_xfer;
    int64_t n;
    int64_t max_nrhs_chunk;
    int64_t factor_bytes;        /* device bytes of all factor + amplitude arrays */
    int64_t workspace_bytes;     /* device bytes of the plan-owned coefficient workspace */
    int32_t launches_per_chunk;  /* kernels one full RHS chunk (max_nrhs_chunk columns) launches */
    int32_t device;
    int32_t class_launches[6];   /* per kernel class (see bf_plan_timing): launches per full chunk */
    int32_t class_levels[6];     /* per kernel class: transfer levels those launches perform */
    int32_t world;               /* index shards (1 unless sharded) */
    int32_t shard_rank;          /* this plan's shard (BF_SHARD_NCCL) */
    int32_t sharding;            /* BF_SHARD_NONE / BF_SHARD_NCCL / BF_SHARD_EMULATED */
    int64_t rows_local;          /* rows of F and G bf_apply expects: N, or N/world for BF_SHARD_NCCL */
    int64_t tc_weight_bytes;     /* device bytes of the tensor-core leaf weight images (0 if not built) */
    int32_t tc_class_mask;       /* bit c set: kernel class c (bf_plan_timing numbering) runs on the tensor
                                    cores (3xTF32) for a full chunk of max_nrhs_chunk columns */
    int32_t structured;          /* 1: the plan applies structured factors (bf_plan_create_structured) */
} bf_plan_info_t;

/* index sharding modes */
#define BF_SHARD_NONE 0
#define BF_SHARD_NCCL 1      /* one shard per process/GPU; the level-h exchange is an NCCL all-to-all */
#define BF_SHARD_EMULATED 2  /* all `world` shards on one device; the exchange is device copies */

/* Create a plan on `device` from complete factor arrays.  The plan deep-copies
 * every array into device memory it owns (the caller may free its arrays when
 * the call returns) and allocates a coefficient workspace for RHS chunks of at
 * most max_nrhs_chunk columns (2 arrays of N r max_nrhs_chunk n_amp complex64).
 * The plan is immutable afterwards. */
bf_status_t bf_plan_create(const bf_desc_t *desc, int device, int64_t max_nrhs_chunk, bf_plan_t *out);

/* The adjoint plan: G = K* F with K*(xi_j, x_i) = conj(K(x_i, xi_j)), i.e.
 *      G = sum_k conj(b_k) o BF*(conj(a_k) o F),   BF* = (eqn:BFM)^*  (P:613-619),
 * the operator Scenario 2 and FIO composition need.  F is indexed by x, G by xi (both
 * N x nrhs column-major, as for bf_apply).  Built on the device from the finalized forward plan `fwd`
 * (unsharded): the conjugate-transposed factors in reverse order ARE a butterfly of the same shape once the
 * two trees swap roles (the adjoint's level-m pair (a, b) is the forward's level-(LN - m) pair (b, a)), so
 * the adjoint plan's blocks are
 *     V0~[a (N/n0) + b] = U[b n0 + a]^*,     U~[a n0 + b] = V0[b (N/n0) + a]^*,
 *     XFER~_m[(a,b)](t, c r + s) = conj(XFER_{LN-m+1}[(2b+c, a>>1)](s, (a&1) r + t)),
 *     amp_a~ = conj(amp_b),  amp_b~ = conj(amp_a)
 * (the switch rides along inside the forward's level-h factor), and every bf_apply entry point and kernel
 * class serves it unchanged.  Exact (data movement and conjugation).  The new plan owns its own copies and
 * workspace (chunks of max_nrhs_chunk columns); `fwd` may be destroyed afterwards.
 * Errors: BF_ERR_STATE if fwd is not finalized, BF_ERR_NOT_SUPPORTED for index-sharded plans, BF_ERR_OOM. */
bf_status_t bf_plan_create_adjoint(bf_plan_t fwd, int64_t max_nrhs_chunk, bf_plan_t *out);

/* ---- structured plans: interpolative factors stored as phases + shared Lagrange ----
 * Every interpolative block of Algorithm 4.1 is diag(phases) . L . diag(phases) with a real Lagrange matrix L
 * that the whole level shares, because the grids of one level are translates of each other (eqn:gdA/gdB
 * P:214-226; eqn:1 P:700, eqn:2 P:750, eqn:3 P:783, eqn:bf3 P:795).  A structured plan stores per pair
 * only one phase diagonal per level -- the row phases of a level merged with the column phases of the next,
 * since both act on the same coefficients -- and per level one L (the builder, bf_plan_build_fio_structured,
 * writes them; DESIGN.md section 5.5 gives the formulas).  The coefficients between levels are then
 *   eta_l  = e(+Phi(c_A, xi_t^B)) o delta_l   (levels l0 .. h-1)     zeta_l = e(-Phi(x_t^A, c_B)) o delta_l (l >= h)
 * and the stages compute (all FP32; complex x real = 2 FMA):
 *   BF_LEVEL_FIRST  (S0)  out[p](t)       = sum_j L(t, j) data[p][j] y_b[j]                    L: r x n0
 *   BF_LEVEL_FIRST  (l)   out[p](t)       = sum_{c,s} L(t, c r + s) data[p][c r + s] in[q_c](s)   L: r x 2r
 *   BF_LEVEL_SECOND (l)   out[p](t)       = sum_c data[p][c r + t] sum_s L_{a&1}(t, s) in[q_c](s)  L: 2 x r x r
 *   BF_LEVEL_FIRST_SWITCH (l) out[p](t)   = sum_s Sw'[p](t, s) sum_{c,s'} L(s, c r + s') psi[p][c r + s'] in[q_c](s')
 *                          data[p] = [psi (2r) | Sw' (r x r)], L: r x 2r   (level h: the switch with its phases)
 *   BF_LEVEL_DENSE  (l)   out[p]          = data[p] [in[q_0]; in[q_1]]        data: [N][2r][r] as bf_desc_t.xfer
 *   BF_LEVEL_DENSE  (S0)  out[p]          = data[p] y_b                       data: [N][n0][r] as bf_desc_t.v0
 *   SL                    G[a n0 + j, c]  = sum_k a_k sum_{b<n0} sl_phase[a n0 + b][j] sum_t sl_lag(j, t) in[a n0+b](t)
 * (q_c = (a>>1) 2^(LN-l+1) + 2b + c; every L column-major; L_e at offset e r^2).  There is no separate switch:
 * the level-h factor must carry it with its neighbouring phases (FIRST_SWITCH or DENSE; V0 DENSE when h == l0).
 * Factor bytes per pair: n0 + 2r per structured level + r^2 (the switch) + n0, against r n0 + 2 r^2 per level + n0 r
 * dense (cfg5: 14.4 GB instead of 110 GB).  Chunks that run on the tensor cores (nv >= 64) use dense blocks expanded from the
 * structured ones at finalization (the plan then frees the structured arrays); every other chunk runs the
 * structured kernels.  Unsharded only; bf_plan_create_adjoint returns BF_ERR_NOT_SUPPORTED for them. */
#define BF_LEVEL_DENSE 0
#define BF_LEVEL_FIRST 1
#define BF_LEVEL_SECOND 2
#define BF_LEVEL_FIRST_SWITCH 3
typedef struct {
    int32_t kind;          /* BF_LEVEL_*                                                              */
    const float *lag;      /* FIRST, FIRST_SWITCH: r x 2r; SECOND: 2 x r x r; DENSE: unused (NULL)    */
    const bf_c64 *data;    /* FIRST / SECOND: [N][2r]; FIRST_SWITCH: [N][2r + r^2]; DENSE: [N][2r][r] */
} bf_slevel_t;
typedef struct {
    int32_t abi_version;   /* BF_ABI_VERSION */
    int32_t log2n, log2leaf, rank, n_amp;   /* as bf_desc_t */
    int32_t memory;        /* BF_MEM_HOST / BF_MEM_DEVICE: where the arrays below live (lag arrays too)  */
    const bf_c64 *amp_a, *amp_b;            /* [n_amp][N] */
    int32_t s0_kind;       /* BF_LEVEL_FIRST (s0_lag r x n0, s0_data [N][n0]) or BF_LEVEL_DENSE (s0_data [N][n0][r]) */
    const float *s0_lag;
    const bf_c64 *s0_data;
    const bf_slevel_t *xfer;                /* D - l0 levels, level l0 + 1 + i */
    const float *sl_lag;   /* n0 x r */
    const bf_c64 *sl_phase;                 /* [N][n0] */
} bf_sdesc_t;
/* Deep-copies the arrays (the caller may free them on return) and finalizes.  BF_ERR_INVALID_ARG for a missing
 * array or an unknown kind; otherwise as bf_plan_create. */
bf_status_t bf_plan_create_structured(const bf_sdesc_t *desc, int device, int64_t max_nrhs_chunk, bf_plan_t *out);

/* Recompression ("structure-preserving sweeping matrix compression", deferred by the
 * paper to [IBF]): a new plan of rank `rank` <= r whose factors are the balanced truncation of src's.  Every
 * coefficient space delta_l[p] of eqn:BFM carries the block K(A,B) = S_p R_p (input -> delta_l[p] -> output);
 * with Gamma_out = S_p^H S_p (top-down) and Gamma_in = R_p R_p^H (bottom-up over the already truncated levels)
 * the sweep keeps the `rank` dominant singular directions of Gamma_out^{1/2} Gamma_in^{1/2}, i.e. the best
 * rank-`rank` approximation of each block, and rewrites V0' = P V0, W'_l = P_l W_l diag(Q_{l-1}), U' = U Q_D
 * (R21).  Built on the device in FP64 at plan construction (untimed, like the switch fold); scratch
 * (D - l0 + 1) N r^2 complex doubles.  src: finalized, unsharded, dense (not structured), r <= 12; rank in the
 * supported set; the new plan owns everything (src may be destroyed).  The interpolative rank 12 recompressed
 * to 8 stays within eps/2 = 5e-7 of the direct sum (tests/test_oracle_recompress.py) with 2/3 the transfer
 * flops of the rank-10 interpolative factorization. */
bf_status_t bf_plan_recompress(bf_plan_t src, int32_t rank, int64_t max_nrhs_chunk, bf_plan_t *out);

/* Streaming construction (factors larger than host RAM): allocate the plan from the
 * shape fields of `meta` (array pointers ignored), upload stage blocks in any order
 * and ranges, then finalize.  block_begin/block_count count blocks of the stage
 * (pairs; for BF_STAGE_AMP_* the amplitude rows).  src is host (pageable or pinned)
 * or device memory per src_memory; the copy is complete when the call returns. */
bf_status_t bf_plan_alloc(const bf_desc_t *meta, int device, int64_t max_nrhs_chunk, bf_plan_t *out);
bf_status_t bf_plan_upload(bf_plan_t plan, int32_t stage, int64_t block_begin, int64_t block_count,
                           const bf_c64 *src, int32_t src_memory);
/* Fails with BF_ERR_STATE unless every block of every stage was uploaded. */
bf_status_t bf_plan_finalize(bf_plan_t plan);

/* G = sum_k a_k o BF(b_k o F) for nrhs columns.  F and G are DEVICE buffers,
 * column-major N x nrhs with leading dimension N, 16-byte aligned, not aliasing.
 * Only enqueues work on `stream` (a cudaStream_t; NULL = legacy default stream):
 * no allocation, no synchronization, CUDA-graph capturable.  RHS are processed in
 * chunks of at most max_nrhs_chunk columns.  nrhs = 0 is a no-op.  One apply per
 * plan may be in flight at a time (the workspace is shared) unless bf_apply_ex is
 * given its own workspace. */
bf_status_t bf_apply(bf_plan_t plan, const bf_c64 *F, bf_c64 *G, int64_t nrhs, void *stream);

/* As bf_apply with leading dimensions (ldf, ldg >= N, even) and an optional
 * caller workspace (device, 16-byte aligned, >= bf_workspace_bytes(plan, chunk)).
 * F or G not 16-byte aligned, or an odd ldf / ldg: BF_ERR_ALIGNMENT. */
bf_status_t bf_apply_ex(bf_plan_t plan, const bf_c64 *F, int64_t ldf, bf_c64 *G, int64_t ldg, int64_t nrhs,
                        void *workspace, size_t workspace_bytes, void *stream);

/* bf_apply as ONE graph launch (same operation, eqn:tg P:24-28 with BF in the form eqn:BFM P:613-619, same
 * arguments and errors).  The first call with a given (F, G, nrhs) captures bf_apply's kernel sequence into a
 * CUDA graph on a private stream and instantiates it (host work of a few hundred microseconds, nothing
 * runs); every call then launches that graph on `stream`, so a step of several kernels costs one launch — for
 * the small configurations, whose kernels run for microseconds, the host launch rate otherwise bounds the
 * step.  The plan keeps ONE graph: a call with other F, G or nrhs re-captures, and bf_plan_set_option /
 * bf_plan_set_timing drop it (with timing on, the call is an eager bf_apply so every launch is timed).  F and
 * G must stay allocated while the graph is cached; their contents are read / written at every launch.
 * BF_ERR_NOT_SUPPORTED for NCCL index-sharded plans. */
bf_status_t bf_apply_graph(bf_plan_t plan, const bf_c64 *F, bf_c64 *G, int64_t nrhs, void *stream);

/* End-to-end apply with HOST buffers (N x nrhs column-major, ld = N; pinned memory
 * recommended): per RHS chunk, host->device copy of F, the apply, device->host copy
 * of G, all on `stream`; returns after the stream has completed the work. */
bf_status_t bf_apply_host(bf_plan_t plan, const bf_c64 *F_host, bf_c64 *G_host, int64_t nrhs, void *stream);

/* Asynchronous end-to-end apply with HOST buffers (pinned: cudaHostAlloc / cudaHostRegister; pageable memory
 * works but the copies then serialize): per RHS chunk of <= max_nrhs_chunk columns, host->device copy of F on the
 * plan's copy stream, the apply on `stream`, device->host copy of G on a second copy stream, through two device
 * staging slots used alternately -- and returns at once.  Consecutive calls (and chunks) therefore overlap the
 * copies of one chunk with the apply of its neighbours (PCIe is full duplex), which bf_apply_host cannot do
 * across calls.  F_host and G_host must stay valid and untouched until bf_apply_host_wait returns (or the
 * plan's work is otherwise known complete).  Uses the plan workspace: one async call stream per plan. */
bf_status_t bf_apply_host_async(bf_plan_t plan, const bf_c64 *F_host, bf_c64 *G_host, int64_t nrhs, void *stream);
/* Wait until every G copy issued by bf_apply_host_async has landed on the host. */
bf_status_t bf_apply_host_wait(bf_plan_t plan);

/* Workspace bytes one chunk of `nrhs_chunk` columns needs. */
size_t bf_workspace_bytes(bf_plan_t plan, int64_t nrhs_chunk);

bf_status_t bf_plan_get_info(bf_plan_t plan, bf_plan_info_t *info);

/* Per-kernel device timing (for the roofline report).  When enabled, every launch
 * of bf_apply is bracketed by CUDA events on the launching stream; bf_plan_timing
 * synchronizes on the last event and returns the accumulated milliseconds and
 * launch counts per kernel class: [0] S0, [1] first-half transfer, [2] switch-fused
 * transfer / switch, [3] second-half transfer, [4] SL, [5] level-h exchange (index-
 * sharded plans).  Arrays have BF_NUM_KCLASS entries.  Enabling resets the accumulators. */
#define BF_NUM_KCLASS 6
bf_status_t bf_plan_set_timing(bf_plan_t plan, int32_t enable);
bf_status_t bf_plan_timing(bf_plan_t plan, double *ms, int64_t *launches);

/* Plan options (take effect at the next bf_apply; not thread-safe against an apply in flight).
 *   BF_OPT_TENSOR_CORES  1 (default): stages whose vector batch makes them a dense contraction
 *                        (nv = nrhs n_amp >= 64 per chunk, n0 in {32, 64}) run on the tcgen05
 *                        tensor cores in 3xTF32 with FP32 accumulation;
 *                        0: every stage runs the FP32 FFMA (SIMT) kernels.
 * Returns BF_ERR_INVALID_ARG for an unknown option or value. */
#define BF_OPT_TENSOR_CORES 1
/*   BF_OPT_EXCHANGE (index-sharded plans): 0 (default) = the level-h exchange is a separate step (NCCL
 *                        grouped send/recv, or device copies between emulated shards); 1 = fused exchange:
 *                        the launch that produces level h stores each output pair directly into its
 *                        destination shard's receive array (peer memory over NVLink via CUDA IPC for one
 *                        shard per GPU; the same device for emulated shards), ordered by stream-ordered
 *                        barriers.  Enabling it is collective for NCCL plans (every rank must call it).
 *                        Not available when h == l0 (BF_ERR_NOT_SUPPORTED).  While it is on, bf_apply_ex with a
 *                        caller workspace returns BF_ERR_NOT_SUPPORTED (the peers store into the plan workspace). */
#define BF_OPT_EXCHANGE 4
/*   BF_OPT_BAND_COMPOSE  1 (default): the tensor-core band applies its two transfer levels as one composed
 *                        4 x 4 block operator per group of 4 pairs (C = W_{l+1} W_l per block path, formed
 *                        in FP32 on chip; same MAC count, one accumulation chain per tile);
 *                        0: the level-by-level band kernel (band_tc_kernel). */
#define BF_OPT_BAND_COMPOSE 5
/*   BF_OPT_HOST_PIECES   2 (default), 1..16: bf_apply_host splits each chunk into this many equal pieces whose
 *                        host<->device copies overlap the apply of the neighbouring pieces; 3 = tapered
 *                        pieces of 1/4, 1/2, 1/4 of a chunk (measured at cfg4: 2 pieces 137.5 ms, tapered
 *                        140 ms, 4 pieces 145 ms: smaller pieces re-read the factors and fall below the
 *                        tensor-core tiles). */
#define BF_OPT_HOST_PIECES 8
/*   BF_OPT_LEAF_MULTICAST 1 (default): the 3xTF32 leaf stages S0 and SL run as clusters of two CTAs working
 *                        on the two halves of a leaf's vector tiles, each loading half of every weight-image
 *                        tile (V0x / Ux) and multicasting it to both (needs an even number of 128-vector tiles
 *                        per chunk; else one CTA per tile); 0: off. */
#define BF_OPT_LEAF_MULTICAST 9
/*   BF_OPT_SMALL_BATCH   1 (default): chunks of few vectors (nv % 8 == 0) run the persistent small-batch kernels
 *                        (bf_small.cu: a producer warp bulk-copies weight blocks into a shared-memory ring, one job
 *                        per consumer warp): transfer levels two per launch for 8 <= nv < 128,
 *                        S0 for nv <= 56, SL for nv in {8, 16, 32}; 0: the FP32 kernels of bf_kernels.cu (one
 *                        transfer level per launch).  Both compute every output with the same FP32 operation order
 *                        (bitwise equal). */
#define BF_OPT_SMALL_BATCH 10
/*   BF_OPT_BAND_PRECOMPOSE 1 (default): plans whose chunks hold at most 256 vectors compose each tensor-core
 *                        band's two-level operator once at finalization (FP64 products, complex64 result, the
 *                        same bytes as the two levels' blocks; counted in factor_bytes) and the band kernel only
 *                        embeds and splits it; 0: the band composes on chip per group (the default for larger
 *                        chunks, where each group's operator serves several vector tiles). */
#define BF_OPT_BAND_PRECOMPOSE 11
/*   BF_OPT_BAND3         1 (default): unsharded dense plans with r in {6, 8} whose chunks hold >= 128 vectors run
 *                        the transfer levels as three-level tensor-core bands where they leave no lone level
 *                        (8 levels: 3 + 3 + 2; bf_band3.cu): three adjacent factors of eqn:BFM applied
 *                        as one 8 x 8 block operator per group of 8 pairs, composed once at finalization in FP64
 *                        (64 r^2 complex per group, counted in factor_bytes); 0: two-level bands only.  The
 *                        operators are built at finalization whatever the option; without the memory for all of
 *                        them none is built and the plan runs two-level bands. */
#define BF_OPT_BAND3 12
bf_status_t bf_plan_set_option(bf_plan_t plan, int32_t option, int64_t value);

/* Wait for the plan's outstanding work (the last bf_apply enqueued outside a CUDA-graph capture; replays of a
 * graph that captured bf_apply must be synchronized by the caller), then free everything it owns.
 * bf_apply / bf_apply_ex only enqueue work (no allocation, no host synchronization), so they can be captured
 * into a CUDA graph (tests/test_gpu_tc.py::test_cuda_graph_capture).  Index-sharded (NCCL) plans: this wait and
 * the one inside bf_apply_host poll the communicator; an asynchronous NCCL error, or no progress within
 * BF_NCCL_TIMEOUT_S seconds (default 300), aborts the communicator and returns BF_ERR_NCCL (bf_apply also returns
 * BF_ERR_NCCL when an asynchronous error is already pending). */
bf_status_t bf_plan_destroy(bf_plan_t plan);

/* ---- index-sharded plans: one long vector split by index over world = 2^g ranks ----
 * (no paper passage: the paper is serial.)  Rank q owns the xi-rows
 * [q N/G, (q+1) N/G) of F (levels l <= h: pairs whose b has top g bits q) and the x-rows
 * [q N/G, (q+1) N/G) of G (levels l > h: pairs whose a has top g bits q).  The only
 * communication is one all-to-all of the level-h coefficients (N r nv / G^2 complex per
 * rank pair), issued by bf_apply on its stream as grouped ncclSend/ncclRecv.
 * Local factor blocks (desc of bf_plan_create_sharded), each stage in local pair order:
 *   first-half stages (V0, XFER of levels l <= h, SW): local pair a 2^(LN-l-g) + b_l is
 *       global pair a 2^(LN-l) + q 2^(LN-l-g) + b_l;
 *   second-half stages (XFER of levels l > h, U): local pair i is global pair q N/G + i;
 *   amp_b: b_k on xi-rows [q N/G, (q+1) N/G); amp_a: a_k on x-rows [q N/G, (q+1) N/G).
 * bf_apply on such a plan takes the LOCAL rows: F and G are (N/G) x nrhs (ld >= N/G).
 * world = 1 is allowed (no communication).  Requires h - g >= 2 and LN - g >= 2 l0. */
bf_status_t bf_nccl_get_unique_id(void *id128);   /* 128 bytes, to be broadcast to all ranks */
bf_status_t bf_plan_alloc_sharded(const bf_desc_t *meta, int device, int64_t max_nrhs_chunk, int32_t rank,
                                  int32_t world, const void *nccl_unique_id, bf_plan_t *out);
bf_status_t bf_plan_create_sharded(const bf_desc_t *local, int device, int64_t max_nrhs_chunk, int32_t rank,
                                   int32_t world, const void *nccl_unique_id, bf_plan_t *out);
/* Host-only layout query (for tests of the exchange): the N/G global level-h pair indices of rank
 * `rank` in the order of its send buffer (which = 0), its receive buffer (which = 1), or its
 * second-half local order (which = 2). */
bf_status_t bf_shard_pairs(int32_t log2n, int32_t log2leaf, int32_t world, int32_t rank, int32_t which,
                           int64_t *out);

/* Thread-local description of the last non-OK status ("" if none). */
const char *bf_last_error(void);

int32_t bf_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BF_H_ */
