// bf_plan.cu -- the C ABI of include/bf.h: plan creation / streaming upload,
// bf_apply orchestration (one stream, RHS chunks, no allocation), end-to-end
// host apply, per-kernel event timing, and the index-sharded plan (NCCL
// all-to-all at level h, or G shards emulated on one device).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <string>
#include <utility>
#include <vector>

#include "../../include/bf.h"
#include "bf_internal.h"
#include "bf_plan_internal.h"
#include "bf_shard.h"

namespace {

thread_local std::string g_err;

bf_status_t fail(bf_status_t s, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
bf_status_t fail(bf_status_t s, const char* fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

bf_status_t cuda_fail(cudaError_t e, const char* what)
{
    return fail(BF_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

// Restores the caller's current device on scope exit.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev)
    {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard()
    {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// ---------------------------------------------------------------------------
// NCCL, loaded on first use (only index-sharded plans need it; the library has
// no link-time dependency on it).  Types as in nccl.h.
// ---------------------------------------------------------------------------
typedef struct ncclComm* ncclComm_t;
typedef struct {
    char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
constexpr int kNcclUint8 = 1;

struct Nccl {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl& nccl()
{
    static Nccl n;
    static bool tried = false;
    if (tried) return n;
    tried = true;
    // BF_NCCL_LIB (the Python binding points it at the NCCL torch loaded), else the standard sonames
    const char* cands[] = {getenv("BF_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
    void* h = nullptr;
    for (const char* c : cands)
        if (c && (h = dlopen(c, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) return n;
#define BF_NCCL_SYM(field, name) n.field = reinterpret_cast<decltype(n.field)>(dlsym(h, name))
    BF_NCCL_SYM(GetUniqueId, "ncclGetUniqueId");
    BF_NCCL_SYM(CommInitRank, "ncclCommInitRank");
    BF_NCCL_SYM(CommDestroy, "ncclCommDestroy");
    BF_NCCL_SYM(CommAbort, "ncclCommAbort");
    BF_NCCL_SYM(CommGetAsyncError, "ncclCommGetAsyncError");
    BF_NCCL_SYM(Send, "ncclSend");
    BF_NCCL_SYM(Recv, "ncclRecv");
    BF_NCCL_SYM(GroupStart, "ncclGroupStart");
    BF_NCCL_SYM(GroupEnd, "ncclGroupEnd");
    BF_NCCL_SYM(GetErrorString, "ncclGetErrorString");
#undef BF_NCCL_SYM
    n.ok = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.Send && n.Recv && n.GroupStart && n.GroupEnd &&
           n.GetErrorString && n.CommGetAsyncError && n.CommAbort;
    return n;
}

bf_status_t nccl_fail(ncclResult_t r, const char* what)
{
    return fail(BF_ERR_NCCL, "%s: NCCL error %d (%s)", what, r, nccl().GetErrorString ? nccl().GetErrorString(r) : "?");
}

// Seconds a synchronizing call waits for NCCL work before aborting the communicator (BF_NCCL_TIMEOUT_S, default 300).
double nccl_timeout_s()
{
    static const double t = [] {
        const char* e = getenv("BF_NCCL_TIMEOUT_S");
        const double v = e ? atof(e) : 0.0;
        return v > 0 ? v : 300.0;
    }();
    return t;
}

}  // namespace

struct TimedLaunch {
    int cls;
    cudaEvent_t start, stop;
};

// The factors and workspace of one index shard (the whole problem when the plan is not sharded).
struct Shard {
    float2* amp_a = nullptr;   // [n_amp][N/G]   a_k on this shard's x rows
    float2* amp_b = nullptr;   // [n_amp][N/G]   b_k on this shard's xi rows
    float2* v0 = nullptr;
    float2* sw = nullptr;
    float2* u = nullptr;
    std::vector<float2*> xfer;
    std::vector<float2*> cmp;  // [level index of a band's first level]: precomposed two-level operator, or null
    std::vector<float2*> cmp3; // [level index of a band's first level]: precomposed three-level operator, or null
    float* v0x = nullptr;      // tensor-core image of V0 / U (bf_tc.cu), built at finalize when used
    float* ux = nullptr;
    float2* ws = nullptr;      // two coefficient arrays of (N/G) R nv_max
    // structured plans (bf_struct.cu, NEXT-1): a stage whose dense array above is null runs on these
    float* s0_lag = nullptr;   // r x n0
    float2* s0_ph = nullptr;   // [N][n0]
    std::vector<int> kind;     // per transfer level: BF_LEVEL_*
    std::vector<float*> lag;   // per transfer level (structured kinds): L1 r x 2r or L2 2 x r x r
    std::vector<float2*> ph;   // per transfer level (structured kinds): [N][2r]
    float* sl_lag = nullptr;   // n0 x r
    float2* sl_ph = nullptr;   // [N][n0]
    bfk::LagP s0_lagh{};            // host copies: the kernels take the Lagrange matrices as parameters
    std::vector<bfk::LagP> lagh;
    bool dense_all() const
    {
        if (!v0 || !u) return false;
        for (auto x : xfer)
            if (!x) return false;
        return true;
    }
};

struct bf_plan_s {
    int device = 0;
    bfk::Dims d{};             // GLOBAL dims
    int64_t max_chunk = 0;
    int world = 1, rank = 0, g = 0;
    int mode = BF_SHARD_NONE;  // BF_SHARD_NONE / BF_SHARD_NCCL / BF_SHARD_EMULATED
    std::vector<Shard> sh;     // 1 shard, or `world` shards when emulated
    ncclComm_t comm = nullptr;
    // fused exchange (BF_OPT_EXCHANGE = 1): the level-h launch stores into the destination shards' arrays
    bool exchange_peer = false;
    float2* peer_ws[bfs::kMaxShards] = {};   // workspace base of every shard (IPC-mapped for NCCL plans)
    bool peer_ipc[bfs::kMaxShards] = {};     // opened with cudaIpcOpenMemHandle (closed at destroy)
    char* bar_buf = nullptr;                 // 2 x world bytes for the stream-ordered NCCL barrier
    // [shard][stage slot]: block ranges [begin, end) uploaded so far (finalize checks their union covers the stage)
    std::vector<std::vector<std::vector<std::pair<int64_t, int64_t>>>> uploaded;
    bool finalized = false;
    bool switch_in_factors = false;   // the factors already contain the switch (adjoint and structured plans)
    bool structured = false;          // built by bf_plan_create_structured
    size_t ws_bytes = 0;       // per shard
    // end-to-end staging (lazily allocated by bf_apply_host)
    float2* dF = nullptr;
    float2* dG = nullptr;
    int64_t staging_elems = 0;   // complex elements of dF / dG each
    cudaStream_t h2d = nullptr, d2h = nullptr;   // copy streams of the pipelined bf_apply_host
    // bf_apply_host_async: two staging slots of max_nrhs_chunk columns, used alternately per chunk
    float2* aF[2] = {nullptr, nullptr};
    float2* aG[2] = {nullptr, nullptr};
    cudaEvent_t a_h2d[2] = {}, a_applied[2] = {}, a_d2h[2] = {};
    int64_t a_uses = 0;                            // chunks issued through the async ring
    bool tensor_cores = true;  // BF_OPT_TENSOR_CORES
    bfk::BandVariant band;     // BF_OPT_BAND_COMPOSE
    int host_pieces = 2;       // BF_OPT_HOST_PIECES: bf_apply_host pipeline pieces per chunk
    bool leaf_multicast = true;  // BF_OPT_LEAF_MULTICAST: TF32 S0 / SL as 2-CTA clusters sharing the weight stream
    bool small_batch = true;      // BF_OPT_SMALL_BATCH: fused bands for small vector batches (bf_small.cu)
    bool precompose = true;      // BF_OPT_BAND_PRECOMPOSE: use the finalize-time composed band operators
    bool band3 = true;           // BF_OPT_BAND3: three-level tensor-core bands (bf_band3.cu) where built
    // timing
    bool timing = false;
    std::vector<TimedLaunch> pending;
    std::vector<cudaEvent_t> pool;
    double ms[BF_NUM_KCLASS] = {0};
    int64_t nlaunch[BF_NUM_KCLASS] = {0};
    cudaEvent_t done = nullptr;
    // bf_apply_graph: the instantiated CUDA graph of one bf_apply with the argument set (g_F, g_G, g_nrhs),
    // captured on the private stream `cap`; dropped by any option change and by bf_plan_set_timing
    cudaGraphExec_t gexec = nullptr;
    cudaStream_t cap = nullptr;
    const void* g_F = nullptr;
    const void* g_G = nullptr;
    int64_t g_nrhs = -1;

    int64_t nloc() const { return d.N >> g; }   // pairs / rows per shard
    bfk::Dims local() const
    {
        bfk::Dims l = d;
        l.LN = d.LN - g;
        l.N = d.N >> g;
        return l;
    }
};

namespace {

constexpr int KC_EXCHANGE = 5;   // timing class of the level-h all-to-all (BF_NUM_KCLASS)

// stage slot index: 0 V0, 1 SW, 2 U, 3 AMP_A, 4 AMP_B, 5 + i XFER i
int slot_of(const bf_plan_s* p, int stage)
{
    if (stage >= BF_STAGE_XFER0) {
        const int i = stage - BF_STAGE_XFER0;
        return i < int(p->sh[0].xfer.size()) ? 5 + i : -1;
    }
    return (stage >= 0 && stage <= 4) ? stage : -1;
}

// blocks of a stage in ONE shard
int64_t stage_blocks(const bf_plan_s* p, int stage)
{
    if (stage == BF_STAGE_AMP_A || stage == BF_STAGE_AMP_B) return p->d.n_amp;
    return p->nloc();
}

int64_t stage_elems(const bf_plan_s* p, int stage)
{
    const int64_t r = p->d.R, n0 = int64_t(1) << p->d.l0;
    switch (stage) {
    case BF_STAGE_V0: return r * n0;
    case BF_STAGE_SW: return r * r;
    case BF_STAGE_U: return n0 * r;
    case BF_STAGE_AMP_A:
    case BF_STAGE_AMP_B: return p->nloc();
    default: return 2 * r * r;
    }
}

float2* stage_base(Shard& s, int stage)
{
    switch (stage) {
    case BF_STAGE_V0: return s.v0;
    case BF_STAGE_SW: return s.sw;
    case BF_STAGE_U: return s.u;
    case BF_STAGE_AMP_A: return s.amp_a;
    case BF_STAGE_AMP_B: return s.amp_b;
    default: return s.xfer[stage - BF_STAGE_XFER0];
    }
}

bf_status_t validate_shape(const bf_desc_t* d)
{
    if (!d) return fail(BF_ERR_INVALID_ARG, "descriptor is NULL");
    if (d->abi_version != BF_ABI_VERSION)
        return fail(BF_ERR_INVALID_ARG, "abi_version %d != %d", d->abi_version, BF_ABI_VERSION);
    const int LN = d->log2n, l0 = d->log2leaf, r = d->rank;
    if (LN < 2 || LN > 26 || LN % 2) return fail(BF_ERR_SHAPE, "log2n=%d must be even in [2,26]", LN);
    if (l0 < 3 || l0 > 7 || 2 * l0 > LN)
        return fail(BF_ERR_SHAPE, "log2leaf=%d must satisfy 3 <= l0 <= 7 and 2 l0 <= log2n=%d", l0, LN);
    if (!bfk::rank_supported(r)) return fail(BF_ERR_NOT_SUPPORTED, "rank=%d not in {6,8,10,12,14,16}", r);
    if (r > (1 << l0)) return fail(BF_ERR_SHAPE, "rank=%d exceeds the leaf size %d", r, 1 << l0);
    if (!(d->n_amp == 1 || d->n_amp == 2 || d->n_amp == 4))
        return fail(BF_ERR_NOT_SUPPORTED, "n_amp=%d not in {1,2,4}", d->n_amp);
    return BF_OK;
}

// index sharding over world = 2^g ranks: the first half on a shard is the butterfly of size 2^(LN-g), the
// exchange needs >= 4 b's per source block at level h (h - g >= 2: a band group of 4 pairs never straddles
// two sources), and every shard holds whole leaves on both sides (LN - g >= 2 l0).
bf_status_t validate_sharding(const bf_desc_t* d, int world, int rank)
{
    if (world < 1 || (world & (world - 1))) return fail(BF_ERR_INVALID_ARG, "world=%d is not a power of two", world);
    if (rank < 0 || rank >= world) return fail(BF_ERR_INVALID_ARG, "rank=%d not in [0,%d)", rank, world);
    int g = 0;
    while ((1 << g) < world) g++;
    const int h = d->log2n / 2;
    if (g > 0 && (h - g < 2 || d->log2n - g < 2 * d->log2leaf))
        return fail(BF_ERR_SHAPE, "world=%d too large for log2n=%d, log2leaf=%d", world, d->log2n, d->log2leaf);
    return BF_OK;
}

void drop_graph(bf_plan_s* p)
{
    if (p->gexec) {
        DeviceGuard g(p->device);
        if (p->done) cudaEventSynchronize(p->done);   // no replay may still be running
        cudaGraphExecDestroy(p->gexec);
    }
    p->gexec = nullptr;
    p->g_F = p->g_G = nullptr;
    p->g_nrhs = -1;
}

void free_plan(bf_plan_s* p)
{
    if (!p) return;
    DeviceGuard g(p->device);
    for (int i = 0; i < bfs::kMaxShards; i++)
        if (p->peer_ipc[i]) cudaIpcCloseMemHandle(p->peer_ws[i]);
    cudaFree(p->bar_buf);
    if (p->done) cudaEventSynchronize(p->done);
    for (auto& tl : p->pending) {
        cudaEventDestroy(tl.start);
        cudaEventDestroy(tl.stop);
    }
    for (auto e : p->pool) cudaEventDestroy(e);
    if (p->done) cudaEventDestroy(p->done);
    for (auto& s : p->sh) {
        cudaFree(s.amp_a);
        cudaFree(s.amp_b);
        cudaFree(s.v0);
        cudaFree(s.sw);
        cudaFree(s.v0x);
        cudaFree(s.ux);
        cudaFree(s.u);
        for (auto x : s.xfer) cudaFree(x);
        for (auto x : s.cmp) cudaFree(x);
        for (auto x : s.cmp3) cudaFree(x);
        cudaFree(s.ws);
        cudaFree(s.s0_lag);
        cudaFree(s.s0_ph);
        cudaFree(s.sl_lag);
        cudaFree(s.sl_ph);
        for (auto x : s.lag) cudaFree(x);
        for (auto x : s.ph) cudaFree(x);
    }
    cudaFree(p->dF);
    cudaFree(p->dG);
    for (int i = 0; i < 2; i++) {
        if (p->a_d2h[i]) cudaEventSynchronize(p->a_d2h[i]);
        cudaFree(p->aF[i]);
        cudaFree(p->aG[i]);
        for (cudaEvent_t ev : {p->a_h2d[i], p->a_applied[i], p->a_d2h[i]})
            if (ev) cudaEventDestroy(ev);
    }
    if (p->h2d) cudaStreamDestroy(p->h2d);
    if (p->d2h) cudaStreamDestroy(p->d2h);
    if (p->gexec) cudaGraphExecDestroy(p->gexec);
    if (p->cap) cudaStreamDestroy(p->cap);
    if (p->comm) nccl().CommDestroy(p->comm);
    delete p;
}

bf_status_t dalloc(float2** ptr, int64_t elems, const char* what)
{
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(ptr), size_t(elems) * sizeof(float2));
    if (e != cudaSuccess) {
        cudaGetLastError();
        *ptr = nullptr;
        return fail(BF_ERR_OOM, "cudaMalloc(%s, %lld B) failed: %s", what, (long long)(elems * 8),
                    cudaGetErrorString(e));
    }
    return BF_OK;
}

cudaEvent_t pool_get(bf_plan_s* p)
{
    if (!p->pool.empty()) {
        cudaEvent_t e = p->pool.back();
        p->pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// Launch with optional event bracketing.
template <class F>
cudaError_t timed(bf_plan_s* p, int cls, cudaStream_t s, F&& launch)
{
    if (!p->timing) return launch();
    TimedLaunch tl{cls, pool_get(p), pool_get(p)};
    cudaEventRecord(tl.start, s);
    cudaError_t e = launch();
    cudaEventRecord(tl.stop, s);
    p->pending.push_back(tl);
    return e;
}

// One kernel launch of the apply: what it runs and how it is accounted.
struct Step {
    enum Kind { S0, XFER, BAND, SL, EXCHANGE } kind;
    int l_first = 0;   // XFER: the level; BAND: first level (global level numbering)
    int K = 1;         // BAND: levels fused
    int cls = 0;       // bfk::KClass or KC_EXCHANGE
    int levels = 0;    // transfer levels this launch performs
};

// K = 3 where can3(l) (three-level tensor-core bands): 3s while they leave no lone level behind (8 levels:
// 3 + 3 + 2, 10: 3 + 3 + 2 + 2).
template <class Ok, class Ok3>
void push_levels(std::vector<Step>& st, const bfk::Dims& d, int lo, int hi, bool band, Ok&& pair_ok, Ok3&& can3)
{
    for (int l = lo; l <= hi;) {
        const int rem = hi - l + 1;
        int K = (band && l < hi && pair_ok(l)) ? 2 : 1;
        if (K == 2 && rem >= 3 && rem != 4 && can3(l)) K = 3;
        const int last = l + K - 1;
        const bool has_h = (l <= d.h && d.h <= last);
        const int cls = has_h ? bfk::KC_SWITCH : (last < d.h ? bfk::KC_XFER1 : bfk::KC_XFER2);
        st.push_back({band ? Step::BAND : Step::XFER, l, K, cls, K});
        l += K;
    }
}

// The launch sequence of one RHS chunk of nv vectors: S0, transfer levels l0+1..D (fused in bands of 2
// when the band kernel supports the shape, the switch applied inside the launch that produces level h),
// SL.  With no transfer level (h == l0) the switch runs alone after S0.  Sharded: the bands stop at h,
// the exchange follows, then the second half.
std::vector<Step> schedule(const bf_plan_s* p, int nv, bool plan3 = false)
{
    const bfk::Dims& d = p->d;
    const bool sharded = p->mode != BF_SHARD_NONE, small_batch = p->small_batch;
    std::vector<Step> st;
    st.push_back({Step::S0, 0, 1, bfk::KC_S0, 0});
    // structured plans without dense blocks: bands of the structured kernels (bf_struct.cu) for small batches
    const bool band = p->sh[0].dense_all()
                          ? (bfk::band_supported(d.R, nv) || (small_batch && bfk::band_sv_supported(d, nv)))
                          : (small_batch && bfk::band_st_supported(d, nv));
    // structured levels: only the kind pairs the structured band fuses
    const Shard& s0 = p->sh[0];
    auto kind_of = [&](int l) { return s0.xfer[l - d.l0 - 1] ? 0 : s0.kind[l - d.l0 - 1]; };
    auto pair_ok = [&](int l) { return s0.dense_all() || bfk::band_st_kinds(kind_of(l), kind_of(l + 1)); };
    // three-level bands: unsharded dense plans on the tensor cores whose operator was composed at finalization
    // (plan3: the schedule finalization builds those operators for)
    const bool use3 = !sharded && p->band3 && p->tensor_cores && s0.dense_all() && bfk::band3_supported(d, nv);
    auto can3 = [&](int l) { return use3 && (plan3 || s0.cmp3[l - d.l0 - 1] != nullptr); };
    if (!sharded) {
        push_levels(st, d, d.l0 + 1, d.D, band, pair_ok, can3);
    } else {
        push_levels(st, d, d.l0 + 1, d.h, band, pair_ok, can3);
        st.push_back({Step::EXCHANGE, 0, 1, KC_EXCHANGE, 0});
        push_levels(st, d, d.h + 1, d.D, band, pair_ok, can3);
    }
    st.push_back({Step::SL, 0, 1, bfk::KC_SL, 0});
    return st;
}

// Level-h exchange of one RHS chunk: block d (of G equal blocks) of every shard's send buffer goes to
// shard d's receive buffer at block q.  ws[i] is shard i's workspace base.
bf_status_t exchange(bf_plan_s* p, float2* const* ws, int send_buf, int nv, cudaStream_t s)
{
    const int G = p->world;
    const int64_t blk_pairs = p->nloc() / G;
    const int64_t bel = blk_pairs * p->d.R * nv;   // elements of one block
    const size_t blk_bytes = size_t(bel) * sizeof(float2);
    const int64_t arr = p->nloc() * p->d.R * nv;   // elements of one coefficient array of a shard
    if (p->mode == BF_SHARD_EMULATED) {
        for (int q = 0; q < G; q++)
            for (int dd = 0; dd < G; dd++) {
                cudaError_t e = cudaMemcpyAsync(ws[dd] + (1 - send_buf) * arr + q * bel, ws[q] + send_buf * arr + dd * bel,
                                                blk_bytes, cudaMemcpyDeviceToDevice, s);
                if (e != cudaSuccess) return cuda_fail(e, "exchange copy");
            }
        return BF_OK;
    }
    // NCCL: grouped send/recv with every peer (the last first-half launch wrote the blocks in destination order)
    const float2* sb = ws[0] + send_buf * arr;
    float2* rb = ws[0] + (1 - send_buf) * arr;
    cudaError_t e = cudaMemcpyAsync(rb + p->rank * bel, sb + p->rank * bel, blk_bytes, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e, "exchange self copy");
    if (G == 1) return BF_OK;
    Nccl& n = nccl();
    ncclResult_t r = n.GroupStart();
    if (r) return nccl_fail(r, "ncclGroupStart");
    for (int peer = 0; peer < G; peer++) {
        if (peer == p->rank) continue;
        if ((r = n.Send(sb + peer * bel, blk_bytes, kNcclUint8, peer, p->comm, s))) break;
        if ((r = n.Recv(rb + peer * bel, blk_bytes, kNcclUint8, peer, p->comm, s))) break;
    }
    ncclResult_t r2 = n.GroupEnd();
    if (r) return nccl_fail(r, "ncclSend/ncclRecv");
    if (r2) return nccl_fail(r2, "ncclGroupEnd");
    return BF_OK;
}

// Run steps [s_begin, s_end) of the schedule for one shard; `cur` is the coefficient buffer (0/1) holding
// the current level, updated in place.  remap_first: the first transfer launch reads the receive layout.
bf_status_t run_steps(bf_plan_s* p, Shard& sh, const std::vector<Step>& st, size_t s_begin, size_t s_end,
                      const float2* F, int64_t ldf, float2* G, int64_t ldg, int nv, int& cur, bool remap_first,
                      float2* ws, cudaStream_t s, const bfs::PeerOut* po = nullptr)
{
    const bfk::Dims dl = p->local();
    const int64_t arr = p->nloc() * p->d.R * nv;
    bool remap = remap_first;
    for (size_t k = s_begin; k < s_end; k++) {
        const Step& stp = st[k];
        float2* in = ws + cur * arr;
        float2* out = ws + (1 - cur) * arr;
        // kernel level: first half runs at the global level, second half at level - g (bf_shard.h)
        const int lk = (stp.l_first > p->d.h) ? stp.l_first - p->g : stp.l_first;
        const int rh = remap ? p->d.h : 0, rhg = remap ? p->d.h - p->g : 0;
        cudaError_t e = timed(p, stp.cls, s, [&]() -> cudaError_t {
            switch (stp.kind) {
            case Step::S0:
                if (p->tensor_cores && sh.v0x && bfk::s0_tc_supported(dl, nv, ldf))
                    return bfk::launch_s0_tc(dl, F, ldf, sh.amp_b, sh.v0x, in, nv, s, p->leaf_multicast);
                if (!sh.v0) return bfk::launch_s0_st(dl, F, ldf, sh.amp_b, sh.s0_lagh, sh.s0_ph, in, nv, s);
                if (p->small_batch && nv < 64 && bfk::s0_sv_supported(dl, nv))
                    return bfk::launch_s0_sv(dl, F, ldf, sh.amp_b, sh.v0, in, nv, s);
                return bfk::launch_s0(dl, F, ldf, sh.amp_b, sh.v0, in, nv, s);
            case Step::XFER: {
                const int li = stp.l_first - p->d.l0 - 1;
                if (!sh.xfer[li]) return bfk::launch_xfer_st(dl, lk, sh.kind[li], sh.lagh[li], sh.ph[li], in, out, nv, s);
                if (p->small_batch && bfk::band_sv_supported(dl, nv)) {   // a lone dense level (structured plans)
                    const float2* W1[2] = {sh.xfer[li], nullptr};
                    return bfk::launch_band_sv(dl, lk, 1, in, out, W1, nv, s, rh, rhg, po);
                }
                return bfk::launch_xfer(dl, lk, in, out, sh.xfer[li], nv, s, rh, rhg, po);
            }
            case Step::BAND: {
                const int li = stp.l_first - p->d.l0 - 1;
                if (!sh.dense_all()) {   // structured plan (bf_struct.cu)
                    if (stp.K == 1) {
                        if (sh.xfer[li]) {
                            const float2* W1[2] = {sh.xfer[li], nullptr};
                            return bfk::launch_band_sv(dl, lk, 1, in, out, W1, nv, s, rh, rhg, po);
                        }
                        return bfk::launch_xfer_st(dl, lk, sh.kind[li], sh.lagh[li], sh.ph[li], in, out, nv, s);
                    }
                    bfk::LagP L2{};
                    const int r2 = 2 * p->d.R * p->d.R;
                    for (int i = 0; i < r2; i++) {
                        L2.v[i] = sh.lagh[li].v[i];
                        L2.v[512 + i] = sh.lagh[li + 1].v[i];
                    }
                    const int k1 = sh.xfer[li] ? 0 : sh.kind[li], k2 = sh.xfer[li + 1] ? 0 : sh.kind[li + 1];
                    return bfk::launch_band_st(dl, lk, k1, k2, L2, sh.xfer[li] ? sh.xfer[li] : sh.ph[li],
                                               sh.xfer[li + 1] ? sh.xfer[li + 1] : sh.ph[li + 1], in, out, nv, s);
                }
                if (stp.K == 3) return bfk::launch_band3(dl, lk, in, out, sh.cmp3[li], nv, s);
                const float2* W[2] = {sh.xfer[li], stp.K > 1 ? sh.xfer[li + 1] : nullptr};
                if (stp.K == 2 && p->tensor_cores && bfk::band_tc_supported(dl, nv))
                    return bfk::launch_band_tc(dl, lk, in, out, W, nv, s, rh, rhg, po, p->band,
                                               p->precompose ? sh.cmp[stp.l_first - p->d.l0 - 1] : nullptr);
                if (p->small_batch && bfk::band_sv_supported(dl, nv))
                    return bfk::launch_band_sv(dl, lk, stp.K, in, out, W, nv, s, rh, rhg, po);
                return bfk::launch_band(dl, lk, stp.K, in, out, W, nv, s, rh, rhg, po);
            }
            case Step::SL:
                if (p->tensor_cores && sh.ux && bfk::sl_tc_supported(dl, nv))
                    return bfk::launch_sl_tc(dl, in, sh.ux, sh.amp_a, G, ldg, nv, s, p->leaf_multicast);
                if (!sh.u) return bfk::launch_sl_st(dl, in, sh.sl_lag, sh.sl_ph, sh.amp_a, G, ldg, nv, s);
                if (p->small_batch && bfk::sl_sv_supported(dl, nv))
                    return bfk::launch_sl_sv(dl, in, sh.u, sh.amp_a, G, ldg, nv, s);
                return bfk::launch_sl(dl, in, sh.u, sh.amp_a, G, ldg, nv, s);
            default: return cudaErrorInvalidValue;
            }
        });
        if (e != cudaSuccess) {
            static const char* kinds[] = {"S0", "transfer", "band", "SL", "exchange"};
            char what[96];
            snprintf(what, sizeof what, "kernel launch (%s, level %d, K %d, nv %d)", kinds[stp.kind], stp.l_first, stp.K,
                     nv);
            return cuda_fail(e, what);
        }
        if (stp.kind == Step::XFER || stp.kind == Step::BAND) {
            cur = 1 - cur;
            remap = false;
        }
    }
    return BF_OK;
}

// Stream-ordered barrier over the NCCL ranks: every rank sends one byte to and receives one byte from
// every peer; the group completes on a rank's stream only after every peer has reached the same point.
bf_status_t nccl_barrier(bf_plan_s* p, cudaStream_t s)
{
    if (p->mode != BF_SHARD_NCCL || p->world == 1) return BF_OK;
    Nccl& n = nccl();
    ncclResult_t r = n.GroupStart();
    if (r) return nccl_fail(r, "ncclGroupStart");
    for (int peer = 0; peer < p->world; peer++) {
        if (peer == p->rank) continue;
        if ((r = n.Send(p->bar_buf + p->rank, 1, kNcclUint8, peer, p->comm, s))) break;
        if ((r = n.Recv(p->bar_buf + p->world + peer, 1, kNcclUint8, peer, p->comm, s))) break;
    }
    ncclResult_t r2 = n.GroupEnd();
    if (r) return nccl_fail(r, "barrier send/recv");
    if (r2) return nccl_fail(r2, "barrier ncclGroupEnd");
    return BF_OK;
}

// One RHS chunk of a sharded plan with the fused exchange: (A) every shard runs its first half up to the
// launch that produces level h; (B) that launch stores its output pairs straight into the destination
// shards' receive arrays (peer memory over NVLink for one shard per GPU); (C) the second halves read their
// receive arrays in place.  NCCL plans order A/B/C across the ranks with stream-ordered barriers (B writes
// into arrays the peers' last phase-A launch reads; C reads what every peer's B wrote).
bf_status_t apply_chunk_peer(bf_plan_s* p, const std::vector<Step>& st, size_t ex, const std::vector<float2*>& ws,
                             const float2* Fc, int64_t ldf, float2* Gc, int64_t ldg, int nv, cudaStream_t s)
{
    const int nsh = int(p->sh.size());
    const int64_t arr = p->nloc() * p->d.R * nv;
    std::vector<int> cur(nsh, 0);
    for (int i = 0; i < nsh; i++) {   // (A)
        const int64_t off = (p->mode == BF_SHARD_EMULATED) ? int64_t(i) * p->nloc() : 0;
        bf_status_t r = run_steps(p, p->sh[i], st, 0, ex - 1, Fc + off, ldf, nullptr, ldg, nv, cur[i], false, ws[i], s);
        if (r != BF_OK) return r;
    }
    bf_status_t r = nccl_barrier(p, s);
    if (r != BF_OK) return r;
    const int c = cur[0];   // every shard runs the same schedule: the same array parity
    int lb = 0;
    while ((int64_t(1) << lb) < p->nloc() / p->world) lb++;
    for (int i = 0; i < nsh; i++) {   // (B)
        bfs::PeerOut po{};
        po.on = 1;
        po.lb = lb;
        po.src = (p->mode == BF_SHARD_EMULATED) ? i : p->rank;
        for (int d = 0; d < p->world; d++) po.dst[d] = p->peer_ws[d] + (1 - c) * arr;
        int ci = cur[i];
        if ((r = run_steps(p, p->sh[i], st, ex - 1, ex, nullptr, ldf, nullptr, ldg, nv, ci, false, ws[i], s, &po)) !=
            BF_OK)
            return r;
        cur[i] = ci;
    }
    if ((r = nccl_barrier(p, s)) != BF_OK) return r;
    for (int i = 0; i < nsh; i++) {   // (C)
        const int64_t off = (p->mode == BF_SHARD_EMULATED) ? int64_t(i) * p->nloc() : 0;
        int ci = cur[i];   // the receive array is the level-h output array of this shard
        if ((r = run_steps(p, p->sh[i], st, ex + 1, st.size(), nullptr, ldf, Gc + off, ldg, nv, ci, true, ws[i], s)) !=
            BF_OK)
            return r;
    }
    return BF_OK;
}

// NCCL plans: an asynchronous communicator error (a peer died, a network fault) is reported instead of
// enqueueing more collectives on a broken communicator.
bf_status_t nccl_check(bf_plan_s* p)
{
    if (p->mode != BF_SHARD_NCCL || !p->comm) return BF_OK;
    ncclResult_t r = 0;
    const ncclResult_t q = nccl().CommGetAsyncError(p->comm, &r);
    if (q) return nccl_fail(q, "ncclCommGetAsyncError");
    if (r) return nccl_fail(r, "NCCL asynchronous error");
    return BF_OK;
}

// Wait for `ev` (work enqueued on the plan's stream).  For NCCL plans the wait polls the communicator: an
// asynchronous error or no progress within nccl_timeout_s() aborts it (the peers' collectives then fail
// instead of hanging) and returns BF_ERR_NCCL.
bf_status_t wait_event_nccl(bf_plan_s* p, cudaEvent_t ev)
{
    if (p->mode != BF_SHARD_NCCL || !p->comm || p->world == 1) {
        const cudaError_t e = cudaEventSynchronize(ev);
        return e == cudaSuccess ? BF_OK : cuda_fail(e, "synchronize");
    }
    struct timespec ts0;
    clock_gettime(CLOCK_MONOTONIC, &ts0);
    for (;;) {
        const cudaError_t e = cudaEventQuery(ev);
        if (e == cudaSuccess) return BF_OK;
        if (e != cudaErrorNotReady) return cuda_fail(e, "synchronize");
        bf_status_t st = nccl_check(p);
        struct timespec ts;
        clock_gettime(CLOCK_MONOTONIC, &ts);
        const double dt = double(ts.tv_sec - ts0.tv_sec) + 1e-9 * double(ts.tv_nsec - ts0.tv_nsec);
        if (st == BF_OK && dt > nccl_timeout_s())
            st = fail(BF_ERR_NCCL, "NCCL exchange made no progress for %.0f s (BF_NCCL_TIMEOUT_S)", dt);
        if (st != BF_OK) {
            nccl().CommAbort(p->comm);
            p->comm = nullptr;
            return st;
        }
        struct timespec nap = {0, 100000};
        nanosleep(&nap, nullptr);
    }
}

bf_status_t apply_impl(bf_plan_s* p, const float2* F, int64_t ldf, float2* G, int64_t ldg, int64_t nrhs, float2* ws0,
                       cudaStream_t s)
{
    const int64_t chunk = p->max_chunk;
    const bool sharded = p->mode != BF_SHARD_NONE;
    if (bf_status_t st = nccl_check(p); st != BF_OK) return st;
    const int nsh = int(p->sh.size());
    std::vector<float2*> ws(nsh);
    for (int i = 0; i < nsh; i++) ws[i] = (i == 0) ? ws0 : p->sh[i].ws;
    for (int64_t c0 = 0; c0 < nrhs; c0 += chunk) {
        const int64_t nc = std::min(chunk, nrhs - c0);
        const int nv = int(nc * p->d.n_amp);
        const auto st = schedule(p, nv);
        const float2* Fc = F + c0 * ldf;
        float2* Gc = G + c0 * ldg;
        if (!sharded) {
            int cur = 0;
            bf_status_t r = run_steps(p, p->sh[0], st, 0, st.size(), Fc, ldf, Gc, ldg, nv, cur, false, ws[0], s);
            if (r != BF_OK) return r;
            continue;
        }
        size_t ex = 0;
        while (st[ex].kind != Step::EXCHANGE) ex++;
        if (p->exchange_peer && ws0 == p->sh[0].ws && ex >= 2 && st[ex - 1].kind != Step::S0) {
            bf_status_t r = apply_chunk_peer(p, st, ex, ws, Fc, ldf, Gc, ldg, nv, s);
            if (r != BF_OK) return r;
            continue;
        }
        // rows of shard i: emulated plans take the full F/G (shard i at row offset i N/G), NCCL plans the
        // local rows
        int cur = 0;
        for (int i = 0; i < nsh; i++) {
            const int64_t off = (p->mode == BF_SHARD_EMULATED) ? int64_t(i) * p->nloc() : 0;
            cur = 0;
            bf_status_t r = run_steps(p, p->sh[i], st, 0, ex, Fc + off, ldf, nullptr, ldg, nv, cur, false, ws[i], s);
            if (r != BF_OK) return r;
        }
        bf_status_t xr = BF_OK;
        cudaError_t e = timed(p, KC_EXCHANGE, s, [&]() -> cudaError_t {
            xr = exchange(p, ws.data(), cur, nv, s);
            return cudaSuccess;
        });
        if (xr != BF_OK) return xr;
        if (e != cudaSuccess) return cuda_fail(e, "exchange");
        for (int i = 0; i < nsh; i++) {
            const int64_t off = (p->mode == BF_SHARD_EMULATED) ? int64_t(i) * p->nloc() : 0;
            int c = 1 - cur;   // the exchange wrote the other buffer
            bf_status_t r = run_steps(p, p->sh[i], st, ex + 1, st.size(), nullptr, ldf, Gc + off, ldg, nv, c, true,
                                      ws[i], s);
            if (r != BF_OK) return r;
        }
    }
    // completion marker for bf_plan_destroy; not recorded while the stream is being captured into a CUDA
    // graph (the replays are the caller's to synchronize before destroying the plan)
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cap) == cudaSuccess && cap == cudaStreamCaptureStatusNone)
        cudaEventRecord(p->done, s);
    return BF_OK;
}

bf_status_t alloc_plan(const bf_desc_t* meta, int device, int64_t max_nrhs_chunk, int world, int rank, int mode,
                       bf_plan_t* out, bool dense_factors = true)
{
    if (!out) return fail(BF_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    bf_status_t st = validate_shape(meta);
    if (st != BF_OK) return st;
    if ((st = validate_sharding(meta, world, rank)) != BF_OK) return st;
    if (max_nrhs_chunk < 1) return fail(BF_ERR_INVALID_ARG, "max_nrhs_chunk=%lld < 1", (long long)max_nrhs_chunk);
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
    if (device < 0 || device >= ndev) return fail(BF_ERR_INVALID_ARG, "device %d not in [0,%d)", device, ndev);
    DeviceGuard dg(device);

    auto* p = new bf_plan_s();
    p->device = device;
    p->d.LN = meta->log2n;
    p->d.l0 = meta->log2leaf;
    p->d.R = meta->rank;
    p->d.n_amp = meta->n_amp;
    p->d.N = int64_t(1) << p->d.LN;
    p->d.h = p->d.LN / 2;
    p->d.D = p->d.LN - p->d.l0;
    p->max_chunk = max_nrhs_chunk;
    p->world = world;
    p->rank = rank;
    while ((1 << p->g) < world) p->g++;
    p->mode = mode;
    const int nsh = (mode == BF_SHARD_EMULATED) ? world : 1;
    p->sh.resize(nsh);
    const int nx = p->d.D - p->d.l0;
    p->uploaded.assign(nsh, std::vector<std::vector<std::pair<int64_t, int64_t>>>(5 + nx));
    const int64_t n = p->nloc(), r = p->d.R, n0 = int64_t(1) << p->d.l0;
    const int64_t nv = max_nrhs_chunk * p->d.n_amp;
    p->ws_bytes = size_t(2) * size_t(n * r) * size_t(nv) * sizeof(float2);
    for (auto& s : p->sh) {
        s.xfer.assign(nx, nullptr);
        s.cmp.assign(nx, nullptr);
        s.cmp3.assign(nx, nullptr);
        s.kind.assign(nx, BF_LEVEL_DENSE);
        s.lag.assign(nx, nullptr);
        s.lagh.assign(nx, bfk::LagP{});
        s.ph.assign(nx, nullptr);
        if ((st = dalloc(&s.amp_a, p->d.n_amp * n, "amp_a")) || (st = dalloc(&s.amp_b, p->d.n_amp * n, "amp_b")) ||
            (st = dalloc(&s.ws, int64_t(p->ws_bytes / sizeof(float2)), "workspace"))) {
            free_plan(p);
            return st;
        }
        if (!dense_factors) continue;   // structured plans allocate per stage (bf_plan_create_structured)
        if ((st = dalloc(&s.v0, n * r * n0, "v0")) || (st = dalloc(&s.sw, n * r * r, "sw")) ||
            (st = dalloc(&s.u, n * r * n0, "u"))) {
            free_plan(p);
            return st;
        }
        for (int i = 0; i < nx; i++)
            if ((st = dalloc(&s.xfer[i], n * 2 * r * r, "xfer"))) {
                free_plan(p);
                return st;
            }
    }
    if ((e = cudaEventCreateWithFlags(&p->done, cudaEventDisableTiming)) != cudaSuccess) {
        free_plan(p);
        return cuda_fail(e, "cudaEventCreate");
    }
    *out = p;
    return BF_OK;
}

bf_status_t upload_desc(const bf_desc_t* desc, bf_plan_t p);

}  // namespace

// ---------------------------------------------------------------------------
// internal helpers for the streaming builder (bf_build.cpp)
// ---------------------------------------------------------------------------
bf_status_t bfp_stage_dst(bf_plan_t p, int shard, int32_t stage, int64_t begin, int64_t count, void** dst)
{
    if (!p || !dst) return fail(BF_ERR_INVALID_ARG, "NULL argument");
    if (p->finalized) return fail(BF_ERR_STATE, "plan already finalized");
    if (shard < 0 || shard >= int(p->sh.size())) return fail(BF_ERR_INVALID_ARG, "bad shard %d", shard);
    const int slot = slot_of(p, stage);
    if (slot < 0) return fail(BF_ERR_INVALID_ARG, "bad stage id %d", stage);
    if (begin < 0 || count < 0 || begin + count > stage_blocks(p, stage))
        return fail(BF_ERR_INVALID_ARG, "block range [%lld,%lld) out of [0,%lld)", (long long)begin,
                    (long long)(begin + count), (long long)stage_blocks(p, stage));
    *dst = stage_base(p->sh[shard], stage) + begin * stage_elems(p, stage);
    if (count > 0) p->uploaded[shard][slot].push_back({begin, begin + count});
    return BF_OK;
}

int bfp_device(bf_plan_t p) { return p ? p->device : -1; }
int bfp_num_shards(bf_plan_t p) { return p ? int(p->sh.size()) : 0; }
int bfp_rank(bf_plan_t p) { return p ? p->rank : 0; }

bf_status_t bfp_fail(bf_status_t s, const char* msg) { return fail(s, "%s", msg); }

bf_status_t bfp_plan_alloc_sharded(const bf_desc_t* meta, int device, int64_t max_nrhs_chunk, int world, int rank,
                                   int mode, const void* nccl_id, bf_plan_t* out)
{
    bf_status_t st = alloc_plan(meta, device, max_nrhs_chunk, world, rank, mode, out);
    if (st != BF_OK || mode != BF_SHARD_NCCL) return st;
    Nccl& n = nccl();
    if (!n.ok || !nccl_id) {
        free_plan(*out);
        *out = nullptr;
        return n.ok ? fail(BF_ERR_INVALID_ARG, "nccl_unique_id is NULL")
                    : fail(BF_ERR_NCCL, "NCCL library not found (set BF_NCCL_LIB)");
    }
    DeviceGuard dg(device);
    ncclUniqueId id;
    memcpy(&id, nccl_id, sizeof id);
    ncclResult_t r = n.CommInitRank(&(*out)->comm, world, id, rank);
    if (r) {
        (*out)->comm = nullptr;
        free_plan(*out);
        *out = nullptr;
        return nccl_fail(r, "ncclCommInitRank");
    }
    return BF_OK;
}

void bfp_plan_free(bf_plan_t p) { free_plan(p); }

// ---------------------------------------------------------------------------
// ABI
// ---------------------------------------------------------------------------
extern "C" {

int32_t bf_abi_version(void) { return BF_ABI_VERSION; }

const char* bf_last_error(void) { return g_err.c_str(); }

bf_status_t bf_nccl_get_unique_id(void* id128)
{
    if (!id128) return fail(BF_ERR_INVALID_ARG, "id is NULL");
    Nccl& n = nccl();
    if (!n.ok) return fail(BF_ERR_NCCL, "NCCL library not found (set BF_NCCL_LIB)");
    ncclUniqueId id;
    ncclResult_t r = n.GetUniqueId(&id);
    if (r) return nccl_fail(r, "ncclGetUniqueId");
    memcpy(id128, &id, sizeof id);
    return BF_OK;
}

bf_status_t bf_plan_alloc(const bf_desc_t* meta, int device, int64_t max_nrhs_chunk, bf_plan_t* out)
{
    return alloc_plan(meta, device, max_nrhs_chunk, 1, 0, BF_SHARD_NONE, out);
}

bf_status_t bf_plan_alloc_sharded(const bf_desc_t* meta, int device, int64_t max_nrhs_chunk, int32_t rank,
                                  int32_t world, const void* nccl_unique_id, bf_plan_t* out)
{
    return bfp_plan_alloc_sharded(meta, device, max_nrhs_chunk, world, rank, BF_SHARD_NCCL, nccl_unique_id, out);
}

bf_status_t bf_plan_upload(bf_plan_t p, int32_t stage, int64_t block_begin, int64_t block_count, const bf_c64* src,
                           int32_t src_memory)
{
    if (!p || (!src && block_count > 0)) return fail(BF_ERR_INVALID_ARG, "NULL argument");
    if (src_memory != BF_MEM_HOST && src_memory != BF_MEM_DEVICE)
        return fail(BF_ERR_INVALID_ARG, "src_memory=%d", src_memory);
    if (p->sh.size() != 1) return fail(BF_ERR_STATE, "emulated plans are built by bf_plan_build_fio_emulated");
    DeviceGuard g(p->device);
    void* dst = nullptr;
    bf_status_t st = bfp_stage_dst(p, 0, stage, block_begin, block_count, &dst);
    if (st != BF_OK) return st;
    const size_t bytes = size_t(block_count) * size_t(stage_elems(p, stage)) * sizeof(float2);
    cudaError_t e = cudaMemcpy(dst, src, bytes,
                               src_memory == BF_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(upload)");
    return BF_OK;
}

namespace {
// The tensor-core leaf images (s0_tc_kernel, sl_tc_kernel): TF32 hi/lo tiles, real-embedded.  Without memory
// for an image the SIMT kernel serves that stage.
bf_status_t build_leaf_images(bf_plan_s* p, Shard& s)
{
    const bfk::Dims dl = p->local();
    auto alloc = [](float** x, size_t bytes) {
        if (cudaMalloc(x, bytes) == cudaSuccess) return true;
        cudaGetLastError();
        *x = nullptr;
        return false;
    };
    cudaError_t e = cudaSuccess;
    if (!s.v0x && alloc(&s.v0x, size_t(bfk::v0x_floats(dl)) * sizeof(float))) e = bfk::expand_leaf_weights(dl, s.v0, s.u, s.v0x, nullptr, 0);
    if (e == cudaSuccess && !s.ux && alloc(&s.ux, size_t(bfk::ux_floats(dl)) * sizeof(float)))
        e = bfk::expand_leaf_weights(dl, s.v0, s.u, nullptr, s.ux, 0);
    return e == cudaSuccess ? BF_OK : cuda_fail(e, "leaf weight images");
}
}  // namespace

}  // extern "C"

namespace {
// Dense blocks from a structured plan's stages (bf_struct.cu expand_st_kernel), structured arrays released.
bf_status_t expand_structured(bf_plan_s* p)
{
    const bfk::Dims d = p->local();
    const int64_t n = p->nloc(), r = d.R, n0 = int64_t(1) << d.l0;
    Shard& s = p->sh[0];
    bf_status_t st = BF_OK;
    cudaError_t e = cudaSuccess;
    if (!s.v0) {
        if ((st = dalloc(&s.v0, n * r * n0, "v0 (expanded)")) != BF_OK) return st;
        e = bfk::launch_expand_st(d, 0, 0, s.s0_lag, s.s0_ph, s.v0, 0);
    }
    for (size_t i = 0; i < s.xfer.size() && e == cudaSuccess; i++) {
        if (s.xfer[i]) continue;
        if ((st = dalloc(&s.xfer[i], n * 2 * r * r, "xfer (expanded)")) != BF_OK) return st;
        e = bfk::launch_expand_st(d, s.kind[i], d.l0 + 1 + int(i), s.lag[i], s.ph[i], s.xfer[i], 0);
    }
    if (e == cudaSuccess && !s.u) {
        if ((st = dalloc(&s.u, n * r * n0, "u (expanded)")) != BF_OK) return st;
        e = bfk::launch_expand_st(d, 4, 0, s.sl_lag, s.sl_ph, s.u, 0);
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(e, "structured factor expansion");
    for (float** x : {&s.s0_lag, &s.sl_lag}) {
        cudaFree(*x);
        *x = nullptr;
    }
    for (float2** x : {&s.s0_ph, &s.sl_ph}) {
        cudaFree(*x);
        *x = nullptr;
    }
    for (size_t i = 0; i < s.xfer.size(); i++) {
        cudaFree(s.lag[i]);
        cudaFree(s.ph[i]);
        s.lag[i] = nullptr;
        s.ph[i] = nullptr;
        s.kind[i] = BF_LEVEL_DENSE;
    }
    return BF_OK;
}

// copy `bytes` from host or device memory (UVA) into a new device array
bf_status_t dcopy_v(void** dst, const void* src, size_t bytes, const char* what)
{
    if (!src) return fail(BF_ERR_INVALID_ARG, "structured descriptor: %s is NULL", what);
    cudaError_t e = cudaMalloc(dst, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *dst = nullptr;
        return fail(BF_ERR_OOM, "cudaMalloc(%s, %zu B) failed", what, bytes);
    }
    e = cudaMemcpy(*dst, src, bytes, cudaMemcpyDefault);
    return e == cudaSuccess ? BF_OK : cuda_fail(e, what);
}
bf_status_t dcopy(float** dst, const void* src, size_t bytes, const char* what)
{
    return dcopy_v(reinterpret_cast<void**>(dst), src, bytes, what);
}
bf_status_t dcopy(float2** dst, const void* src, size_t bytes, const char* what)
{
    return dcopy_v(reinterpret_cast<void**>(dst), src, bytes, what);
}
}  // namespace

extern "C" {

bf_status_t bf_plan_create_structured(const bf_sdesc_t* sd, int device, int64_t max_nrhs_chunk, bf_plan_t* out)
{
    if (!out) return fail(BF_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (!sd) return fail(BF_ERR_INVALID_ARG, "descriptor is NULL");
    bf_desc_t meta{};
    meta.abi_version = sd->abi_version;
    meta.log2n = sd->log2n;
    meta.log2leaf = sd->log2leaf;
    meta.rank = sd->rank;
    meta.n_amp = sd->n_amp;
    meta.memory = sd->memory;
    if (sd->memory != BF_MEM_HOST && sd->memory != BF_MEM_DEVICE) return fail(BF_ERR_INVALID_ARG, "memory=%d", sd->memory);
    if (sd->s0_kind != BF_LEVEL_FIRST && sd->s0_kind != BF_LEVEL_DENSE)
        return fail(BF_ERR_INVALID_ARG, "s0_kind=%d", sd->s0_kind);
    if (sd->log2leaf > 6 || sd->rank > 16)
        return fail(BF_ERR_NOT_SUPPORTED, "structured plans: leaf <= 64 and rank <= 16");
    bf_plan_t p = nullptr;
    bf_status_t st = alloc_plan(&meta, device, max_nrhs_chunk, 1, 0, BF_SHARD_NONE, &p, false);
    if (st != BF_OK) return st;
    DeviceGuard g(device);
    p->structured = true;
    p->switch_in_factors = true;
    Shard& s = p->sh[0];
    const int64_t N = p->d.N, r = p->d.R, n0 = int64_t(1) << p->d.l0, c8 = sizeof(float2);
    const int nx = int(s.xfer.size());
    auto done = [&](bf_status_t r2) {
        if (r2 != BF_OK) free_plan(p);
        return r2;
    };
    if (!sd->amp_a || !sd->amp_b || (nx > 0 && !sd->xfer)) return done(fail(BF_ERR_INVALID_ARG, "structured descriptor: NULL array"));
    cudaError_t e = cudaMemcpy(s.amp_a, sd->amp_a, size_t(p->d.n_amp * N * c8), cudaMemcpyDefault);
    if (e == cudaSuccess) e = cudaMemcpy(s.amp_b, sd->amp_b, size_t(p->d.n_amp * N * c8), cudaMemcpyDefault);
    if (e != cudaSuccess) return done(cuda_fail(e, "amplitudes"));
    if (sd->s0_kind == BF_LEVEL_DENSE) {
        if ((st = dcopy(&s.v0, sd->s0_data, size_t(N * r * n0 * c8), "s0_data (dense)")) != BF_OK) return done(st);
    } else if ((st = dcopy(&s.s0_lag, sd->s0_lag, size_t(r * n0 * 4), "s0_lag")) != BF_OK ||
               (st = dcopy(&s.s0_ph, sd->s0_data, size_t(N * n0 * c8), "s0_data")) != BF_OK) {
        return done(st);
    } else if ((e = cudaMemcpy(s.s0_lagh.v, s.s0_lag, size_t(r * n0 * 4), cudaMemcpyDeviceToHost)) != cudaSuccess) {
        return done(cuda_fail(e, "s0_lag"));
    }
    for (int i = 0; i < nx; i++) {
        const bf_slevel_t& lv = sd->xfer[i];
        if (lv.kind == BF_LEVEL_DENSE) {
            if ((st = dcopy(&s.xfer[i], lv.data, size_t(N * 2 * r * r * c8), "xfer data (dense)")) != BF_OK) return done(st);
        } else if (lv.kind == BF_LEVEL_FIRST || lv.kind == BF_LEVEL_SECOND || lv.kind == BF_LEVEL_FIRST_SWITCH) {
            s.kind[i] = lv.kind;
            const int64_t per = lv.kind == BF_LEVEL_FIRST_SWITCH ? 2 * r + r * r : 2 * r;
            if ((st = dcopy(&s.lag[i], lv.lag, size_t(2 * r * r * 4), "xfer lag")) != BF_OK ||
                (st = dcopy(&s.ph[i], lv.data, size_t(N * per * c8), "xfer data")) != BF_OK)
                return done(st);
            if ((e = cudaMemcpy(s.lagh[i].v, s.lag[i], size_t(2 * r * r * 4), cudaMemcpyDeviceToHost)) != cudaSuccess)
                return done(cuda_fail(e, "xfer lag"));
        } else {
            return done(fail(BF_ERR_INVALID_ARG, "xfer[%d].kind=%d", i, lv.kind));
        }
    }
    if ((st = dcopy(&s.sl_lag, sd->sl_lag, size_t(n0 * r * 4), "sl_lag")) != BF_OK ||
        (st = dcopy(&s.sl_ph, sd->sl_phase, size_t(N * n0 * c8), "sl_phase")) != BF_OK)
        return done(st);
    if ((st = bf_plan_finalize(p)) != BF_OK) return done(st);
    *out = p;
    return BF_OK;
}

bf_status_t bf_plan_finalize(bf_plan_t p)
{
    if (!p) return fail(BF_ERR_INVALID_ARG, "plan is NULL");
    if (p->finalized) return fail(BF_ERR_STATE, "plan already finalized");
    const int nx = int(p->sh[0].xfer.size());
    for (size_t i = 0; i < p->sh.size() && !p->structured; i++)
        for (int slot = 0; slot < 5 + nx; slot++) {
            const int stage = slot < 5 ? slot : BF_STAGE_XFER0 + (slot - 5);
            // union of the uploaded ranges: the first block not covered (overlapping or repeated uploads of
            // one range do not count twice)
            auto rs = p->uploaded[i][slot];
            std::sort(rs.begin(), rs.end());
            int64_t covered = 0;
            for (const auto& r : rs) {
                if (r.first > covered) break;
                covered = std::max(covered, r.second);
            }
            if (covered < stage_blocks(p, stage))
                return fail(BF_ERR_STATE, "shard %zu stage %d: block %lld of %lld not uploaded", i, stage,
                            (long long)covered, (long long)stage_blocks(p, stage));
        }
    DeviceGuard g(p->device);
    // fold the switch into the factor that produces level h: XFER_h, or V0 when h == l0 (no transfer level
    // precedes h); the apply then has no separate switch product
    for (Shard& s : p->sh) {
        if (p->switch_in_factors) break;
        const int n0 = 1 << p->d.l0;
        float2* target = (p->d.h > p->d.l0) ? s.xfer[p->d.h - p->d.l0 - 1] : s.v0;
        const int cols = (p->d.h > p->d.l0) ? 2 * p->d.R : n0;
        cudaError_t e = bfk::launch_fold_switch(s.sw, target, p->nloc(), p->d.R, cols, 0);
        if (e != cudaSuccess) return cuda_fail(e, "switch fold");
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(e, "finalize");
    for (Shard& s : p->sh) {   // the switch blocks now live inside the level-h factor
        cudaFree(s.sw);
        s.sw = nullptr;
    }
    // structured plans whose chunks run on the tensor cores: those kernels take dense blocks -- expand every
    // structured stage once (the structured arrays are then released; the plan behaves as a dense one)
    const bfk::Dims dl0 = p->local();
    if (p->structured && p->tensor_cores && bfk::leaf_tc_shape(dl0) && p->max_chunk * p->d.n_amp >= 64) {
        if (bf_status_t st = expand_structured(p); st != BF_OK) return st;
    }
    // tensor-core leaf weights: only when a chunk can be a dense contraction (nv >= 64 vectors)
    const bfk::Dims dl = p->local();
    if (p->tensor_cores && bfk::leaf_tc_shape(dl) && p->max_chunk * p->d.n_amp >= 64) {
        for (Shard& s : p->sh)
            if (bf_status_t st = build_leaf_images(p, s); st != BF_OK) return st;
        e = cudaDeviceSynchronize();
        if (e != cudaSuccess) return cuda_fail(e, "leaf weight expansion");
    }
    // three-level tensor-core bands (bf_band3.cu): compose each band's 8 x 8 block operator per group of 8 pairs
    // once (FP64 products).  Without the memory for one, that band's levels fall back to two-level bands.
    {
        const int nvf = int(p->max_chunk * p->d.n_amp);
        for (const auto& stp : schedule(p, nvf, true)) {
            if (stp.kind != Step::BAND || stp.K != 3) continue;
            const int li = stp.l_first - p->d.l0 - 1;
            for (Shard& s : p->sh) {
                if (s.cmp3[li]) continue;
                if (cudaMalloc(&s.cmp3[li], size_t(bfk::band3_operator_elems(dl)) * sizeof(float2)) != cudaSuccess) {
                    cudaGetLastError();
                    s.cmp3[li] = nullptr;
                    continue;
                }
                e = bfk::launch_compose3(dl, stp.l_first, s.xfer[li], s.xfer[li + 1], s.xfer[li + 2], s.cmp3[li], 0);
                if (e != cudaSuccess) return cuda_fail(e, "band3 precompose");
            }
        }
        e = cudaDeviceSynchronize();
        if (e != cudaSuccess) return cuda_fail(e, "band3 precompose");
        // a band whose operator is missing would break the 3-level grouping of the ones after it: keep all or none
        bool all = true;
        for (const auto& stp : schedule(p, nvf, true))
            if (stp.kind == Step::BAND && stp.K == 3)
                for (Shard& s : p->sh) all = all && s.cmp3[stp.l_first - p->d.l0 - 1] != nullptr;
        if (!all)
            for (Shard& s : p->sh)
                for (auto& x : s.cmp3) {
                    cudaFree(x);
                    x = nullptr;
                }
    }
    // small vector batches (<= 2 tiles of 128 vectors per chunk): precompose every tensor-core band's two-level
    // operator once (FP64 products), so the band kernel only embeds and splits it per group instead of
    // composing it on chip -- with one vector tile per group the on-chip compose was the band's critical path
    // (ncu: weight warps' compose loop; 0.41 of HBM at nv = 64).  Same bytes per group as the compact blocks.
    {
        const int nvf = int(p->max_chunk * p->d.n_amp);
        if (p->tensor_cores && nvf <= 256 && bfk::band_tc_supported(dl, nvf)) {
            for (const auto& stp : schedule(p, nvf)) {
                if (stp.kind != Step::BAND || stp.K != 2) continue;
                const int li = stp.l_first - p->d.l0 - 1;
                const int lk = (stp.l_first > p->d.h) ? stp.l_first - p->g : stp.l_first;
                for (Shard& s : p->sh) {
                    if (s.cmp[li]) continue;
                    if (cudaMalloc(&s.cmp[li], size_t(p->nloc()) * 4 * p->d.R * p->d.R * sizeof(float2)) != cudaSuccess) {
                        cudaGetLastError();   // no memory: that band composes on chip
                        s.cmp[li] = nullptr;
                        continue;
                    }
                    e = bfk::launch_compose_band(dl, lk, s.xfer[li], s.xfer[li + 1], s.cmp[li], 0);
                    if (e != cudaSuccess) return cuda_fail(e, "band precompose");
                }
            }
            e = cudaDeviceSynchronize();
            if (e != cudaSuccess) return cuda_fail(e, "band precompose");
        }
    }
    p->finalized = true;
    return BF_OK;
}

bf_status_t bf_plan_create(const bf_desc_t* desc, int device, int64_t max_nrhs_chunk, bf_plan_t* out)
{
    if (!out) return fail(BF_ERR_INVALID_ARG, "out is NULL");
    bf_plan_t p = nullptr;
    bf_status_t st = bf_plan_alloc(desc, device, max_nrhs_chunk, &p);
    if (st != BF_OK) return st;
    if ((st = upload_desc(desc, p)) != BF_OK) {
        free_plan(p);
        return st;
    }
    *out = p;
    return BF_OK;
}

bf_status_t bf_plan_create_adjoint(bf_plan_t fwd, int64_t max_nrhs_chunk, bf_plan_t* out)
{
    if (!out) return fail(BF_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (!fwd) return fail(BF_ERR_INVALID_ARG, "plan is NULL");
    if (!fwd->finalized) return fail(BF_ERR_STATE, "forward plan not finalized");
    if (fwd->mode != BF_SHARD_NONE) return fail(BF_ERR_NOT_SUPPORTED, "adjoint of an index-sharded plan");
    if (!fwd->sh[0].dense_all()) return fail(BF_ERR_NOT_SUPPORTED, "adjoint of a structured plan");
    const bfk::Dims& d = fwd->d;
    bf_desc_t meta{};
    meta.abi_version = BF_ABI_VERSION;
    meta.log2n = d.LN;
    meta.log2leaf = d.l0;
    meta.rank = d.R;
    meta.n_amp = d.n_amp;
    meta.memory = BF_MEM_DEVICE;
    bf_plan_t p = nullptr;
    bf_status_t st = alloc_plan(&meta, fwd->device, max_nrhs_chunk, 1, 0, BF_SHARD_NONE, &p);
    if (st != BF_OK) return st;
    DeviceGuard g(p->device);
    Shard& s = p->sh[0];
    const Shard& f = fwd->sh[0];
    cudaFree(s.sw);   // the forward's level-h factor carries the switch; its adjoint carries the adjoint switch
    s.sw = nullptr;
    p->switch_in_factors = true;
    cudaError_t e = bfk::launch_adjoint_factors(d, f.amp_a, f.amp_b, f.v0, f.u, f.xfer.data(), s.amp_a, s.amp_b, s.v0,
                                                s.u, s.xfer.data(), 0);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        free_plan(p);
        return cuda_fail(e, "adjoint factors");
    }
    for (size_t slot = 0; slot < p->uploaded[0].size(); slot++) {
        const int stage = slot < 5 ? int(slot) : BF_STAGE_XFER0 + int(slot) - 5;
        p->uploaded[0][slot].push_back({0, stage_blocks(p, stage)});
    }
    if ((st = bf_plan_finalize(p)) != BF_OK) {
        free_plan(p);
        return st;
    }
    *out = p;
    return BF_OK;
}

bf_status_t bf_plan_recompress(bf_plan_t src, int32_t rank, int64_t max_nrhs_chunk, bf_plan_t* out)
{
    if (!out) return fail(BF_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (!src) return fail(BF_ERR_INVALID_ARG, "plan is NULL");
    if (!src->finalized) return fail(BF_ERR_STATE, "source plan not finalized");
    if (src->mode != BF_SHARD_NONE) return fail(BF_ERR_NOT_SUPPORTED, "recompression of an index-sharded plan");
    if (!src->sh[0].dense_all()) return fail(BF_ERR_NOT_SUPPORTED, "recompression of a structured plan");
    if (src->d.R > 12) return fail(BF_ERR_NOT_SUPPORTED, "recompression: source rank %d > 12", src->d.R);
    if (rank > src->d.R || !bfk::rank_supported(rank))
        return fail(BF_ERR_NOT_SUPPORTED, "recompression to rank %d (source %d)", rank, src->d.R);
    const bfk::Dims& d = src->d;
    bf_desc_t meta{};
    meta.abi_version = BF_ABI_VERSION;
    meta.log2n = d.LN;
    meta.log2leaf = d.l0;
    meta.rank = rank;
    meta.n_amp = d.n_amp;
    meta.memory = BF_MEM_DEVICE;
    bf_plan_t p = nullptr;
    bf_status_t st = alloc_plan(&meta, src->device, max_nrhs_chunk, 1, 0, BF_SHARD_NONE, &p);
    if (st != BF_OK) return st;
    DeviceGuard g(p->device);
    Shard& s = p->sh[0];
    const Shard& f = src->sh[0];
    cudaFree(s.sw);   // the source's level-h factor carries the switch, and so does the recompressed one
    s.sw = nullptr;
    p->switch_in_factors = true;
    const int64_t N = d.N, r = d.R, rp = rank, nl = d.D - d.l0 + 1;
    void *gout = nullptr, *q2 = nullptr, *gin2 = nullptr;
    const size_t zb = 16;   // complex double
    cudaError_t e = cudaMalloc(&gout, size_t(nl) * N * r * r * zb);
    if (e == cudaSuccess) e = cudaMalloc(&q2, size_t(2) * N * r * rp * zb);
    if (e == cudaSuccess) e = cudaMalloc(&gin2, size_t(2) * N * rp * rp * zb);
    if (e == cudaSuccess) e = cudaMemcpy(s.amp_a, f.amp_a, size_t(d.n_amp * N) * 8, cudaMemcpyDeviceToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(s.amp_b, f.amp_b, size_t(d.n_amp * N) * 8, cudaMemcpyDeviceToDevice);
    if (e == cudaSuccess) {
        bfk::Dims ds = d;
        e = bfk::launch_recompress(ds, int(rp), f.v0, f.xfer.data(), f.u, s.v0, s.xfer.data(), s.u, gout, q2, gin2, 0);
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    cudaFree(gout);
    cudaFree(q2);
    cudaFree(gin2);
    if (e != cudaSuccess) {
        cudaGetLastError();
        free_plan(p);
        return e == cudaErrorMemoryAllocation ? fail(BF_ERR_OOM, "recompression scratch: out of device memory")
                                              : cuda_fail(e, "recompression");
    }
    for (size_t slot = 0; slot < p->uploaded[0].size(); slot++) {
        const int stage = slot < 5 ? int(slot) : BF_STAGE_XFER0 + int(slot) - 5;
        p->uploaded[0][slot].push_back({0, stage_blocks(p, stage)});
    }
    if ((st = bf_plan_finalize(p)) != BF_OK) {
        free_plan(p);
        return st;
    }
    *out = p;
    return BF_OK;
}

bf_status_t bf_plan_create_sharded(const bf_desc_t* local, int device, int64_t max_nrhs_chunk, int32_t rank,
                                   int32_t world, const void* nccl_unique_id, bf_plan_t* out)
{
    if (!out) return fail(BF_ERR_INVALID_ARG, "out is NULL");
    bf_plan_t p = nullptr;
    bf_status_t st = bf_plan_alloc_sharded(local, device, max_nrhs_chunk, rank, world, nccl_unique_id, &p);
    if (st != BF_OK) return st;
    if ((st = upload_desc(local, p)) != BF_OK) {
        free_plan(p);
        return st;
    }
    *out = p;
    return BF_OK;
}

size_t bf_workspace_bytes(bf_plan_t p, int64_t nrhs_chunk)
{
    if (!p || nrhs_chunk < 1) return 0;
    return size_t(2) * size_t(p->nloc() * p->d.R) * size_t(nrhs_chunk * p->d.n_amp) * sizeof(float2);
}

bf_status_t bf_apply_ex(bf_plan_t p, const bf_c64* F, int64_t ldf, bf_c64* G, int64_t ldg, int64_t nrhs,
                        void* workspace, size_t workspace_bytes, void* stream)
{
    if (!p) return fail(BF_ERR_INVALID_ARG, "plan is NULL");
    if (!p->finalized) return fail(BF_ERR_STATE, "plan not finalized");
    if (nrhs < 0) return fail(BF_ERR_INVALID_ARG, "nrhs=%lld < 0", (long long)nrhs);
    if (nrhs == 0) return BF_OK;
    if (!F || !G) return fail(BF_ERR_INVALID_ARG, "F or G is NULL");
    const int64_t rows = (p->mode == BF_SHARD_NCCL) ? p->nloc() : p->d.N;
    if (ldf < rows || ldg < rows)
        return fail(BF_ERR_ALIGNMENT, "ldf=%lld / ldg=%lld < rows=%lld", (long long)ldf, (long long)ldg,
                    (long long)rows);
    // 16-byte aligned columns (the tensor-core S0 bulk-copies F columns; cp.async.bulk needs a 16-B source)
    if ((reinterpret_cast<uintptr_t>(F) | reinterpret_cast<uintptr_t>(G)) % 16)
        return fail(BF_ERR_ALIGNMENT, "F/G not 16-byte aligned");
    if ((ldf | ldg) & 1) return fail(BF_ERR_ALIGNMENT, "ldf=%lld / ldg=%lld not even", (long long)ldf, (long long)ldg);
    float2* ws = p->sh[0].ws;
    if (workspace) {
        if (p->mode == BF_SHARD_EMULATED) return fail(BF_ERR_NOT_SUPPORTED, "emulated plans use their own workspace");
        // the fused exchange stores into the peers' plan workspaces (IPC-mapped): every rank must use its plan
        // workspace, else the ranks would run different exchange protocols and hang
        if (p->exchange_peer)
            return fail(BF_ERR_NOT_SUPPORTED, "a caller workspace cannot be used with the fused exchange (BF_OPT_EXCHANGE = 1)");
        if (reinterpret_cast<uintptr_t>(workspace) % 16) return fail(BF_ERR_ALIGNMENT, "workspace not 16-byte aligned");
        if (workspace_bytes < bf_workspace_bytes(p, std::min(nrhs, p->max_chunk)))
            return fail(BF_ERR_INVALID_ARG, "workspace of %zu B < %zu B", workspace_bytes,
                        bf_workspace_bytes(p, std::min(nrhs, p->max_chunk)));
        ws = static_cast<float2*>(workspace);
    }
    // F and G must not alias
    const char* f0 = reinterpret_cast<const char*>(F);
    const char* g0 = reinterpret_cast<const char*>(G);
    const size_t fb = size_t((nrhs - 1) * ldf + rows) * 8, gb = size_t((nrhs - 1) * ldg + rows) * 8;
    if (f0 < g0 + gb && g0 < f0 + fb) return fail(BF_ERR_INVALID_ARG, "F and G overlap");
    DeviceGuard g(p->device);
    return apply_impl(p, reinterpret_cast<const float2*>(F), ldf, reinterpret_cast<float2*>(G), ldg, nrhs, ws,
                      static_cast<cudaStream_t>(stream));
}

bf_status_t bf_apply(bf_plan_t p, const bf_c64* F, bf_c64* G, int64_t nrhs, void* stream)
{
    if (!p) return fail(BF_ERR_INVALID_ARG, "plan is NULL");
    const int64_t rows = (p->mode == BF_SHARD_NCCL) ? p->nloc() : p->d.N;
    return bf_apply_ex(p, F, rows, G, rows, nrhs, nullptr, 0, stream);
}

bf_status_t bf_apply_graph(bf_plan_t p, const bf_c64* F, bf_c64* G, int64_t nrhs, void* stream)
{
    if (!p) return fail(BF_ERR_INVALID_ARG, "plan is NULL");
    if (!p->finalized) return fail(BF_ERR_STATE, "plan not finalized");
    if (p->mode == BF_SHARD_NCCL) return fail(BF_ERR_NOT_SUPPORTED, "bf_apply_graph on an NCCL plan");
    if (nrhs <= 0) return bf_apply(p, F, G, nrhs, stream);   // argument errors and the empty batch as bf_apply
    if (p->timing) return bf_apply(p, F, G, nrhs, stream);   // per-launch events need the eager launches
    DeviceGuard g(p->device);
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!(p->gexec && p->g_F == F && p->g_G == G && p->g_nrhs == nrhs)) {
        drop_graph(p);
        cudaError_t e = cudaSuccess;
        if (!p->cap && (e = cudaStreamCreateWithFlags(&p->cap, cudaStreamNonBlocking)) != cudaSuccess)
            return cuda_fail(e, "capture stream");
        // the capture stream must see the caller's prior work on `stream` only at replay time: the graph is
        // launched on `stream`, so nothing is ordered here
        if ((e = cudaStreamBeginCapture(p->cap, cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
            return cuda_fail(e, "begin capture");
        const bf_status_t st = bf_apply(p, F, G, nrhs, p->cap);
        cudaGraph_t graph = nullptr;
        e = cudaStreamEndCapture(p->cap, &graph);
        if (st != BF_OK) {
            if (graph) cudaGraphDestroy(graph);
            return st;
        }
        if (e != cudaSuccess) return cuda_fail(e, "end capture");
        e = cudaGraphInstantiate(&p->gexec, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) {
            p->gexec = nullptr;
            return cuda_fail(e, "graph instantiate");
        }
        p->g_F = F;
        p->g_G = G;
        p->g_nrhs = nrhs;
    }
    cudaError_t e = cudaGraphLaunch(p->gexec, s);
    if (e != cudaSuccess) return cuda_fail(e, "graph launch");
    cudaEventRecord(p->done, s);
    return BF_OK;
}

bf_status_t bf_apply_host(bf_plan_t p, const bf_c64* F_host, bf_c64* G_host, int64_t nrhs, void* stream)
{
    if (!p) return fail(BF_ERR_INVALID_ARG, "plan is NULL");
    if (!p->finalized) return fail(BF_ERR_STATE, "plan not finalized");
    if (nrhs < 0 || (nrhs > 0 && (!F_host || !G_host))) return fail(BF_ERR_INVALID_ARG, "bad arguments");
    if (nrhs == 0) return BF_OK;
    DeviceGuard g(p->device);
    const int64_t rows = (p->mode == BF_SHARD_NCCL) ? p->nloc() : p->d.N, chunk = p->max_chunk;
    bf_status_t st;
    cudaError_t e;
    if (!p->h2d && ((e = cudaStreamCreateWithFlags(&p->h2d, cudaStreamNonBlocking)) != cudaSuccess ||
                    (e = cudaStreamCreateWithFlags(&p->d2h, cudaStreamNonBlocking)) != cudaSuccess))
        return cuda_fail(e, "copy streams");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // Pipeline over pieces (BF_OPT_HOST_PIECES = NP): the host->device copy of piece i+1 and the
    // device->host copy of piece i-1 run on their own streams while piece i is applied on `stream` (PCIe is
    // full duplex).  NP = 3 ("tapered"): per chunk-sized span, pieces of 1/4, 1/2, 1/4 -- only the small
    // first and last pieces' copies are exposed; otherwise NP equal pieces.  Staging parts form a ring of
    // NB parts; hazards are ordered with events: a part is refilled only after the apply that read it, and
    // rewritten only after the copy-out that read it.
    std::vector<std::pair<int64_t, int64_t>> pcs;   // (first column, columns)
    int NB;
    int64_t part;
    if (p->host_pieces == 3 && chunk >= 4) {
        NB = 2;
        part = (chunk + 1) / 2;
        for (int64_t c = 0; c < nrhs; c += chunk) {
            const int64_t span = std::min(chunk, nrhs - c), q = span / 4;
            if (q == 0) {
                pcs.push_back({c, span});
                continue;
            }
            pcs.push_back({c, q});
            pcs.push_back({c + q, span - 2 * q});
            pcs.push_back({c + span - q, q});
        }
    } else {
        NB = int(std::min<int64_t>(std::max(p->host_pieces, 1), chunk));
        part = (chunk + NB - 1) / NB;
        for (int64_t c = 0; c < nrhs; c += part) pcs.push_back({c, std::min(part, nrhs - c)});
    }
    const int64_t npieces = int64_t(pcs.size());
    // staging ring: NB slots of the largest piece (the pieces of one span are not all equal)
    for (const auto& pc : pcs) part = std::max(part, pc.second);
    const int64_t need = rows * NB * part;
    if (p->staging_elems < need) {
        cudaFree(p->dF);
        cudaFree(p->dG);
        p->dF = p->dG = nullptr;
        p->staging_elems = 0;
        if ((st = dalloc(&p->dF, need, "e2e F")) || (st = dalloc(&p->dG, need, "e2e G"))) return st;
        p->staging_elems = need;
    }
    std::vector<cudaEvent_t> ev(3 * size_t(npieces), nullptr);   // [h2d done, apply done, d2h done] per piece
    for (auto& x : ev)
        if ((e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming)) != cudaSuccess) break;
    auto cleanup = [&]() {
        for (auto& x : ev)
            if (x) cudaEventDestroy(x);
    };
    if (e != cudaSuccess) {
        cleanup();
        return cuda_fail(e, "events");
    }
    st = BF_OK;
    for (int64_t i = 0; i < npieces && st == BF_OK; i++) {
        const int64_t c0 = pcs[size_t(i)].first, nc = pcs[size_t(i)].second, buf = i % NB;
        const size_t bytes = size_t(rows * nc) * sizeof(float2);
        float2* dF = p->dF + buf * part * rows;
        float2* dG = p->dG + buf * part * rows;
        cudaEvent_t* E = &ev[3 * size_t(i)];
        if (i >= NB) cudaStreamWaitEvent(p->h2d, ev[3 * size_t(i - NB) + 1], 0);
        if ((e = cudaMemcpyAsync(dF, F_host + c0 * rows, bytes, cudaMemcpyHostToDevice, p->h2d)) != cudaSuccess) {
            st = cuda_fail(e, "H2D");
            break;
        }
        cudaEventRecord(E[0], p->h2d);
        cudaStreamWaitEvent(s, E[0], 0);
        if (i >= NB) cudaStreamWaitEvent(s, ev[3 * size_t(i - NB) + 2], 0);
        if ((st = apply_impl(p, dF, rows, dG, rows, nc, p->sh[0].ws, s)) != BF_OK) break;
        cudaEventRecord(E[1], s);
        cudaStreamWaitEvent(p->d2h, E[1], 0);
        if ((e = cudaMemcpyAsync(G_host + c0 * rows, dG, bytes, cudaMemcpyDeviceToHost, p->d2h)) != cudaSuccess) {
            st = cuda_fail(e, "D2H");
            break;
        }
        cudaEventRecord(E[2], p->d2h);
    }
    // the apply stream (with its NCCL exchanges) first, polled for communicator errors on sharded plans
    if (st == BF_OK && npieces > 0) st = wait_event_nccl(p, ev[3 * size_t(npieces - 1) + 1]);
    cudaError_t e1 = cudaStreamSynchronize(p->h2d), e2 = cudaStreamSynchronize(p->d2h), e3 = cudaStreamSynchronize(s);
    cleanup();
    if (st != BF_OK) return st;
    if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess)
        return cuda_fail(e1 != cudaSuccess ? e1 : e2 != cudaSuccess ? e2 : e3, "bf_apply_host");
    return BF_OK;
}

bf_status_t bf_apply_host_async(bf_plan_t p, const bf_c64* F_host, bf_c64* G_host, int64_t nrhs, void* stream)
{
    if (!p) return fail(BF_ERR_INVALID_ARG, "plan is NULL");
    if (!p->finalized) return fail(BF_ERR_STATE, "plan not finalized");
    if (nrhs < 0 || (nrhs > 0 && (!F_host || !G_host))) return fail(BF_ERR_INVALID_ARG, "bad arguments");
    if (nrhs == 0) return BF_OK;
    DeviceGuard g(p->device);
    const int64_t rows = (p->mode == BF_SHARD_NCCL) ? p->nloc() : p->d.N, chunk = p->max_chunk;
    cudaError_t e = cudaSuccess;
    if (!p->h2d && ((e = cudaStreamCreateWithFlags(&p->h2d, cudaStreamNonBlocking)) != cudaSuccess ||
                    (e = cudaStreamCreateWithFlags(&p->d2h, cudaStreamNonBlocking)) != cudaSuccess))
        return cuda_fail(e, "copy streams");
    for (int i = 0; i < 2; i++) {
        if (p->aF[i]) continue;
        bf_status_t st;
        if ((st = dalloc(&p->aF[i], rows * chunk, "async F")) || (st = dalloc(&p->aG[i], rows * chunk, "async G")))
            return st;
        for (cudaEvent_t* ev : {&p->a_h2d[i], &p->a_applied[i], &p->a_d2h[i]})
            if ((e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming)) != cudaSuccess) return cuda_fail(e, "events");
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // per chunk: slot = use % 2.  H2D into slot's F once the apply two chunks back has read it; the apply (on
    // `stream`) once that H2D landed and the slot's previous G has been copied out; D2H after the apply.  The
    // host returns at once: the copies of chunk i+1 and i-1 run while chunk i is applied.
    for (int64_t c0 = 0; c0 < nrhs; c0 += chunk) {
        const int64_t nc = std::min(chunk, nrhs - c0);
        const int sl = int(p->a_uses & 1);
        const bool reuse = p->a_uses >= 2;
        p->a_uses++;
        const size_t bytes = size_t(rows * nc) * sizeof(float2);
        if (reuse) cudaStreamWaitEvent(p->h2d, p->a_applied[sl], 0);
        if ((e = cudaMemcpyAsync(p->aF[sl], F_host + c0 * rows, bytes, cudaMemcpyHostToDevice, p->h2d)) != cudaSuccess)
            return cuda_fail(e, "H2D");
        cudaEventRecord(p->a_h2d[sl], p->h2d);
        cudaStreamWaitEvent(s, p->a_h2d[sl], 0);
        if (reuse) cudaStreamWaitEvent(s, p->a_d2h[sl], 0);
        if (bf_status_t st = apply_impl(p, p->aF[sl], rows, p->aG[sl], rows, nc, p->sh[0].ws, s); st != BF_OK) return st;
        cudaEventRecord(p->a_applied[sl], s);
        cudaStreamWaitEvent(p->d2h, p->a_applied[sl], 0);
        if ((e = cudaMemcpyAsync(G_host + c0 * rows, p->aG[sl], bytes, cudaMemcpyDeviceToHost, p->d2h)) != cudaSuccess)
            return cuda_fail(e, "D2H");
        cudaEventRecord(p->a_d2h[sl], p->d2h);
    }
    return BF_OK;
}

bf_status_t bf_apply_host_wait(bf_plan_t p)
{
    if (!p) return fail(BF_ERR_INVALID_ARG, "plan is NULL");
    DeviceGuard g(p->device);
    for (int i = 0; i < 2; i++)
        if (p->a_d2h[i] && p->a_uses > i) {
            if (bf_status_t st = wait_event_nccl(p, p->a_d2h[i]); st != BF_OK) return st;
        }
    return BF_OK;
}

bf_status_t bf_plan_get_info(bf_plan_t p, bf_plan_info_t* info)
{
    if (!p || !info) return fail(BF_ERR_INVALID_ARG, "NULL argument");
    const int64_t n = p->nloc(), r = p->d.R, n0 = int64_t(1) << p->d.l0;
    const int nx = int(p->sh[0].xfer.size());
    const int64_t nsh = int64_t(p->sh.size());
    info->log2n = p->d.LN;
    info->log2leaf = p->d.l0;
    info->rank = p->d.R;
    info->n_amp = p->d.n_amp;
    info->switch_level = p->d.h;
    info->n_xfer = nx;
    info->n = p->d.N;
    info->max_nrhs_chunk = p->max_chunk;
    // the switch blocks are folded into the level-h factor at finalize (freed afterwards)
    info->factor_bytes = 0;
    for (const Shard& s : p->sh) {
        int64_t f = 2 * p->d.n_amp * n + (s.sw ? n * r * r : 0) + (s.v0 ? n * r * n0 : 0) + (s.u ? n * r * n0 : 0) +
                    (s.s0_ph ? n * n0 : 0) + (s.sl_ph ? n * n0 : 0);
        for (int i = 0; i < nx; i++)
            f += (s.xfer[i] ? n * 2 * r * r : 0) +
                 (s.ph[i] ? n * (s.kind[i] == BF_LEVEL_FIRST_SWITCH ? 2 * r + r * r : 2 * r) : 0);
        info->factor_bytes += 8 * f;
        info->factor_bytes += 4 * ((s.s0_lag ? r * n0 : 0) + (s.sl_lag ? r * n0 : 0));
        for (int i = 0; i < nx; i++) info->factor_bytes += s.lag[i] ? 4 * 2 * r * r : 0;
    }
    for (const Shard& s : p->sh)
        for (auto c : s.cmp)
            if (c) info->factor_bytes += 8 * n * 4 * r * r;   // precomposed band operators
    for (const Shard& s : p->sh)
        for (auto c : s.cmp3)
            if (c) info->factor_bytes += 8 * n * 8 * r * r;   // precomposed three-level band operators
    info->workspace_bytes = nsh * int64_t(p->ws_bytes);
    info->tc_weight_bytes = 0;
    for (const Shard& s : p->sh) {
        if (s.v0x) info->tc_weight_bytes += bfk::v0x_floats(p->local()) * int64_t(sizeof(float));
        if (s.ux) info->tc_weight_bytes += bfk::ux_floats(p->local()) * int64_t(sizeof(float));
    }
    {
        const bfk::Dims dl = p->local();
        const int nvf = int(p->max_chunk * p->d.n_amp);
        int mask = 0;
        if (p->tensor_cores && p->sh[0].v0x && bfk::s0_tc_supported(dl, nvf, dl.N))
            mask |= 1 << bfk::KC_S0;
        if (p->tensor_cores && p->sh[0].ux && bfk::sl_tc_supported(dl, nvf)) mask |= 1 << bfk::KC_SL;
        if (p->tensor_cores && bfk::band_tc_supported(dl, nvf))
            for (const auto& stp : schedule(p, nvf))
                if (stp.kind == Step::BAND && stp.K >= 2) mask |= 1 << stp.cls;
        info->tc_class_mask = mask;
    }
    const auto st = schedule(p, int(p->max_chunk * p->d.n_amp));
    info->launches_per_chunk = 0;
    for (int i = 0; i < BF_NUM_KCLASS; i++) info->class_launches[i] = info->class_levels[i] = 0;
    for (const auto& x : st) {
        const int mult = (x.kind == Step::EXCHANGE) ? 1 : int(nsh);   // emulated: every shard launches
        info->class_launches[x.cls] += mult;
        info->class_levels[x.cls] += mult * x.levels;
        if (x.kind != Step::EXCHANGE) info->launches_per_chunk += mult;
    }
    info->device = p->device;
    info->world = p->world;
    info->shard_rank = p->rank;
    info->sharding = p->mode;
    info->rows_local = (p->mode == BF_SHARD_NCCL) ? n : p->d.N;
    info->structured = p->structured ? 1 : 0;
    return BF_OK;
}

namespace {
// Fused-exchange destinations: each shard's workspace base.  Emulated shards share the device; for one
// shard per GPU the plans exchange CUDA IPC handles of their workspaces (NCCL send/recv of the 64-byte
// handles) and map the peers' workspaces (NVLink peer access).  Collective for NCCL plans.
bf_status_t setup_peer_exchange(bf_plan_s* p)
{
    DeviceGuard g(p->device);
    if (p->mode == BF_SHARD_EMULATED) {
        for (int i = 0; i < p->world; i++) p->peer_ws[i] = p->sh[i].ws;
        return BF_OK;
    }
    if (p->peer_ws[p->rank]) return BF_OK;   // already mapped
    cudaError_t e;
    if (!p->bar_buf && (e = cudaMalloc(&p->bar_buf, 2 * size_t(p->world))) != cudaSuccess) return cuda_fail(e, "barrier");
    cudaMemset(p->bar_buf, 0, 2 * size_t(p->world));
    if (p->world == 1) {
        p->peer_ws[0] = p->sh[0].ws;
        return BF_OK;
    }
    std::vector<cudaIpcMemHandle_t> hs(p->world);
    if ((e = cudaIpcGetMemHandle(&hs[p->rank], p->sh[0].ws)) != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
    char* hb = nullptr;
    const size_t hsz = sizeof(cudaIpcMemHandle_t);
    if ((e = cudaMalloc(&hb, hsz * p->world)) != cudaSuccess) return cuda_fail(e, "handle buffer");
    cudaStream_t s = nullptr;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaMemcpyAsync(hb + hsz * p->rank, &hs[p->rank], hsz, cudaMemcpyHostToDevice, s);
    Nccl& n = nccl();
    ncclResult_t r = n.GroupStart();
    for (int peer = 0; peer < p->world && !r; peer++) {
        if (peer == p->rank) continue;
        if ((r = n.Send(hb + hsz * p->rank, hsz, kNcclUint8, peer, p->comm, s))) break;
        r = n.Recv(hb + hsz * peer, hsz, kNcclUint8, peer, p->comm, s);
    }
    ncclResult_t r2 = n.GroupEnd();
    cudaMemcpyAsync(hs.data(), hb, hsz * p->world, cudaMemcpyDeviceToHost, s);
    e = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    cudaFree(hb);
    if (r || r2) return nccl_fail(r ? r : r2, "IPC handle exchange");
    if (e != cudaSuccess) return cuda_fail(e, "IPC handle exchange");
    for (int d = 0; d < p->world; d++) {
        if (d == p->rank) {
            p->peer_ws[d] = p->sh[0].ws;
            continue;
        }
        void* ptr = nullptr;
        if ((e = cudaIpcOpenMemHandle(&ptr, hs[d], cudaIpcMemLazyEnablePeerAccess)) != cudaSuccess)
            return cuda_fail(e, "cudaIpcOpenMemHandle");
        p->peer_ws[d] = static_cast<float2*>(ptr);
        p->peer_ipc[d] = true;
    }
    return BF_OK;
}
}  // namespace

bf_status_t bf_plan_set_option(bf_plan_t p, int32_t option, int64_t value)
{
    if (!p) return fail(BF_ERR_INVALID_ARG, "plan is NULL");
    drop_graph(p);   // the captured launch sequence depends on the options
    if (option == BF_OPT_TENSOR_CORES) {
        if (value != 0 && value != 1) return fail(BF_ERR_INVALID_ARG, "BF_OPT_TENSOR_CORES takes 0 or 1");
        p->tensor_cores = value != 0;
        return BF_OK;
    }
    if (option == BF_OPT_EXCHANGE) {
        if (value != 0 && value != 1) return fail(BF_ERR_INVALID_ARG, "BF_OPT_EXCHANGE takes 0 or 1");
        if (value == 1) {
            if (p->mode == BF_SHARD_NONE) return fail(BF_ERR_NOT_SUPPORTED, "the fused exchange needs a sharded plan");
            if (p->world > bfs::kMaxShards) return fail(BF_ERR_NOT_SUPPORTED, "more than %d shards", bfs::kMaxShards);
            if (p->d.h == p->d.l0) return fail(BF_ERR_NOT_SUPPORTED, "no transfer level produces level h (h == l0)");
            bf_status_t st = setup_peer_exchange(p);
            if (st != BF_OK) return st;
        }
        p->exchange_peer = value != 0;
        return BF_OK;
    }
    if (option == BF_OPT_LEAF_MULTICAST) {
        if (value != 0 && value != 1) return fail(BF_ERR_INVALID_ARG, "BF_OPT_LEAF_MULTICAST takes 0 or 1");
        p->leaf_multicast = value != 0;
        return BF_OK;
    }
    if (option == BF_OPT_BAND3) {
        if (value != 0 && value != 1) return fail(BF_ERR_INVALID_ARG, "BF_OPT_BAND3 takes 0 or 1");
        p->band3 = value != 0;
        return BF_OK;
    }
    if (option == BF_OPT_BAND_PRECOMPOSE) {
        if (value != 0 && value != 1) return fail(BF_ERR_INVALID_ARG, "BF_OPT_BAND_PRECOMPOSE takes 0 or 1");
        p->precompose = value != 0;
        return BF_OK;
    }
    if (option == BF_OPT_SMALL_BATCH) {
        if (value != 0 && value != 1) return fail(BF_ERR_INVALID_ARG, "BF_OPT_SMALL_BATCH takes 0 or 1");
        p->small_batch = value != 0;
        return BF_OK;
    }
    if (option == BF_OPT_HOST_PIECES) {
        if (value < 1 || value > 16) return fail(BF_ERR_INVALID_ARG, "BF_OPT_HOST_PIECES takes 1..16");
        p->host_pieces = int(value);
        return BF_OK;
    }
    if (option == BF_OPT_BAND_COMPOSE) {
        if (value != 0 && value != 1) return fail(BF_ERR_INVALID_ARG, "BF_OPT_BAND_COMPOSE takes 0 or 1");
        p->band.compose = value != 0;
        return BF_OK;
    }
    return fail(BF_ERR_INVALID_ARG, "unknown plan option");
}

bf_status_t bf_plan_set_timing(bf_plan_t p, int32_t enable)
{
    if (!p) return fail(BF_ERR_INVALID_ARG, "plan is NULL");
    drop_graph(p);
    DeviceGuard g(p->device);
    for (auto& tl : p->pending) {
        cudaEventSynchronize(tl.stop);
        p->pool.push_back(tl.start);
        p->pool.push_back(tl.stop);
    }
    p->pending.clear();
    std::fill(p->ms, p->ms + BF_NUM_KCLASS, 0.0);
    std::fill(p->nlaunch, p->nlaunch + BF_NUM_KCLASS, 0);
    p->timing = enable != 0;
    return BF_OK;
}

bf_status_t bf_plan_timing(bf_plan_t p, double* ms, int64_t* launches)
{
    if (!p || !ms || !launches) return fail(BF_ERR_INVALID_ARG, "NULL argument");
    DeviceGuard g(p->device);
    for (auto& tl : p->pending) {
        cudaError_t e = cudaEventSynchronize(tl.stop);
        if (e != cudaSuccess) return cuda_fail(e, "timing event");
        float t = 0.f;
        cudaEventElapsedTime(&t, tl.start, tl.stop);
        p->ms[tl.cls] += t;
        p->nlaunch[tl.cls] += 1;
        p->pool.push_back(tl.start);
        p->pool.push_back(tl.stop);
    }
    p->pending.clear();
    for (int i = 0; i < BF_NUM_KCLASS; i++) {
        ms[i] = p->ms[i];
        launches[i] = p->nlaunch[i];
    }
    return BF_OK;
}

bf_status_t bf_plan_destroy(bf_plan_t p)
{
    if (!p) return BF_OK;
    bf_status_t st = BF_OK;
    {
        DeviceGuard g(p->device);
        if (p->done) st = wait_event_nccl(p, p->done);
    }
    free_plan(p);
    return st;
}

bf_status_t bf_shard_pairs(int32_t log2n, int32_t log2leaf, int32_t world, int32_t rank, int32_t which, int64_t* out)
{
    bf_desc_t d{};
    d.abi_version = BF_ABI_VERSION;
    d.log2n = log2n;
    d.log2leaf = log2leaf;
    bf_status_t st = validate_sharding(&d, world, rank);
    if (st != BF_OK) return st;
    if (!out || which < 0 || which > 2) return fail(BF_ERR_INVALID_ARG, "bad arguments");
    int g = 0;
    while ((1 << g) < world) g++;
    const int h = log2n / 2;
    const int64_t n = (int64_t(1) << log2n) >> g;
    for (int64_t loc = 0; loc < n; loc++) {
        if (which == 0)   // send buffer = first-half local order at level h
            out[loc] = bfs::first_half_global(loc, log2n, h, g, rank);
        else if (which == 2)   // second-half local order at level h
            out[loc] = bfs::second_half_global(loc, log2n, g, rank);
        else   // receive buffer: position recv_index(p) holds second-half local pair p
            out[bfs::recv_index(loc, h, h - g)] = bfs::second_half_global(loc, log2n, g, rank);
    }
    return BF_OK;
}

}  // extern "C"

namespace {

bf_status_t upload_desc(const bf_desc_t* desc, bf_plan_t p)
{
    const int nx = desc->log2n - 2 * desc->log2leaf;
    if (!desc->amp_a || !desc->amp_b || !desc->v0 || !desc->sw || !desc->u || (nx > 0 && !desc->xfer))
        return fail(BF_ERR_INVALID_ARG, "a factor array pointer is NULL");
    for (int i = 0; i < nx; i++)
        if (!desc->xfer[i]) return fail(BF_ERR_INVALID_ARG, "xfer[%d] is NULL", i);
    const int mem = desc->memory;
    const int64_t n = p->nloc();
    bf_status_t st;
    if ((st = bf_plan_upload(p, BF_STAGE_AMP_A, 0, p->d.n_amp, desc->amp_a, mem)) ||
        (st = bf_plan_upload(p, BF_STAGE_AMP_B, 0, p->d.n_amp, desc->amp_b, mem)) ||
        (st = bf_plan_upload(p, BF_STAGE_V0, 0, n, desc->v0, mem)) ||
        (st = bf_plan_upload(p, BF_STAGE_SW, 0, n, desc->sw, mem)) ||
        (st = bf_plan_upload(p, BF_STAGE_U, 0, n, desc->u, mem)))
        return st;
    for (int i = 0; i < nx; i++)
        if ((st = bf_plan_upload(p, BF_STAGE_XFER0 + i, 0, n, desc->xfer[i], mem))) return st;
    return bf_plan_finalize(p);
}

}  // namespace
