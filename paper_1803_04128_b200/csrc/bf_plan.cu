// bf_plan.cu -- the C ABI of include/bf.h: plan creation / streaming upload,
// bf_apply orchestration (one stream, RHS chunks, no allocation), end-to-end
// host apply, per-kernel event timing.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/bf.h"
#include "bf_internal.h"
#include "bf_plan_internal.h"

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

}  // namespace

struct TimedLaunch {
    int cls;
    cudaEvent_t start, stop;
};

struct bf_plan_s {
    int device = 0;
    bfk::Dims d{};
    int64_t max_chunk = 0;
    // factors (device)
    float2* amp_a = nullptr;
    float2* amp_b = nullptr;
    float2* v0 = nullptr;
    float2* sw = nullptr;
    float2* u = nullptr;
    std::vector<float2*> xfer;
    std::vector<int64_t> uploaded;   // blocks uploaded per stage slot
    bool finalized = false;
    // workspace (two coefficient arrays)
    float2* ws = nullptr;
    size_t ws_bytes = 0;
    // end-to-end staging (lazily allocated by bf_apply_host)
    float2* dF = nullptr;
    float2* dG = nullptr;
    // timing
    bool timing = false;
    std::vector<TimedLaunch> pending;
    std::vector<cudaEvent_t> pool;
    double ms[BF_NUM_KCLASS] = {0};
    int64_t nlaunch[BF_NUM_KCLASS] = {0};
    cudaEvent_t done = nullptr;
};

namespace {

// stage slot index: 0 V0, 1 SW, 2 U, 3 AMP_A, 4 AMP_B, 5 + i XFER i
int slot_of(const bf_plan_s* p, int stage)
{
    if (stage >= BF_STAGE_XFER0) {
        const int i = stage - BF_STAGE_XFER0;
        return i < int(p->xfer.size()) ? 5 + i : -1;
    }
    return (stage >= 0 && stage <= 4) ? stage : -1;
}

int64_t stage_blocks(const bf_plan_s* p, int stage)
{
    if (stage == BF_STAGE_AMP_A || stage == BF_STAGE_AMP_B) return p->d.n_amp;
    return p->d.N;
}

int64_t stage_elems(const bf_plan_s* p, int stage)
{
    const int64_t r = p->d.R, n0 = int64_t(1) << p->d.l0;
    switch (stage) {
    case BF_STAGE_V0: return r * n0;
    case BF_STAGE_SW: return r * r;
    case BF_STAGE_U: return n0 * r;
    case BF_STAGE_AMP_A:
    case BF_STAGE_AMP_B: return p->d.N;
    default: return 2 * r * r;
    }
}

float2* stage_base(bf_plan_s* p, int stage)
{
    switch (stage) {
    case BF_STAGE_V0: return p->v0;
    case BF_STAGE_SW: return p->sw;
    case BF_STAGE_U: return p->u;
    case BF_STAGE_AMP_A: return p->amp_a;
    case BF_STAGE_AMP_B: return p->amp_b;
    default: return p->xfer[stage - BF_STAGE_XFER0];
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

void free_plan(bf_plan_s* p)
{
    if (!p) return;
    DeviceGuard g(p->device);
    if (p->done) cudaEventSynchronize(p->done);
    for (auto& tl : p->pending) {
        cudaEventDestroy(tl.start);
        cudaEventDestroy(tl.stop);
    }
    for (auto e : p->pool) cudaEventDestroy(e);
    if (p->done) cudaEventDestroy(p->done);
    cudaFree(p->amp_a);
    cudaFree(p->amp_b);
    cudaFree(p->v0);
    cudaFree(p->sw);
    cudaFree(p->u);
    for (auto x : p->xfer) cudaFree(x);
    cudaFree(p->ws);
    cudaFree(p->dF);
    cudaFree(p->dG);
    delete p;
}

bf_status_t dalloc(float2** ptr, int64_t elems, const char* what)
{
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(ptr), size_t(elems) * sizeof(float2));
    if (e != cudaSuccess) {
        cudaGetLastError();
        *ptr = nullptr;
        return fail(BF_ERR_OOM, "cudaMalloc(%s, %lld B) failed: %s", what, (long long)(elems * 8), cudaGetErrorString(e));
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
    enum Kind { S0, SWITCH, XFER, BAND, SL } kind;
    int l_first = 0;   // XFER: the level; BAND: first level
    int K = 1;         // BAND: levels fused
    int m_sw = 0;      // BAND: band level after which the switch applies (0 = none)
    int cls = 0;       // bfk::KClass
    int levels = 0;    // transfer levels this launch performs
};

// The launch sequence of one RHS chunk of nv vectors: S0, transfer levels l0+1..D (fused in bands of 2
// when the band kernel supports the shape, the switch applied inside the launch that produces level h),
// SL.  With no transfer level (h == l0) the switch runs alone after S0.
std::vector<Step> schedule(const bfk::Dims& d, int nv)
{
    std::vector<Step> st;
    st.push_back({Step::S0, 0, 1, 0, bfk::KC_S0, 0});
    if (d.h == d.l0) st.push_back({Step::SWITCH, 0, 1, 0, bfk::KC_SWITCH, 0});
    const bool band = bfk::band_supported(d.R, nv);
    for (int l = d.l0 + 1; l <= d.D;) {
        const int K = band ? std::min(2, d.D - l + 1) : 1;
        const int last = l + K - 1;
        const int cls = (l <= d.h && d.h <= last) ? bfk::KC_SWITCH : (last < d.h ? bfk::KC_XFER1 : bfk::KC_XFER2);
        const int m_sw = (l <= d.h && d.h <= last) ? d.h - l + 1 : 0;
        st.push_back({band ? Step::BAND : Step::XFER, l, K, m_sw, cls, K});
        l += K;
    }
    st.push_back({Step::SL, 0, 1, 0, bfk::KC_SL, 0});
    return st;
}

bf_status_t apply_impl(bf_plan_s* p, const float2* F, int64_t ldf, float2* G, int64_t ldg, int64_t nrhs, float2* ws,
                       cudaStream_t s)
{
    const bfk::Dims& d = p->d;
    const int64_t chunk = p->max_chunk;
    const int64_t pair_elems = d.N * d.R;   // complex per vector per coefficient array
    for (int64_t c0 = 0; c0 < nrhs; c0 += chunk) {
        const int64_t nc = std::min(chunk, nrhs - c0);
        const int nv = int(nc * d.n_amp);
        float2* cur = ws;
        float2* oth = ws + pair_elems * nv;
        for (const Step& stp : schedule(d, nv)) {
            cudaError_t e = timed(p, stp.cls, s, [&]() -> cudaError_t {
                switch (stp.kind) {
                case Step::S0: return bfk::launch_s0(d, F + c0 * ldf, ldf, p->amp_b, p->v0, cur, nv, s);
                case Step::SWITCH: return bfk::launch_switch(d, cur, oth, p->sw, nv, s);
                case Step::XFER:
                    return bfk::launch_xfer(d, stp.l_first, cur, oth, p->xfer[stp.l_first - d.l0 - 1],
                                            stp.l_first == d.h ? p->sw : nullptr, nv, s);
                case Step::BAND: {
                    const float2* W[2] = {p->xfer[stp.l_first - d.l0 - 1],
                                          stp.K > 1 ? p->xfer[stp.l_first - d.l0] : nullptr};
                    return bfk::launch_band(d, stp.l_first, stp.K, cur, oth, W, p->sw, stp.m_sw, nv, s);
                }
                default: return bfk::launch_sl(d, cur, p->u, p->amp_a, G + c0 * ldg, ldg, nv, s);
                }
            });
            if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
            if (stp.kind == Step::SWITCH || stp.kind == Step::XFER || stp.kind == Step::BAND) std::swap(cur, oth);
        }
    }
    cudaEventRecord(p->done, s);
    return BF_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// internal helpers for the streaming builder (bf_build.cpp)
// ---------------------------------------------------------------------------
bf_status_t bfp_stage_dst(bf_plan_t p, int32_t stage, int64_t begin, int64_t count, void** dst)
{
    if (!p || !dst) return fail(BF_ERR_INVALID_ARG, "NULL argument");
    if (p->finalized) return fail(BF_ERR_STATE, "plan already finalized");
    const int slot = slot_of(p, stage);
    if (slot < 0) return fail(BF_ERR_INVALID_ARG, "bad stage id %d", stage);
    if (begin < 0 || count < 0 || begin + count > stage_blocks(p, stage))
        return fail(BF_ERR_INVALID_ARG, "block range [%lld,%lld) out of [0,%lld)", (long long)begin,
                    (long long)(begin + count), (long long)stage_blocks(p, stage));
    *dst = stage_base(p, stage) + begin * stage_elems(p, stage);
    p->uploaded[slot] += count;
    return BF_OK;
}

int bfp_device(bf_plan_t p) { return p ? p->device : -1; }

bf_status_t bfp_fail(bf_status_t s, const char* msg) { return fail(s, "%s", msg); }

// ---------------------------------------------------------------------------
// ABI
// ---------------------------------------------------------------------------
extern "C" {

int32_t bf_abi_version(void) { return BF_ABI_VERSION; }

const char* bf_last_error(void) { return g_err.c_str(); }

bf_status_t bf_plan_alloc(const bf_desc_t* meta, int device, int64_t max_nrhs_chunk, bf_plan_t* out)
{
    if (!out) return fail(BF_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    bf_status_t st = validate_shape(meta);
    if (st != BF_OK) return st;
    if (max_nrhs_chunk < 1) return fail(BF_ERR_INVALID_ARG, "max_nrhs_chunk=%lld < 1", (long long)max_nrhs_chunk);
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
    if (device < 0 || device >= ndev) return fail(BF_ERR_INVALID_ARG, "device %d not in [0,%d)", device, ndev);
    DeviceGuard g(device);

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
    const int nx = p->d.D - p->d.l0;
    p->xfer.assign(nx, nullptr);
    p->uploaded.assign(5 + nx, 0);
    const int64_t N = p->d.N, r = p->d.R, n0 = int64_t(1) << p->d.l0;
    if ((st = dalloc(&p->amp_a, p->d.n_amp * N, "amp_a")) || (st = dalloc(&p->amp_b, p->d.n_amp * N, "amp_b")) ||
        (st = dalloc(&p->v0, N * r * n0, "v0")) || (st = dalloc(&p->sw, N * r * r, "sw")) ||
        (st = dalloc(&p->u, N * r * n0, "u"))) {
        free_plan(p);
        return st;
    }
    for (int i = 0; i < nx; i++)
        if ((st = dalloc(&p->xfer[i], N * 2 * r * r, "xfer"))) {
            free_plan(p);
            return st;
        }
    const int64_t nv = max_nrhs_chunk * p->d.n_amp;
    p->ws_bytes = size_t(2) * size_t(N * r) * size_t(nv) * sizeof(float2);
    if ((st = dalloc(&p->ws, int64_t(p->ws_bytes / sizeof(float2)), "workspace"))) {
        free_plan(p);
        return st;
    }
    if ((e = cudaEventCreateWithFlags(&p->done, cudaEventDisableTiming)) != cudaSuccess) {
        free_plan(p);
        return cuda_fail(e, "cudaEventCreate");
    }
    *out = p;
    return BF_OK;
}

bf_status_t bf_plan_upload(bf_plan_t p, int32_t stage, int64_t block_begin, int64_t block_count, const bf_c64* src,
                           int32_t src_memory)
{
    if (!p || (!src && block_count > 0)) return fail(BF_ERR_INVALID_ARG, "NULL argument");
    if (src_memory != BF_MEM_HOST && src_memory != BF_MEM_DEVICE)
        return fail(BF_ERR_INVALID_ARG, "src_memory=%d", src_memory);
    DeviceGuard g(p->device);
    void* dst = nullptr;
    bf_status_t st = bfp_stage_dst(p, stage, block_begin, block_count, &dst);
    if (st != BF_OK) return st;
    const size_t bytes = size_t(block_count) * size_t(stage_elems(p, stage)) * sizeof(float2);
    cudaError_t e = cudaMemcpy(dst, src, bytes, src_memory == BF_MEM_HOST ? cudaMemcpyHostToDevice
                                                                          : cudaMemcpyDeviceToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(upload)");
    return BF_OK;
}

bf_status_t bf_plan_finalize(bf_plan_t p)
{
    if (!p) return fail(BF_ERR_INVALID_ARG, "plan is NULL");
    if (p->finalized) return fail(BF_ERR_STATE, "plan already finalized");
    const int nx = int(p->xfer.size());
    for (int slot = 0; slot < 5 + nx; slot++) {
        const int stage = slot < 5 ? slot : BF_STAGE_XFER0 + (slot - 5);
        if (p->uploaded[slot] < stage_blocks(p, stage))
            return fail(BF_ERR_STATE, "stage %d: %lld of %lld blocks uploaded", stage, (long long)p->uploaded[slot],
                        (long long)stage_blocks(p, stage));
    }
    DeviceGuard g(p->device);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(e, "finalize");
    p->finalized = true;
    return BF_OK;
}

bf_status_t bf_plan_create(const bf_desc_t* desc, int device, int64_t max_nrhs_chunk, bf_plan_t* out)
{
    bf_status_t st = validate_shape(desc);
    if (st != BF_OK) return st;
    const int nx = desc->log2n - 2 * desc->log2leaf;
    if (!desc->amp_a || !desc->amp_b || !desc->v0 || !desc->sw || !desc->u || (nx > 0 && !desc->xfer))
        return fail(BF_ERR_INVALID_ARG, "a factor array pointer is NULL");
    for (int i = 0; i < nx; i++)
        if (!desc->xfer[i]) return fail(BF_ERR_INVALID_ARG, "xfer[%d] is NULL", i);
    bf_plan_t p = nullptr;
    if ((st = bf_plan_alloc(desc, device, max_nrhs_chunk, &p)) != BF_OK) return st;
    const int mem = desc->memory;
    const int64_t N = p->d.N;
    if ((st = bf_plan_upload(p, BF_STAGE_AMP_A, 0, p->d.n_amp, desc->amp_a, mem)) ||
        (st = bf_plan_upload(p, BF_STAGE_AMP_B, 0, p->d.n_amp, desc->amp_b, mem)) ||
        (st = bf_plan_upload(p, BF_STAGE_V0, 0, N, desc->v0, mem)) ||
        (st = bf_plan_upload(p, BF_STAGE_SW, 0, N, desc->sw, mem)) ||
        (st = bf_plan_upload(p, BF_STAGE_U, 0, N, desc->u, mem))) {
        free_plan(p);
        return st;
    }
    for (int i = 0; i < nx; i++)
        if ((st = bf_plan_upload(p, BF_STAGE_XFER0 + i, 0, N, desc->xfer[i], mem))) {
            free_plan(p);
            return st;
        }
    if ((st = bf_plan_finalize(p))) {
        free_plan(p);
        return st;
    }
    *out = p;
    return BF_OK;
}

size_t bf_workspace_bytes(bf_plan_t p, int64_t nrhs_chunk)
{
    if (!p || nrhs_chunk < 1) return 0;
    return size_t(2) * size_t(p->d.N * p->d.R) * size_t(nrhs_chunk * p->d.n_amp) * sizeof(float2);
}

bf_status_t bf_apply_ex(bf_plan_t p, const bf_c64* F, int64_t ldf, bf_c64* G, int64_t ldg, int64_t nrhs,
                        void* workspace, size_t workspace_bytes, void* stream)
{
    if (!p) return fail(BF_ERR_INVALID_ARG, "plan is NULL");
    if (!p->finalized) return fail(BF_ERR_STATE, "plan not finalized");
    if (nrhs < 0) return fail(BF_ERR_INVALID_ARG, "nrhs=%lld < 0", (long long)nrhs);
    if (nrhs == 0) return BF_OK;
    if (!F || !G) return fail(BF_ERR_INVALID_ARG, "F or G is NULL");
    if (ldf < p->d.N || ldg < p->d.N)
        return fail(BF_ERR_ALIGNMENT, "ldf=%lld / ldg=%lld < N=%lld", (long long)ldf, (long long)ldg,
                    (long long)p->d.N);
    if ((reinterpret_cast<uintptr_t>(F) | reinterpret_cast<uintptr_t>(G)) % 8)
        return fail(BF_ERR_ALIGNMENT, "F/G not 8-byte aligned");
    float2* ws = p->ws;
    if (workspace) {
        if (reinterpret_cast<uintptr_t>(workspace) % 16) return fail(BF_ERR_ALIGNMENT, "workspace not 16-byte aligned");
        if (workspace_bytes < bf_workspace_bytes(p, std::min(nrhs, p->max_chunk)))
            return fail(BF_ERR_INVALID_ARG, "workspace of %zu B < %zu B", workspace_bytes,
                        bf_workspace_bytes(p, std::min(nrhs, p->max_chunk)));
        ws = static_cast<float2*>(workspace);
    }
    // F and G must not alias
    const char* f0 = reinterpret_cast<const char*>(F);
    const char* g0 = reinterpret_cast<const char*>(G);
    const size_t fb = size_t((nrhs - 1) * ldf + p->d.N) * 8, gb = size_t((nrhs - 1) * ldg + p->d.N) * 8;
    if (f0 < g0 + gb && g0 < f0 + fb) return fail(BF_ERR_INVALID_ARG, "F and G overlap");
    DeviceGuard g(p->device);
    return apply_impl(p, reinterpret_cast<const float2*>(F), ldf, reinterpret_cast<float2*>(G), ldg, nrhs, ws,
                      static_cast<cudaStream_t>(stream));
}

bf_status_t bf_apply(bf_plan_t p, const bf_c64* F, bf_c64* G, int64_t nrhs, void* stream)
{
    if (!p) return fail(BF_ERR_INVALID_ARG, "plan is NULL");
    return bf_apply_ex(p, F, p->d.N, G, p->d.N, nrhs, nullptr, 0, stream);
}

bf_status_t bf_apply_host(bf_plan_t p, const bf_c64* F_host, bf_c64* G_host, int64_t nrhs, void* stream)
{
    if (!p) return fail(BF_ERR_INVALID_ARG, "plan is NULL");
    if (!p->finalized) return fail(BF_ERR_STATE, "plan not finalized");
    if (nrhs < 0 || (nrhs > 0 && (!F_host || !G_host))) return fail(BF_ERR_INVALID_ARG, "bad arguments");
    if (nrhs == 0) return BF_OK;
    DeviceGuard g(p->device);
    const int64_t N = p->d.N, chunk = p->max_chunk;
    bf_status_t st;
    if (!p->dF && ((st = dalloc(&p->dF, N * chunk, "e2e F")) || (st = dalloc(&p->dG, N * chunk, "e2e G"))))
        return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    for (int64_t c0 = 0; c0 < nrhs; c0 += chunk) {
        const int64_t nc = std::min(chunk, nrhs - c0);
        const size_t bytes = size_t(N * nc) * sizeof(float2);
        cudaError_t e = cudaMemcpyAsync(p->dF, F_host + c0 * N, bytes, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return cuda_fail(e, "H2D");
        if ((st = apply_impl(p, p->dF, N, p->dG, N, nc, p->ws, s)) != BF_OK) return st;
        e = cudaMemcpyAsync(G_host + c0 * N, p->dG, bytes, cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) return cuda_fail(e, "D2H");
    }
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "bf_apply_host");
    return BF_OK;
}

bf_status_t bf_plan_get_info(bf_plan_t p, bf_plan_info_t* info)
{
    if (!p || !info) return fail(BF_ERR_INVALID_ARG, "NULL argument");
    const int64_t N = p->d.N, r = p->d.R, n0 = int64_t(1) << p->d.l0;
    const int nx = int(p->xfer.size());
    info->log2n = p->d.LN;
    info->log2leaf = p->d.l0;
    info->rank = p->d.R;
    info->n_amp = p->d.n_amp;
    info->switch_level = p->d.h;
    info->n_xfer = nx;
    info->n = N;
    info->max_nrhs_chunk = p->max_chunk;
    info->factor_bytes = 8 * (2 * p->d.n_amp * N + 2 * N * r * n0 + N * r * r + int64_t(nx) * N * 2 * r * r);
    info->workspace_bytes = int64_t(p->ws_bytes);
    const auto st = schedule(p->d, int(p->max_chunk * p->d.n_amp));
    info->launches_per_chunk = int32_t(st.size());
    for (int i = 0; i < BF_NUM_KCLASS; i++) info->class_launches[i] = info->class_levels[i] = 0;
    for (const auto& x : st) {
        info->class_launches[x.cls] += 1;
        info->class_levels[x.cls] += x.levels;
    }
    info->device = p->device;
    return BF_OK;
}

bf_status_t bf_plan_set_timing(bf_plan_t p, int32_t enable)
{
    if (!p) return fail(BF_ERR_INVALID_ARG, "plan is NULL");
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
    cudaError_t e = cudaSuccess;
    {
        DeviceGuard g(p->device);
        if (p->done) e = cudaEventSynchronize(p->done);
    }
    free_plan(p);
    if (e != cudaSuccess) return cuda_fail(e, "outstanding work failed");
    return BF_OK;
}

}  // extern "C"
