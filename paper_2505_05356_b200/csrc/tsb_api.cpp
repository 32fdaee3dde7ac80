// C-ABI implementation (include/tsb.h): contexts, device scenes, reusable
// render-pass workspaces, fused Adam, NCCL gradient reduction.
//
// Host code only; every device operation is stream-ordered.  A render pass
// never waits for the device inside prepare/forward/backward: every depth chunk
// is enqueued and decides on the device whether it has work (tsb_bin.cu
// chunk_live), and the frame's abort word (list-storage overflow, over-long
// fp32 tie run) is read back asynchronously.  The pass is *settled* -- synchronised,
// and on an abort redone with more storage / the exact sort -- before anything
// observes its results or changes what it read (settle / settle_all).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <string>
#include <vector>

#include "tsb_internal.h"

using namespace tsb;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define TSB_CUDA(expr)                                                                      \
    do {                                                                                    \
        cudaError_t e_ = (expr);                                                            \
        if (e_ != cudaSuccess)                                                              \
            return fail(e_ == cudaErrorMemoryAllocation ? TSB_ERR_NOMEM : TSB_ERR_CUDA,     \
                        std::string(#expr) + ": " + cudaGetErrorString(e_));                \
    } while (0)

#define TSB_CHECK_LAUNCH()                                                                  \
    do {                                                                                    \
        cudaError_t e_ = cudaGetLastError();                                                \
        if (e_ != cudaSuccess) return fail(TSB_ERR_CUDA, std::string("kernel launch: ") +  \
                                                             cudaGetErrorString(e_));       \
    } while (0)

template <typename T>
int dev_alloc(T** p, size_t count) {
    *p = nullptr;
    if (count == 0) count = 1;
    cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
    if (e != cudaSuccess) return fail(TSB_ERR_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    return TSB_OK;
}

template <typename T>
void dev_free(T*& p) {
    if (p) cudaFree((void*)p);
    p = nullptr;
}

}  // namespace

namespace tsb {
// error reporting for the host-only TUs (tsb_io.cpp)
int io_fail(int code, const std::string& msg) { return fail(code, msg); }
}  // namespace tsb

struct tsb_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int64_t launches = 0;
    void* pinned = nullptr;  // small pinned staging (K, V readback)
    // stage profiling: event pairs recorded on `stream`
    bool profiling = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    std::vector<std::pair<int, size_t>> ev_marks;  // (stage, index of start event)
    std::vector<tsb_pass*> passes;                 // joined by tsb_ctx_join
    int64_t redos = 0;                             // frames redone after a device-side abort
    unsigned long long* work = nullptr;            // raster work counters (profiling)
    bool use_graphs = true;                        // forward as a CUDA graph (TSB_NO_GRAPHS=1 disables)
    // nearest-prefix cap learned by any pass of the context (a pass whose prefix ran out
    // grows it; the others start their next frame from it instead of rediscovering it)
    int kcap_learned = 0;
    bool prefix_off = false;  // some pass needed the full order at every cap
};

namespace {
// RAII stage marker: records a start event on construction and a stop event on
// destruction, both on the context stream (only when profiling is enabled).
struct Stage {
    tsb_ctx* c;
    int stage;
    size_t idx = 0;
    bool on;
    cudaStream_t stream;
    static bool debug_sync() {  // TSB_DEBUG_SYNC=1 (with TSB_NO_GRAPHS=1): each stage synchronised and checked
        static const bool on_ = std::getenv("TSB_DEBUG_SYNC") != nullptr;
        return on_;
    }
    Stage(tsb_ctx* ctx, int s, cudaStream_t st) : c(ctx), stage(s), on(ctx->profiling), stream(st) {
        if (!on) return;
        if (c->ev_used + 2 > c->ev_pool.size()) {
            for (int i = 0; i < 64; ++i) {
                cudaEvent_t e;
                cudaEventCreate(&e);
                c->ev_pool.push_back(e);
            }
        }
        idx = c->ev_used;
        c->ev_used += 2;
        cudaEventRecord(c->ev_pool[idx], stream);
    }
    ~Stage() {
        if (debug_sync()) {
            cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
            cudaStreamIsCapturing(stream, &cs);
            const cudaError_t e = cs == cudaStreamCaptureStatusNone ? cudaStreamSynchronize(stream) : cudaSuccess;
            if (e != cudaSuccess) std::fprintf(stderr, "tsb debug: stage %d failed: %s\n", stage, cudaGetErrorString(e));
        }
        if (!on) return;
        cudaEventRecord(c->ev_pool[idx + 1], stream);
        c->ev_marks.emplace_back(stage, idx);
    }
};
}  // namespace

struct tsb_scene {
    tsb_ctx* ctx = nullptr;
    tsb_scene_desc d{};
    int narrays = 0;
    float4* params = nullptr;
    float4* grads = nullptr;
    float4* m = nullptr;
    float4* v = nullptr;
    float* densify = nullptr;
    double* stats = nullptr;  // kStats: bg grads (quad 4*nf, phasor 2*nf) at kStatBg, loss at kStatLoss
    float* staging = nullptr; // 4n floats for host<->device (un)packing
    double* pcache = nullptr; // [7][n] doubles: cov3d (6 planes) + opacity, then [6][n] floats: fp32 cov3d
                              // (SceneK::cov6 / opac / cov6f); kPcacheWords doubles per Gaussian
    int64_t step = 0;
    int64_t densify_count = 0;
    cudaEvent_t params_ev = nullptr;  // last parameter write (ctx stream)
    cudaEvent_t grads_ev = nullptr;   // last gradient/stats write (any stream)
};

struct tsb_pass {
    tsb_ctx* ctx = nullptr;
    cudaStream_t stream = nullptr;   // each pass runs on its own stream (frames overlap)
    cudaEvent_t done_ev = nullptr;   // recorded after every enqueue (tsb_ctx_join)
    // per scene this pass has read: an event after its last enqueue reading it (a parameter
    // upload waits for the readers of its own scene only)
    std::vector<std::pair<const tsb_scene*, cudaEvent_t>> scene_evs;
    cudaEvent_t fwd_ev = nullptr;    // end of the last forward (its abort word is final): settle waits here,
                                     // not for the frame's backward or downloads
    void* pinned = nullptr;          // per-pass pinned staging
    tsb_scene* scene = nullptr;
    CamK cam{};
    OptK opt{};
    FrameK frame{};
    uint32_t channels = 0;
    int nf = 1, W = 0, H = 0, ntiles = 0, nblocks = 0;
    bool prepared = false, forwarded = false, have_loss = false;
    int32_t V = -1;  // visible count (read back lazily)
    // capacities
    int n_cap = 0, px_cap = 0, blk_cap = 0, tiles_cap = 0;
    size_t temp_bytes = 0;

    // per Gaussian
    uint32_t *key_a = nullptr, *key_b = nullptr;  // fp32 depth keys
    double* depth64 = nullptr;
    uint32_t *gidx_a = nullptr, *gidx_b = nullptr;
    uint32_t* sorted = nullptr;  // global (depth, index) order: gidx_b, or gidx_a after the exact fallback
    uint32_t* order_dbg = nullptr;  // debug copy of the exact order (equal-key runs resolved)
    int order_dbg_cap = 0;
    uint32_t* touched = nullptr;
    uint2* rect = nullptr;
    RecK rec{};
    double* screen = nullptr;  // [8][n] screen-space gradients, accumulated in fp64 across blocks
    double* screen_keep = nullptr;  // debug copy of screen (tsb_pass_debug_keep_screen)
    bool keep_screen = false;
    // the rank order the raster blocks scan (ScanK): Gaussian and tile rect per rank
    uint32_t* ord = nullptr;
    uint2* trect = nullptr;
    // super-tile lists (ScanK::sl_*): per super-tile the ranks meeting it, in rank order
    uint32_t *sl_hist = nullptr, *sl_off = nullptr, *sl_rank = nullptr;
    uint2* sl_rect = nullptr;
    int sl_cap = 0, sl_hist_cap = 0, sl_off_cap = 0;
    int sup_x = 1, sup_log = 3, nsup = 1;
    bool sl_lists = false;  // the current frame's order is long enough for the lists (kSlMinRanks)
    bool force_lists = false;  // test hook (tsb_pass_debug_set_list_capacity): lists at any length
    int2* blk_term = nullptr;  // per raster block: where its forward scan stopped
    uint32_t* blk_list = nullptr;  // per raster block: the list entries its forward consumed (kBlkListCap)
    // deterministic backward (TSB_CH_DETERMINISTIC): slot offsets per rank, slots, fix-up pixel index
    uint32_t* det_off = nullptr;
    float* det_part = nullptr;
    size_t det_cap = 0;
    int det_off_cap = 0;
    int* fix_idx = nullptr;
    // per pixel
    float* out = nullptr;
    int32_t *n_contrib = nullptr, *n_processed = nullptr, *last = nullptr;
    float* T_pre = nullptr;
    float* d_quad = nullptr;
    float* up_extra = nullptr;  // [8][npx] host-uploaded upstreams: phasor (2*nf), depth_raw, weight, distortion, T
    double* dist3 = nullptr;    // [3][npx] distortion moments (PixK::dist3)
    float* target = nullptr;
    int32_t* flagged = nullptr;
    // misc
    int32_t* counters = nullptr;  // [0] n_visible, [1] n_flagged, [2] abort word, [4] prefix end, [5] key range
    // Nearest-prefix depth order (tsb_sort.cu): a frame sorts only its nearest kcap
    // Gaussians; one that runs past them is redone with the full order and the pass's
    // cap grows (x4, then the full sort).
    int kcap = 0;               // prefix cap of the next frames (0: full sort)
    bool prefix = false;        // the prepared frame's order is only a prefix
    int32_t* n_bin = nullptr;   // end of the sorted order: counters + 4 (prefix) or counters
    uint32_t *sel_keys = nullptr, *sel_vals = nullptr, *sel_scratch = nullptr;
    int sel_cap = 0;
    double* loss_part = nullptr;
    double* bg_part = nullptr;
    double* loss_dev = nullptr;
    float* chw = nullptr;
    uint32_t* sort_scratch = nullptr;
    // fp64 fix-up record cache
    int* fx_stamp = nullptr;
    int* fx_work = nullptr;
    int* fx_work_n = nullptr;
    Rec64* fx_cache = nullptr;
    FixState* fx_state = nullptr;  // [fx_state_cap] fp64 end state of recomposited pixels (k_fixup_bwd)
    int fx_state_cap = 0;
    double* out64 = nullptr;       // TSB_CH_EXACT: fp64 output planes (out64_cap pixels)
    double* ext_out64 = nullptr;   // TSB_CH_EXACT with colour / flow: [9][H][W]
    int out64_cap = 0, ext_out64_cap = 0;
    int frame_stamp = 0;
    // deferred settle: what was enqueued since the last check of the abort word
    bool pending = false;
    bool pend_loss = false, pend_bwd = false;
    const float* pend_target = nullptr;
    ChW pend_chw{};
    double pend_mix = 0.0;
    double pend_chw_full[8] = {0};  // the loss's channel weights before the (1 - lambda) mse scaling
    double mix = 0.0;          // SSIM weight of the current forward's image loss
    double* ssim_g = nullptr;  // SSIM gradient planes [4 * nf][3][npx]
    double* ssim_part = nullptr;
    int ssim_cap_px = 0, ssim_cap_blocks = 0;
    UpK pend_up{};
    struct Download {
        int which;
        void* host;
        size_t bytes;
    };
    std::vector<Download> pend_dl;  // asynchronous output downloads of the unsettled frame
    // forward CUDA graph, rebuilt when forward_key changes
    cudaStream_t cap_stream = nullptr;
    FrameDev* frame_dev = nullptr;
    struct FwdGraph {
        cudaGraphExec_t exec = nullptr;
        std::string key;
        int fixed = 0;
    };
    FwdGraph fwd[2];            // [0]: forward only, [1]: deferred prepare + forward
    // colour / flow channels (tsb_ext.cu), allocated on first use
    float4 *ext_col = nullptr, *ext_mf = nullptr, *ext_mb = nullptr, *ext_dmotion = nullptr;
    float *ext_out = nullptr, *ext_screen = nullptr, *ext_up = nullptr;
    double* ext_bg_part = nullptr;
    float *ext_dmacc = nullptr, *ext_ftgt = nullptr;  // flow loss: d_motion_*_acc [6][npx], targets [6][npx]
    double *ext_fl_part = nullptr, *ext_fl_res = nullptr;
    bool fl_grad[2] = {false, false};
    int ext_n_cap = 0, ext_px_cap = 0, ext_blk_cap = 0;
    bool has_mf = false, has_mb = false;
    bool prep_deferred = false; // prepare's device work not issued yet
};

namespace {
constexpr size_t kFrameSlot = 3072;  // FrameDev staging offset in tsb_pass::pinned
constexpr int kPrefixCap0 = 4096;   // initial nearest-prefix cap of the depth order (c3 terminates within ~3 K ranks)
}

extern "C" {

const char* tsb_last_error(void) { return g_err.c_str(); }
int tsb_abi_version(void) { return TSB_ABI_VERSION; }

int tsb_ctx_create(int device, tsb_ctx** out) {
    if (!out) return fail(TSB_ERR_INVALID, "tsb_ctx_create: out is null");
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        return fail(TSB_ERR_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    if (device < 0 || device >= count) return fail(TSB_ERR_INVALID, "tsb_ctx_create: bad device index");
    cudaDeviceProp prop;
    TSB_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
        return fail(TSB_ERR_CUDA, "tsb_ctx_create: device is not sm_100 (B200); this build has no other path");
    TSB_CUDA(cudaSetDevice(device));
    tsb_ctx* c = new tsb_ctx();
    c->device = device;
    if (const char* ng = std::getenv("TSB_NO_GRAPHS")) c->use_graphs = !(ng[0] == '1');
    e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete c;
        return fail(TSB_ERR_CUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
    }
    e = cudaMallocHost(&c->pinned, 4096);
    if (e == cudaSuccess) e = cudaMalloc(&c->work, 4 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemset(c->work, 0, 4 * sizeof(unsigned long long));
    if (e != cudaSuccess) {
        cudaStreamDestroy(c->stream);
        delete c;
        return fail(TSB_ERR_NOMEM, "cudaMallocHost failed");
    }
    *out = c;
    return TSB_OK;
}

int tsb_ctx_set_profiling(tsb_ctx* c, int enabled) {
    if (!c) return fail(TSB_ERR_INVALID, "null context");
    c->profiling = enabled != 0;
    return TSB_OK;
}

int tsb_ctx_stage_times(tsb_ctx* c, double* ms, int64_t* calls) {
    if (!c) return fail(TSB_ERR_INVALID, "null context");
    TSB_CUDA(cudaStreamSynchronize(c->stream));
    for (int i = 0; i < TSB_NUM_STAGES; ++i) {
        if (ms) ms[i] = 0.0;
        if (calls) calls[i] = 0;
    }
    for (const auto& m : c->ev_marks) {
        float t = 0.f;
        TSB_CUDA(cudaEventElapsedTime(&t, c->ev_pool[m.second], c->ev_pool[m.second + 1]));
        if (ms) ms[m.first] += t;
        if (calls) calls[m.first] += 1;
    }
    c->ev_marks.clear();
    c->ev_used = 0;
    return TSB_OK;
}

void tsb_ctx_destroy(tsb_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    cudaFreeHost(c->pinned);
    if (c->work) cudaFree(c->work);
    cudaStreamDestroy(c->stream);
    delete c;
}

int tsb_ctx_raster_counts(tsb_ctx* c, int64_t* evaluations, int64_t* contributions) {
    if (!c) return fail(TSB_ERR_INVALID, "null context");
    int rc = tsb_ctx_synchronize(c);
    if (rc) return rc;
    unsigned long long h[2];
    TSB_CUDA(cudaMemcpy(h, c->work, sizeof h, cudaMemcpyDeviceToHost));
    TSB_CUDA(cudaMemset(c->work, 0, sizeof h));
    if (evaluations) *evaluations = (int64_t)h[0];
    if (contributions) *contributions = (int64_t)h[1];
    return TSB_OK;
}

int tsb_ctx_scan_counts(tsb_ctx* c, int64_t* ranks, int64_t* list_entries) {
    if (!c) return fail(TSB_ERR_INVALID, "null context");
    int rc = tsb_ctx_synchronize(c);
    if (rc) return rc;
    unsigned long long h[2];
    TSB_CUDA(cudaMemcpy(h, c->work + 2, sizeof h, cudaMemcpyDeviceToHost));
    TSB_CUDA(cudaMemset(c->work + 2, 0, sizeof h));
    if (ranks) *ranks = (int64_t)h[0];
    if (list_entries) *list_entries = (int64_t)h[1];
    return TSB_OK;
}

namespace {
int settle(tsb_pass* p);
int flush_prepare(tsb_pass* p);
// done_ev, and the event of the pass's scene (the enqueued work may read it)
cudaError_t record_done(tsb_pass* p, cudaStream_t st) {
    cudaError_t e = cudaEventRecord(p->done_ev, st);
    if (e != cudaSuccess || !p->scene) return e;
    for (auto& se : p->scene_evs)
        if (se.first == p->scene) return cudaEventRecord(se.second, st);
    cudaEvent_t ev;
    if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return e;
    p->scene_evs.push_back({p->scene, ev});
    return cudaEventRecord(ev, st);
}
// The context stream waits for every enqueue that read scene s (passes prepared with s are
// settled first: a redone frame must see the parameters it was prepared with).
int scene_join(tsb_scene* s) {
    tsb_ctx* c = s->ctx;
    for (tsb_pass* p : c->passes) {
        if (p->scene == s) {
            int rc = flush_prepare(p);
            if (!rc) rc = settle(p);
            if (rc) return rc;
        }
        for (auto& se : p->scene_evs)
            if (se.first == s) TSB_CUDA(cudaStreamWaitEvent(c->stream, se.second, 0));
    }
    return TSB_OK;
}
int settle_all(tsb_ctx* c) {
    for (tsb_pass* p : c->passes) {
        int rc = flush_prepare(p);  // a prepared frame reads the scene as it is now
        if (!rc) rc = settle(p);
        if (rc) return rc;
    }
    return TSB_OK;
}
}  // namespace

int tsb_ctx_join(tsb_ctx* c) {
    if (!c) return fail(TSB_ERR_INVALID, "null context");
    int rc = settle_all(c);
    if (rc) return rc;
    for (tsb_pass* p : c->passes) TSB_CUDA(cudaStreamWaitEvent(c->stream, p->done_ev, 0));
    return TSB_OK;
}

int64_t tsb_ctx_redo_count(tsb_ctx* c) { return c ? c->redos : 0; }

int tsb_ctx_synchronize(tsb_ctx* c) {
    int rc = tsb_ctx_join(c);
    if (rc) return rc;
    TSB_CUDA(cudaStreamSynchronize(c->stream));
    return TSB_OK;
}

void* tsb_ctx_stream(tsb_ctx* c) { return c ? (void*)c->stream : nullptr; }
void* tsb_pass_stream(tsb_pass* p) { return p ? (void*)p->stream : nullptr; }
int64_t tsb_ctx_launch_count(tsb_ctx* c) { return c ? c->launches : 0; }

// ---------------------------------------------------------------------------
// scene
// ---------------------------------------------------------------------------
namespace {
SceneK scenek(const tsb_scene* s);
int color_base(const tsb_scene* s);
// Refresh the time-independent cache after a parameter change (ctx stream).
int refresh_param_cache(tsb_scene* s) {
    const SceneK S = scenek(s);
    launch_param_cache(S, s->pcache, s->pcache + 6 * (size_t)s->d.n,
                       reinterpret_cast<float*>(s->pcache + 7 * (size_t)s->d.n), s->ctx->stream);
    if (s->d.n > 0) s->ctx->launches++;
    TSB_CHECK_LAUNCH();
    return TSB_OK;
}
}  // namespace

int tsb_scene_create(tsb_ctx* ctx, const tsb_scene_desc* d, tsb_scene** out) {
    if (!ctx || !d || !out) return fail(TSB_ERR_INVALID, "tsb_scene_create: null argument");
    *out = nullptr;
    if (d->n < 0) return fail(TSB_ERR_INVALID, "scene: negative Gaussian count");
    if (d->n_keyframes < 0 || d->n_keyframes == 1 || d->n_keyframes > kMaxKeyframes)
        return fail(TSB_ERR_INVALID, "scene: n_keyframes must be 0 or in [2, 16]");
    if (d->sh_degree < 0 || d->sh_degree > 3) return fail(TSB_ERR_INVALID, "scene: sh_degree must be in [0, 3]");
    if (d->n_freq < 1 || d->n_freq > 2) return fail(TSB_ERR_INVALID, "scene: n_freq must be 1 or 2");
    for (int f = 0; f < d->n_freq; ++f)
        if (!(d->frequency[f] > 0.0)) return fail(TSB_ERR_INVALID, "scene: modulation frequency must be > 0");
    if (!(d->source_intensity > 0.0) || !(d->speed_of_light > 0.0))
        return fail(TSB_ERR_INVALID, "scene: invalid ToF config");
    TSB_CUDA(cudaSetDevice(ctx->device));
    tsb_scene* s = new tsb_scene();
    s->ctx = ctx;
    s->d = *d;
    if (d->color != 0 && d->color != 1) return fail(TSB_ERR_INVALID, "scene: color must be 0 or 1");
    s->narrays = 3 + d->n_keyframes + (d->sh_degree > 0 ? 4 : 0) + (d->color ? kColorArrays : 0);
    const size_t nel = (size_t)s->narrays * (size_t)std::max(d->n, 1);
    int rc = TSB_OK;
    if ((rc = dev_alloc(&s->params, nel)) || (rc = dev_alloc(&s->grads, nel)) || (rc = dev_alloc(&s->m, nel)) ||
        (rc = dev_alloc(&s->v, nel)) || (rc = dev_alloc(&s->densify, (size_t)std::max(d->n, 1))) ||
        (rc = dev_alloc(&s->stats, kStats)) || (rc = dev_alloc(&s->staging, 4 * (size_t)std::max(d->n, 1))) ||
        (rc = dev_alloc(&s->pcache, kPcacheWords * (size_t)std::max(d->n, 1)))) {
        tsb_scene_destroy(s);
        return rc;
    }
    cudaStream_t st = ctx->stream;
    if (cudaEventCreateWithFlags(&s->params_ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&s->grads_ev, cudaEventDisableTiming) != cudaSuccess) {
        tsb_scene_destroy(s);
        return fail(TSB_ERR_CUDA, "tsb_scene_create: event creation failed");
    }
    cudaMemsetAsync(s->params, 0, nel * sizeof(float4), st);
    cudaMemsetAsync(s->grads, 0, nel * sizeof(float4), st);
    cudaMemsetAsync(s->m, 0, nel * sizeof(float4), st);
    cudaMemsetAsync(s->v, 0, nel * sizeof(float4), st);
    cudaMemsetAsync(s->densify, 0, sizeof(float) * std::max(d->n, 1), st);
    cudaMemsetAsync(s->stats, 0, sizeof(double) * kStats, st);
    if (int rc2 = refresh_param_cache(s)) {
        tsb_scene_destroy(s);
        return rc2;
    }
    cudaEventRecord(s->params_ev, st);
    cudaEventRecord(s->grads_ev, st);
    TSB_CUDA(cudaStreamSynchronize(st));
    *out = s;
    return TSB_OK;
}

void tsb_scene_destroy(tsb_scene* s) {
    if (!s) return;
    cudaSetDevice(s->ctx->device);
    cudaStreamSynchronize(s->ctx->stream);
    dev_free(s->params);
    dev_free(s->grads);
    dev_free(s->m);
    dev_free(s->v);
    dev_free(s->densify);
    dev_free(s->stats);
    dev_free(s->staging);
    dev_free(s->pcache);
    if (s->params_ev) cudaEventDestroy(s->params_ev);
    if (s->grads_ev) cudaEventDestroy(s->grads_ev);
    delete s;
}

namespace {

// Pack one SoA parameter array (comps floats per Gaussian) into lanes
// comp0..comp0+comps-1 of float4 array `dst`.
int pack_one(tsb_scene* s, float4* dst, const float* src, int where, int comps, int comp0) {
    const int n = s->d.n;
    if (n == 0 || !src) return TSB_OK;
    cudaStream_t st = s->ctx->stream;
    const float* dsrc = src;
    if (where == TSB_HOST) {
        TSB_CUDA(cudaMemcpyAsync(s->staging, src, sizeof(float) * comps * (size_t)n, cudaMemcpyHostToDevice, st));
        dsrc = s->staging;
    }
    launch_pack_params(dst, dsrc, n, comps, comp0, 4, st);
    s->ctx->launches++;
    TSB_CHECK_LAUNCH();
    // (the next component's copy into the staging buffer is ordered after this pack on the
    // same stream; callers that return to the host sync once at the end)
    return TSB_OK;
}

int unpack_one(tsb_scene* s, const float4* src, float* host, int comps, int comp0) {
    const int n = s->d.n;
    if (n == 0 || !host) return TSB_OK;
    cudaStream_t st = s->ctx->stream;
    launch_unpack(src, s->staging, n, comps, comp0, st);
    s->ctx->launches++;
    TSB_CHECK_LAUNCH();
    TSB_CUDA(cudaMemcpyAsync(host, s->staging, sizeof(float) * comps * (size_t)n, cudaMemcpyDeviceToHost, st));
    TSB_CUDA(cudaStreamSynchronize(st));
    return TSB_OK;
}

}  // namespace


int tsb_scene_set_params(tsb_scene* s, int where, const float* position, const float* log_scale,
                         const float* rotation, const float* opacity_logit, const float* reflectivity_dc,
                         const float* motion) {
    if (!s) return fail(TSB_ERR_INVALID, "null scene");
    if (where != TSB_HOST && where != TSB_DEVICE) return fail(TSB_ERR_INVALID, "bad memory kind");
    TSB_CUDA(cudaSetDevice(s->ctx->device));
    const int n = s->d.n;
    int rc;
    if ((rc = scene_join(s))) return rc;  // passes may still be reading this scene's parameters
    if ((rc = pack_one(s, s->params, position, where, 3, 0))) return rc;
    if ((rc = pack_one(s, s->params, opacity_logit, where, 1, 3))) return rc;
    if ((rc = pack_one(s, s->params + n, log_scale, where, 3, 0))) return rc;
    if ((rc = pack_one(s, s->params + n, reflectivity_dc, where, 1, 3))) return rc;
    if ((rc = pack_one(s, s->params + 2 * (size_t)n, rotation, where, 4, 0))) return rc;
    if (motion)
        for (int k = 0; k < s->d.n_keyframes; ++k)
            if ((rc = pack_one(s, s->params + (size_t)(3 + k) * n, motion + (size_t)k * 3 * n, where, 3, 0)))
                return rc;
    if ((rc = refresh_param_cache(s))) return rc;
    TSB_CUDA(cudaEventRecord(s->params_ev, s->ctx->stream));
    // host sources are read by asynchronous copies: they are free again on return
    if (where == TSB_HOST) TSB_CUDA(cudaStreamSynchronize(s->ctx->stream));
    return TSB_OK;
}

int tsb_scene_get_params(tsb_scene* s, float* position, float* log_scale, float* rotation, float* opacity_logit,
                         float* reflectivity_dc, float* motion) {
    if (!s) return fail(TSB_ERR_INVALID, "null scene");
    TSB_CUDA(cudaSetDevice(s->ctx->device));
    const int n = s->d.n;
    int rc;
    if ((rc = unpack_one(s, s->params, position, 3, 0))) return rc;
    if ((rc = unpack_one(s, s->params, opacity_logit, 1, 3))) return rc;
    if ((rc = unpack_one(s, s->params + n, log_scale, 3, 0))) return rc;
    if ((rc = unpack_one(s, s->params + n, reflectivity_dc, 1, 3))) return rc;
    if ((rc = unpack_one(s, s->params + 2 * (size_t)n, rotation, 4, 0))) return rc;
    if (motion)
        for (int k = 0; k < s->d.n_keyframes; ++k)
            if ((rc = unpack_one(s, s->params + (size_t)(3 + k) * n, motion + (size_t)k * 3 * n, 3, 0))) return rc;
    return TSB_OK;
}

int tsb_scene_get_grads(tsb_scene* s, float* d_position, float* d_log_scale, float* d_rotation,
                        float* d_opacity_logit, float* d_reflectivity_dc, float* d_motion, double* d_bg_quad,
                        double* loss) {
    if (!s) return fail(TSB_ERR_INVALID, "null scene");
    {
        int rc0 = settle_all(s->ctx);
        if (rc0) return rc0;
    }
    TSB_CUDA(cudaSetDevice(s->ctx->device));
    const int n = s->d.n;
    int rc;
    TSB_CUDA(cudaStreamWaitEvent(s->ctx->stream, s->grads_ev, 0));
    if ((rc = unpack_one(s, s->grads, d_position, 3, 0))) return rc;
    if ((rc = unpack_one(s, s->grads, d_opacity_logit, 1, 3))) return rc;
    if ((rc = unpack_one(s, s->grads + n, d_log_scale, 3, 0))) return rc;
    if ((rc = unpack_one(s, s->grads + n, d_reflectivity_dc, 1, 3))) return rc;
    if ((rc = unpack_one(s, s->grads + 2 * (size_t)n, d_rotation, 4, 0))) return rc;
    if (d_motion)
        for (int k = 0; k < s->d.n_keyframes; ++k)
            if ((rc = unpack_one(s, s->grads + (size_t)(3 + k) * n, d_motion + (size_t)k * 3 * n, 3, 0))) return rc;
    double st[kStats];
    TSB_CUDA(cudaMemcpyAsync(st, s->stats, sizeof st, cudaMemcpyDeviceToHost, s->ctx->stream));
    TSB_CUDA(cudaStreamSynchronize(s->ctx->stream));
    if (d_bg_quad) std::memcpy(d_bg_quad, st + kStatBg, sizeof(double) * 4 * s->d.n_freq);
    if (loss) *loss = st[kStatLoss];
    return TSB_OK;
}

int tsb_scene_get_bg_grads(tsb_scene* s, double* d_bg_quad, double* d_bg_phasor) {
    if (!s) return fail(TSB_ERR_INVALID, "null scene");
    {
        int rc0 = settle_all(s->ctx);
        if (rc0) return rc0;
    }
    TSB_CUDA(cudaSetDevice(s->ctx->device));
    TSB_CUDA(cudaStreamWaitEvent(s->ctx->stream, s->grads_ev, 0));
    double st[kStats];
    TSB_CUDA(cudaMemcpyAsync(st, s->stats, sizeof st, cudaMemcpyDeviceToHost, s->ctx->stream));
    TSB_CUDA(cudaStreamSynchronize(s->ctx->stream));
    const int nf = s->d.n_freq;
    if (d_bg_quad) std::memcpy(d_bg_quad, st + kStatBg, sizeof(double) * 4 * nf);
    if (d_bg_phasor) std::memcpy(d_bg_phasor, st + kStatBg + 4 * nf, sizeof(double) * 2 * nf);
    return TSB_OK;
}

int tsb_scene_set_sh(tsb_scene* s, int where, const float* refl_sh) {
    if (!s || !refl_sh) return fail(TSB_ERR_INVALID, "tsb_scene_set_sh: null argument");
    if (s->d.sh_degree == 0) return fail(TSB_ERR_INVALID, "tsb_scene_set_sh: scene has sh_degree 0");
    if (where != TSB_HOST && where != TSB_DEVICE) return fail(TSB_ERR_INVALID, "bad memory kind");
    TSB_CUDA(cudaSetDevice(s->ctx->device));
    int rc;
    if ((rc = tsb_ctx_join(s->ctx))) return rc;
    const int n = s->d.n;
    if (n == 0) return TSB_OK;
    cudaStream_t st = s->ctx->stream;
    const float* src = refl_sh;
    float* tmp = nullptr;
    if (where == TSB_HOST) {
        if ((rc = dev_alloc(&tmp, (size_t)16 * n))) return rc;
        TSB_CUDA(cudaMemcpyAsync(tmp, refl_sh, sizeof(float) * 16 * (size_t)n, cudaMemcpyHostToDevice, st));
        src = tmp;
    }
    launch_pack_sh(s->params + (3 + (size_t)s->d.n_keyframes) * n, s->params + n, src, n, st);
    s->ctx->launches += 1;
    TSB_CHECK_LAUNCH();
    TSB_CUDA(cudaStreamSynchronize(st));
    if (tmp) cudaFree(tmp);
    TSB_CUDA(cudaEventRecord(s->params_ev, st));
    return TSB_OK;
}

int tsb_scene_get_sh(tsb_scene* s, float* refl_sh, int grads) {
    if (!s || !refl_sh) return fail(TSB_ERR_INVALID, "tsb_scene_get_sh: null argument");
    if (grads) {
        int rc0 = settle_all(s->ctx);
        if (rc0) return rc0;
    }
    TSB_CUDA(cudaSetDevice(s->ctx->device));
    const int n = s->d.n;
    if (n == 0) return TSB_OK;
    cudaStream_t st = s->ctx->stream;
    const float4* base = grads ? s->grads : s->params;
    if (grads) TSB_CUDA(cudaStreamWaitEvent(st, s->grads_ev, 0));
    float* tmp = nullptr;
    int rc;
    if ((rc = dev_alloc(&tmp, (size_t)16 * n))) return rc;
    TSB_CUDA(cudaMemsetAsync(tmp, 0, sizeof(float) * 16 * (size_t)n, st));
    if (s->d.sh_degree > 0) launch_unpack_sh(base + (3 + (size_t)s->d.n_keyframes) * n, tmp, n, st);
    s->ctx->launches += 1;
    TSB_CUDA(cudaMemcpyAsync(refl_sh, tmp, sizeof(float) * 16 * (size_t)n, cudaMemcpyDeviceToHost, st));
    TSB_CUDA(cudaStreamSynchronize(st));
    cudaFree(tmp);
    // coefficient 0 from scale_amp.w
    std::vector<float> dc(n);
    if ((rc = unpack_one(s, base + n, dc.data(), 1, 3))) return rc;
    for (int i = 0; i < n; ++i) refl_sh[16 * (size_t)i] = dc[i];
    return TSB_OK;
}

int tsb_scene_set_color(tsb_scene* s, int where, const float* color_sh) {
    if (s && s->d.n == 0 && s->d.color) return TSB_OK;  // nothing to copy (empty vector data may be null)
    if (!s || !color_sh) return fail(TSB_ERR_INVALID, "tsb_scene_set_color: null argument");
    if (!s->d.color) return fail(TSB_ERR_INVALID, "tsb_scene_set_color: scene was created without colour");
    if (where != TSB_HOST && where != TSB_DEVICE) return fail(TSB_ERR_INVALID, "bad memory kind");
    TSB_CUDA(cudaSetDevice(s->ctx->device));
    int rc;
    if ((rc = tsb_ctx_join(s->ctx))) return rc;
    const int n = s->d.n;
    if (n == 0) return TSB_OK;
    cudaStream_t st = s->ctx->stream;
    const float* src = color_sh;
    float* tmp = nullptr;
    if (where == TSB_HOST) {
        if ((rc = dev_alloc(&tmp, (size_t)48 * n))) return rc;
        TSB_CUDA(cudaMemcpyAsync(tmp, color_sh, sizeof(float) * 48 * (size_t)n, cudaMemcpyHostToDevice, st));
        src = tmp;
    }
    launch_pack_rows(s->params + (size_t)color_base(s) * n, src, n, kColorArrays, 4, st);
    s->ctx->launches += 1;
    TSB_CHECK_LAUNCH();
    TSB_CUDA(cudaStreamSynchronize(st));
    if (tmp) cudaFree(tmp);
    TSB_CUDA(cudaEventRecord(s->params_ev, st));
    return TSB_OK;
}

int tsb_scene_get_color(tsb_scene* s, float* color_sh, int grads) {
    if (s && s->d.n == 0 && s->d.color) return TSB_OK;
    if (!s || !color_sh) return fail(TSB_ERR_INVALID, "tsb_scene_get_color: null argument");
    if (!s->d.color) return fail(TSB_ERR_INVALID, "tsb_scene_get_color: scene was created without colour");
    if (grads) {
        int rc0 = settle_all(s->ctx);
        if (rc0) return rc0;
    }
    TSB_CUDA(cudaSetDevice(s->ctx->device));
    const int n = s->d.n;
    if (n == 0) return TSB_OK;
    cudaStream_t st = s->ctx->stream;
    if (grads) TSB_CUDA(cudaStreamWaitEvent(st, s->grads_ev, 0));
    float* tmp = nullptr;
    int rc;
    if ((rc = dev_alloc(&tmp, (size_t)48 * n))) return rc;
    launch_unpack_rows((grads ? s->grads : s->params) + (size_t)color_base(s) * n, tmp, n, kColorArrays, 4, st);
    s->ctx->launches += 1;
    TSB_CUDA(cudaMemcpyAsync(color_sh, tmp, sizeof(float) * 48 * (size_t)n, cudaMemcpyDeviceToHost, st));
    TSB_CUDA(cudaStreamSynchronize(st));
    cudaFree(tmp);
    return TSB_OK;
}

int tsb_scene_get_bg_color_grad(tsb_scene* s, double* d_bg_color) {
    if (!s || !d_bg_color) return fail(TSB_ERR_INVALID, "null argument");
    {
        int rc0 = settle_all(s->ctx);
        if (rc0) return rc0;
    }
    TSB_CUDA(cudaSetDevice(s->ctx->device));
    TSB_CUDA(cudaStreamWaitEvent(s->ctx->stream, s->grads_ev, 0));
    double* h = d_bg_color;
    TSB_CUDA(cudaMemcpyAsync(h, s->stats + kStatBgColor, sizeof(double) * 3, cudaMemcpyDeviceToHost, s->ctx->stream));
    TSB_CUDA(cudaStreamSynchronize(s->ctx->stream));
    return TSB_OK;
}

int tsb_scene_zero_grads(tsb_scene* s) {
    if (!s) return fail(TSB_ERR_INVALID, "null scene");
    {
        int rc0 = settle_all(s->ctx);
        if (rc0) return rc0;
    }
    TSB_CUDA(cudaSetDevice(s->ctx->device));
    const size_t nel = (size_t)s->narrays * (size_t)std::max(s->d.n, 1);
    TSB_CUDA(cudaStreamWaitEvent(s->ctx->stream, s->grads_ev, 0));
    TSB_CUDA(cudaMemsetAsync(s->grads, 0, nel * sizeof(float4), s->ctx->stream));
    TSB_CUDA(cudaMemsetAsync(s->stats, 0, sizeof(double) * kStats, s->ctx->stream));
    TSB_CUDA(cudaEventRecord(s->grads_ev, s->ctx->stream));
    return TSB_OK;
}

int tsb_scene_get_adam_state(tsb_scene* s, float* m_position, float* v_position) {
    if (!s) return fail(TSB_ERR_INVALID, "null scene");
    int rc;
    if ((rc = unpack_one(s, s->m, m_position, 3, 0))) return rc;
    if ((rc = unpack_one(s, s->v, v_position, 3, 0))) return rc;
    return TSB_OK;
}

int tsb_scene_get_densify_stat(tsb_scene* s, float* grad_norm_sum, int64_t* count) {
    if (!s) return fail(TSB_ERR_INVALID, "null scene");
    {
        int rc0 = settle_all(s->ctx);
        if (rc0) return rc0;
    }
    TSB_CUDA(cudaSetDevice(s->ctx->device));
    if (grad_norm_sum && s->d.n > 0) {
        TSB_CUDA(cudaStreamWaitEvent(s->ctx->stream, s->grads_ev, 0));
        TSB_CUDA(cudaMemcpyAsync(grad_norm_sum, s->densify, sizeof(float) * s->d.n, cudaMemcpyDeviceToHost,
                                 s->ctx->stream));
        TSB_CUDA(cudaStreamSynchronize(s->ctx->stream));
    }
    if (count) *count = s->densify_count;
    return TSB_OK;
}

int tsb_scene_adam_step(tsb_scene* s, const tsb_adam_config* cfg) {
    if (!s || !cfg) return fail(TSB_ERR_INVALID, "tsb_scene_adam_step: null argument");
    TSB_CUDA(cudaSetDevice(s->ctx->device));
    {
        int rc = tsb_ctx_join(s->ctx);
        if (rc) return rc;
    }
    TSB_CUDA(cudaStreamWaitEvent(s->ctx->stream, s->grads_ev, 0));
    s->step += 1;
    const double t = (double)s->step;
    const double bc1 = 1.0 - std::pow(cfg->beta1, t);
    const double bc2 = 1.0 - std::pow(cfg->beta2, t);
    std::vector<double> lr((size_t)s->narrays * 4, 0.0);
    for (int c = 0; c < 3; ++c) lr[c] = cfg->position;
    lr[3] = cfg->opacity;
    for (int c = 0; c < 3; ++c) lr[4 + c] = cfg->log_scale;
    lr[7] = cfg->reflectivity;
    for (int c = 0; c < 4; ++c) lr[8 + c] = cfg->rotation;
    for (int k = 0; k < s->d.n_keyframes; ++k)
        for (int c = 0; c < 3; ++c) lr[(size_t)(3 + k) * 4 + c] = cfg->motion;
    if (s->d.sh_degree > 0)  // reflectivity SH coefficients 1..15 use the reflectivity rate
        for (int a = 0; a < 4; ++a)
            for (int c = 0; c < (a < 3 ? 4 : 3); ++c) lr[(size_t)(3 + s->d.n_keyframes + a) * 4 + c] = cfg->reflectivity;
    if (s->d.color)  // colour SH: LrTable::color (trainer.cpp:363-365)
        for (int a = 0; a < kColorArrays; ++a)
            for (int c = 0; c < 4; ++c) lr[(size_t)(color_base(s) + a) * 4 + c] = cfg->color;
    {
        Stage sg(s->ctx, TSB_STAGE_ADAM, s->ctx->stream);
        launch_adam(s->params, s->grads, s->m, s->v, s->d.n, s->narrays, lr.data(), cfg->beta1, cfg->beta2,
                    cfg->eps, bc1, bc2, s->densify, s->ctx->stream);
    }
    s->ctx->launches++;
    TSB_CHECK_LAUNCH();
    s->densify_count++;
    {
        int rc = refresh_param_cache(s);
        if (rc) return rc;
    }
    TSB_CUDA(cudaMemsetAsync(s->stats, 0, sizeof(double) * kStats, s->ctx->stream));
    TSB_CUDA(cudaEventRecord(s->params_ev, s->ctx->stream));
    TSB_CUDA(cudaEventRecord(s->grads_ev, s->ctx->stream));
    return TSB_OK;
}

int tsb_scene_densify(tsb_scene* s, const tsb_densify_config* cfg, double scene_extent, int32_t* n_new_out) {
    if (!s || !cfg) return fail(TSB_ERR_INVALID, "tsb_scene_densify: null argument");
    if (!(cfg->split_shrink > 0.0)) return fail(TSB_ERR_INVALID, "densify: split_shrink must be > 0");
    TSB_CUDA(cudaSetDevice(s->ctx->device));
    int rc = tsb_ctx_join(s->ctx);  // every pass is settled and has finished reading the scene
    if (rc) return rc;
    cudaStream_t st = s->ctx->stream;
    TSB_CUDA(cudaStreamWaitEvent(st, s->grads_ev, 0));
    const int n = s->d.n;
    const size_t nn = (size_t)std::max(n, 1);
    DensifyScratch w{};
    const size_t nb = nn / 1024 + 2;
    if ((rc = dev_alloc(&w.transparent, nn)) || (rc = dev_alloc(&w.tprefix, nn)) || (rc = dev_alloc(&w.keep, nn)) ||
        (rc = dev_alloc(&w.extra, nn)) || (rc = dev_alloc(&w.kpos, nn)) || (rc = dev_alloc(&w.epos, nn)) ||
        (rc = dev_alloc(&w.scan_tmp, nb)) || (rc = dev_alloc(&w.totals, 4)) || (rc = dev_alloc(&w.decision, nn))) {
        dev_free(w.transparent); dev_free(w.tprefix); dev_free(w.keep); dev_free(w.extra); dev_free(w.kpos);
        dev_free(w.epos); dev_free(w.scan_tmp); dev_free(w.totals); dev_free(w.decision);
        return rc;
    }
    DensifyK D{};
    D.grad_sum = s->densify;
    D.count = s->densify_count;
    D.grad_threshold = cfg->grad_threshold;
    D.opacity_floor = cfg->opacity_floor;
    D.split_scale = cfg->split_scale_fraction * scene_extent;
    D.split_shrink = cfg->split_shrink;
    D.min_count = cfg->min_count;
    const SceneK S = scenek(s);
    launch_densify_plan(S, D, w, st);
    s->ctx->launches += n > 0 ? 11 : 0;
    uint32_t tot[3] = {0, 0, 0};
    cudaError_t e = cudaMemcpyAsync(tot, w.totals, sizeof tot, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    const uint32_t n_kept = tot[0], n_extra = tot[1];
    const int n_new = (int)(n_kept + n_extra);
    float4 *P2 = nullptr, *G2 = nullptr, *M2 = nullptr, *V2 = nullptr;
    float *dens2 = nullptr, *stg2 = nullptr;
    double* pc2 = nullptr;
    const size_t nel2 = (size_t)s->narrays * (size_t)std::max(n_new, 1);
    if (e == cudaSuccess && !((rc = dev_alloc(&P2, nel2)) || (rc = dev_alloc(&G2, nel2)) || (rc = dev_alloc(&M2, nel2)) ||
                              (rc = dev_alloc(&V2, nel2)) || (rc = dev_alloc(&dens2, (size_t)std::max(n_new, 1))) ||
                              (rc = dev_alloc(&stg2, 4 * (size_t)std::max(n_new, 1))) ||
                              (rc = dev_alloc(&pc2, kPcacheWords * (size_t)std::max(n_new, 1))))) {
        launch_densify_scatter(S, D, w, n_kept, s->narrays, s->params, s->m, s->v, P2, M2, V2, n_new, st);
        s->ctx->launches += n > 0 ? 1 : 0;
        cudaMemsetAsync(G2, 0, nel2 * sizeof(float4), st);
        cudaMemsetAsync(dens2, 0, sizeof(float) * std::max(n_new, 1), st);
        e = cudaStreamSynchronize(st);
    }
    dev_free(w.transparent); dev_free(w.tprefix); dev_free(w.keep); dev_free(w.extra); dev_free(w.kpos);
    dev_free(w.epos); dev_free(w.scan_tmp); dev_free(w.totals); dev_free(w.decision);
    if (e != cudaSuccess || rc) {
        dev_free(P2); dev_free(G2); dev_free(M2); dev_free(V2); dev_free(dens2); dev_free(stg2); dev_free(pc2);
        if (rc) return rc;
        return fail(TSB_ERR_CUDA, std::string("densify: ") + cudaGetErrorString(e));
    }
    dev_free(s->params); dev_free(s->grads); dev_free(s->m); dev_free(s->v); dev_free(s->densify);
    dev_free(s->staging); dev_free(s->pcache);
    s->params = P2; s->grads = G2; s->m = M2; s->v = V2; s->densify = dens2; s->staging = stg2; s->pcache = pc2;
    s->d.n = n_new;
    s->densify_count = 0;
    TSB_CUDA(cudaMemsetAsync(s->stats, 0, sizeof(double) * kStats, st));
    if ((rc = refresh_param_cache(s))) return rc;
    TSB_CUDA(cudaEventRecord(s->params_ev, st));
    TSB_CUDA(cudaEventRecord(s->grads_ev, st));
    if (n_new_out) *n_new_out = n_new;
    return TSB_OK;
}

int tsb_adam_step_flat(tsb_ctx* ctx, int where, float* params, const float* grads, float* m, float* v, size_t n,
                       int64_t t, double lr, double beta1, double beta2, double eps) {
    if (!ctx || (n && (!params || !grads || !m || !v))) return fail(TSB_ERR_INVALID, "adam_step: null argument");
    if (t < 1) return fail(TSB_ERR_INVALID, "adam_step: step count must be >= 1");
    if (n == 0) return TSB_OK;
    TSB_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    const double bc1 = 1.0 - std::pow(beta1, (double)t), bc2 = 1.0 - std::pow(beta2, (double)t);
    if (where == TSB_DEVICE) {
        launch_adam_flat(params, grads, m, v, n, lr, beta1, beta2, eps, bc1, bc2, st);
        ctx->launches++;
        TSB_CHECK_LAUNCH();
        return TSB_OK;
    }
    if (where != TSB_HOST) return fail(TSB_ERR_INVALID, "bad memory kind");
    float* d = nullptr;
    int rc = dev_alloc(&d, 4 * n);
    if (rc) return rc;
    const size_t b = n * sizeof(float);
    cudaMemcpyAsync(d, params, b, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d + n, grads, b, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d + 2 * n, m, b, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d + 3 * n, v, b, cudaMemcpyHostToDevice, st);
    launch_adam_flat(d, d + n, d + 2 * n, d + 3 * n, n, lr, beta1, beta2, eps, bc1, bc2, st);
    ctx->launches++;
    cudaMemcpyAsync(params, d, b, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(m, d + 2 * n, b, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(v, d + 3 * n, b, cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    cudaFree(d);
    if (e != cudaSuccess) return fail(TSB_ERR_CUDA, std::string("adam_step: ") + cudaGetErrorString(e));
    return TSB_OK;
}

int tsb_adam_reindex_flat(tsb_ctx* ctx, int where, const float* m, const float* v, size_t n_old, const int32_t* src,
                          size_t n_new, int32_t stride, float* m_out, float* v_out) {
    if (!ctx || stride < 1 || (n_new && (!src || !m_out || !v_out)) || (n_old && (!m || !v)))
        return fail(TSB_ERR_INVALID, "adam_reindex: bad argument");
    if (where != TSB_HOST && where != TSB_DEVICE) return fail(TSB_ERR_INVALID, "bad memory kind");
    if (where == TSB_HOST)  // the device gather reads only valid sources
        for (size_t i = 0; i < n_new; ++i)
            if (src[i] >= (int64_t)n_old) return fail(TSB_ERR_INVALID, "adam_reindex: source index out of range");
    if (n_new == 0) return TSB_OK;
    TSB_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    const size_t S = (size_t)stride;
    if (where == TSB_DEVICE) {
        launch_adam_reindex(m, v, src, n_new, stride, m_out, v_out, st);
        ctx->launches++;
        TSB_CHECK_LAUNCH();
        return TSB_OK;
    }
    float* d = nullptr;
    int32_t* ds = nullptr;
    int rc;
    if ((rc = dev_alloc(&d, 2 * n_old * S + 2 * n_new * S + 1)) || (rc = dev_alloc(&ds, n_new))) {
        dev_free(d);
        return rc;
    }
    float *dm = d, *dv = d + n_old * S, *dm2 = d + 2 * n_old * S, *dv2 = dm2 + n_new * S;
    if (n_old) {
        cudaMemcpyAsync(dm, m, sizeof(float) * n_old * S, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(dv, v, sizeof(float) * n_old * S, cudaMemcpyHostToDevice, st);
    }
    cudaMemcpyAsync(ds, src, sizeof(int32_t) * n_new, cudaMemcpyHostToDevice, st);
    launch_adam_reindex(dm, dv, ds, n_new, stride, dm2, dv2, st);
    ctx->launches++;
    cudaMemcpyAsync(m_out, dm2, sizeof(float) * n_new * S, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(v_out, dv2, sizeof(float) * n_new * S, cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    dev_free(d);
    dev_free(ds);
    if (e != cudaSuccess) return fail(TSB_ERR_CUDA, std::string("adam_reindex: ") + cudaGetErrorString(e));
    return TSB_OK;
}

// ---------------------------------------------------------------------------
// render pass
// ---------------------------------------------------------------------------
int tsb_pass_create(tsb_ctx* ctx, tsb_pass** out) {
    if (!ctx || !out) return fail(TSB_ERR_INVALID, "tsb_pass_create: null argument");
    TSB_CUDA(cudaSetDevice(ctx->device));
    tsb_pass* p = new tsb_pass();
    p->ctx = ctx;
    if (cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->done_ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->fwd_ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaMallocHost(&p->pinned, 4096) != cudaSuccess) {
        tsb_pass_destroy(p);
        return fail(TSB_ERR_CUDA, "tsb_pass_create: stream/event/pinned allocation failed");
    }
    int rc;
    if ((rc = dev_alloc(&p->counters, 8)) || (rc = dev_alloc(&p->loss_dev, 1)) || (rc = dev_alloc(&p->chw, 8)) ||
        (rc = dev_alloc(&p->fx_work_n, 1)) || (rc = dev_alloc(&p->frame_dev, 1))) {
        tsb_pass_destroy(p);
        return rc;
    }
    p->n_bin = p->counters;
    static const int prefix_cap = [] {
        const char* e = std::getenv("TSB_PREFIX");  // initial prefix cap; 0 disables
        return e ? std::max(0, std::atoi(e)) : kPrefixCap0;
    }();
    p->kcap = prefix_cap;
    raster_init();
    ssim_init();
    ctx->passes.push_back(p);
    *out = p;
    return TSB_OK;
}

namespace {

void free_gauss(tsb_pass* p) {
    dev_free(p->key_a); dev_free(p->key_b); dev_free(p->gidx_a); dev_free(p->gidx_b);
    dev_free(p->depth64); dev_free(p->sort_scratch);
    dev_free(p->fx_stamp); dev_free(p->fx_work); dev_free(p->fx_cache);
    dev_free(p->touched); dev_free(p->rect);
    dev_free(p->rec.A); dev_free(p->rec.B); dev_free(p->rec.C); dev_free(p->rec.D); dev_free(p->screen); dev_free(p->screen_keep);
    dev_free(p->ord); dev_free(p->trect);
}
void free_super(tsb_pass* p) {
    dev_free(p->sl_hist); dev_free(p->sl_off); dev_free(p->sl_rank); dev_free(p->sl_rect);
    p->sl_cap = p->sl_hist_cap = p->sl_off_cap = 0;
}
void free_pixels(tsb_pass* p) {
    dev_free(p->out); dev_free(p->n_contrib); dev_free(p->n_processed); dev_free(p->last);
    dev_free(p->T_pre); dev_free(p->d_quad); dev_free(p->target); dev_free(p->flagged);
    dev_free(p->up_extra); dev_free(p->dist3);
    dev_free(p->fx_state); dev_free(p->fix_idx);
    p->fx_state_cap = 0;
    dev_free(p->out64); dev_free(p->ext_out64);
    p->out64_cap = p->ext_out64_cap = 0;
}

int ensure_gauss(tsb_pass* p, int n) {
    if (n <= p->n_cap) return TSB_OK;
    free_gauss(p);
    const int cap = std::max(n, 1);
    int rc;
    if ((rc = dev_alloc(&p->key_a, cap)) || (rc = dev_alloc(&p->key_b, cap)) || (rc = dev_alloc(&p->gidx_a, cap)) ||
        (rc = dev_alloc(&p->depth64, cap)) ||
        (rc = dev_alloc(&p->gidx_b, cap)) || (rc = dev_alloc(&p->touched, cap)) || (rc = dev_alloc(&p->rect, cap)) ||
        (rc = dev_alloc(&p->rec.A, cap)) || (rc = dev_alloc(&p->rec.B, cap)) || (rc = dev_alloc(&p->rec.C, cap)) ||
        (rc = dev_alloc(&p->rec.D, cap)) || (rc = dev_alloc(&p->screen, (size_t)8 * cap)) ||
        (rc = dev_alloc(&p->ord, cap)) || (rc = dev_alloc(&p->trect, cap)))
        return rc;
    p->rec.rect = p->rect;
    TSB_CUDA(cudaMemsetAsync(p->screen, 0, sizeof(double) * 8 * (size_t)cap, p->stream));
    p->n_cap = cap;
    if ((rc = dev_alloc(&p->sort_scratch, radix_sort_scratch_words(cap))) || (rc = dev_alloc(&p->fx_stamp, cap)) ||
        (rc = dev_alloc(&p->fx_work, cap)) || (rc = dev_alloc(&p->fx_cache, cap)))
        return rc;
    TSB_CUDA(cudaMemsetAsync(p->fx_stamp, 0, sizeof(int) * (size_t)cap, p->stream));
    p->frame_stamp = 0;
    return TSB_OK;
}

int ensure_pixels(tsb_pass* p, int W, int H, int ntiles, int nblocks) {
    const int npx = W * H;
    const int nch = out_channels(2);
    if (npx >= (1 << 24)) return fail(TSB_ERR_UNSUPPORTED, "render: more than 16M pixels");
    if (npx > p->px_cap) {
        free_pixels(p);
        int rc;
        if ((rc = dev_alloc(&p->out, (size_t)nch * npx)) || (rc = dev_alloc(&p->n_contrib, npx)) ||
            (rc = dev_alloc(&p->n_processed, npx)) || (rc = dev_alloc(&p->last, npx)) ||
            (rc = dev_alloc(&p->T_pre, npx)) || (rc = dev_alloc(&p->d_quad, (size_t)8 * npx)) ||
            (rc = dev_alloc(&p->target, (size_t)8 * npx)) || (rc = dev_alloc(&p->flagged, npx)) ||
            (rc = dev_alloc(&p->up_extra, (size_t)8 * npx)) || (rc = dev_alloc(&p->dist3, (size_t)3 * npx)) ||
            (rc = dev_alloc(&p->fx_state, std::min(npx, kFixStateCap))) || (rc = dev_alloc(&p->fix_idx, npx)))
            return rc;
        p->fx_state_cap = std::min(npx, kFixStateCap);
        p->px_cap = npx;
    }
    if (nblocks > p->blk_cap) {
        dev_free(p->loss_part);
        dev_free(p->bg_part);
        dev_free(p->blk_term);
        dev_free(p->blk_list);
        int rc;
        if ((rc = dev_alloc(&p->loss_part, nblocks)) || (rc = dev_alloc(&p->bg_part, (size_t)12 * nblocks)) ||
            (rc = dev_alloc(&p->blk_term, nblocks)) || (rc = dev_alloc(&p->blk_list, (size_t)kBlkListCap * nblocks)))
            return rc;
        TSB_CUDA(cudaMemsetAsync(p->blk_term, 0, sizeof(int2) * (size_t)nblocks, p->stream));
        p->blk_cap = nblocks;
    }
    (void)ntiles;
    return TSB_OK;
}

// Super-tile geometry of the current camera / tiling and the list storage: the histogram
// for n ranks, `entries` list entries (0: the default 2n + 64K; grown when a frame's
// lists overflow -- abort bit 1, settle()).
int ensure_super(tsb_pass* p, int n, int64_t entries) {
    int lg = 3;
    auto sups = [&](int l) {
        return ((p->opt.tiles_x + (1 << l) - 1) >> l) * ((p->opt.tiles_y + (1 << l) - 1) >> l);
    };
    while (sups(lg) > kSlMaxSup || ((p->opt.tiles_x + (1 << lg) - 1) >> lg) > kSlMaxSupSide ||
           ((p->opt.tiles_y + (1 << lg) - 1) >> lg) > kSlMaxSupSide)
        ++lg;
    p->sup_log = lg;
    p->sup_x = (p->opt.tiles_x + (1 << lg) - 1) >> lg;
    p->nsup = sups(lg);
    int rc;
    if (p->nsup * (kSlMaxBlocks + 1) > p->sl_hist_cap) {  // + the row totals
        dev_free(p->sl_hist); dev_free(p->sl_off);
        p->sl_hist_cap = p->sl_off_cap = 0;
        if ((rc = dev_alloc(&p->sl_hist, (size_t)p->nsup * (kSlMaxBlocks + 1))) ||
            (rc = dev_alloc(&p->sl_off, (size_t)p->nsup + 1)))
            return rc;
        p->sl_hist_cap = p->nsup * (kSlMaxBlocks + 1);
        p->sl_off_cap = p->nsup + 1;
    }
    static const int64_t cap0 = [] {  // TSB_SL_CAP: initial list capacity (tests of the overflow redo)
        const char* e = std::getenv("TSB_SL_CAP");
        return e ? (int64_t)std::atoll(e) : (int64_t)0;
    }();
    const int64_t want = std::min<int64_t>(INT32_MAX / 2, entries > 0 ? entries
                                                          : cap0 > 0 ? cap0 : 2 * (int64_t)n + 65536);
    if (want > p->sl_cap) {
        dev_free(p->sl_rank); dev_free(p->sl_rect);
        p->sl_cap = 0;
        if ((rc = dev_alloc(&p->sl_rank, (size_t)want)) || (rc = dev_alloc(&p->sl_rect, (size_t)want))) return rc;
        p->sl_cap = (int)want;
    }
    return TSB_OK;
}

// Upper bound of the frame's order length (*n_bin): the prefix cap or every Gaussian.
int rank_bound(tsb_pass* p) {
    return p->prefix ? std::min(p->kcap, p->scene->d.n) : p->scene->d.n;
}

SuperK superk(tsb_pass* p) {
    SuperK k;
    k.hist = p->sl_hist;
    k.hist_stride = kSlMaxBlocks;
    k.row_total = p->sl_hist + (size_t)p->nsup * kSlMaxBlocks;
    k.off = p->sl_off;
    k.rank = p->sl_rank;
    k.rect = p->sl_rect;
    k.cap = p->sl_cap;
    k.total = p->counters + 7;
    k.sup_x = p->sup_x;
    k.sup_log = p->sup_log;
    k.nsup = p->sl_lists ? p->nsup : 0;
    k.work = p->ctx->profiling ? p->ctx->work : nullptr;
    return k;
}

PixK pixk(tsb_pass* p) {
    PixK px{};
    px.out = p->out;
    const bool counts = (p->channels & TSB_CH_COUNTS) != 0;
    px.n_contrib = counts ? p->n_contrib : nullptr;
    px.n_processed = counts ? p->n_processed : nullptr;
    px.last = p->last;
    px.T_pre = p->T_pre;
    px.d_quad = p->d_quad;
    px.dist3 = (p->channels & TSB_CH_DISTORTION) ? p->dist3 : nullptr;
    px.flagged = p->flagged;
    px.out64 = (p->channels & TSB_CH_EXACT) ? p->out64 : nullptr;
    px.n_flagged = p->counters + 1;
    px.abort = p->counters + 2;
    return px;
}

// first colour SH array: after pos_op, scale_amp, quat, the keyframe offsets and the reflectivity SH
int color_base(const tsb_scene* s) { return 3 + s->d.n_keyframes + (s->d.sh_degree > 0 ? 4 : 0); }

SceneK scenek(const tsb_scene* s) {
    SceneK k{};
    k.n = s->d.n;
    k.nk = s->d.n_keyframes;
    k.nf = s->d.n_freq;
    k.sh_degree = s->d.sh_degree;
    k.freq[0] = s->d.frequency[0];
    k.freq[1] = s->d.n_freq > 1 ? s->d.frequency[1] : 0.0;
    k.s_int = s->d.source_intensity;
    k.c = s->d.speed_of_light;
    const size_t n = (size_t)s->d.n;
    k.pos_op = s->params;
    k.scale_amp = s->params + n;
    k.quat = s->params + 2 * n;
    k.motion = s->params + 3 * n;
    k.sh = s->d.sh_degree > 0 ? s->params + (3 + (size_t)s->d.n_keyframes) * n : nullptr;
    k.color_sh = s->d.color ? s->params + (size_t)color_base(s) * n : nullptr;
    k.cov6 = s->pcache;
    k.opac = s->pcache + 6 * n;
    k.cov6f = reinterpret_cast<const float*>(s->pcache + 7 * n);
    return k;
}

int ensure_ext(tsb_pass* p);
int tile_counts(tsb_pass* p, std::vector<uint32_t>& counts);

int read_visible(tsb_pass* p) {
    int rc0 = flush_prepare(p);
    if (rc0) return rc0;
    rc0 = settle(p);
    if (rc0) return rc0;
    if (p->V >= 0) return TSB_OK;
    int32_t* h = (int32_t*)((char*)p->pinned + 1024);
    TSB_CUDA(cudaMemcpyAsync(h, p->counters, 4, cudaMemcpyDeviceToHost, p->stream));
    TSB_CUDA(cudaStreamSynchronize(p->stream));
    p->V = h[0];
    return TSB_OK;
}

}  // namespace

void tsb_pass_destroy(tsb_pass* p) {
    if (!p) return;
    cudaSetDevice(p->ctx->device);
    if (p->stream) cudaStreamSynchronize(p->stream);
    auto& v = p->ctx->passes;
    v.erase(std::remove(v.begin(), v.end(), p), v.end());
    free_gauss(p);
    free_pixels(p);
    free_super(p);
    dev_free(p->blk_term); dev_free(p->blk_list);
    dev_free(p->det_off); dev_free(p->det_part);
    dev_free(p->counters); dev_free(p->fx_work_n);
    dev_free(p->sel_keys); dev_free(p->sel_vals); dev_free(p->sel_scratch);
    dev_free(p->loss_part); dev_free(p->bg_part); dev_free(p->loss_dev); dev_free(p->chw);
    dev_free(p->ssim_g); dev_free(p->ssim_part); dev_free(p->order_dbg);
    dev_free(p->ext_col); dev_free(p->ext_mf); dev_free(p->ext_mb); dev_free(p->ext_dmotion);
    dev_free(p->ext_out); dev_free(p->ext_screen); dev_free(p->ext_up); dev_free(p->ext_bg_part);
    dev_free(p->ext_dmacc); dev_free(p->ext_ftgt); dev_free(p->ext_fl_part); dev_free(p->ext_fl_res);
    if (p->pinned) cudaFreeHost(p->pinned);
    if (p->done_ev) cudaEventDestroy(p->done_ev);
    for (auto& e : p->scene_evs) cudaEventDestroy(e.second);
    if (p->fwd_ev) cudaEventDestroy(p->fwd_ev);
    for (auto& fg : p->fwd)
        if (fg.exec) cudaGraphExecDestroy(fg.exec);
    dev_free(p->frame_dev);
    if (p->cap_stream) cudaStreamDestroy(p->cap_stream);
    if (p->stream) cudaStreamDestroy(p->stream);
    delete p;
}

int tsb_pass_prepare(tsb_pass* p, tsb_scene* s, const tsb_camera* cam, const tsb_render_options* opt,
                     const tsb_frame* frame) {
    if (!p) return fail(TSB_ERR_INVALID, "null pass");
    {
        int rc0 = settle(p);  // the previous frame of this pass (its buffers are reused)
        if (rc0) return rc0;
    }
    p->prepared = p->forwarded = p->have_loss = false;
    p->pend_loss = p->pend_bwd = false;
    // RenderPassImpl ctor checks (splat.cpp:91-100)
    if (!s || !cam) return fail(TSB_ERR_INVALID, "render: scene and camera required");
    if (!(cam->fx > 0 && cam->fy > 0 && cam->width > 0 && cam->height > 0 && cam->near_plane > 0 &&
          cam->far_plane > cam->near_plane))
        return fail(TSB_ERR_INVALID, "render: invalid camera");
    if (!opt) return fail(TSB_ERR_INVALID, "render: options required");
    if (s->ctx != p->ctx) return fail(TSB_ERR_INVALID, "render: scene and pass belong to different contexts");
    if (cam->width > 32767 || cam->height > 32767)
        return fail(TSB_ERR_UNSUPPORTED, "render: image dimensions above 32767 are not supported");
    TSB_CUDA(cudaSetDevice(p->ctx->device));

    p->scene = s;
    p->nf = s->d.n_freq;
    p->W = cam->width;
    p->H = cam->height;
    p->channels = opt->channels;
    CamK& C = p->cam;
    C.fx = cam->fx; C.fy = cam->fy; C.cx = cam->cx; C.cy = cam->cy;
    C.W = cam->width; C.H = cam->height;
    C.near_plane = cam->near_plane;
    for (int i = 0; i < 9; ++i) C.R[i] = cam->R[i];
    for (int i = 0; i < 3; ++i) C.t[i] = cam->t[i];
    C.lim_x = 1.3 * (0.5 * cam->width / cam->fx);
    C.lim_y = 1.3 * (0.5 * cam->height / cam->fy);
    for (int i = 0; i < 9; ++i) C.Rf[i] = (float)C.R[i];
    C.fxf = (float)C.fx; C.fyf = (float)C.fy; C.cxf = (float)C.cx; C.cyf = (float)C.cy;
    C.limxf = (float)C.lim_x; C.limyf = (float)C.lim_y;
    C.Wf = (float)C.W; C.Hf = (float)C.H;
    for (int i = 0; i < 3; ++i)
        C.center[i] = -(cam->R[0 * 3 + i] * cam->t[0] + cam->R[1 * 3 + i] * cam->t[1] + cam->R[2 * 3 + i] * cam->t[2]);
    OptK& O = p->opt;
    O.alpha_thr = opt->alpha_threshold;
    O.floor_T = opt->transmittance_floor;
    O.dilation = opt->dilation;
    O.sigma_cutoff = opt->sigma_cutoff;
    O.cov_eps = opt->coverage_eps;
    O.cut2 = opt->sigma_cutoff * opt->sigma_cutoff;
    O.ts = std::max(1, opt->tile_size);
    O.tiles_x = (cam->width + O.ts - 1) / O.ts;
    O.tiles_y = (cam->height + O.ts - 1) / O.ts;
    O.sub = (O.ts + kTile - 1) / kTile;
    O.alpha_thr_f = (float)O.alpha_thr;
    O.floor_f = (float)O.floor_T;
    O.cut2_f = (float)O.cut2;
    O.cov_eps_f = (float)O.cov_eps;
    O.dilation_f = (float)O.dilation;
    O.sigma_cutoff_f = (float)O.sigma_cutoff;
    for (int c = 0; c < 8; ++c) O.bg_quad[c] = c < 4 * p->nf ? opt->bg_quad[c] : 0.0;
    for (int c = 0; c < 4; ++c) O.bg_phasor[c] = c < 2 * p->nf ? opt->bg_phasor[c] : 0.0;
    O.dist = (opt->channels & TSB_CH_DISTORTION) ? 1 : 0;
    O.exact = (opt->channels & TSB_CH_EXACT) ? 1 : 0;
    static const float trel = [] {  // TSB_TREL: A/B override of the fix-up's T error threshold
        const char* e = std::getenv("TSB_TREL");
        return e ? (float)std::atof(e) : kTrelFlag;
    }();
    O.trel_flag = trel;
    {  // the raster's thresholds (tsb_raster.cu k_raster_fwd), fp32 as the kernel used them
        const float coarse_m = kCoarseMaha * O.cut2_f, coarse_a = kCoarseAlpha * O.alpha_thr_f;
        O.coarse_m_f = coarse_m;
        O.coarse_a_f = coarse_a;
        O.outside_f = O.cut2_f + coarse_m;
        O.m_lo_f = O.cut2_f - 2.f * coarse_m;
        O.a_hi_f = O.alpha_thr_f + 2.f * coarse_a;
    }
    for (int c = 0; c < 3; ++c) O.bg_color[c] = opt->bg_color[c];
    p->ntiles = O.tiles_x * O.tiles_y;
    if (p->ntiles > 65536) return fail(TSB_ERR_UNSUPPORTED, "render: more than 65536 tiles");
    p->nblocks = p->ntiles * O.sub * O.sub;
    if (frame) {
        if (s->d.n_keyframes > 0 && (frame->key < 0 || frame->key > s->d.n_keyframes - 2))
            return fail(TSB_ERR_INVALID, "render: frame keyframe index out of range");
        p->frame.key = frame->key;
        p->frame.w = frame->w;
    } else {
        p->frame.key = 0;
        p->frame.w = 0.0;
    }

    const int n = s->d.n;
    int rc;
    if ((rc = ensure_gauss(p, n))) return rc;
    if ((rc = ensure_pixels(p, p->W, p->H, p->ntiles, p->nblocks))) return rc;
    if ((rc = ensure_super(p, n, 0))) return rc;
    p->has_mf = p->has_mb = false;  // RenderInput::motion_* belong to one frame
    if ((p->channels & (TSB_CH_COLOR | TSB_CH_FLOW)) && (rc = ensure_ext(p))) return rc;
    if (p->channels & TSB_CH_EXACT) {  // every pixel recomposited (and back-propagated) in fp64
        const int npx = p->W * p->H;
        if (p->fx_state_cap < npx) {
            dev_free(p->fx_state);
            p->fx_state_cap = 0;
            if ((rc = dev_alloc(&p->fx_state, npx))) return rc;
            p->fx_state_cap = npx;
        }
        if (p->out64_cap < npx) {
            dev_free(p->out64);
            p->out64_cap = 0;
            if ((rc = dev_alloc(&p->out64, (size_t)out_channels(2) * npx))) return rc;
            p->out64_cap = npx;
        }
        if ((p->channels & (TSB_CH_COLOR | TSB_CH_FLOW)) && p->ext_out64_cap < npx) {
            dev_free(p->ext_out64);
            p->ext_out64_cap = 0;
            if ((rc = dev_alloc(&p->ext_out64, (size_t)9 * npx))) return rc;
            p->ext_out64_cap = npx;
        }
    }

    // The device work (preprocess + depth sort) is deferred: it becomes the head of
    // the forward graph, or is issued eagerly by flush_prepare when something reads
    // prepare's results before a forward.
    FrameDev* slot = (FrameDev*)((char*)p->pinned + kFrameSlot);
    slot->F = p->frame;
    slot->target = nullptr;
    slot->stamp = ++p->frame_stamp;
    slot->pad = 0;
    p->prep_deferred = true;
    p->sorted = p->gidx_b;  // launch_sort_depth's result buffer
    {
        const int n = p->scene->d.n;
        if (p->ctx->prefix_off) p->kcap = 0;
        else if (p->kcap > 0) p->kcap = std::max(p->kcap, p->ctx->kcap_learned);
        p->prefix = !(p->channels & TSB_CH_FULL_LISTS) && p->kcap > 0 && n > p->kcap;
        if (p->prefix && p->kcap > p->sel_cap) {
            dev_free(p->sel_keys); dev_free(p->sel_vals); dev_free(p->sel_scratch);
            p->sel_cap = 0;
            int rc1;
            if ((rc1 = dev_alloc(&p->sel_keys, p->kcap)) || (rc1 = dev_alloc(&p->sel_vals, p->kcap)) ||
                (rc1 = dev_alloc(&p->sel_scratch, prefix_sort_scratch_words(p->kcap))))
                return rc1;
            p->sel_cap = p->kcap;
        }
        p->n_bin = p->prefix ? p->counters + 4 : p->counters;
    }
    p->V = -1;
    p->prepared = true;
    return TSB_OK;
}

int tsb_pass_visible_count(tsb_pass* p, int32_t* out) {
    if (!p || !out) return fail(TSB_ERR_INVALID, "null argument");
    if (!p->prepared) return fail(TSB_ERR_INVALID, "pass not prepared");
    int rc = read_visible(p);
    if (rc) return rc;
    *out = p->V;
    return TSB_OK;
}

int tsb_pass_num_keys(tsb_pass* p, int64_t* out) {
    if (!p || !out) return fail(TSB_ERR_INVALID, "null argument");
    if (!p->forwarded) return fail(TSB_ERR_INVALID, "tile lists are built by forward()");
    int rc = settle(p);
    if (rc) return rc;
    std::vector<uint32_t> counts;
    if ((rc = tile_counts(p, counts))) return rc;
    int64_t k = 0;
    for (uint32_t c : counts) k += c;
    *out = k;
    return TSB_OK;
}

namespace {

// Equal-key runs of the depth order are resolved where it is read (tsb_ties.cuh); after the
// exact 64-bit fallback (sorted == gidx_a) the order has none.
TieK tiek(tsb_pass* p) {
    TieK t;
    t.keys = p->sorted == p->gidx_a ? nullptr : p->key_b;
    t.depth64 = p->depth64;
    t.abort = p->counters + 2;
    return t;
}

// The rank order the raster kernels scan (ScanK) of the pass's current frame.
ScanK scank(tsb_pass* p) {
    ScanK sc;
    sc.ord = p->ord;
    sc.trect = p->trect;
    sc.n_rank = p->n_bin;
    sc.n_all = p->counters;
    sc.blk_term = p->blk_term;
    sc.blk_list = p->blk_list;
    sc.abort = p->counters + 2;
    sc.work = p->ctx->profiling ? p->ctx->work : nullptr;
    sc.det_off = nullptr;
    sc.det_part = nullptr;
    sc.nsub2 = p->opt.sub * p->opt.sub;
    sc.sl_off = p->sl_lists ? p->sl_off : nullptr;
    sc.sl_rank = p->sl_lists ? p->sl_rank : nullptr;
    sc.sl_rect = p->sl_lists ? p->sl_rect : p->trect;
    sc.sup_x = p->sup_x;
    sc.sup_log = p->sup_log;
    return sc;
}

// fp64 fix-up arguments of the pass's current frame.
FixupK fixk(tsb_pass* p) {
    FixupK fx;
    fx.sc = scank(p);
    fx.overflow = p->counters + 2;
    fx.stamp = p->fx_stamp;
    fx.work = p->fx_work;
    fx.work_n = p->fx_work_n;
    fx.cache = p->fx_cache;
    fx.state = p->fx_state;
    fx.state_cap = p->fx_state_cap;
    fx.fix_idx = p->fix_idx;
    return fx;
}

// Colour / flow buffers, allocated on first use.
int ensure_ext(tsb_pass* p) {
    const int n = std::max(p->scene->d.n, 1), npx = std::max(p->W * p->H, 1), nb = std::max(p->nblocks, 1);
    int rc;
    if (n > p->ext_n_cap) {
        dev_free(p->ext_col); dev_free(p->ext_mf); dev_free(p->ext_mb); dev_free(p->ext_dmotion);
        dev_free(p->ext_screen);
        p->ext_n_cap = 0;
        if ((rc = dev_alloc(&p->ext_col, n)) || (rc = dev_alloc(&p->ext_mf, n)) || (rc = dev_alloc(&p->ext_mb, n)) ||
            (rc = dev_alloc(&p->ext_dmotion, (size_t)2 * n)) || (rc = dev_alloc(&p->ext_screen, (size_t)9 * n)))
            return rc;
        TSB_CUDA(cudaMemsetAsync(p->ext_screen, 0, sizeof(float) * 9 * (size_t)n, p->stream));
        TSB_CUDA(cudaMemsetAsync(p->ext_dmotion, 0, sizeof(float4) * 2 * (size_t)n, p->stream));
        p->ext_n_cap = n;
    }
    if (npx > p->ext_px_cap) {
        dev_free(p->ext_out); dev_free(p->ext_up); dev_free(p->ext_dmacc); dev_free(p->ext_ftgt);
        dev_free(p->ext_fl_part); dev_free(p->ext_fl_res);
        p->ext_px_cap = 0;
        if ((rc = dev_alloc(&p->ext_out, (size_t)kExtPlanes * npx)) || (rc = dev_alloc(&p->ext_up, (size_t)9 * npx)) ||
            (rc = dev_alloc(&p->ext_dmacc, (size_t)6 * npx)) || (rc = dev_alloc(&p->ext_ftgt, (size_t)6 * npx)) ||
            (rc = dev_alloc(&p->ext_fl_part, (size_t)4 * flow_loss_parts(npx))) ||
            (rc = dev_alloc(&p->ext_fl_res, 4)))
            return rc;
        p->ext_px_cap = npx;
    }
    if (nb > p->ext_blk_cap) {
        dev_free(p->ext_bg_part);
        p->ext_blk_cap = 0;
        if ((rc = dev_alloc(&p->ext_bg_part, (size_t)3 * nb))) return rc;
        p->ext_blk_cap = nb;
    }
    return TSB_OK;
}

ExtK extk(tsb_pass* p) {
    ExtK E{};
    E.col = (p->channels & TSB_CH_COLOR) && p->scene->d.color ? p->ext_col : nullptr;
    E.mf = p->has_mf ? p->ext_mf : nullptr;
    E.mb = p->has_mb ? p->ext_mb : nullptr;
    E.out = p->ext_out;
    E.screen = p->ext_screen;
    E.d_motion = p->ext_dmotion;
    E.bg_part = p->ext_bg_part;
    E.flow = (p->channels & TSB_CH_FLOW) ? 1 : 0;
    E.out64 = (p->channels & TSB_CH_EXACT) ? p->ext_out64 : nullptr;
    return E;
}

// Chunked binning + forward composite (+ fused loss); see tsb_bin.cu.  Enqueues
// every planned chunk; chunks without work return on the device.  Ends with an
// asynchronous read-back of the counters (visible count, abort word) that
// settle() inspects.
// prepare's device work: per-frame values H2D, counters, preprocess, depth order.
int record_prepare(tsb_pass* p, cudaStream_t st, int* launches) {
    const int n = p->scene->d.n;
    TSB_CUDA(cudaMemcpyAsync(p->frame_dev, (char*)p->pinned + kFrameSlot, sizeof(FrameDev), cudaMemcpyHostToDevice,
                             st));
    TSB_CUDA(cudaMemsetAsync(p->counters, 0, sizeof(int32_t) * 8, st));
    TSB_CUDA(cudaMemsetAsync(p->counters + 5, 0xff, sizeof(int32_t), st));  // key range min
    uint32_t* key_range = reinterpret_cast<uint32_t*>(p->counters + 5);
    {
        Stage sg(p->ctx, TSB_STAGE_PREPROCESS, st);
        launch_preprocess(scenek(p->scene), p->cam, p->opt, p->frame_dev, p->key_a, p->depth64, p->gidx_a, p->touched,
                          p->rect, p->rec, p->counters, key_range, p->prefix, st);
    }
    int l = n > 0 ? 1 : 0;
    {
        Stage sg(p->ctx, TSB_STAGE_DEPTH_SORT, st);
        if (p->prefix) {
            l += radix_sort24_prefix(p->key_a, p->key_b, p->gidx_b, p->sel_keys, p->sel_vals, n, p->kcap,
                                     p->sort_scratch, p->sel_scratch, key_range, p->counters, p->counters + 4,
                                     p->counters + 2, st);
            // records of the prefix (the lean preprocess wrote keys only)
            l += launch_records(scenek(p->scene), p->cam, p->opt, p->frame_dev, p->gidx_b, p->counters + 4,
                                p->kcap, p->key_a, p->depth64, p->gidx_a, p->rect, p->rec, p->counters + 2, st);
        } else
            l += launch_sort_depth(p->key_a, p->key_b, p->gidx_a, p->gidx_b, key_range, n, p->sort_scratch, st);
    }
    TSB_CHECK_LAUNCH();
    *launches = l;
    return TSB_OK;
}

// Issue a deferred prepare eagerly (something reads its results before a forward).
int flush_prepare(tsb_pass* p) {
    if (!p->prep_deferred) return TSB_OK;
    TSB_CUDA(cudaSetDevice(p->ctx->device));
    TSB_CUDA(cudaStreamWaitEvent(p->stream, p->scene->params_ev, 0));
    int l = 0;
    int rc = record_prepare(p, p->stream, &l);
    if (rc) return rc;
    p->ctx->launches += l;
    p->prep_deferred = false;
    TSB_CUDA(record_done(p, p->stream));
    return TSB_OK;
}

// Issue the forward's device work on `st`: per-frame values H2D, the scan arrays of
// the frame's order, the raster (one launch: every block scans the order for its own
// tile), the fp64 fix-up, the pass-local part of the loss and the counters read-back.
int record_forward(tsb_pass* p, cudaStream_t st, bool loss, const ChW& chw, bool graph, bool with_prep,
                   int* fixed_launches) {
    (void)graph;
    PixK px = pixk(p);
    int fixed = 0;
    const FrameDev* fd = p->frame_dev;
    if (with_prep) {
        int rc = record_prepare(p, st, &fixed);
        if (rc) return rc;
    } else {
        TSB_CUDA(cudaMemcpyAsync(p->frame_dev, (char*)p->pinned + kFrameSlot, sizeof(FrameDev),
                                 cudaMemcpyHostToDevice, st));
    }
    // counters[2] (abort word) is not cleared here: the depth sort of prepare may have set it
    TSB_CUDA(cudaMemsetAsync(p->counters + 1, 0, sizeof(int32_t), st));
    {
        Stage sg(p->ctx, TSB_STAGE_BINNING, st);
        fixed += launch_order_ranks(p->sorted, tiek(p), p->rect, p->opt.ts, p->n_bin, rank_bound(p), p->ord,
                                    p->trect, superk(p), st);
    }
    {
        Stage sg(p->ctx, TSB_STAGE_RASTER_FWD, st);
        launch_raster_fwd(p->rec, scank(p), p->opt, p->W, p->H, p->nf, px, fd, loss, chw, p->loss_part, st);
        fixed += 1;
    }
    const FixupK fx = fixk(p);
    {
        Stage sg(p->ctx, TSB_STAGE_FIXUP, st);
        fixed += launch_fixup(scenek(p->scene), p->cam, p->opt, fd, fx, px, p->nf, st);
    }
    if (loss) {
        Stage sg(p->ctx, TSB_STAGE_LOSS, st);
        TSB_CUDA(cudaMemsetAsync(p->loss_dev, 0, sizeof(double), st));
        launch_fixup_loss(px, p->W, p->H, p->nf, fd, chw, p->loss_dev, (p->channels & TSB_CH_DETERMINISTIC) != 0,
                          st);
        launch_reduce_partials(p->loss_part, p->nblocks, 1, p->loss_dev, 1.0 / ((double)p->W * p->H), px.abort, st);
        fixed += 2;
        if (p->mix > 0.0) {  // lambda (1 - SSIM) per weighted quad channel (losses.cpp:148-166)
            SsimArgs sa{};
            const double npx = (double)p->W * p->H;
            for (int c = 0; c < 4 * p->nf; ++c) {
                const double w = p->pend_chw_full[c];
                if (w == 0.0) continue;
                sa.chans[sa.nz] = c;
                sa.scale[sa.nz] = -w * p->mix / npx;
                sa.lam_w[sa.nz] = w * p->mix;
                ++sa.nz;
            }
            sa.g = p->ssim_g;
            sa.part = p->ssim_part;
            sa.d_quad = p->d_quad;
            sa.loss = p->loss_dev;
            sa.abort = px.abort;
            sa.fd = fd;
            launch_ssim(p->out, p->W, p->H, sa, st);
            fixed += 3;
        }
    }
    TSB_CHECK_LAUNCH();
    int32_t* hc = (int32_t*)((char*)p->pinned + 2048);
    TSB_CUDA(cudaMemcpyAsync(hc, p->counters, sizeof(int32_t) * 8, cudaMemcpyDeviceToHost, st));
    *fixed_launches = fixed;
    return TSB_OK;
}

// Everything a captured forward graph depends on, as bytes (a change rebuilds it).
std::string forward_key(tsb_pass* p, bool loss, const ChW& chw) {
    std::string k;
    auto add = [&k](const void* d, size_t n) { k.append((const char*)d, n); };
    const SceneK S = scenek(p->scene);
    const PixK px = pixk(p);
    const void* ptrs[] = {p->sorted, p->rect, p->counters, p->ord, p->trect, p->blk_term, p->blk_list, p->rec.A, p->rec.B,
                          p->rec.C, p->rec.D, p->loss_part, p->loss_dev, p->fx_stamp, p->fx_work, p->fx_work_n,
                          p->fx_cache, p->frame_dev, p->pinned, p->fx_state, p->sl_hist, p->sl_off, p->sl_rank,
                          p->sl_rect};
    add(ptrs, sizeof ptrs);
    const int sl[] = {p->sl_cap, p->sup_x, p->sup_log, p->nsup, (int)p->sl_lists};
    add(sl, sizeof sl);
    add(&p->fx_state_cap, sizeof p->fx_state_cap);
    add(&S, sizeof S);
    add(&px, sizeof px);
    add(&p->cam, sizeof p->cam);
    add(&p->opt, sizeof p->opt);
    add(&chw, sizeof chw);
    add(&p->mix, sizeof p->mix);
    add(p->pend_chw_full, sizeof p->pend_chw_full);
    const void* sptrs[] = {p->ssim_g, p->ssim_part};
    add(sptrs, sizeof sptrs);
    const void* prep_ptrs[] = {p->key_a, p->key_b, p->depth64, p->gidx_a, p->gidx_b, p->touched, p->sort_scratch,
                               p->n_bin, p->sel_keys, p->sel_vals, p->sel_scratch};
    add(prep_ptrs, sizeof prep_ptrs);
    const int ints[] = {p->W, p->H, p->nf, (int)p->channels, p->ntiles, p->nblocks, loss ? 1 : 0,
                        p->ctx->profiling ? 1 : 0, p->prep_deferred ? 1 : 0, p->prefix ? p->kcap : 0,
                        p->scene->d.n};
    add(ints, sizeof ints);
    return k;
}

int enqueue_forward(tsb_pass* p, const float* target, bool loss, const ChW& chw, bool allow_graph = true) {
    TSB_CUDA(cudaSetDevice(p->ctx->device));
    cudaStream_t st = p->stream;
    FrameDev* slot = (FrameDev*)((char*)p->pinned + kFrameSlot);
    slot->target = loss ? target : nullptr;
    const bool with_prep = p->prep_deferred;
    if (with_prep) TSB_CUDA(cudaStreamWaitEvent(st, p->scene->params_ev, 0));
    static const int sl_min = [] {  // TSB_SL_MIN: order length above which the lists are built (tests: 0)
        const char* e = std::getenv("TSB_SL_MIN");
        return e ? std::atoi(e) : kSlMinRanks;
    }();
    // (fixed for the frame: its backward and debug reads follow it)
    p->sl_lists = p->force_lists || rank_bound(p) > sl_min;
    int fixed = 0;
    // Graphs: not while stage events are being recorded (profiling runs the same kernels eagerly).
    const bool use_graph = allow_graph && p->ctx->use_graphs && !p->ctx->profiling;
    if (use_graph) {
        std::string key = forward_key(p, loss, chw);
        tsb_pass::FwdGraph& fg = p->fwd[with_prep ? 1 : 0];
        if (!fg.exec || key != fg.key) {
            if (fg.exec) cudaGraphExecDestroy(fg.exec);
            fg.exec = nullptr;
            TSB_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            int rc = record_forward(p, st, loss, chw, true, with_prep, &fixed);
            cudaGraph_t g = nullptr;
            cudaError_t e = cudaStreamEndCapture(st, &g);
            if (rc) {
                if (g) cudaGraphDestroy(g);
                return rc;
            }
            if (e != cudaSuccess) return fail(TSB_ERR_CUDA, std::string("forward graph capture: ") + cudaGetErrorString(e));
            e = cudaGraphInstantiate(&fg.exec, g, 0);
            cudaGraphDestroy(g);
            if (e != cudaSuccess) {
                fg.exec = nullptr;
                return fail(TSB_ERR_CUDA, std::string("forward graph instantiate: ") + cudaGetErrorString(e));
            }
            fg.key = std::move(key);
            fg.fixed = fixed;
        }
        TSB_CUDA(cudaGraphLaunch(fg.exec, st));
        p->ctx->launches += fg.fixed;
    } else {
        int rc = record_forward(p, st, loss, chw, false, with_prep, &fixed);
        if (rc) return rc;
        p->ctx->launches += fixed;
    }
    p->prep_deferred = false;
    if (p->channels & (TSB_CH_COLOR | TSB_CH_FLOW)) {
        // colour / flow channels beside the graph (tsb_ext.cu); an aborted frame skips them
        const ExtK E = extk(p);
        const SceneK S = scenek(p->scene);
        launch_ext_prep(S, p->cam, p->frame_dev, p->touched, E, p->counters + 2, st);
        launch_ext_fwd(p->rec, S, p->cam, p->opt, p->frame_dev, scank(p), fixk(p), pixk(p), p->nf, E, st);
        p->ctx->launches += (E.col && S.n > 0 ? 1 : 0) + 1;
        TSB_CHECK_LAUNCH();
    }
    if (loss) {
        // scene loss accumulator += this pass's loss (serialised with other gradient writers)
        TSB_CUDA(cudaStreamWaitEvent(st, p->scene->grads_ev, 0));
        launch_reduce_partials(p->loss_dev, 1, 1, p->scene->stats + kStatLoss, 1.0, p->counters + 2, st);
        TSB_CUDA(cudaEventRecord(p->scene->grads_ev, st));
        p->ctx->launches += 1;
        TSB_CHECK_LAUNCH();
    }
    p->forwarded = true;
    p->have_loss = loss;
    p->pending = true;
    p->pend_loss = loss;
    p->pend_target = loss ? target : nullptr;
    p->pend_chw = chw;
    p->pend_bwd = false;
    p->pend_dl.clear();
    TSB_CUDA(cudaEventRecord(p->fwd_ev, st));
    TSB_CUDA(record_done(p, st));
    return TSB_OK;
}

int output_ptr(tsb_pass* p, int which, void** dptr, size_t* bytes);

int enqueue_backward(tsb_pass* p, const UpK& up);

// Wait for the pass's enqueued forward (not its backward or downloads: they stay
// in flight behind it on the pass stream) and check its abort word.  An aborted
// frame wrote nothing (every kernel after the abort returns at entry); it is
// redone with more list storage / the exact 64-bit depth sort, including its
// loss and backward.  Its inputs are still intact: everything that changes the
// scene settles all passes first.
// A prefix-sorted frame's full order, for a redo or a debug read: records of every
// visible Gaussian (the lean preprocess skipped them) and the full depth sort
// (exact64: the exact 64-bit sort instead).  The raw keys are intact.
void full_order(tsb_pass* p, bool exact64, cudaStream_t st) {
    const int n = p->scene->d.n;
    p->ctx->launches += launch_records(scenek(p->scene), p->cam, p->opt, p->frame_dev, nullptr, nullptr, n, p->key_a,
                                       p->depth64, p->gidx_a, p->rect, p->rec, p->counters + 2, st);
    if (exact64) {
        p->ctx->launches += launch_sort_depth64(p->depth64, p->touched, p->key_a, p->key_b, p->gidx_a, p->gidx_b, n,
                                                p->sort_scratch, st);
        p->sorted = p->gidx_a;
    } else {
        p->ctx->launches += launch_sort_depth(p->key_a, p->key_b, p->gidx_a, p->gidx_b,
                                              reinterpret_cast<uint32_t*>(p->counters + 5), n, p->sort_scratch, st);
        p->sorted = p->gidx_b;
    }
    p->prefix = false;
    p->n_bin = p->counters;
}

// The frame from the exact (non-lean) preprocess and the full depth sort: the redo of a
// frame whose lean visibility test disagreed with prep64 (abort bit 16).
void exact_order(tsb_pass* p, cudaStream_t st) {
    const int n = p->scene->d.n;
    uint32_t* key_range = reinterpret_cast<uint32_t*>(p->counters + 5);
    cudaMemsetAsync(p->counters, 0, sizeof(int32_t) * 8, st);
    cudaMemsetAsync(key_range, 0xff, sizeof(int32_t), st);
    launch_preprocess(scenek(p->scene), p->cam, p->opt, p->frame_dev, p->key_a, p->depth64, p->gidx_a, p->touched,
                      p->rect, p->rec, p->counters, key_range, false, st);
    p->ctx->launches += 1 + launch_sort_depth(p->key_a, p->key_b, p->gidx_a, p->gidx_b, key_range, n,
                                              p->sort_scratch, st);
    p->sorted = p->gidx_b;
    p->prefix = false;
    p->n_bin = p->counters;
}

int settle(tsb_pass* p) {
    for (int attempt = 0; p->pending; ++attempt) {
        TSB_CUDA(cudaSetDevice(p->ctx->device));
        TSB_CUDA(cudaEventSynchronize(p->fwd_ev));
        p->pending = false;
        const int32_t* hc = (const int32_t*)((const char*)p->pinned + 2048);
        p->V = hc[0];
        const int ab = hc[2];
        static const bool trace = std::getenv("TSB_TRACE") != nullptr;
        if (trace)
            std::fprintf(stderr, "tsb trace: pass %p settle attempt %d ab %d V %d nbin %d kcap %d prefix %d\n", (void*)p,
                         attempt, ab, hc[0], hc[4], p->kcap, (int)p->prefix);
        if (!ab) return TSB_OK;
        if (attempt >= 8) return fail(TSB_ERR_UNSUPPORTED, "render: frame kept aborting (depth order)");
        p->ctx->redos++;
        cudaStream_t st = p->stream;
        if (ab & 1) {  // the super-tile lists overflowed: grow them to the frame's total
            int rc = ensure_super(p, p->scene->d.n, (int64_t)hc[7] + hc[7] / 4 + 4096);
            if (rc) return rc;
        }
        if (ab & 16) {  // lean / exact visibility disagreed: exact preprocess + full sort
            exact_order(p, st);  // an over-long tie run of this order aborts the next attempt (bit 2)
        } else if (p->prefix && (ab & (8 | 2))) {  // the full order (+ the records the lean preprocess skipped)
            if (ab & 8) {  // the prefix ran out before every pixel terminated: later frames sort a longer one
                const int n = p->scene->d.n;
                p->kcap = (int64_t)p->kcap * 4 >= n ? 0 : p->kcap * 4;
                if (p->kcap == 0) p->ctx->prefix_off = true;
                else p->ctx->kcap_learned = std::max(p->ctx->kcap_learned, p->kcap);
            }
            full_order(p, (ab & 2) != 0, st);
        } else if (ab & 2) {  // an equal-key run too long to resolve on read: exact 64-bit sort
            p->ctx->launches += launch_sort_depth64(p->depth64, p->touched, p->key_a, p->key_b, p->gidx_a, p->gidx_b,
                                                    p->scene->d.n, p->sort_scratch, st);
            p->sorted = p->gidx_a;
        }
        TSB_CUDA(cudaMemsetAsync(p->counters + 2, 0, sizeof(int32_t), st));
        const bool bwd = p->pend_bwd;
        const UpK up = p->pend_up;
        const std::vector<tsb_pass::Download> dls = p->pend_dl;
        int rc = enqueue_forward(p, p->pend_target, p->pend_loss, p->pend_chw, false);
        if (rc) return rc;
        if (bwd && (rc = enqueue_backward(p, up))) return rc;
        for (const auto& d : dls) {  // re-issue the frame's asynchronous downloads
            void* dp = nullptr;
            size_t b = 0;
            if ((rc = output_ptr(p, d.which, &dp, &b))) return rc;
            TSB_CUDA(cudaMemcpyAsync(d.host, dp, std::min(b, d.bytes), cudaMemcpyDeviceToHost, st));
            p->pend_dl.push_back(d);
        }
        TSB_CUDA(record_done(p, st));
    }
    return TSB_OK;
}

int run_forward(tsb_pass* p, const float* target, bool loss, const ChW& chw) {
    if (!p->prepared) return fail(TSB_ERR_INVALID, "pass not prepared");
    if (p->pending) {  // a second forward of the same prepared frame
        int rc = settle(p);
        if (rc) return rc;
    }
    return enqueue_forward(p, target, loss, chw);
}

}  // namespace

int tsb_pass_forward(tsb_pass* p) {
    if (!p) return fail(TSB_ERR_INVALID, "null pass");
    if (p->pending) {
        int rc0 = settle(p);
        if (rc0) return rc0;
    }
    p->mix = 0.0;
    return run_forward(p, nullptr, false, ChW{});
}

int tsb_pass_forward_loss(tsb_pass* p, int where, const float* target, const double* channel_weight,
                          double* loss_out) {
    return tsb_pass_forward_image_loss(p, where, target, channel_weight, 0.0, loss_out);
}

int tsb_pass_forward_image_loss(tsb_pass* p, int where, const float* target, const double* channel_weight,
                                double ssim_mix, double* loss_out) {
    if (!p || !target || !channel_weight) return fail(TSB_ERR_INVALID, "tsb_pass_forward_loss: null argument");
    if (!(ssim_mix >= 0.0 && ssim_mix <= 1.0)) return fail(TSB_ERR_INVALID, "forward_loss: ssim_mix must be in [0, 1]");
    if (!p->prepared) return fail(TSB_ERR_INVALID, "pass not prepared");
    TSB_CUDA(cudaSetDevice(p->ctx->device));
    cudaStream_t st = p->stream;
    const size_t nq = (size_t)4 * p->nf * p->W * p->H;
    const float* dt = target;
    if (where == TSB_HOST) {
        TSB_CUDA(cudaMemcpyAsync(p->target, target, nq * sizeof(float), cudaMemcpyHostToDevice, st));
        dt = p->target;
    } else if (where != TSB_DEVICE) {
        return fail(TSB_ERR_INVALID, "bad memory kind");
    }
    ChW w{};
    for (int c = 0; c < 4 * p->nf; ++c) w.w[c] = (float)(channel_weight[c] * (1.0 - ssim_mix));
    if (p->pending) {  // a second forward of the same prepared frame
        int rc0 = settle(p);
        if (rc0) return rc0;
    }
    for (int c = 0; c < 8; ++c) p->pend_chw_full[c] = c < 4 * p->nf ? channel_weight[c] : 0.0;
    p->mix = ssim_mix;
    if (ssim_mix > 0.0) {
        const int npx = p->W * p->H, nb = ssim_blocks(p->W, p->H);
        if (npx > p->ssim_cap_px || nb > p->ssim_cap_blocks) {
            dev_free(p->ssim_g);
            dev_free(p->ssim_part);
            p->ssim_cap_px = p->ssim_cap_blocks = 0;
            int rc1;
            if ((rc1 = dev_alloc(&p->ssim_g, (size_t)8 * 3 * npx)) || (rc1 = dev_alloc(&p->ssim_part, (size_t)8 * nb)))
                return rc1;
            p->ssim_cap_px = npx;
            p->ssim_cap_blocks = nb;
        }
    }
    int rc = run_forward(p, dt, true, w);
    if (rc) return rc;
    if (loss_out) {
        if ((rc = settle(p))) return rc;
        double* hl = (double*)((char*)p->pinned + 256);
        TSB_CUDA(cudaMemcpyAsync(hl, p->loss_dev, sizeof(double), cudaMemcpyDeviceToHost, st));
        TSB_CUDA(cudaStreamSynchronize(st));
        *loss_out = *hl;
    }
    return TSB_OK;
}

namespace {
// Device address and size of output `which` (no settle).
int output_ptr(tsb_pass* p, int which, void** dptr, size_t* bytes) {
    if (!p || !dptr) return fail(TSB_ERR_INVALID, "null argument");
    if (!p->prepared) return fail(TSB_ERR_INVALID, "pass not prepared");
    const size_t HW = (size_t)p->W * p->H;
    void* ptr = nullptr;
    size_t b = 0;
    switch (which) {
        case TSB_OUT_QUAD: ptr = p->out; b = 4 * p->nf * HW * 4; break;
        case TSB_OUT_DEPTH_RAW: ptr = p->out + ch_depth_raw(p->nf) * HW; b = HW * 4; break;
        case TSB_OUT_DEPTH: ptr = p->out + ch_depth(p->nf) * HW; b = HW * 4; break;
        case TSB_OUT_WEIGHT: ptr = p->out + ch_weight(p->nf) * HW; b = HW * 4; break;
        case TSB_OUT_TRANSM: ptr = p->out + ch_T(p->nf) * HW; b = HW * 4; break;
        case TSB_OUT_N_CONTRIB:
            if (!(p->channels & TSB_CH_COUNTS)) return fail(TSB_ERR_INVALID, "counts channel not enabled");
            ptr = p->n_contrib; b = HW * 4; break;
        case TSB_OUT_N_PROCESSED:
            if (!(p->channels & TSB_CH_COUNTS)) return fail(TSB_ERR_INVALID, "counts channel not enabled");
            ptr = p->n_processed; b = HW * 4; break;
        case TSB_OUT_D_QUAD: ptr = p->d_quad; b = 4 * p->nf * HW * 4; break;
        case TSB_OUT_PHASOR: ptr = p->out + ch_phasor(p->nf) * HW; b = 2 * p->nf * HW * 4; break;
        case TSB_OUT_DISTORTION:
            if (!(p->channels & TSB_CH_DISTORTION)) return fail(TSB_ERR_INVALID, "distortion channel not enabled");
            ptr = p->out + ch_distortion(p->nf) * HW; b = HW * 4; break;
        case TSB_OUT_COLOR:
            if (!(p->channels & TSB_CH_COLOR)) return fail(TSB_ERR_INVALID, "colour channel not enabled");
            ptr = p->ext_out; b = 3 * HW * 4; break;
        case TSB_OUT_MOTION_FWD_ACC:
        case TSB_OUT_MOTION_BWD_ACC:
        case TSB_OUT_FLOW_FWD:
        case TSB_OUT_FLOW_BWD:
        case TSB_OUT_FLOW_VALID: {
            if (!(p->channels & TSB_CH_FLOW)) return fail(TSB_ERR_INVALID, "flow channel not enabled");
            static const int plane[5] = {3, 6, 9, 11, 13}, planes[5] = {3, 3, 2, 2, 2};
            const int i = which - TSB_OUT_MOTION_FWD_ACC;
            ptr = p->ext_out + plane[i] * HW; b = planes[i] * HW * 4; break;
        }
        case TSB_OUT_D_MOTION_FWD_ACC:
        case TSB_OUT_D_MOTION_BWD_ACC: {
            const int k = which - TSB_OUT_D_MOTION_FWD_ACC;
            if (!p->fl_grad[k]) return fail(TSB_ERR_INVALID, "no flow-loss gradient for this direction");
            ptr = p->ext_dmacc + (size_t)3 * k * HW; b = 3 * HW * 4; break;
        }
        case TSB_OUT_F64:
            if (!(p->channels & TSB_CH_EXACT)) return fail(TSB_ERR_INVALID, "exact (fp64) mode not enabled");
            ptr = p->out64; b = (size_t)out_channels(p->nf) * HW * 8; break;
        case TSB_OUT_EXT_F64:
            if (!(p->channels & TSB_CH_EXACT) || !(p->channels & (TSB_CH_COLOR | TSB_CH_FLOW)))
                return fail(TSB_ERR_INVALID, "exact (fp64) mode with colour / flow not enabled");
            ptr = p->ext_out64; b = 9 * HW * 8; break;
        default: return fail(TSB_ERR_INVALID, "unknown output");
    }
    *dptr = ptr;
    if (bytes) *bytes = b;
    return TSB_OK;
}
}  // namespace

int tsb_pass_output(tsb_pass* p, int which, void** dptr, size_t* bytes) {
    if (!p || !dptr) return fail(TSB_ERR_INVALID, "null argument");
    if (!p->prepared) return fail(TSB_ERR_INVALID, "pass not prepared");
    int rc = settle(p);
    if (rc) return rc;
    return output_ptr(p, which, dptr, bytes);
}

int tsb_pass_download_async(tsb_pass* p, int which, void* host, size_t bytes) {
    if (!p || !host) return fail(TSB_ERR_INVALID, "null argument");
    if (!p->forwarded) return fail(TSB_ERR_INVALID, "download requires a forward pass");
    void* d = nullptr;
    size_t b = 0;
    int rc = output_ptr(p, which, &d, &b);
    if (rc) return rc;
    if (bytes < b) return fail(TSB_ERR_INVALID, "tsb_pass_download_async: host buffer too small");
    TSB_CUDA(cudaMemcpyAsync(host, d, b, cudaMemcpyDeviceToHost, p->stream));
    TSB_CUDA(record_done(p, p->stream));
    if (p->pending) p->pend_dl.push_back({which, host, bytes});
    return TSB_OK;
}

int tsb_pass_wait(tsb_pass* p) {
    if (!p) return fail(TSB_ERR_INVALID, "null pass");
    int rc = settle(p);
    if (rc) return rc;
    TSB_CUDA(cudaStreamSynchronize(p->stream));
    return TSB_OK;
}

int tsb_pass_download(tsb_pass* p, int which, void* host, size_t bytes) {
    void* d = nullptr;
    size_t b = 0;
    int rc = tsb_pass_output(p, which, &d, &b);
    if (rc) return rc;
    if (!host || bytes < b) return fail(TSB_ERR_INVALID, "tsb_pass_download: host buffer too small");
    TSB_CUDA(cudaMemcpyAsync(host, d, b, cudaMemcpyDeviceToHost, p->stream));
    TSB_CUDA(cudaStreamSynchronize(p->stream));
    return TSB_OK;
}

namespace {
int enqueue_backward(tsb_pass* p, const UpK& up) {
    cudaStream_t st = p->stream;
    tsb_scene* s = p->scene;
    float dpsi[2];
    for (int f = 0; f < p->nf; ++f) dpsi[f] = (float)(4.0 * M_PI * s->d.frequency[f] / s->d.speed_of_light);
    const PixK px = pixk(p);
    const bool ext = up.color || up.mf || up.mb;
    const ExtK E = extk(p);
    {
        // per-pass outputs only (screen gradients, background partials): overlaps other passes
        Stage sg(p->ctx, TSB_STAGE_RASTER_BWD, st);
        ScanK sc = scank(p);
        FixupK fx = fixk(p);
        const bool det = (p->channels & TSB_CH_DETERMINISTIC) != 0;
        if (det) {  // slots: offsets over the frame's ranks, sized on the host (one sync), cleared
            const int n = s->d.n;
            if (p->det_off_cap < p->n_cap + 2) {
                dev_free(p->det_off);
                p->det_off_cap = 0;
                int rc;
                if ((rc = dev_alloc(&p->det_off, (size_t)p->n_cap + 2))) return rc;
                p->det_off_cap = p->n_cap + 2;
            }
            uint32_t* total = p->det_off + p->det_off_cap - 1;  // past every rank's offset
            launch_det_offsets(sc, p->det_off, total, st);
            uint32_t* h = (uint32_t*)((char*)p->pinned + 1072);
            TSB_CUDA(cudaMemcpyAsync(h, total, 4, cudaMemcpyDeviceToHost, st));
            TSB_CUDA(cudaStreamSynchronize(st));
            const size_t slots = std::max<size_t>(h[0], 1);
            if (slots > p->det_cap) {
                dev_free(p->det_part);
                p->det_cap = 0;
                int rc;
                if ((rc = dev_alloc(&p->det_part, 8 * slots))) return rc;
                p->det_cap = slots;
            }
            TSB_CUDA(cudaMemsetAsync(p->det_part, 0, sizeof(float) * 8 * slots, st));
            sc.det_off = p->det_off;
            sc.det_part = p->det_part;
            fx.sc = sc;
            p->ctx->launches += 1;
            (void)n;
        }
        launch_raster_bwd(p->rec, sc, p->opt, p->W, p->H, p->nf, dpsi, px, up, p->screen, s->d.n, p->bg_part, st);
        // the recomposited pixels, whose backward follows their fp64 forward
        if (det) {
            launch_fixup_bwd_det(scenek(s), p->cam, p->opt, p->frame_dev, fx, px, up, p->nf, st);
            launch_det_reduce(sc, s->d.n, p->screen, s->d.n, st);
            p->ctx->launches += 2;
        } else {
            launch_fixup_bwd(scenek(s), p->cam, p->opt, p->frame_dev, fx, px, up, p->nf, p->screen, s->d.n, st);
            p->ctx->launches += 1;
        }
        if (ext) {  // colour / motion upstreams: adds to the same screen gradients (tsb_ext.cu)
            TSB_CUDA(cudaMemsetAsync(p->ext_dmotion, 0, sizeof(float4) * 2 * (size_t)std::max(s->d.n, 1), st));
            launch_ext_bwd(p->rec, p->opt, p->W, p->H, p->nf, scank(p), px, up, E, p->screen, s->d.n, st);
            p->ctx->launches += 1;
        }
    }
    // scene gradient writers are serialised by the scene's event chain
    TSB_CUDA(cudaStreamWaitEvent(st, s->grads_ev, 0));
    launch_reduce_partials(p->bg_part, p->nblocks, 6 * p->nf, s->stats + kStatBg, 1.0, px.abort, st);
    if (ext) {
        launch_reduce_partials(p->ext_bg_part, p->nblocks, 3, s->stats + kStatBgColor, 1.0, px.abort, st);
        p->ctx->launches += 1;
    }
    if (p->keep_screen) {
        dev_free(p->screen_keep);
        int rc;
        if ((rc = dev_alloc(&p->screen_keep, (size_t)8 * s->d.n))) return rc;
        TSB_CUDA(cudaMemcpyAsync(p->screen_keep, p->screen, sizeof(double) * 8 * (size_t)s->d.n,
                                 cudaMemcpyDeviceToDevice, st));
    }
    {
        Stage sg(p->ctx, TSB_STAGE_CHAIN, st);
        // an aborted frame left the screen gradients zero: the chain adds nothing
        launch_chain(scenek(s), p->cam, p->opt, p->frame, p->touched, p->screen, s->grads, st);
        if (ext) {
            launch_chain_ext(scenek(s), p->cam, p->frame, p->touched, E, s->grads, st);
            p->ctx->launches += 1;
        }
    }
    p->ctx->launches += 3;
    TSB_CHECK_LAUNCH();
    TSB_CUDA(cudaEventRecord(s->grads_ev, st));
    TSB_CUDA(record_done(p, st));
    p->pend_bwd = true;
    p->pend_up = up;
    return TSB_OK;
}

int run_backward(tsb_pass* p, const UpK& up) {
    if (p->pend_bwd && p->pending) {  // a second backward of one unsettled frame: settle the first
        int rc = settle(p);
        if (rc) return rc;
    }
    return enqueue_backward(p, up);
}
}  // namespace

int tsb_pass_backward(tsb_pass* p, int where, const float* d_quad) {
    if (!p) return fail(TSB_ERR_INVALID, "null pass");
    if (!p->forwarded) return fail(TSB_ERR_INVALID, "backward requires a forward pass");
    TSB_CUDA(cudaSetDevice(p->ctx->device));
    cudaStream_t st = p->stream;
    const float* up = p->d_quad;
    if (d_quad) {
        const size_t nq = (size_t)4 * p->nf * p->W * p->H;
        if (where == TSB_HOST) {
            TSB_CUDA(cudaMemcpyAsync(p->d_quad, d_quad, nq * sizeof(float), cudaMemcpyHostToDevice, st));
        } else if (where == TSB_DEVICE) {
            up = d_quad;
        } else {
            return fail(TSB_ERR_INVALID, "bad memory kind");
        }
    } else if (!p->have_loss) {
        return fail(TSB_ERR_INVALID, "backward: no upstream gradient and no loss was evaluated");
    }
    UpK u{};
    u.quad = up;
    return run_backward(p, u);
}

int tsb_pass_backward_buffers(tsb_pass* p, int where, const float* d_quad, const float* d_phasor,
                              const float* d_depth_raw, const float* d_weight, const float* d_distortion,
                              const float* d_transmittance) {
    return tsb_pass_backward_ext(p, where, d_quad, d_phasor, d_depth_raw, d_weight, d_distortion, d_transmittance,
                                 nullptr, nullptr, nullptr);
}

int tsb_pass_backward_ext(tsb_pass* p, int where, const float* d_quad, const float* d_phasor,
                          const float* d_depth_raw, const float* d_weight, const float* d_distortion,
                          const float* d_transmittance, const float* d_color, const float* d_motion_fwd_acc,
                          const float* d_motion_bwd_acc) {
    if (!p) return fail(TSB_ERR_INVALID, "null pass");
    if (d_color && !(p->channels & TSB_CH_COLOR))
        return fail(TSB_ERR_INVALID, "backward: a colour upstream needs the colour channel in the forward");
    if ((d_motion_fwd_acc || d_motion_bwd_acc) && !(p->channels & TSB_CH_FLOW))
        return fail(TSB_ERR_INVALID, "backward: a motion upstream needs the flow channel in the forward");
    if (!p->forwarded) return fail(TSB_ERR_INVALID, "backward requires a forward pass");
    if (where != TSB_HOST && where != TSB_DEVICE) return fail(TSB_ERR_INVALID, "bad memory kind");
    if (d_distortion && !(p->channels & TSB_CH_DISTORTION))
        return fail(TSB_ERR_INVALID, "backward: a distortion upstream needs the distortion channel in the forward");
    TSB_CUDA(cudaSetDevice(p->ctx->device));
    cudaStream_t st = p->stream;
    const size_t HW = (size_t)p->W * p->H;
    UpK u{};
    u.quad = d_quad; u.phasor = d_phasor; u.depth_raw = d_depth_raw; u.weight = d_weight;
    u.distortion = d_distortion; u.transm = d_transmittance;
    u.color = d_color; u.mf = d_motion_fwd_acc; u.mb = d_motion_bwd_acc;
    if (where == TSB_HOST) {
        const float* srcs[9] = {d_quad, d_phasor, d_depth_raw, d_weight, d_distortion, d_transmittance,
                                d_color, d_motion_fwd_acc, d_motion_bwd_acc};
        float* dsts[9] = {p->d_quad, p->up_extra, p->up_extra + 4 * HW, p->up_extra + 5 * HW,
                          p->up_extra + 6 * HW, p->up_extra + 7 * HW, p->ext_up, p->ext_up + 3 * HW,
                          p->ext_up + 6 * HW};
        const size_t planes[9] = {(size_t)4 * p->nf, (size_t)2 * p->nf, 1, 1, 1, 1, 3, 3, 3};
        const float** outs[9] = {&u.quad, &u.phasor, &u.depth_raw, &u.weight, &u.distortion, &u.transm,
                                 &u.color, &u.mf, &u.mb};
        for (int i = 0; i < 9; ++i) {
            if (!srcs[i]) continue;
            TSB_CUDA(cudaMemcpyAsync(dsts[i], srcs[i], planes[i] * HW * sizeof(float), cudaMemcpyHostToDevice, st));
            *outs[i] = dsts[i];
        }
    }
    return run_backward(p, u);
}

int tsb_pass_set_motion(tsb_pass* p, int where, const float* motion_fwd, const float* motion_bwd) {
    if (!p) return fail(TSB_ERR_INVALID, "null pass");
    if (!p->prepared) return fail(TSB_ERR_INVALID, "pass not prepared");
    if (where != TSB_HOST && where != TSB_DEVICE) return fail(TSB_ERR_INVALID, "bad memory kind");
    TSB_CUDA(cudaSetDevice(p->ctx->device));
    if (p->pending) {  // the motions belong to the next forward of this frame
        int rc0 = settle(p);
        if (rc0) return rc0;
    }
    int rc;
    if ((rc = ensure_ext(p))) return rc;
    const int n = p->scene->d.n;
    cudaStream_t st = p->stream;
    const float* src[2] = {motion_fwd, motion_bwd};
    float4* dst[2] = {p->ext_mf, p->ext_mb};
    for (int k = 0; k < 2; ++k) {
        if (!src[k] || n == 0) continue;
        const float* d = src[k];
        if (where == TSB_HOST) {  // stage through the (idle) screen buffer's first 3n floats
            TSB_CUDA(cudaMemcpyAsync(p->ext_screen, src[k], sizeof(float) * 3 * (size_t)n, cudaMemcpyHostToDevice, st));
            d = p->ext_screen;
        }
        launch_pack_rows(dst[k], d, n, 1, 3, st);
        p->ctx->launches += 1;
        if (where == TSB_HOST)
            TSB_CUDA(cudaMemsetAsync(p->ext_screen, 0, sizeof(float) * 3 * (size_t)n, st));
    }
    TSB_CHECK_LAUNCH();
    p->has_mf = motion_fwd != nullptr;
    p->has_mb = motion_bwd != nullptr;
    return TSB_OK;
}

int tsb_pass_flow_loss(tsb_pass* p, int where, const float* target_fwd, const float* target_bwd, double weight,
                       double* value, int64_t* valid_pixels, int32_t* has_grads) {
    if (!p) return fail(TSB_ERR_INVALID, "null pass");
    if (!p->forwarded || !(p->channels & TSB_CH_FLOW))
        return fail(TSB_ERR_INVALID, "flow_loss: render lacks flow channels");
    if (where != TSB_HOST && where != TSB_DEVICE) return fail(TSB_ERR_INVALID, "bad memory kind");
    TSB_CUDA(cudaSetDevice(p->ctx->device));
    int rc = settle(p);  // the loss reads a finished (not aborted) forward
    if (rc) return rc;
    cudaStream_t st = p->stream;
    const size_t HW = (size_t)p->W * p->H;
    FlowK F{};
    const float* tg[2] = {target_fwd, target_bwd};
    for (int k = 0; k < 2; ++k) {
        p->fl_grad[k] = false;
        if (!tg[k]) continue;
        if (where == TSB_HOST) {
            TSB_CUDA(cudaMemcpyAsync(p->ext_ftgt + 3 * k * HW, tg[k], sizeof(float) * 3 * HW, cudaMemcpyHostToDevice, st));
            F.target[k] = p->ext_ftgt + 3 * k * HW;
        } else {
            F.target[k] = tg[k];
        }
    }
    double res[4] = {0.0, 0.0, 0.0, 0.0};
    if (F.target[0] || F.target[1]) {
        F.d_macc = p->ext_dmacc;
        F.part = p->ext_fl_part;
        F.res = p->ext_fl_res;
        F.abort = p->counters + 2;
        launch_flow_loss(p->cam, p->nf, p->out, p->ext_out, F, weight, st);
        p->ctx->launches += 3;
        TSB_CHECK_LAUNCH();
        double* h = (double*)((char*)p->pinned + 320);
        TSB_CUDA(cudaMemcpyAsync(h, p->ext_fl_res, sizeof(double) * 4, cudaMemcpyDeviceToHost, st));
        TSB_CUDA(cudaStreamSynchronize(st));
        std::memcpy(res, h, sizeof res);
        const bool used = res[1] > 0.0;
        for (int k = 0; k < 2; ++k) p->fl_grad[k] = used && F.target[k] != nullptr;
    }
    if (value) *value = res[0];
    if (valid_pixels) *valid_pixels = (int64_t)res[1];
    if (has_grads) *has_grads = (p->fl_grad[0] ? 1 : 0) | (p->fl_grad[1] ? 2 : 0);
    return TSB_OK;
}

int tsb_pass_render_stack(tsb_pass* p, const char* dir, int quartet) {
    if (!p || !dir) return fail(TSB_ERR_INVALID, "tsb_pass_render_stack: null argument");
    if (!p->forwarded) return fail(TSB_ERR_INVALID, "render_stack: requires a forward pass");
    if (!(p->channels & TSB_CH_DISTORTION))
        return fail(TSB_ERR_INVALID, "render_stack: needs the distortion channel (eval.cpp:104)");
    if (quartet < 0 || quartet > 99999) return fail(TSB_ERR_INVALID, "render_stack: quartet index out of range");
    int rc = settle(p);
    if (rc) return rc;
    std::error_code ec;
    std::filesystem::create_directories(dir, ec);
    if (ec) return fail(TSB_ERR_INVALID, std::string("render_stack: cannot create ") + dir + ": " + ec.message());
    const int npx = p->W * p->H;
    const size_t HW = (size_t)npx;
    float* planes = nullptr;
    if ((rc = dev_alloc(&planes, 2 * HW))) return rc;
    cudaStream_t st = p->stream;
    launch_stack_planes(p->out, p->nf, npx, p->scene->d.frequency[0], p->scene->d.speed_of_light, planes, st);
    p->ctx->launches += 1;
    TSB_CHECK_LAUNCH();
    // host copies: quad (first frequency), gated depth + d_ToF, distortion, colour
    const bool color = (p->channels & TSB_CH_COLOR) != 0;
    std::vector<float> h((size_t)(4 + 2 + 1 + (color ? 3 : 0)) * HW);
    TSB_CUDA(cudaMemcpyAsync(h.data(), p->out, sizeof(float) * 4 * HW, cudaMemcpyDeviceToHost, st));
    TSB_CUDA(cudaMemcpyAsync(h.data() + 4 * HW, planes, sizeof(float) * 2 * HW, cudaMemcpyDeviceToHost, st));
    TSB_CUDA(cudaMemcpyAsync(h.data() + 6 * HW, p->out + ch_distortion(p->nf) * HW, sizeof(float) * HW,
                             cudaMemcpyDeviceToHost, st));
    if (color)
        TSB_CUDA(cudaMemcpyAsync(h.data() + 7 * HW, p->ext_out, sizeof(float) * 3 * HW, cudaMemcpyDeviceToHost, st));
    TSB_CUDA(cudaStreamSynchronize(st));
    cudaFree(planes);
    // file names of write_render_stacks (eval.cpp:78-82, 168-184)
    auto name = [&](const char* stem, const char* suffix) {
        char buf[64];
        std::snprintf(buf, sizeof buf, "%s_%05d%s.pfm", stem, quartet, suffix);
        return (std::filesystem::path(dir) / buf).string();
    };
    static const char* kPhase[4] = {"_p0", "_p90", "_p180", "_p270"};
    for (int m = 0; m < 4; ++m)
        if ((rc = tsb_write_pfm(name("quad", kPhase[m]).c_str(), h.data() + m * HW, p->W, p->H, 1))) return rc;
    if ((rc = tsb_write_pfm(name("depth", "").c_str(), h.data() + 4 * HW, p->W, p->H, 1))) return rc;
    if ((rc = tsb_write_pfm(name("dtof", "").c_str(), h.data() + 5 * HW, p->W, p->H, 1))) return rc;
    if ((rc = tsb_write_pfm(name("dd", "").c_str(), h.data() + 6 * HW, p->W, p->H, 1))) return rc;
    if (color && (rc = tsb_write_pfm(name("color", "").c_str(), h.data() + 7 * HW, p->W, p->H, 3))) return rc;
    return TSB_OK;
}

int tsb_pass_get_motion_grads(tsb_pass* p, float* d_motion_fwd, float* d_motion_bwd) {
    if (!p) return fail(TSB_ERR_INVALID, "null pass");
    if (!p->ext_dmotion) return fail(TSB_ERR_INVALID, "no colour / flow backward has run on this pass");
    int rc = settle(p);
    if (rc) return rc;
    const int n = p->scene->d.n;
    if (n == 0) return TSB_OK;
    cudaStream_t st = p->stream;
    float* out[2] = {d_motion_fwd, d_motion_bwd};
    for (int k = 0; k < 2; ++k) {
        if (!out[k]) continue;
        float* tmp = nullptr;
        if ((rc = dev_alloc(&tmp, (size_t)3 * n))) return rc;
        launch_unpack_rows(p->ext_dmotion + (size_t)k * n, tmp, n, 1, 3, st);
        TSB_CUDA(cudaMemcpyAsync(out[k], tmp, sizeof(float) * 3 * (size_t)n, cudaMemcpyDeviceToHost, st));
        TSB_CUDA(cudaStreamSynchronize(st));
        cudaFree(tmp);
    }
    return TSB_OK;
}

// ---- debug / parity ----
namespace {
// The scan arrays (ord / trect / super-tile lists) of the pass's current order, outside a
// frame: synchronous, the lists grown until they fit (a debug path must not leave the
// abort word set for the frame's later kernels).
int order_ranks_sync(tsb_pass* p) {
    for (int attempt = 0; attempt < 4; ++attempt) {
        int32_t ab0 = 0;
        TSB_CUDA(cudaMemcpyAsync(&ab0, p->counters + 2, 4, cudaMemcpyDeviceToHost, p->stream));
        TSB_CUDA(cudaStreamSynchronize(p->stream));
        if (ab0) return fail(TSB_ERR_INVALID, "debug order: the frame aborted");
        launch_order_ranks(p->sorted, tiek(p), p->rect, p->opt.ts, p->n_bin, rank_bound(p), p->ord, p->trect,
                           superk(p), p->stream);
        TSB_CHECK_LAUNCH();
        int32_t h[8];
        TSB_CUDA(cudaMemcpyAsync(h, p->counters, sizeof h, cudaMemcpyDeviceToHost, p->stream));
        TSB_CUDA(cudaStreamSynchronize(p->stream));
        if (!(h[2] & 1)) return TSB_OK;
        TSB_CUDA(cudaMemsetAsync(p->counters + 2, 0, 4, p->stream));
        int rc = ensure_super(p, p->scene->d.n, (int64_t)h[7] + h[7] / 4 + 4096);
        if (rc) return rc;
    }
    return fail(TSB_ERR_UNSUPPORTED, "debug order: super-tile lists");
}
// The exact (depth, index) order of the prepared frame on the device (runs of equal
// compressed keys resolved as the binning resolves them).
int order_device(tsb_pass* p, const uint32_t** out) {
    const int n = std::max(p->scene->d.n, 1);
    if (n > p->order_dbg_cap) {
        dev_free(p->order_dbg);
        p->order_dbg_cap = 0;
        int rc0;
        if ((rc0 = dev_alloc(&p->order_dbg, n))) return rc0;
        p->order_dbg_cap = n;
    }
    if (p->prefix) full_order(p, false, p->stream);  // the frame sorted only its nearest prefix
    // the scan arrays over the full order (its first ranks are the prefix's, and lead every
    // super-tile list: the forward's scan positions stay valid for a backward that follows)
    int rc = order_ranks_sync(p);
    if (rc) return rc;
    launch_materialize_order(p->sorted, tiek(p), p->counters, p->scene->d.n, p->order_dbg, p->stream);
    TSB_CHECK_LAUNCH();
    *out = p->order_dbg;
    return TSB_OK;
}
// Complete tile-list lengths (splat.cpp:187-200) over the full order.
int tile_counts(tsb_pass* p, std::vector<uint32_t>& counts) {
    const uint32_t* od = nullptr;
    int rc = order_device(p, &od);
    if (rc) return rc;
    const int nt = p->ntiles;
    uint32_t* dc = nullptr;
    if ((rc = dev_alloc(&dc, (size_t)nt))) return rc;
    launch_tile_counts(scank(p), p->opt.tiles_x, nt, dc, p->stream);
    counts.assign((size_t)nt, 0u);
    TSB_CUDA(cudaMemcpyAsync(counts.data(), dc, sizeof(uint32_t) * nt, cudaMemcpyDeviceToHost, p->stream));
    cudaError_t e = cudaStreamSynchronize(p->stream);
    dev_free(dc);
    if (e != cudaSuccess) return fail(TSB_ERR_CUDA, std::string("tile counts: ") + cudaGetErrorString(e));
    return TSB_OK;
}
}  // namespace

int tsb_pass_debug_prepared(tsb_pass* p, int32_t* gidx, int32_t* rect) {
    if (!p || !p->prepared) return fail(TSB_ERR_INVALID, "pass not prepared");
    int rc = read_visible(p);
    if (rc) return rc;
    cudaStream_t st = p->stream;
    const int V = p->V;
    std::vector<uint32_t> g(V > 0 ? V : 1);
    const uint32_t* order = nullptr;
    if ((rc = order_device(p, &order))) return rc;
    if (V > 0) TSB_CUDA(cudaMemcpyAsync(g.data(), order, sizeof(uint32_t) * V, cudaMemcpyDeviceToHost, st));
    std::vector<uint2> r((size_t)std::max(p->scene->d.n, 1));
    if (rect && p->scene->d.n > 0)
        TSB_CUDA(cudaMemcpyAsync(r.data(), p->rect, sizeof(uint2) * p->scene->d.n, cudaMemcpyDeviceToHost, st));
    TSB_CUDA(cudaStreamSynchronize(st));
    for (int i = 0; i < V; ++i) {
        if (gidx) gidx[i] = (int32_t)g[i];
        if (rect) {
            const uint2 rc2 = r[g[i]];
            rect[4 * i + 0] = rc2.x & 0xffff;
            rect[4 * i + 1] = rc2.x >> 16;
            rect[4 * i + 2] = rc2.y & 0xffff;
            rect[4 * i + 3] = rc2.y >> 16;
        }
    }
    return TSB_OK;
}

int tsb_pass_debug_tiles(tsb_pass* p, int32_t* tiles_x, int32_t* tiles_y, int64_t* offsets, int32_t* ids) {
    if (!p || !p->forwarded) return fail(TSB_ERR_INVALID, "tile lists are built by forward()");
    if (tiles_x) *tiles_x = p->opt.tiles_x;
    if (tiles_y) *tiles_y = p->opt.tiles_y;
    int rc = settle(p);
    if (rc) return rc;
    std::vector<uint32_t> counts;
    if ((rc = tile_counts(p, counts))) return rc;  // over the full order
    const int nt = p->ntiles;
    std::vector<int64_t> off((size_t)nt + 1, 0);
    for (int t = 0; t < nt; ++t) off[t + 1] = off[t] + counts[t];
    if (offsets)
        for (int t = 0; t <= nt; ++t) offsets[t] = off[t];
    if (ids && off[nt] > 0) {
        cudaStream_t st = p->stream;
        int64_t* doff = nullptr;
        uint32_t* dids = nullptr;
        if ((rc = dev_alloc(&doff, (size_t)nt + 1)) || (rc = dev_alloc(&dids, (size_t)off[nt]))) {
            dev_free(doff);
            return rc;
        }
        TSB_CUDA(cudaMemcpyAsync(doff, off.data(), sizeof(int64_t) * (nt + 1), cudaMemcpyHostToDevice, st));
        launch_tile_lists(scank(p), p->opt.tiles_x, nt, doff, dids, st);
        TSB_CUDA(cudaMemcpyAsync(ids, dids, sizeof(uint32_t) * (size_t)off[nt], cudaMemcpyDeviceToHost, st));
        cudaError_t e = cudaStreamSynchronize(st);
        dev_free(doff);
        dev_free(dids);
        if (e != cudaSuccess) return fail(TSB_ERR_CUDA, std::string("debug_tiles: ") + cudaGetErrorString(e));
    }
    return TSB_OK;
}

int tsb_pass_debug_records(tsb_pass* p, float* rec12) {
    if (!p || !p->prepared) return fail(TSB_ERR_INVALID, "pass not prepared");
    int rc = read_visible(p);
    if (rc) return rc;
    cudaStream_t st = p->stream;
    const int n = p->scene->d.n, V = p->V;
    std::vector<float4> A(std::max(n, 1)), B(std::max(n, 1)), C(std::max(n, 1)), D(std::max(n, 1));
    std::vector<uint32_t> g(std::max(V, 1));
    {
        // first: on a prefix-sorted frame order_device() runs full_order, whose k_records
        // writes the records of every visible Gaussian past the prefix
        const uint32_t* od = nullptr;
        int rc2;
        if ((rc2 = order_device(p, &od))) return rc2;
        if (V > 0) TSB_CUDA(cudaMemcpyAsync(g.data(), od, sizeof(uint32_t) * V, cudaMemcpyDeviceToHost, st));
    }
    if (n > 0) {
        TSB_CUDA(cudaMemcpyAsync(A.data(), p->rec.A, sizeof(float4) * n, cudaMemcpyDeviceToHost, st));
        TSB_CUDA(cudaMemcpyAsync(B.data(), p->rec.B, sizeof(float4) * n, cudaMemcpyDeviceToHost, st));
        TSB_CUDA(cudaMemcpyAsync(C.data(), p->rec.C, sizeof(float4) * n, cudaMemcpyDeviceToHost, st));
        if (p->nf > 1) TSB_CUDA(cudaMemcpyAsync(D.data(), p->rec.D, sizeof(float4) * n, cudaMemcpyDeviceToHost, st));
    }
    TSB_CUDA(cudaStreamSynchronize(st));
    for (int r = 0; r < V; ++r) {
        const uint32_t i = g[r];
        float* o = rec12 + 12 * (size_t)r;
        const float l11 = B[i].x, l12 = B[i].y, l22 = B[i].z;
        o[0] = A[i].x + A[i].z;  // mean x (rounded sum of base and offset)
        o[1] = A[i].y + A[i].w;
        o[2] = l11 * l11;              // conic a
        o[3] = l11 * l12;              // conic b
        o[4] = l12 * l12 + l22 * l22;  // conic c
        o[5] = B[i].w;                 // opacity
        o[6] = C[i].x;                 // coef
        o[7] = C[i].y;                 // depth
        o[8] = C[i].z;
        o[9] = C[i].w;
        o[10] = p->nf > 1 ? D[i].x : 0.f;
        o[11] = p->nf > 1 ? D[i].y : 0.f;
    }
    return TSB_OK;
}

int tsb_pass_debug_set_list_capacity(tsb_pass* p, uint32_t entries) {
    if (!p || entries == 0) return fail(TSB_ERR_INVALID, "tsb_pass_debug_set_list_capacity: bad argument");
    int rc = settle(p);
    if (rc) return rc;
    // the super-tile list storage shrunk to `entries`: a frame that needs more aborts on the
    // device and is redone with grown lists when the pass settles
    dev_free(p->sl_rank); dev_free(p->sl_rect);
    p->sl_cap = 0;
    if ((rc = dev_alloc(&p->sl_rank, (size_t)entries)) || (rc = dev_alloc(&p->sl_rect, (size_t)entries))) return rc;
    p->sl_cap = (int)std::min<uint32_t>(entries, INT32_MAX / 2);
    p->force_lists = true;
    return TSB_OK;
}

int tsb_pass_debug_keep_screen(tsb_pass* p, int enabled) {
    if (!p) return fail(TSB_ERR_INVALID, "null pass");
    p->keep_screen = enabled != 0;
    return TSB_OK;
}

int tsb_pass_debug_screen_grads(tsb_pass* p, float* g8) {
    if (!p || !g8) return fail(TSB_ERR_INVALID, "null argument");
    if (!p->keep_screen || !p->screen_keep)
        return fail(TSB_ERR_INVALID, "screen gradients are consumed by the chain kernel; "
                                     "enable tsb_pass_debug_keep_screen before backward");
    int rc = read_visible(p);
    if (rc) return rc;
    const int n = p->scene->d.n, V = p->V;
    std::vector<double> sc((size_t)8 * std::max(n, 1));
    std::vector<uint32_t> g((size_t)std::max(V, 1));
    TSB_CUDA(cudaMemcpyAsync(sc.data(), p->screen_keep, sizeof(double) * 8 * (size_t)n, cudaMemcpyDeviceToHost,
                             p->stream));
    {
        const uint32_t* od = nullptr;
        int rc2;
        if ((rc2 = order_device(p, &od))) return rc2;
        if (V > 0) TSB_CUDA(cudaMemcpyAsync(g.data(), od, sizeof(uint32_t) * V, cudaMemcpyDeviceToHost, p->stream));
    }
    TSB_CUDA(cudaStreamSynchronize(p->stream));
    for (int i = 0; i < V; ++i)
        for (int c = 0; c < 8; ++c) g8[8 * (size_t)i + c] = sc[(size_t)c * n + g[i]];
    return TSB_OK;
}

int tsb_pass_debug_fixups(tsb_pass* p, int32_t* count) {
    if (!p || !count) return fail(TSB_ERR_INVALID, "null argument");
    int rc0 = settle(p);
    if (rc0) return rc0;
    int32_t* h = (int32_t*)((char*)p->pinned + 512);
    TSB_CUDA(cudaMemcpyAsync(h, p->counters + 1, 4, cudaMemcpyDeviceToHost, p->stream));
    TSB_CUDA(cudaStreamSynchronize(p->stream));
    *count = *h;
    return TSB_OK;
}

int tsb_pass_debug_fixup_list(tsb_pass* p, int32_t* entries, int32_t capacity, int32_t* count) {
    int32_t n = 0;
    int rc = tsb_pass_debug_fixups(p, &n);
    if (rc) return rc;
    if (count) *count = n;
    if (entries && n > 0) {
        TSB_CUDA(cudaMemcpy(entries, p->flagged, sizeof(int32_t) * std::min(n, capacity), cudaMemcpyDeviceToHost));
    }
    return TSB_OK;
}

// ---------------------------------------------------------------------------
// NCCL
// ---------------------------------------------------------------------------
// NCCL is resolved with dlopen on first use instead of being a link-time
// dependency: a process that already loaded an NCCL (e.g. PyTorch's bundled
// libnccl.so.2) keeps using that one, and pure render users never load it.
namespace {
struct NcclApi {
    bool tried = false, ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;

bool nccl_load() {
    if (g_nccl.tried) return g_nccl.ok;
    g_nccl.tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        g_err = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
        return false;
    }
#define TSB_SYM(field, name) g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name))
    TSB_SYM(GetUniqueId, "ncclGetUniqueId");
    TSB_SYM(CommInitRank, "ncclCommInitRank");
    TSB_SYM(CommDestroy, "ncclCommDestroy");
    TSB_SYM(AllReduce, "ncclAllReduce");
    TSB_SYM(GroupStart, "ncclGroupStart");
    TSB_SYM(GroupEnd, "ncclGroupEnd");
    TSB_SYM(GetErrorString, "ncclGetErrorString");
#undef TSB_SYM
    g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.CommDestroy && g_nccl.AllReduce &&
                g_nccl.GroupStart && g_nccl.GroupEnd && g_nccl.GetErrorString;
    if (!g_nccl.ok) g_err = "libnccl.so.2 lacks required symbols";
    return g_nccl.ok;
}
}  // namespace

struct tsb_comm {
    ncclComm_t comm = nullptr;
    tsb_ctx* ctx = nullptr;
};

int tsb_comm_unique_id(void* out) {
    if (!out) return fail(TSB_ERR_INVALID, "null argument");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    if (!nccl_load()) return TSB_ERR_NCCL;
    ncclUniqueId id;
    ncclResult_t r = g_nccl.GetUniqueId(&id);
    if (r != ncclSuccess) return fail(TSB_ERR_NCCL, std::string("ncclGetUniqueId: ") + g_nccl.GetErrorString(r));
    std::memcpy(out, &id, sizeof id);
    return TSB_OK;
}

int tsb_comm_create(tsb_ctx* ctx, const void* unique_id, int nranks, int rank, tsb_comm** out) {
    if (!ctx || !unique_id || !out) return fail(TSB_ERR_INVALID, "tsb_comm_create: null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(TSB_ERR_INVALID, "tsb_comm_create: bad rank");
    TSB_CUDA(cudaSetDevice(ctx->device));
    if (!nccl_load()) return TSB_ERR_NCCL;
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof id);
    tsb_comm* c = new tsb_comm();
    c->ctx = ctx;
    ncclResult_t r = g_nccl.CommInitRank(&c->comm, nranks, id, rank);
    if (r != ncclSuccess) {
        delete c;
        return fail(TSB_ERR_NCCL, std::string("ncclCommInitRank: ") + g_nccl.GetErrorString(r));
    }
    *out = c;
    return TSB_OK;
}

void tsb_comm_destroy(tsb_comm* c) {
    if (!c) return;
    if (c->comm && g_nccl.ok) g_nccl.CommDestroy(c->comm);
    delete c;
}

int tsb_scene_allreduce_grads(tsb_scene* s, tsb_comm* c) {
    if (!s || !c) return fail(TSB_ERR_INVALID, "null argument");
    {
        int rc0 = settle_all(s->ctx);  // a redone frame must add its gradients before the reduction
        if (rc0) return rc0;
    }
    const size_t nel = (size_t)s->narrays * (size_t)s->d.n * 4;
    cudaStream_t st = s->ctx->stream;
    TSB_CUDA(cudaStreamWaitEvent(st, s->grads_ev, 0));
    Stage sg(s->ctx, TSB_STAGE_ALLREDUCE, st);
    ncclResult_t r = g_nccl.GroupStart();
    if (r == ncclSuccess && nel > 0)
        r = g_nccl.AllReduce(s->grads, s->grads, nel, ncclFloat, ncclSum, c->comm, st);
    if (r == ncclSuccess) r = g_nccl.AllReduce(s->stats, s->stats, kStats, ncclDouble, ncclSum, c->comm, st);
    ncclResult_t r2 = g_nccl.GroupEnd();
    if (r != ncclSuccess || r2 != ncclSuccess)
        return fail(TSB_ERR_NCCL,
                    std::string("ncclAllReduce: ") + g_nccl.GetErrorString(r != ncclSuccess ? r : r2));
    TSB_CUDA(cudaEventRecord(s->grads_ev, st));
    return TSB_OK;
}

// ---------------------------------------------------------------------------
// DeformNet (tsb_mlp.cu)
// ---------------------------------------------------------------------------
struct tsb_deform {
    tsb_ctx* ctx = nullptr;
    tsb_deform_config cfg{};
    int din = 0, L = 0, width = 0;  // input dim, hidden layers, units
    std::vector<int> rows, cols;    // per layer: W is rows x cols
    std::vector<int64_t> w_off, b_off;
    int64_t P = 0;
    float *params = nullptr, *grads = nullptr, *m = nullptr, *v = nullptr;
    int64_t step = 0;
    struct Slot {
        int64_t cap = 0, n = 0;
        float* X = nullptr;            // [cap][din] encodings (column c*ex = scaled position)
        std::vector<float*> H;         // [L][cap][width] post-ReLU activations
        std::vector<uint32_t*> Hb;     // [L][cap][width / 32] their ReLU gates as bits (fused forward only)
        bool bits_valid = false;
        bool valid = false;
    } slots[TSB_DEFORM_SLOTS];
    int64_t dcap = 0;
    float *delta_a = nullptr, *delta_b = nullptr;  // [dcap][max(width, din)]
    float* io = nullptr;                           // [dcap][3] host-staged positions / offsets / grads
    int64_t io_cap = 0;
    float* part = nullptr;                         // split-K partials
    int64_t part_cap = 0;
    // fused forward (k_mlp_fwd_fused): weights pre-split / pre-laid-out per K chunk
    bool fused = false;
    MlpLayout lay{};
    char* wpack = nullptr;
    bool packed = false;
};

namespace {
constexpr int kDeformMaxSlices = 148;  // one CTA per SM (the dW kernel holds ~192 KB of shared memory)

int deform_slot_alloc(tsb_deform* d, tsb_deform::Slot& s, int64_t n) {
    if (n <= s.cap) return TSB_OK;
    dev_free(s.X);
    for (float*& h : s.H) dev_free(h);
    for (uint32_t*& h : s.Hb) dev_free(h);
    s.H.assign(d->L, nullptr);
    s.Hb.assign(d->L, nullptr);
    s.cap = 0;
    int rc;
    if ((rc = dev_alloc(&s.X, (size_t)n * d->din))) return rc;
    for (int l = 0; l < d->L; ++l) {
        if ((rc = dev_alloc(&s.H[l], (size_t)n * d->width))) return rc;
        if (d->width % 32 == 0 && (rc = dev_alloc(&s.Hb[l], (size_t)n * (d->width / 32)))) return rc;
    }
    s.cap = n;
    return TSB_OK;
}

int deform_scratch(tsb_deform* d, int64_t n) {
    const int wmax = std::max(d->width, d->din);
    if (n > d->dcap) {
        dev_free(d->delta_a);
        dev_free(d->delta_b);
        int rc;
        if ((rc = dev_alloc(&d->delta_a, (size_t)n * wmax)) || (rc = dev_alloc(&d->delta_b, (size_t)n * wmax)))
            return rc;
        d->dcap = n;
    }
    const int64_t need = (int64_t)kDeformMaxSlices * 128 * 128 + (int64_t)kDeformMaxSlices * 128;  // + row sums
    if (need > d->part_cap) {
        dev_free(d->part);
        int rc;
        if ((rc = dev_alloc(&d->part, (size_t)need))) return rc;
        d->part_cap = need;
    }
    return TSB_OK;
}

int deform_io(tsb_deform* d, int64_t n) {
    if (3 * n <= d->io_cap) return TSB_OK;
    dev_free(d->io);
    int rc;
    if ((rc = dev_alloc(&d->io, (size_t)3 * n))) return rc;
    d->io_cap = 3 * n;
    return TSB_OK;
}

int deform_gemm(tsb_deform* d, GemmArgs g, int slices) {
    const int r = launch_gemm_tf32x3(g, slices, d->ctx->stream);
    if (r < 0) return fail(TSB_ERR_UNSUPPORTED, "deform: GEMM N > 128");
    d->ctx->launches += r;
    TSB_CHECK_LAUNCH();
    return TSB_OK;
}

// Forward of `n` positions (pos[i * pos_stride + c]) at time t into out[i * out_stride + c].
int deform_forward(tsb_deform* d, int slot, const float* pos, int64_t pos_stride, int64_t n, double t, float* out,
                   int64_t out_stride) {
    if (slot < 0 || slot >= TSB_DEFORM_SLOTS) return fail(TSB_ERR_INVALID, "deform: bad slot");
    tsb_deform::Slot& s = d->slots[slot];
    int rc;
    if ((rc = deform_slot_alloc(d, s, std::max<int64_t>(n, 1)))) return rc;
    cudaStream_t st = d->ctx->stream;
    DeformEnc te{};
    te.n = 1 + 2 * d->cfg.l_t;
    te.v[0] = (float)t;
    double f = M_PI;
    for (int l = 0; l < d->cfg.l_t; ++l, f *= 2.0) {
        te.v[1 + 2 * l] = (float)std::sin(f * t);
        te.v[2 + 2 * l] = (float)std::cos(f * t);
    }
    static const bool unfused = [] {
        const char* e = std::getenv("TSB_MLP_UNFUSED");
        return e && e[0] == '1';
    }();
    if (d->fused && !unfused) {
        if (!d->packed) {
            launch_pack_weights(d->lay, d->params, d->wpack, st);
            d->ctx->launches++;
            d->packed = true;
        }
        MlpFwdArgs a{};
        a.lay = d->lay;
        a.pos = pos;
        a.pos_stride = pos_stride;
        a.n = n;
        a.inv_scale = 1.0 / d->cfg.coord_scale;
        a.l_x = d->cfg.l_x;
        a.din = d->din;
        a.te = te;
        a.wpack = d->wpack;
        a.params = d->params;
        a.X = s.X;
        a.ldx = d->din;
        for (int l = 0; l < d->L; ++l) {
            a.H[l] = s.H[l];
            a.Hbits[l] = d->width % 32 == 0 ? s.Hb[l] : nullptr;
        }
        a.ldh = d->width;
        a.out = out;
        a.out_stride = out_stride;
        launch_mlp_fwd_fused(a, st);
        d->ctx->launches++;
        TSB_CHECK_LAUNCH();
        s.n = n;
        s.valid = true;
        s.bits_valid = d->width % 32 == 0;
        return TSB_OK;
    }
    launch_deform_encode(pos, pos_stride, n, 1.0 / d->cfg.coord_scale, d->cfg.l_x, te, s.X, d->din, st);
    d->ctx->launches++;
    const float* prev = s.X;
    int64_t ld = d->din;
    for (int l = 0; l <= d->L; ++l) {
        const bool last = l == d->L;
        GemmArgs g{};
        g.A = prev; g.a_m = ld; g.a_k = 1;
        g.B = d->params + d->w_off[l]; g.b_n = d->cols[l]; g.b_k = 1;
        g.M = (int)n; g.N = d->rows[l]; g.K = d->cols[l]; g.k_per_slice = ((g.K + 31) / 32) * 32;
        g.C = last ? out : s.H[l];
        g.ldc = last ? out_stride : d->width;
        g.bias = d->params + d->b_off[l];
        g.relu = last ? 0 : 1;
        if ((rc = deform_gemm(d, g, 1))) return rc;
        if (!last) {
            prev = s.H[l];
            ld = d->width;
        }
    }
    s.n = n;
    s.valid = true;
    s.bits_valid = false;  // (the layer-by-layer forward writes no gate bits)
    return TSB_OK;
}

// Backward of the slot's forward for d_out[i * dstride + o] (o < 3); d_pos (nullable)
// receives d(offsets)/d(position) (accumulated when `accumulate`).
int deform_backward(tsb_deform* d, int slot, const float* d_out, int64_t dstride, float* d_pos, int64_t pstride,
                    bool accumulate) {
    if (slot < 0 || slot >= TSB_DEFORM_SLOTS || !d->slots[slot].valid)
        return fail(TSB_ERR_INVALID, "deform: backward without a cached forward in this slot");
    tsb_deform::Slot& s = d->slots[slot];
    const int64_t n = s.n;
    int rc;
    if ((rc = deform_scratch(d, std::max<int64_t>(n, 1)))) return rc;
    cudaStream_t st = d->ctx->stream;
    const float* delta = d_out;
    int64_t dld = dstride;
    float* bufs[2] = {d->delta_a, d->delta_b};
    int flip = 0;
    const int slices = (int)std::max<int64_t>(1, std::min<int64_t>(kDeformMaxSlices, (n + 4095) / 4096));
    const int kps = (int)(((n + slices - 1) / slices + 31) / 32 * 32);
    const int used = (int)std::max<int64_t>(1, (n + kps - 1) / kps);
    for (int l = d->L; l >= 0; --l) {
        const float* below = l == 0 ? s.X : s.H[l - 1];
        const int K = d->cols[l], O = d->rows[l];
        // dW_l += delta^T below  (reduction over the n rows, split into row slices)
        GemmArgs g{};
        g.A = delta; g.a_m = 1; g.a_k = dld;
        g.B = below; g.b_n = 1; g.b_k = K;
        g.M = O; g.N = K; g.K = (int)n; g.k_per_slice = kps;
        g.C = d->part; g.ldc = K; g.slice_stride = (int64_t)O * K;
        float* rowsum = d->part + (int64_t)kDeformMaxSlices * 128 * 128;  // db_l = column sums of delta (fused)
        g.rowsum = rowsum;
        if ((rc = deform_gemm(d, g, used))) return rc;
        launch_reduce_slices(d->part, used, (int64_t)O * K, (int64_t)O * K, d->grads + d->w_off[l], true, st);
        launch_reduce_slices(rowsum, used, O, O, d->grads + d->b_off[l], true, st);
        d->ctx->launches += 2;
        if (l == 0 && !d_pos) break;
        // d_below = delta W_l (gated by the ReLU of the layer below, or the input gradient)
        float* out = bufs[flip];
        flip ^= 1;
        GemmArgs h{};
        h.A = delta; h.a_m = dld; h.a_k = 1;
        h.B = d->params + d->w_off[l]; h.b_n = 1; h.b_k = K;
        h.M = (int)n; h.N = K; h.K = O; h.k_per_slice = ((O + 31) / 32) * 32;
        h.C = out; h.ldc = K;
        if (l > 0 && s.bits_valid) {  // the gate of the layer below, 1 bit per unit
            h.maskbits = s.Hb[l - 1];
            h.ldmaskbits = d->width / 32;
        } else if (l > 0) {
            h.mask = s.H[l - 1];
            h.ldmask = d->width;
        }
        if (l == 0) {
            // the encoding chain fused into the input-gradient epilogue (no d_input round trip)
            // where the launch allows it, else the GEMM then k_deform_chain
            GemmArgs hc = h;
            if (d->cfg.l_x == 10) {
                hc.chain_x = s.X;
                hc.chain_ldx = d->din;
                hc.chain_inv_scale = 1.0 / d->cfg.coord_scale;
                hc.chain_dpos = d_pos;
                hc.chain_pstride = pstride;
                hc.chain_acc = accumulate ? 1 : 0;
                const int r = launch_gemm_tf32x3(hc, 1, st);
                if (r >= 0) {
                    d->ctx->launches += r;
                    TSB_CHECK_LAUNCH();
                    break;
                }
                if (r != kGemmNoChain) return fail(TSB_ERR_CUDA, "deform: GEMM launch");
            }
            if ((rc = deform_gemm(d, h, 1))) return rc;
            launch_deform_chain(out, K, s.X, d->din, n, 1.0 / d->cfg.coord_scale, d->cfg.l_x, d_pos, pstride,
                                accumulate, st);
            d->ctx->launches++;
            break;
        }
        if ((rc = deform_gemm(d, h, 1))) return rc;
        delta = out;
        dld = K;
    }
    TSB_CHECK_LAUNCH();
    return TSB_OK;
}
}  // namespace

int tsb_deform_create(tsb_ctx* ctx, const tsb_deform_config* cfg, tsb_deform** out) {
    if (!ctx || !cfg || !out) return fail(TSB_ERR_INVALID, "tsb_deform_create: null argument");
    *out = nullptr;
    if (cfg->hidden_layers < 0 || cfg->width <= 0 || cfg->l_x < 0 || cfg->l_t < 0 || !(cfg->coord_scale > 0.0))
        return fail(TSB_ERR_INVALID, "DeformNet: invalid config");  // deform.cpp:29-31
    const int din = 3 * (1 + 2 * cfg->l_x) + 1 + 2 * cfg->l_t;
    if (cfg->width > 128 || din > 128 || 1 + 2 * cfg->l_t > 64)
        return fail(TSB_ERR_UNSUPPORTED, "DeformNet: width and input_dim must be <= 128 on this build");
    TSB_CUDA(cudaSetDevice(ctx->device));
    tsb_deform* d = new tsb_deform();
    d->ctx = ctx;
    d->cfg = *cfg;
    d->din = din;
    d->L = cfg->hidden_layers;
    d->width = cfg->width;
    int prev = din;
    for (int l = 0; l <= d->L; ++l) {
        const int r = l == d->L ? 3 : d->width;
        d->rows.push_back(r);
        d->cols.push_back(prev);
        d->w_off.push_back(d->P);
        d->P += (int64_t)r * prev;
        d->b_off.push_back(d->P);
        d->P += r;
        prev = r;
    }
    int rc;
    if ((rc = dev_alloc(&d->params, d->P)) || (rc = dev_alloc(&d->grads, d->P)) || (rc = dev_alloc(&d->m, d->P)) ||
        (rc = dev_alloc(&d->v, d->P))) {
        tsb_deform_destroy(d);
        return rc;
    }
    // fused forward: hidden width a multiple of 32, the encoding halves within the kernel's buffers
    const int ex = 1 + 2 * cfg->l_x, et = 1 + 2 * cfg->l_t;
    d->fused = d->L + 1 <= kMlpMaxLayers && d->width % 32 == 0 && 2 * ex <= 64 && ex + et <= 64;
    if (d->fused) {
        MlpLayout& lay = d->lay;
        lay.layers = d->L + 1;
        lay.total_chunks = 0;
        int64_t off = 0;
        for (int l = 0; l <= d->L; ++l) {
            lay.rows[l] = d->rows[l];
            lay.cols[l] = d->cols[l];
            lay.cols_pad[l] = (d->cols[l] + 31) / 32 * 32;
            lay.nt[l] = l == d->L ? 16 : d->width;
            lay.chunks[l] = lay.cols_pad[l] / 32;
            lay.w_off[l] = d->w_off[l];
            lay.b_off[l] = d->b_off[l];
            lay.chunk_off[l] = off;
            off += (int64_t)lay.chunks[l] * lay.nt[l] * 32 * 8;
            lay.total_chunks += lay.chunks[l];
        }
        if ((rc = dev_alloc(&d->wpack, (size_t)off))) {
            tsb_deform_destroy(d);
            return rc;
        }
    }
    cudaStream_t st = ctx->stream;
    cudaMemsetAsync(d->params, 0, sizeof(float) * d->P, st);
    cudaMemsetAsync(d->grads, 0, sizeof(float) * d->P, st);
    cudaMemsetAsync(d->m, 0, sizeof(float) * d->P, st);
    cudaMemsetAsync(d->v, 0, sizeof(float) * d->P, st);
    *out = d;
    return TSB_OK;
}

void tsb_deform_destroy(tsb_deform* d) {
    if (!d) return;
    cudaSetDevice(d->ctx->device);
    cudaStreamSynchronize(d->ctx->stream);
    dev_free(d->params); dev_free(d->grads); dev_free(d->m); dev_free(d->v);
    for (auto& s : d->slots) {
        dev_free(s.X);
        for (float*& h : s.H) dev_free(h);
        for (uint32_t*& h : s.Hb) dev_free(h);
    }
    dev_free(d->delta_a); dev_free(d->delta_b); dev_free(d->io); dev_free(d->part); dev_free(d->wpack);
    delete d;
}

int64_t tsb_deform_param_count(const tsb_deform* d) { return d ? d->P : 0; }

int tsb_deform_set_params(tsb_deform* d, int where, const float* flat) {
    if (!d || !flat) return fail(TSB_ERR_INVALID, "tsb_deform_set_params: null argument");
    TSB_CUDA(cudaSetDevice(d->ctx->device));
    TSB_CUDA(cudaMemcpyAsync(d->params, flat, sizeof(float) * d->P,
                             where == TSB_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, d->ctx->stream));
    d->packed = false;
    TSB_CUDA(cudaStreamSynchronize(d->ctx->stream));
    return TSB_OK;
}

int tsb_deform_get_params(tsb_deform* d, float* flat) {
    if (!d || !flat) return fail(TSB_ERR_INVALID, "tsb_deform_get_params: null argument");
    TSB_CUDA(cudaSetDevice(d->ctx->device));
    TSB_CUDA(cudaMemcpyAsync(flat, d->params, sizeof(float) * d->P, cudaMemcpyDeviceToHost, d->ctx->stream));
    TSB_CUDA(cudaStreamSynchronize(d->ctx->stream));
    return TSB_OK;
}

int tsb_deform_get_grads(tsb_deform* d, float* flat) {
    if (!d || !flat) return fail(TSB_ERR_INVALID, "tsb_deform_get_grads: null argument");
    TSB_CUDA(cudaSetDevice(d->ctx->device));
    TSB_CUDA(cudaMemcpyAsync(flat, d->grads, sizeof(float) * d->P, cudaMemcpyDeviceToHost, d->ctx->stream));
    TSB_CUDA(cudaStreamSynchronize(d->ctx->stream));
    return TSB_OK;
}

int tsb_deform_zero_grads(tsb_deform* d) {
    if (!d) return fail(TSB_ERR_INVALID, "null network");
    TSB_CUDA(cudaMemsetAsync(d->grads, 0, sizeof(float) * d->P, d->ctx->stream));
    return TSB_OK;
}

int tsb_deform_offsets(tsb_deform* d, int slot, int where, const float* positions, int64_t n, double t,
                       float* offsets) {
    if (!d || !positions || !offsets || n < 0) return fail(TSB_ERR_INVALID, "tsb_deform_offsets: bad argument");
    if (n > 0x7fffffff) return fail(TSB_ERR_UNSUPPORTED, "tsb_deform_offsets: too many points");
    TSB_CUDA(cudaSetDevice(d->ctx->device));
    cudaStream_t st = d->ctx->stream;
    int rc;
    const float* pos = positions;
    float* out = offsets;
    if (where == TSB_HOST) {
        if ((rc = deform_io(d, std::max<int64_t>(n, 1)))) return rc;
        TSB_CUDA(cudaMemcpyAsync(d->io, positions, sizeof(float) * 3 * n, cudaMemcpyHostToDevice, st));
        pos = d->io;
        out = d->io;  // overwritten after the encoding read it (stream order)
    } else if (where != TSB_DEVICE) {
        return fail(TSB_ERR_INVALID, "bad memory kind");
    }
    if ((rc = deform_forward(d, slot, pos, 3, n, t, out, 3))) return rc;
    if (where == TSB_HOST) {
        TSB_CUDA(cudaMemcpyAsync(offsets, d->io, sizeof(float) * 3 * n, cudaMemcpyDeviceToHost, st));
        TSB_CUDA(cudaStreamSynchronize(st));
    }
    return TSB_OK;
}

int tsb_deform_backward(tsb_deform* d, int slot, int where, const float* d_offsets, float* d_positions) {
    if (!d || !d_offsets) return fail(TSB_ERR_INVALID, "tsb_deform_backward: null argument");
    if (slot < 0 || slot >= TSB_DEFORM_SLOTS || !d->slots[slot].valid)
        return fail(TSB_ERR_INVALID, "deform: backward without a cached forward in this slot");
    TSB_CUDA(cudaSetDevice(d->ctx->device));
    cudaStream_t st = d->ctx->stream;
    const int64_t n = d->slots[slot].n;
    int rc;
    if (where == TSB_HOST) {
        if ((rc = deform_io(d, 2 * std::max<int64_t>(n, 1)))) return rc;
        TSB_CUDA(cudaMemcpyAsync(d->io, d_offsets, sizeof(float) * 3 * n, cudaMemcpyHostToDevice, st));
        float* dpos = d_positions ? d->io + 3 * n : nullptr;
        if ((rc = deform_backward(d, slot, d->io, 3, dpos, 3, false))) return rc;
        if (d_positions)
            TSB_CUDA(cudaMemcpyAsync(d_positions, dpos, sizeof(float) * 3 * n, cudaMemcpyDeviceToHost, st));
        TSB_CUDA(cudaStreamSynchronize(st));
        return TSB_OK;
    }
    if (where != TSB_DEVICE) return fail(TSB_ERR_INVALID, "bad memory kind");
    return deform_backward(d, slot, d_offsets, 3, d_positions, 3, false);
}

int tsb_deform_scene_offsets(tsb_deform* d, int slot, tsb_scene* s, int keyframe, double t) {
    if (!d || !s) return fail(TSB_ERR_INVALID, "tsb_deform_scene_offsets: null argument");
    if (s->ctx != d->ctx) return fail(TSB_ERR_INVALID, "deform: scene and network belong to different contexts");
    if (keyframe < 0 || keyframe >= s->d.n_keyframes) return fail(TSB_ERR_INVALID, "deform: keyframe out of range");
    TSB_CUDA(cudaSetDevice(d->ctx->device));
    int rc = tsb_ctx_join(d->ctx);  // passes may still read the keyframe offsets
    if (rc) return rc;
    const size_t n = (size_t)s->d.n;
    // positions: pos_op lanes xyz; offsets: keyframe plane lanes xyz (lane w stays 0)
    if ((rc = deform_forward(d, slot, reinterpret_cast<const float*>(s->params), 4, (int64_t)n, t,
                             reinterpret_cast<float*>(s->params + (size_t)(3 + keyframe) * n), 4)))
        return rc;
    TSB_CUDA(cudaEventRecord(s->params_ev, d->ctx->stream));
    return TSB_OK;
}

int tsb_deform_scene_backward(tsb_deform* d, int slot, tsb_scene* s, int keyframe) {
    if (!d || !s) return fail(TSB_ERR_INVALID, "tsb_deform_scene_backward: null argument");
    if (s->ctx != d->ctx) return fail(TSB_ERR_INVALID, "deform: scene and network belong to different contexts");
    if (keyframe < 0 || keyframe >= s->d.n_keyframes) return fail(TSB_ERR_INVALID, "deform: keyframe out of range");
    TSB_CUDA(cudaSetDevice(d->ctx->device));
    int rc = settle_all(d->ctx);  // every frame's gradients are in (a redone frame adds later otherwise)
    if (rc) return rc;
    cudaStream_t st = d->ctx->stream;
    TSB_CUDA(cudaStreamWaitEvent(st, s->grads_ev, 0));
    const size_t n = (size_t)s->d.n;
    // trainer.cpp:329-331: canonical position += dX + din; the chain already added dX
    if ((rc = deform_backward(d, slot, reinterpret_cast<const float*>(s->grads + (size_t)(3 + keyframe) * n), 4,
                              reinterpret_cast<float*>(s->grads), 4, true)))
        return rc;
    TSB_CUDA(cudaEventRecord(s->grads_ev, st));
    return TSB_OK;
}

int tsb_deform_debug_activation(tsb_deform* d, int slot, int layer, float* host_out) {
    if (!d || !host_out || slot < 0 || slot >= TSB_DEFORM_SLOTS || !d->slots[slot].valid || layer < 0 ||
        layer >= d->L)
        return fail(TSB_ERR_INVALID, "tsb_deform_debug_activation: bad argument");
    const tsb_deform::Slot& s = d->slots[slot];
    TSB_CUDA(cudaMemcpyAsync(host_out, s.H[layer], sizeof(float) * (size_t)s.n * d->width, cudaMemcpyDeviceToHost,
                             d->ctx->stream));
    TSB_CUDA(cudaStreamSynchronize(d->ctx->stream));
    return TSB_OK;
}

int tsb_deform_adam_step(tsb_deform* d, double lr, double beta1, double beta2, double eps) {
    if (!d) return fail(TSB_ERR_INVALID, "null network");
    d->step += 1;
    d->packed = false;
    return tsb_adam_step_flat(d->ctx, TSB_DEVICE, d->params, d->grads, d->m, d->v, (size_t)d->P, d->step, lr, beta1,
                              beta2, eps);
}

int tsb_debug_gemm(tsb_ctx* ctx, int M, int N, int K, int slices, const float* A, int64_t a_m, int64_t a_k,
                   const float* B, int64_t b_n, int64_t b_k, const float* bias, int relu, const float* mask,
                   float* C) {
    if (!ctx || !A || !B || !C || M <= 0 || N <= 0 || N > 128 || K < 0 || slices < 1)
        return fail(TSB_ERR_INVALID, "tsb_debug_gemm: bad argument");
    TSB_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    const size_t na = (size_t)std::max<int64_t>(1, (int64_t)(M - 1) * a_m + (int64_t)std::max(K - 1, 0) * a_k + 1);
    const size_t nb = (size_t)std::max<int64_t>(1, (int64_t)(N - 1) * b_n + (int64_t)std::max(K - 1, 0) * b_k + 1);
    const int kps = ((K + slices - 1) / slices + 31) / 32 * 32;
    const int used = std::max(1, (K + std::max(kps, 32) - 1) / std::max(kps, 32));
    float *dA = nullptr, *dB = nullptr, *dC = nullptr, *dP = nullptr, *dbias = nullptr, *dmask = nullptr;
    int rc;
    if ((rc = dev_alloc(&dA, na)) || (rc = dev_alloc(&dB, nb)) || (rc = dev_alloc(&dC, (size_t)M * N)) ||
        (rc = dev_alloc(&dP, (size_t)used * M * N)) || (rc = dev_alloc(&dbias, N)) || (rc = dev_alloc(&dmask, (size_t)M * N)))
        return rc;
    cudaMemcpyAsync(dA, A, na * 4, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(dB, B, nb * 4, cudaMemcpyHostToDevice, st);
    if (bias) cudaMemcpyAsync(dbias, bias, (size_t)N * 4, cudaMemcpyHostToDevice, st);
    if (mask) cudaMemcpyAsync(dmask, mask, (size_t)M * N * 4, cudaMemcpyHostToDevice, st);
    GemmArgs g{};
    g.A = dA; g.a_m = a_m; g.a_k = a_k;
    g.B = dB; g.b_n = b_n; g.b_k = b_k;
    g.M = M; g.N = N; g.K = K; g.k_per_slice = std::max(kps, 32);
    g.C = dP; g.ldc = N; g.slice_stride = (int64_t)M * N;
    g.bias = used == 1 && bias ? dbias : nullptr;
    g.relu = used == 1 ? relu : 0;
    g.mask = used == 1 && mask ? dmask : nullptr;
    g.ldmask = N;
    launch_gemm_tf32x3(g, used, st);
    ctx->launches++;
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) {
        launch_reduce_slices(dP, used, (int64_t)M * N, (int64_t)M * N, dC, false, st);
        cudaMemcpyAsync(C, dC, (size_t)M * N * 4, cudaMemcpyDeviceToHost, st);
        e = cudaStreamSynchronize(st);
    }
    cudaFree(dA); cudaFree(dB); cudaFree(dC); cudaFree(dP); cudaFree(dbias); cudaFree(dmask);
    if (e != cudaSuccess) return fail(TSB_ERR_CUDA, std::string("tsb_debug_gemm: ") + cudaGetErrorString(e));
    return TSB_OK;
}

// ---------------------------------------------------------------------------
// host helpers (tof.hpp)
// ---------------------------------------------------------------------------
static double freq_or_default(double f) { return f > 0 ? f : 29.9792458e6; }

double tsb_unambiguous_range(double frequency) { return 299792458.0 / (2.0 * freq_or_default(frequency)); }

double tsb_quad_to_depth(double q0, double q90, double q180, double q270, double frequency) {
    const double re = q90 - q270, im = q0 - q180;
    if (re == 0.0 && im == 0.0) return std::nan("");
    double psi = std::atan2(im, re);
    if (psi < 0.0) psi += 2.0 * M_PI;
    return psi * 299792458.0 / (4.0 * M_PI * freq_or_default(frequency));
}

void tsb_quad_basis(double depth, double frequency, double* out4) {
    const double psi = 4.0 * M_PI * depth * freq_or_default(frequency) / 299792458.0;
    const double s = std::sin(psi), c = std::cos(psi);
    out4[0] = s;
    out4[1] = c;
    out4[2] = -s;
    out4[3] = -c;
}

}  // extern "C"
