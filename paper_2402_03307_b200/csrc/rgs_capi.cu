// C-ABI implementation (include/rgs_cuda.h): contexts, device scenes, the
// forward / backward pipelines and records export.
//
// Forward pipeline per view (render_forward, rasterizer.cpp:308-318):
//   K1 preprocess (FP64)  -> per-Gaussian splat records, tile rects, depth keys
//   depth ranks           -> splat order by (depth, index)
//   tile-major scatter    -> per-chunk tile counts, tile ranges [begin, end), then every
//                            (tile, splat) pair written at its place in the per-tile
//                            (depth, index) order == bin_and_sort
//   (images beyond 256 x 256 / 8192 tiles: pair offsets, duplicate-with-key, stable LSD
//    radix passes by tile, tile ranges)
//   K5 FP32 blend         -> image, final_T, n_contrib, slow-pixel list
//   FP64 fix-up           -> slow pixels recomputed exactly
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_set>
#include <vector>

#include "../../include/rgs_cuda.h"
#include "rgs_internal.cuh"

using namespace rgs_dev;

namespace {

struct CudaError {
    cudaError_t e;
    const char* what;
};

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t _e = (x);                                                   \
        if (_e != cudaSuccess) throw CudaError{_e, #x};                         \
    } while (0)

// Grow-only device buffer, stream-ordered allocation.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void ensure(size_t need, cudaStream_t s) {
        if (need <= bytes) return;
        if (p) CK(cudaFreeAsync(p, s));
        size_t b = std::max(need, bytes + bytes / 2);
        b = (b + 255) & ~size_t(255);
        CK(cudaMallocAsync(&p, b, s));
        bytes = b;
    }
    void release(cudaStream_t s) {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        bytes = 0;
    }
    template <typename T>
    T* as() const {
        return reinterpret_cast<T*>(p);
    }
};

// All per-view device state (one set per render in flight / per retained record).
struct Frame {
    // per Gaussian / input splat
    DevBuf valid, tiles, mean2, conic_ab, color_depth, flow_radius, rect, conic_f, color_f, guard_f, ext_f, src, key,
        dir_dist;
    DevBuf ent_key, ent_id, sorted_ids, sorted_tiles, pair_off;
    // depth buckets
    DevBuf bucket_count, bucket_off, bucket_cur, big_list, big_scratch;
    // tiles / pairs / pixels: pairs ping-pong between (keys_a, pair_vals_buf) and (keys_b, vals_b)
    DevBuf ranges, keys_a, pair_vals_buf, keys_b, vals_b, radix_counts, radix_offsets;
    DevBuf tile_counts;  // tile-major scatter: chunk x tile pair counts, then absolute positions
    DevBuf tile_order;   // K5's tile order (longest list first)
    DevBuf final_T, n_contrib, slow_list;
    DevBuf stats;  // BinState
    DevBuf scan_tmp;
    DevBuf tmp_img;                    // image target when the caller passes none
    BinState* host_stats = nullptr;    // pinned copy of `stats`
    long long pair_cap = 0;            // capacity of the pair buffers (0: not learned yet)
    // results
    int n = 0, n_valid = 0;
    long long n_pairs = 0;
    int width = 0, height = 0, tiles_x = 0, tiles_y = 0;
    bool have_src = false;
    double bg[3] = {0, 0, 0};

    SplatArrays arrays() const {
        SplatArrays a;
        a.valid = valid.as<uint8_t>();
        a.tiles = tiles.as<uint32_t>();
        a.mean2 = mean2.as<double2>();
        a.conic_ab = conic_ab.as<double4>();
        a.color_depth = color_depth.as<double4>();
        a.flow_radius = flow_radius.as<double4>();
        a.rect = rect.as<ushort4>();
        a.conic_f = conic_f.as<float4>();
        a.color_f = color_f.as<float4>();
        a.guard_f = guard_f.as<float4>();
        a.ext_f = ext_f.as<float4>();
        a.source_index = have_src ? src.as<int32_t>() : nullptr;
        a.depth_key = key.as<unsigned long long>();
        a.dir_dist = dir_dist.as<double4>();
        return a;
    }
    const uint32_t* pair_vals() const { return pair_vals_buf.as<uint32_t>(); }
    // tile-major scatter: the tile starts follow the chunk x tile matrix (16-byte aligned)
    uint32_t* tile_starts(int ntiles, int n) const {
        return tile_counts.as<uint32_t>() + ((rgs_launch::tile_count_words(n, ntiles) + 3) & ~size_t(3));
    }
    BinState* dstats() const { return stats.as<BinState>(); }

    void ensure_gaussians(int cap, cudaStream_t s) {
        size_t n1 = std::max(cap, 1);
        valid.ensure(n1, s);
        tiles.ensure(4 * n1, s);
        mean2.ensure(16 * n1, s);
        conic_ab.ensure(32 * n1, s);
        color_depth.ensure(32 * n1, s);
        flow_radius.ensure(32 * n1, s);
        rect.ensure(8 * n1, s);
        conic_f.ensure(16 * n1, s);
        color_f.ensure(16 * n1, s);
        guard_f.ensure(16 * n1, s);
        ext_f.ensure(16 * n1, s);
        dir_dist.ensure(32 * n1, s);
        key.ensure(8 * n1, s);
        ent_key.ensure(8 * n1, s);
        ent_id.ensure(4 * n1, s);
        sorted_ids.ensure(4 * n1, s);
        sorted_tiles.ensure(4 * n1, s);
        pair_off.ensure(4 * n1, s);
        big_scratch.ensure(16 * 2 * n1, s);
        const size_t nb = (size_t)rgs_launch::num_depth_buckets();
        bucket_count.ensure(4 * nb, s);
        bucket_off.ensure(4 * nb, s);
        bucket_cur.ensure(4 * nb, s);
        big_list.ensure(4 * nb, s);
        stats.ensure(sizeof(BinState), s);
        scan_tmp.ensure(4 * (4096 + rgs_launch::scan1_scratch_words((int)n1)), s);
        if (!host_stats) CK(cudaMallocHost(&host_stats, sizeof(BinState)));
    }
    void ensure_pixels(size_t npix, int ntiles, cudaStream_t s) {
        final_T.ensure(8 * std::max<size_t>(npix, 1), s);
        n_contrib.ensure(4 * std::max<size_t>(npix, 1), s);
        slow_list.ensure(4 * std::max<size_t>(npix, 1), s);
        const size_t nt = (size_t)std::max(ntiles, 1) + 1;
        ranges.ensure(8 * nt, s);
        tile_order.ensure(4 * nt, s);
    }
    void ensure_pairs(long long p, bool radix, cudaStream_t s) {
        size_t p1 = (size_t)std::max<long long>(p, 1);
        pair_vals_buf.ensure(4 * p1, s);
        if (!radix) return;  // the tile-major scatter writes the sorted splat ids only
        keys_a.ensure(4 * p1, s);
        keys_b.ensure(4 * p1, s);
        vals_b.ensure(4 * p1, s);
        const size_t e = rgs_launch::radix_count_entries(p);
        radix_counts.ensure(4 * e, s);
        radix_offsets.ensure(4 * e, s);
        scan_tmp.ensure(4 * (e / 1024 + 4096), s);
    }
    void release(cudaStream_t s) {
        DevBuf* all[] = {&valid, &tiles, &mean2, &conic_ab, &color_depth, &flow_radius, &rect, &conic_f,
                         &color_f, &guard_f, &ext_f, &src, &key, &dir_dist, &ent_key, &ent_id, &sorted_ids, &sorted_tiles,
                         &pair_off, &bucket_count, &bucket_off, &bucket_cur, &big_list, &big_scratch, &ranges,
                         &keys_a, &pair_vals_buf, &keys_b, &vals_b, &radix_counts, &radix_offsets, &tile_counts,
                         &tile_order, &final_T,
                         &n_contrib, &slow_list, &stats, &scan_tmp, &tmp_img};
        for (DevBuf* b : all) b->release(s);
        if (host_stats) {
            cudaStreamSynchronize(s);
            cudaFreeHost(host_stats);
            host_stats = nullptr;
        }
        pair_cap = 0;
    }
};

}  // namespace

// Pipeline stages timed by the profiling mode (rgs_ctx_set_profiling).
enum Stage {
    kStPreprocess = 0, kStDepthRank, kStHist, kStTileFill, kStTileSort, kStBlend, kStFixup, kStBwdTiles,
    kStBwdFixup, kStBwdGauss, kStBwdColor, kStImageLoss, kStAdam, kStConsistency, kStTileCounts, kStTileScatter,
    kNumStages
};
static const char* kStageNames[kNumStages] = {
    "preprocess_k1", "depth_rank", "pair_offsets_scan", "duplicate_k3", "tile_radix_sort_k4", "blend_fp32_k5",
    "blend_fp64_fixup", "backward_tiles_k6", "backward_fp64_fixup", "backward_gauss_k7b", "backward_color_k7a",
    "image_loss_k8", "adam_k9", "consistency_k10", "tile_counts", "tile_scatter_k4"};

struct rgs_records;
struct rgs_ctx {
    int device = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;
    std::string err;
    int err_index = -1;
    long long launches = 0;
    Frame scratch;
    std::unordered_set<rgs_records*> live_records;  // orphaned (not freed) when the context goes first
    DevBuf deferred;  // u64 deferred status word (RGS_FLAG_DEFER_CHECKS), ~0 when clean
    unsigned long long* host_word = nullptr;  // pinned
    DevBuf sgrad;     // N x 9 doubles (screen-space gradients)
    DevBuf sgrad_fixed;  // N x 9 x 2 u64 (RGS_FLAG_REPRODUCIBLE fixed-point counters)
    DevBuf cgrad;     // N x 3 doubles (the colour path's d mean3, K7a -> K7b)
    DevBuf tile_grads;  // P x 9 doubles (deterministic backward: per (tile, position))
    DevBuf tmp_img;   // host-buffer staging
    DevBuf tmp_splats, tmp_scan, tmp_ids;
    DevBuf slice_cache;  // t-independent slice of the scene of the current view batch (render_batch)
    BinState* host_stats = nullptr;  // pinned
    // profiling: CUDA events around every stage, on the launching stream
    int timing = 0;  // 1: all stages, serialised views; 2: live K5 timing (see rgs_ctx_set_profiling)
    int binning_mode = 0;  // RGS_BINNING_* (rgs_ctx_set_binning)
    bool count_evals = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    struct Pending {
        int stage;
        cudaEvent_t a, b;
    };
    std::vector<Pending> pending;
    double stage_ms[kNumStages] = {0};
    long long stage_n[kNumStages] = {0};
    DevBuf counters;  // 16 x u64: E, B, E_kernel of the FP32 blend, slow reasons (3-6), warp visits (7, 8)
    // multi-view batches (render_batch)
    static constexpr int kSlots = 12;
    Frame slot_frame[kSlots];
    cudaStream_t slot_stream[kSlots] = {};
    cudaEvent_t slot_done[kSlots] = {};
    cudaEvent_t join_ev = nullptr;
    std::vector<void*> frame_pool;   // PooledFrame* of destroyed records
    void* train = nullptr;           // TrainScratch (training-side buffers), created on first use
    void (*train_free)(void*, cudaStream_t) = nullptr;
    BinState* view_stats = nullptr;  // pinned, one per view of the current batch
    size_t view_stats_cap = 0;
    void ensure_view_stats(size_t n) {
        if (n <= view_stats_cap) return;
        if (view_stats) cudaFreeHost(view_stats);
        CK(cudaMallocHost(&view_stats, sizeof(BinState) * n));
        view_stats_cap = n;
    }
    cudaEvent_t next_event() {
        if (ev_used == ev_pool.size()) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            ev_pool.push_back(e);
        }
        return ev_pool[ev_used++];
    }
    void collect() {
        if (pending.empty()) return;
        for (const Pending& p : pending) {
            float ms = 0;
            CK(cudaEventSynchronize(p.b));
            CK(cudaEventElapsedTime(&ms, p.a, p.b));
            stage_ms[p.stage] += ms;
            stage_n[p.stage] += 1;
        }
        pending.clear();
        ev_used = 0;
    }
};

namespace {
// RAII: brackets one pipeline stage with events when profiling is on.
struct StageTimer {
    rgs_ctx* c;
    int stage;
    cudaStream_t s;
    cudaEvent_t a = nullptr;
    StageTimer(rgs_ctx* ctx, int st, cudaStream_t stream) : c(ctx), stage(st), s(stream) {
        if (c->timing == 1 || (c->timing == 2 && stage == kStBlend)) {
            a = c->next_event();
            CK(cudaEventRecord(a, s));
        }
    }
    ~StageTimer() {
        if (a) {
            cudaEvent_t b = c->next_event();
            cudaEventRecord(b, s);
            c->pending.push_back({stage, a, b});
        }
    }
};
}  // namespace

struct rgs_scene {
    rgs_ctx* ctx = nullptr;
    int n = 0;
    int sh_degree = 0;
    float* params = nullptr;     // FP32 storage
    double* params64 = nullptr;  // RGS_SCENE_F64 storage
};

// A retained view's device state, recycled through the context's pool (rgs_records_destroy
// returns it with an event marking the end of its last use, the next user waits on it), so
// a training loop that creates and destroys one record per view allocates nothing per view.
struct PooledFrame {
    Frame f;
    cudaEvent_t free_ev = nullptr;
};

struct rgs_records {
    rgs_ctx* ctx = nullptr;
    PooledFrame* pf = nullptr;
    Frame* fb = nullptr;
    int retained = 0;
    int n_slow = -1;
    // RGS_FLAG_DEFER_CHECKS: the forward's BinState copy is in flight (fb->host_stats, complete
    // at `ready`); resolve() reads it when host-side counts are first needed
    mutable bool pending = false;
    cudaEvent_t ready = nullptr;
};

namespace {

constexpr size_t kFramePoolMax = 8;

PooledFrame* frame_get(rgs_ctx* c, cudaStream_t s) {
    if (c->frame_pool.empty()) return new PooledFrame;
    PooledFrame* pf = static_cast<PooledFrame*>(c->frame_pool.back());
    c->frame_pool.pop_back();
    if (pf->free_ev) cudaStreamWaitEvent(s, pf->free_ev, 0);  // its last user is done
    return pf;
}

void frame_put(rgs_ctx* c, PooledFrame* pf) {
    if (c->frame_pool.size() >= kFramePoolMax) {
        pf->f.release(c->stream);
        if (pf->free_ev) cudaEventDestroy(pf->free_ev);
        delete pf;
        return;
    }
    if (!pf->free_ev) cudaEventCreateWithFlags(&pf->free_ev, cudaEventDisableTiming);
    cudaEventRecord(pf->free_ev, c->stream);
    c->frame_pool.push_back(pf);
}

int set_err(rgs_ctx* ctx, int code, const std::string& msg) {
    if (ctx) ctx->err = msg;
    return code;
}

// Deferred status word of a pair-buffer overflow: index 0, so it reports before rotor errors.
constexpr unsigned long long kOverflowWord = (unsigned long long)RGS_E_OVERFLOW;

// A deferred-check record's host-side counts (and its overflow), read when first needed.
int resolve(rgs_ctx* c, const rgs_records* r) {
    if (!r->pending) return RGS_OK;
    CK(cudaEventSynchronize(r->ready));
    const BinState st = *r->fb->host_stats;
    r->pending = false;
    r->fb->n_valid = st.n_valid;
    r->fb->n_pairs = st.n_pairs;
    if (st.overflow)
        return set_err(c, RGS_E_OVERFLOW, "deferred-check forward outgrew its pair buffers; re-run it checked");
    return RGS_OK;
}

int cuda_fail(rgs_ctx* ctx, const CudaError& e) {
    return set_err(ctx, RGS_E_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e.e) + " at " + e.what);
}

// camera.hpp:19-24 with the reference's expression order.
int validate_camera(rgs_ctx* ctx, const rgs_camera* c) {
    if (!(c->fx > 0) || !(c->fy > 0)) return set_err(ctx, RGS_E_CAMERA, "camera: focal lengths must be positive");
    const double* w = c->world_to_camera;
    double mx = 0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = w[i * 4 + 0] * w[j * 4 + 0];
            s += w[i * 4 + 1] * w[j * 4 + 1];
            s += w[i * 4 + 2] * w[j * 4 + 2];
            double d = std::fabs(s - (i == j ? 1.0 : 0.0));
            mx = (i == 0 && j == 0) ? d : ((mx < d) ? d : mx);
        }
    if (mx > 1e-6) return set_err(ctx, RGS_E_CAMERA, "camera: rotation block not orthogonal");
    if (c->width <= 0 || c->height <= 0) return set_err(ctx, RGS_E_INVALID, "camera: empty image");
    return RGS_OK;
}

DevCamera make_dev_camera(const rgs_camera* c) {
    DevCamera d;
    d.width = c->width;
    d.height = c->height;
    d.tiles_x = (c->width + kTile - 1) / kTile;
    d.tiles_y = (c->height + kTile - 1) / kTile;
    d.fx = c->fx;
    d.fy = c->fy;
    d.cx = c->cx;
    d.cy = c->cy;
    d.time = c->time;
    const double* w = c->world_to_camera;
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) d.R[i * 3 + j] = w[i * 4 + j];
        d.t[i] = w[i * 4 + 3];
    }
    // center = -R^T t, sequential sum (camera.hpp:17 under the Eigen subset).
    for (int i = 0; i < 3; ++i) {
        volatile double s = (-d.R[0 * 3 + i]) * d.t[0];
        s = s + (-d.R[1 * 3 + i]) * d.t[1];
        s = s + (-d.R[2 * 3 + i]) * d.t[2];
        d.center[i] = s;
    }
    return d;
}

const char* rotor_msg(int code) {
    return code == RGS_E_ZERO_ROTOR ? "normalize: zero rotor" : "normalize: result violates rotor invariants";
}

enum Source { kFromScene, kFromSplats };
}  // namespace
namespace {

// K5 / K6 take the tiles longest list first when the view has the GPU to itself (a single
// view, or one view in flight) and its frame is small enough for its records to stay in L2: the
// spatially scattered tile order costs a 3840x2160 / 2M-Gaussian frame 0.9 % (C4: 379.5 vs 382.8
// FPS) while it saves 2.8 % of K5 at 1352x1014 (0.2513 vs 0.2585 ms).
inline bool use_tile_order(bool batch, bool solo, size_t npix) {
    return (!batch || solo) && npix <= (size_t)2200000;
}

// Enqueues the forward pipeline of one view into frame `f` on stream `s`.
//
// No host synchronisation in the steady state: the pair buffers have a capacity
// (learned from the first view, grown on demand); a view whose pair count exceeds it
// sets BinState::overflow, skips the pair work, and is re-rendered after a sync.  The
// view's BinState is copied asynchronously to `host_stats`.  With `sync` the view is
// resolved before returning (errors reported, overflow re-rendered).
int run_forward(rgs_ctx* ctx, Frame& f, cudaStream_t s, Source src, const rgs_scene* scene, const void* dev_splats,
                int n_splats, bool splats_monotone, const rgs_camera* cam, const double bg[3], unsigned flags,
                float* image, bool flow_mode, bool sync, BinState* host_stats,
                const SliceCacheView* slice_cache = nullptr, bool render_only = false, bool batch = false,
                bool solo = false) {
    const DevCamera dc = make_dev_camera(cam);
    const int n = src == kFromScene ? scene->n : n_splats;
    const size_t npix = (size_t)cam->width * cam->height;
    const int ntiles = dc.tiles_x * dc.tiles_y;
    // tile keys hold ty and tx in 12 bits each (rgs_launch::tile_key_shift); pixel indices are 32-bit
    if (dc.tiles_x > 4096 || dc.tiles_y > 4096 || npix >= ((size_t)1 << 31))
        return set_err(ctx, RGS_E_INVALID, "image too large: at most 65536 x 65536 tiles' worth, < 2^31 pixels");
    f.n = n;
    f.width = cam->width;
    f.height = cam->height;
    f.tiles_x = dc.tiles_x;
    f.tiles_y = dc.tiles_y;
    for (int k = 0; k < 3; ++k) f.bg[k] = bg ? bg[k] : 0.0;
    f.ensure_gaussians(n, s);
    f.ensure_pixels(npix, ntiles, s);
    f.have_src = src == kFromSplats;  // frames are recycled between scene and splat renders
    if (f.have_src) f.src.ensure(4 * (size_t)std::max(n, 1), s);
    const int nb = 1 << rgs_launch::depth_bucket_bits(n);
    // Binning: the tile-major scatter (up to 256 x 256 and 8192 tiles) for single views -- the
    // shorter critical path; K3 + the radix passes for the views of a batch, which overlap the
    // blends of the other views in flight better ("Binning").
    const bool scatter =
        rgs_launch::tile_scatter_usable(dc.tiles_x, dc.tiles_y, n, f.pair_cap, batch, ctx->binning_mode);
    rgs_launch::frame_init(f.dstats(), (uint32_t)std::min<long long>(f.pair_cap, 0xffffffffll),
                           f.bucket_count.as<uint32_t>(), f.bucket_cur.as<uint32_t>(), n, s);
    ctx->launches += 1;
    SplatArrays sa = f.arrays();
    if (render_only && !flow_mode) {
        // no records are kept: the flow / radius records (export, flow renders) and the view
        // directions (backward) are not written
        sa.flow_radius = nullptr;
        sa.dir_dist = nullptr;
    }
    BinState* st_dev = f.dstats();

    // K1: slice + project + SH (or host splats), depth keys, key range.
    {
        StageTimer t(ctx, kStPreprocess, s);
        if (src == kFromScene)
            rgs_launch::preprocess(scene->params, scene->params64, n, scene->sh_degree, dc, sa, st_dev, s, slice_cache);
        else
            rgs_launch::splats_from_host(dev_splats, n, dc, sa, st_dev, s);
        ctx->launches += 1;
    }
    // Global (depth, index) ranks: depth-bucket histogram + scan, scatter, per-bucket sorts.
    uint32_t* scan_tmp = f.scan_tmp.as<uint32_t>();
    {
        StageTimer t(ctx, kStDepthRank, s);
        rgs_launch::bucket_hist(sa.valid, sa.depth_key, n, st_dev, f.bucket_count.as<uint32_t>(), s);
        rgs_launch::exclusive_scan_1p(f.bucket_count.as<uint32_t>(), nb, f.bucket_off.as<uint32_t>(), scan_tmp + 2048,
                                   nullptr, s);
        rgs_launch::depth_ranks(sa.valid, sa.depth_key, sa.tiles, n,
                                (src == kFromSplats && !splats_monotone) ? sa.source_index : nullptr, st_dev,
                                f.bucket_count.as<uint32_t>(), f.bucket_off.as<uint32_t>(),
                                f.bucket_cur.as<uint32_t>(), f.ent_key.as<unsigned long long>(),
                                f.ent_id.as<uint32_t>(), f.sorted_ids.as<uint32_t>(), f.sorted_tiles.as<uint32_t>(),
                                f.big_list.as<uint32_t>(), f.big_scratch.p, s);
        ctx->launches += 6;
    }
    if (scatter) {
        // Per-chunk tile counts -> absolute positions, tile ranges and the pair count.
        StageTimer t(ctx, kStTileCounts, s);
        f.tile_counts.ensure(4 * (rgs_launch::tile_count_words(n, ntiles) + ntiles + 4), s);
        rgs_launch::tile_counts(f.sorted_ids.as<uint32_t>(), f.sorted_tiles.as<uint32_t>(), sa.rect, st_dev, n,
                                dc.tiles_x, dc.tiles_y, f.tile_counts.as<uint32_t>(), f.tile_starts(ntiles, n),
                                f.ranges.as<uint2>(), s);
        ctx->launches += 3;
    } else {
        // Pair offsets in rank order (exclusive scan of tiles-touched; total = pair count).
        StageTimer t(ctx, kStHist, s);
        rgs_launch::exclusive_scan_1p(f.sorted_tiles.as<uint32_t>(), n, f.pair_off.as<uint32_t>(), scan_tmp + 4096,
                                   &st_dev->n_pairs, s, &st_dev->n_valid);
        ctx->launches += 1;
    }
    if (f.pair_cap == 0) {
        // First view of this frame slot: learn the pair count once, size with headroom.
        CK(cudaMemcpyAsync(f.host_stats, st_dev, sizeof(BinState), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        f.pair_cap = std::max<long long>(4096, (long long)f.host_stats->n_pairs * 5 / 4 + 1024);
        const uint32_t cap = (uint32_t)std::min<long long>(f.pair_cap, 0xffffffffll);
        CK(cudaMemcpyAsync(&st_dev->pair_cap, &cap, sizeof cap, cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));
    }
    f.ensure_pairs(f.pair_cap, !scatter, s);
    rgs_launch::check_capacity(st_dev, s);
    ctx->launches += 1;

    if (scatter) {
        StageTimer t(ctx, kStTileScatter, s);
        rgs_launch::tile_scatter(f.sorted_ids.as<uint32_t>(), f.sorted_tiles.as<uint32_t>(), sa.rect, st_dev, n,
                                 dc.tiles_x, dc.tiles_y, f.tile_counts.as<uint32_t>(), f.tile_starts(ntiles, n),
                                 f.ranges.as<uint2>(), f.pair_vals_buf.as<uint32_t>(), s);
        ctx->launches += 1;
    } else {
        // Duplicate-with-key in rank order, then the two stable tile-digit passes.
        {
            StageTimer t(ctx, kStTileFill, s);
            // scan_tmp is free again after the pair-offset scan: it holds the digit histograms
            rgs_launch::duplicate(f.sorted_ids.as<uint32_t>(), f.pair_off.as<uint32_t>(),
                                  f.sorted_tiles.as<uint32_t>(), sa.rect, st_dev, n, dc.tiles_x, dc.tiles_y,
                                  f.keys_a.as<uint32_t>(), f.pair_vals_buf.as<uint32_t>(), f.scan_tmp.as<int>(), s);
            ctx->launches += 1;
        }
        StageTimer t(ctx, kStTileSort, s);
        const int in_b = rgs_launch::tile_radix_sort(
            f.keys_a.as<uint32_t>(), f.pair_vals_buf.as<uint32_t>(), f.keys_b.as<uint32_t>(), f.vals_b.as<uint32_t>(),
            st_dev, f.pair_cap, dc.tiles_x, dc.tiles_y, f.radix_counts.as<uint32_t>(), f.radix_offsets.as<uint32_t>(),
            f.scan_tmp.as<int>(), f.ranges.as<uint2>(), s);
        ctx->launches += in_b ? 5 : 3;
        if (in_b) {  // three passes: the sorted pairs are in the B buffers (roles swapped for this frame)
            std::swap(f.keys_a, f.keys_b);
            std::swap(f.pair_vals_buf, f.vals_b);
        }
    }

    // Blend.
    uint32_t* nc = flow_mode ? nullptr : f.n_contrib.as<uint32_t>();
    double* fT = flow_mode ? nullptr : f.final_T.as<double>();
    int* slow_count = &f.dstats()->slow_count;
    double* image64 = (flags & RGS_FLAG_IMAGE_F64) ? reinterpret_cast<double*>(image) : nullptr;
    float* image32 = image64 ? nullptr : image;
    if (image64) flags |= RGS_FLAG_BLEND_FP64;
    if (!image32 && !image64) {
        f.tmp_img.ensure(npix * 3 * sizeof(float), s);
        image32 = f.tmp_img.as<float>();
    }
    if (flags & RGS_FLAG_BLEND_FP64) {
        rgs_launch::mark_all_slow((int)npix, f.slow_list.as<uint32_t>(), slow_count, s);
        ctx->launches += 1;
    } else {
        unsigned long long* counters = nullptr;
        if (ctx->count_evals && !flow_mode) counters = ctx->counters.as<unsigned long long>();
        StageTimer t(ctx, kStBlend, s);
        rgs_launch::blend_fp32(sa, f.pair_vals(), f.ranges.as<uint2>(), dc,
                               make_float3((float)f.bg[0], (float)f.bg[1], (float)f.bg[2]), flow_mode ? 1 : 0,
                               image32, fT, nc, f.slow_list.as<uint32_t>(), slow_count, counters, s,
                               // longest tiles first when the view has the GPU to itself (single
                               // views, the serialised profiling mode); in a pipelined batch the
                               // other views fill the tail and the order kernel only adds latency
                               use_tile_order(batch, solo, npix) ? f.tile_order.as<uint32_t>() : nullptr);
        ctx->launches += use_tile_order(batch, solo, npix) ? 2 : 1;

    }
    {
        StageTimer t(ctx, kStFixup, s);
        rgs_launch::blend_fp64_pixels(sa, f.pair_vals(), f.ranges.as<uint2>(), dc,
                                      make_double3(f.bg[0], f.bg[1], f.bg[2]), flow_mode ? 1 : 0, image32, image64,
                                      fT, nc, f.slow_list.as<uint32_t>(), slow_count, (int)npix, s);
        ctx->launches += 1;
    }
    CK(cudaGetLastError());
    BinState* hs = host_stats ? host_stats : f.host_stats;
    CK(cudaMemcpyAsync(hs, st_dev, sizeof(BinState), cudaMemcpyDeviceToHost, s));
    if (!sync) return RGS_OK;
    CK(cudaStreamSynchronize(s));
    const BinState st = *hs;
    if (st.err != kNoError) {
        const int code = (int)(st.err & 0xff);
        ctx->err_index = (int)(st.err >> 8);
        return set_err(ctx, code, rotor_msg(code));
    }
    if (st.overflow) {
        f.pair_cap = (long long)st.n_pairs * 5 / 4 + 1024;
        return run_forward(ctx, f, s, src, scene, dev_splats, n_splats, splats_monotone, cam, bg, flags, image,
                           flow_mode, true, host_stats, slice_cache, render_only, batch);
    }
    f.n_valid = st.n_valid;
    f.n_pairs = st.n_pairs;
    return RGS_OK;
}

template <typename F>
int guarded(rgs_ctx* ctx, F&& fn) {
    if (!ctx) return RGS_E_INVALID;
    try {
        CK(cudaSetDevice(ctx->device));
        ctx->err.clear();
        return fn();
    } catch (const CudaError& e) {
        return cuda_fail(ctx, e);
    } catch (const std::exception& e) {
        return set_err(ctx, RGS_E_INVALID, e.what());
    }
}

}  // namespace

extern "C" {

int rgs_abi_version(void) { return RGS_ABI_VERSION; }

int rgs_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int rgs_ctx_create(int device, rgs_ctx** out) {
    if (!out) return RGS_E_INVALID;
    *out = nullptr;
    int n = rgs_device_count();
    if (n <= 0 || device < 0 || device >= n) return RGS_E_NO_DEVICE;
    rgs_ctx* c = new rgs_ctx;
    c->device = device;
    try {
        CK(cudaSetDevice(device));
        CK(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        CK(cudaMallocHost(&c->host_stats, sizeof(BinState)));
        CK(cudaMallocHost(&c->host_word, sizeof(unsigned long long)));
        for (int k = 0; k < rgs_ctx::kSlots; ++k) {
            CK(cudaStreamCreateWithFlags(&c->slot_stream[k], cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&c->slot_done[k], cudaEventDisableTiming));
        }
        CK(cudaEventCreateWithFlags(&c->join_ev, cudaEventDisableTiming));
        if (!rgs_launch::binning_init()) throw CudaError{cudaErrorInvalidValue, "binning_init"};
        c->binning_mode = rgs_launch::default_binning_mode();
        if (!rgs_launch::raster_init()) throw CudaError{cudaErrorInvalidValue, "raster_init"};
        if (!rgs_launch::train_init()) throw CudaError{cudaErrorInvalidValue, "train_init"};
        // Keep freed blocks in the pool: frames re-grow without hitting the driver.
        cudaMemPool_t pool;
        CK(cudaDeviceGetDefaultMemPool(&pool, device));
        unsigned long long thresh = ~0ull;
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh));
        c->deferred.ensure(sizeof(unsigned long long), c->own_stream);
        CK(cudaMemsetAsync(c->deferred.p, 0xff, sizeof(unsigned long long), c->own_stream));
        CK(cudaStreamSynchronize(c->own_stream));
    } catch (const CudaError& e) {
        delete c;
        return RGS_E_CUDA;
    }
    c->stream = c->own_stream;
    *out = c;
    return RGS_OK;
}

void rgs_ctx_destroy(rgs_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    for (rgs_records* r : c->live_records) {  // records outliving their context: orphaned
        r->pf->f.release(c->stream);
        if (r->pf->free_ev) cudaEventDestroy(r->pf->free_ev);
        delete r->pf;
        r->pf = nullptr;
        r->fb = nullptr;
        if (r->ready) cudaEventDestroy(r->ready);
        r->ready = nullptr;
        r->ctx = nullptr;
    }
    c->live_records.clear();
    c->scratch.release(c->stream);
    c->deferred.release(c->stream);
    c->sgrad.release(c->stream);
    c->sgrad_fixed.release(c->stream);
    c->cgrad.release(c->stream);
    c->tmp_img.release(c->stream);
    c->tmp_splats.release(c->stream);
    c->tmp_scan.release(c->stream);
    c->tmp_ids.release(c->stream);
    c->slice_cache.release(c->stream);
    for (void* v : c->frame_pool) {
        PooledFrame* pf = static_cast<PooledFrame*>(v);
        pf->f.release(c->stream);
        if (pf->free_ev) cudaEventDestroy(pf->free_ev);
        delete pf;
    }
    c->frame_pool.clear();
    if (c->train && c->train_free) c->train_free(c->train, c->stream);
    for (int k = 0; k < rgs_ctx::kSlots; ++k) {
        if (!c->slot_stream[k]) continue;
        c->slot_frame[k].release(c->slot_stream[k]);
        cudaStreamSynchronize(c->slot_stream[k]);
        cudaStreamDestroy(c->slot_stream[k]);
        cudaEventDestroy(c->slot_done[k]);
    }
    if (c->join_ev) cudaEventDestroy(c->join_ev);
    if (c->view_stats) cudaFreeHost(c->view_stats);
    for (size_t i = 0; i < c->ev_pool.size(); ++i) cudaEventDestroy(c->ev_pool[i]);
    cudaStreamSynchronize(c->stream);
    if (c->host_stats) cudaFreeHost(c->host_stats);
    if (c->host_word) cudaFreeHost(c->host_word);
    if (c->own_stream) cudaStreamDestroy(c->own_stream);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    delete c;
}

int rgs_ctx_set_stream(rgs_ctx* c, void* stream) {
    if (!c) return RGS_E_INVALID;
    c->stream = stream ? reinterpret_cast<cudaStream_t>(stream) : c->own_stream;
    return RGS_OK;
}
void* rgs_ctx_stream(rgs_ctx* c) { return c ? (void*)c->stream : nullptr; }
const char* rgs_ctx_last_error(const rgs_ctx* c) { return c ? c->err.c_str() : "null context"; }
int rgs_ctx_error_index(const rgs_ctx* c) { return c ? c->err_index : -1; }
long long rgs_ctx_kernel_launches(const rgs_ctx* c) { return c ? c->launches : 0; }

int rgs_profile_num_stages(void) { return kNumStages; }
const char* rgs_profile_stage_name(int k) { return (k >= 0 && k < kNumStages) ? kStageNames[k] : ""; }

int rgs_ctx_set_binning(rgs_ctx* c, int mode) {
    if (!c) return RGS_E_INVALID;
    if (mode < RGS_BINNING_AUTO || mode > RGS_BINNING_SCATTER) return set_err(c, RGS_E_INVALID, "unknown binning mode");
    c->binning_mode = mode;
    return RGS_OK;
}

int rgs_ctx_set_profiling(rgs_ctx* c, int timing, int count_evals) {
    return guarded(c, [&] {
        c->collect();
        c->timing = timing < 0 ? 0 : (timing > 2 ? 1 : timing);
        c->count_evals = count_evals != 0;
        if (c->count_evals) {
            c->counters.ensure(128, c->stream);
            CK(cudaMemsetAsync(c->counters.p, 0, 128, c->stream));
        }
        return RGS_OK;
    });
}

int rgs_measure_fp32_tflops(rgs_ctx* c, double* tflops) {
    if (!tflops) return RGS_E_INVALID;
    return guarded(c, [&] {
        DevBuf out;
        out.ensure(64, c->stream);
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        const int blocks = 148 * 8;
        rgs_launch::ffma_peak(out.as<float>(), blocks, 64, c->stream);  // warm-up
        double best = 0;
        for (int rep = 0; rep < 5; ++rep) {
            CK(cudaEventRecord(a, c->stream));
            const double fmas = rgs_launch::ffma_peak(out.as<float>(), blocks, 4096, c->stream);
            CK(cudaEventRecord(b, c->stream));
            CK(cudaEventSynchronize(b));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, a, b));
            best = std::max(best, 2.0 * fmas / (ms * 1e-3) / 1e12);
        }
        c->launches += 6;
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        out.release(c->stream);
        *tflops = best;
        return RGS_OK;
    });
}

int rgs_measure_fp64_tflops(rgs_ctx* c, double* tflops) {
    if (!tflops) return RGS_E_INVALID;
    return guarded(c, [&] {
        DevBuf out;
        out.ensure(64, c->stream);
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        const int blocks = 148 * 8;
        rgs_launch::dfma_peak(out.as<double>(), blocks, 16, c->stream);  // warm-up
        double best = 0;
        for (int rep = 0; rep < 5; ++rep) {
            CK(cudaEventRecord(a, c->stream));
            const double fmas = rgs_launch::dfma_peak(out.as<double>(), blocks, 256, c->stream);
            CK(cudaEventRecord(b, c->stream));
            CK(cudaEventSynchronize(b));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, a, b));
            best = std::max(best, 2.0 * fmas / (ms * 1e-3) / 1e12);
        }
        c->launches += 6;
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        out.release(c->stream);
        *tflops = best;
        return RGS_OK;
    });
}

int rgs_ctx_profile_reset(rgs_ctx* c) {
    return guarded(c, [&] {
        c->collect();
        for (int k = 0; k < kNumStages; ++k) {
            c->stage_ms[k] = 0;
            c->stage_n[k] = 0;
        }
        if (c->counters.p) CK(cudaMemsetAsync(c->counters.p, 0, 128, c->stream));
        return RGS_OK;
    });
}

int rgs_ctx_profile_read(rgs_ctx* c, double* stage_ms, long long* stage_launches, unsigned long long* evals) {
    return guarded(c, [&] {
        c->collect();
        for (int k = 0; k < kNumStages; ++k) {
            if (stage_ms) stage_ms[k] = c->stage_ms[k];
            if (stage_launches) stage_launches[k] = c->stage_n[k];
        }
        if (evals) {
            evals[0] = evals[1] = evals[2] = 0;
            if (c->counters.p) {
                CK(cudaMemcpyAsync(evals, c->counters.p, 24, cudaMemcpyDeviceToHost, c->stream));
                CK(cudaStreamSynchronize(c->stream));
            }
        }
        return RGS_OK;
    });
}
int rgs_ctx_profile_slow_reasons(rgs_ctx* c, unsigned long long* out4) {
    if (!out4) return RGS_E_INVALID;
    return guarded(c, [&]() -> int {
        for (int k = 0; k < 4; ++k) out4[k] = 0;
        if (!c->counters.p) return RGS_OK;
        CK(cudaMemcpyAsync(out4, c->counters.as<unsigned long long>() + 3, 32, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        return RGS_OK;
    });
}

int rgs_ctx_profile_blend_visits(rgs_ctx* c, unsigned long long* out2) {
    if (!out2) return RGS_E_INVALID;
    return guarded(c, [&]() -> int {
        out2[0] = out2[1] = 0;
        if (!c->counters.p) return RGS_OK;
        CK(cudaMemcpyAsync(out2, c->counters.as<unsigned long long>() + 7, 16, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        return RGS_OK;
    });
}

int rgs_ctx_synchronize(rgs_ctx* c) {
    return guarded(c, [&] {
        CK(cudaStreamSynchronize(c->stream));
        return RGS_OK;
    });
}

void* rgs_malloc(rgs_ctx* c, size_t bytes) {
    if (!c) return nullptr;
    void* p = nullptr;
    if (cudaSetDevice(c->device) != cudaSuccess || cudaMalloc(&p, std::max<size_t>(bytes, 1)) != cudaSuccess) {
        set_err(c, RGS_E_CUDA, "rgs_malloc: out of device memory");
        return nullptr;
    }
    return p;
}
void rgs_free(rgs_ctx* c, void* p) {
    if (!c || !p) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    cudaFree(p);
}
int rgs_memcpy(rgs_ctx* c, void* dst, const void* src, size_t bytes) {
    if (!dst || !src) return RGS_E_INVALID;
    return guarded(c, [&]() -> int {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        return RGS_OK;
    });
}

int rgs_camera_validate(rgs_ctx* c, const rgs_camera* cam) {
    if (!cam) return RGS_E_INVALID;
    return validate_camera(c, cam);
}

// ------------------------------------------------------------------ scene
int rgs_scene_create_ex(rgs_ctx* c, int n, int sh_degree, unsigned scene_flags, rgs_scene** out) {
    if (!out || n < 0 || (scene_flags & ~RGS_SCENE_F64)) return RGS_E_INVALID;
    return guarded(c, [&] {
        rgs_scene* s = new rgs_scene;
        s->ctx = c;
        s->n = n;
        s->sh_degree = sh_degree;
        const size_t cnt = 65 * (size_t)std::max(n, 1);
        if (scene_flags & RGS_SCENE_F64) {
            CK(cudaMalloc(&s->params64, sizeof(double) * cnt));
            CK(cudaMemsetAsync(s->params64, 0, sizeof(double) * cnt, c->stream));
        } else {
            CK(cudaMalloc(&s->params, sizeof(float) * cnt));
            CK(cudaMemsetAsync(s->params, 0, sizeof(float) * cnt, c->stream));
        }
        *out = s;
        return RGS_OK;
    });
}

int rgs_scene_create(rgs_ctx* c, int n, int sh_degree, rgs_scene** out) {
    return rgs_scene_create_ex(c, n, sh_degree, 0u, out);
}

void rgs_scene_destroy(rgs_scene* s) {
    if (!s) return;
    cudaSetDevice(s->ctx->device);
    cudaFree(s->params);
    cudaFree(s->params64);
    delete s;
}
int rgs_scene_size(const rgs_scene* s) { return s ? s->n : 0; }
int rgs_scene_set_sh_degree(rgs_scene* s, int d) {
    if (!s) return RGS_E_INVALID;
    s->sh_degree = d;
    return RGS_OK;
}
float* rgs_scene_params(rgs_scene* s) { return s ? s->params : nullptr; }
double* rgs_scene_params_f64(rgs_scene* s) { return s ? s->params64 : nullptr; }

int rgs_scene_upload_f32(rgs_ctx* c, rgs_scene* s, const float* mean, const float* ls, const float* rot,
                         const float* op, const float* sh) {
    if (!s || !mean || !ls || !rot || !op || !sh) return RGS_E_INVALID;
    return guarded(c, [&] {
        const size_t n = (size_t)s->n;
        if (n == 0) return RGS_OK;
        if (s->params64) {  // widen on the host, then the exact FP64 upload
            std::vector<double> d(65 * n);
            std::vector<float> h(65 * n);
            CK(cudaMemcpy(h.data(), mean, 16 * n, cudaMemcpyDefault));
            CK(cudaMemcpy(h.data() + 4 * n, ls, 16 * n, cudaMemcpyDefault));
            CK(cudaMemcpy(h.data() + 8 * n, rot, 32 * n, cudaMemcpyDefault));
            CK(cudaMemcpy(h.data() + 16 * n, op, 4 * n, cudaMemcpyDefault));
            CK(cudaMemcpy(h.data() + 17 * n, sh, 192 * n, cudaMemcpyDefault));
            for (size_t k = 0; k < 65 * n; ++k) d[k] = h[k];
            return (rgs_status)rgs_scene_upload_f64(c, s, d.data(), d.data() + 4 * n, d.data() + 8 * n, d.data() + 16 * n,
                                        d.data() + 17 * n, nullptr);
        }
        DevBuf tmp;
        tmp.ensure(sizeof(float) * 65 * n, c->stream);
        float* t = tmp.as<float>();
        CK(cudaMemcpyAsync(t, mean, 16 * n, cudaMemcpyDefault, c->stream));
        CK(cudaMemcpyAsync(t + 4 * n, ls, 16 * n, cudaMemcpyDefault, c->stream));
        CK(cudaMemcpyAsync(t + 8 * n, rot, 32 * n, cudaMemcpyDefault, c->stream));
        CK(cudaMemcpyAsync(t + 16 * n, op, 4 * n, cudaMemcpyDefault, c->stream));
        CK(cudaMemcpyAsync(t + 17 * n, sh, 192 * n, cudaMemcpyDefault, c->stream));
        rgs_launch::scene_pack(t, t + 4 * n, t + 8 * n, t + 16 * n, t + 17 * n, (int)n, s->params, c->stream);
        c->launches += 1;
        tmp.release(c->stream);
        CK(cudaStreamSynchronize(c->stream));
        return RGS_OK;
    });
}

int rgs_scene_upload_f64(rgs_ctx* c, rgs_scene* s, const double* mean, const double* ls, const double* rot,
                         const double* op, const double* sh, long long* n_inexact) {
    if (!s || !mean || !ls || !rot || !op || !sh) return RGS_E_INVALID;
    const size_t n = (size_t)s->n;
    if (s->params64) {
        if (n_inexact) *n_inexact = 0;
        return guarded(c, [&] {
            if (n == 0) return RGS_OK;
            DevBuf tmp;
            tmp.ensure(sizeof(double) * 65 * n, c->stream);
            double* t = tmp.as<double>();
            CK(cudaMemcpyAsync(t, mean, 32 * n, cudaMemcpyHostToDevice, c->stream));
            CK(cudaMemcpyAsync(t + 4 * n, ls, 32 * n, cudaMemcpyHostToDevice, c->stream));
            CK(cudaMemcpyAsync(t + 8 * n, rot, 64 * n, cudaMemcpyHostToDevice, c->stream));
            CK(cudaMemcpyAsync(t + 16 * n, op, 8 * n, cudaMemcpyHostToDevice, c->stream));
            CK(cudaMemcpyAsync(t + 17 * n, sh, 384 * n, cudaMemcpyHostToDevice, c->stream));
            rgs_launch::scene_pack64(t, t + 4 * n, t + 8 * n, t + 16 * n, t + 17 * n, (int)n, s->params64,
                                     c->stream);
            c->launches += 1;
            tmp.release(c->stream);
            CK(cudaStreamSynchronize(c->stream));
            return RGS_OK;
        });
    }
    std::vector<float> f(65 * std::max<size_t>(n, 1));
    long long inexact = 0;
    auto conv = [&](const double* src, size_t cnt, float* dst) {
        for (size_t i = 0; i < cnt; ++i) {
            dst[i] = (float)src[i];
            if ((double)dst[i] != src[i] && !(std::isnan(src[i]))) ++inexact;
        }
    };
    conv(mean, 4 * n, f.data());
    conv(ls, 4 * n, f.data() + 4 * n);
    conv(rot, 8 * n, f.data() + 8 * n);
    conv(op, n, f.data() + 16 * n);
    conv(sh, 48 * n, f.data() + 17 * n);
    if (n_inexact) *n_inexact = inexact;
    return rgs_scene_upload_f32(c, s, f.data(), f.data() + 4 * n, f.data() + 8 * n, f.data() + 16 * n,
                                f.data() + 17 * n);
}

int rgs_scene_download_f64(rgs_ctx* c, const rgs_scene* s, double* mean, double* ls, double* rot, double* op,
                           double* sh) {
    if (!s) return RGS_E_INVALID;
    return guarded(c, [&] {
        const size_t n = (size_t)s->n;
        if (n == 0) return RGS_OK;
        DevBuf tmp;
        tmp.ensure(sizeof(double) * 65 * n, c->stream);
        double* t = tmp.as<double>();
        rgs_launch::scene_unpack(s->params, s->params64, (int)n, t, t + 4 * n, t + 8 * n, t + 16 * n, t + 17 * n, c->stream);
        c->launches += 1;
        if (mean) CK(cudaMemcpyAsync(mean, t, 32 * n, cudaMemcpyDeviceToHost, c->stream));
        if (ls) CK(cudaMemcpyAsync(ls, t + 4 * n, 32 * n, cudaMemcpyDeviceToHost, c->stream));
        if (rot) CK(cudaMemcpyAsync(rot, t + 8 * n, 64 * n, cudaMemcpyDeviceToHost, c->stream));
        if (op) CK(cudaMemcpyAsync(op, t + 16 * n, 8 * n, cudaMemcpyDeviceToHost, c->stream));
        if (sh) CK(cudaMemcpyAsync(sh, t + 17 * n, 384 * n, cudaMemcpyDeviceToHost, c->stream));
        tmp.release(c->stream);
        CK(cudaStreamSynchronize(c->stream));
        return RGS_OK;
    });
}

// ------------------------------------------------------------------ forward
static int forward_common(rgs_ctx* c, Source src, const rgs_scene* scene, const rgs_splat* splats, int n_splats,
                          const rgs_camera* cam, const double bg[3], unsigned flags, float* image,
                          rgs_records** records, bool flow) {
    if (!cam) return RGS_E_INVALID;
    return guarded(c, [&]() -> int {
        int rc = validate_camera(c, cam);
        if (rc) return rc;
        c->err_index = -1;
        const size_t npix = (size_t)cam->width * cam->height;
        const size_t chans = flow ? 2 : 3;
        const size_t elem = (flags & RGS_FLAG_IMAGE_F64) ? sizeof(double) : sizeof(float);
        const bool host_io = (flags & RGS_FLAG_HOST_BUFFERS) != 0;
        float* dimg = image;
        if (host_io && image) {
            c->tmp_img.ensure(npix * 3 * sizeof(double), c->stream);
            dimg = c->tmp_img.as<float>();
        }
        const void* dsp = nullptr;
        bool monotone = true;
        if (src == kFromSplats) {
            c->tmp_splats.ensure(sizeof(rgs_splat) * (size_t)std::max(n_splats, 1), c->stream);
            if (n_splats > 0)
                CK(cudaMemcpyAsync(c->tmp_splats.p, splats, sizeof(rgs_splat) * (size_t)n_splats,
                                   host_io ? cudaMemcpyHostToDevice : cudaMemcpyDefault, c->stream));
            dsp = c->tmp_splats.p;
            // Monotone source indices: index order already is the tie-break order.
            std::vector<rgs_splat> h;
            const rgs_splat* hp = splats;
            cudaPointerAttributes attr;
            if (cudaPointerGetAttributes(&attr, splats) == cudaSuccess && attr.type == cudaMemoryTypeDevice) {
                h.resize(n_splats);
                CK(cudaMemcpy(h.data(), splats, sizeof(rgs_splat) * n_splats, cudaMemcpyDeviceToHost));
                hp = h.data();
            }
            cudaGetLastError();
            for (int i = 1; i < n_splats; ++i)
                if (hp[i].source_index <= hp[i - 1].source_index) monotone = false;
        }
        rgs_records* rec = nullptr;
        Frame* f = &c->scratch;
        if (records) {
            rec = new rgs_records;
            rec->ctx = c;
            c->live_records.insert(rec);
            rec->retained = (flags & RGS_FLAG_RETAIN_RECORDS) ? 1 : 0;
            rec->pf = frame_get(c, c->stream);
            rec->fb = &rec->pf->f;
            f = rec->fb;
        }
        // Deferred checks (a retained record whose frame already knows its pair capacity): no
        // host synchronisation; errors and overflow go to the context's deferred status word.
        const bool defer = (flags & RGS_FLAG_DEFER_CHECKS) && rec && !host_io && f->pair_cap > 0;
        if (defer) {
            // no re-render is possible after the fact: 2x headroom over the frame's last checked
            // pair count (an overflow is still reported, as RGS_E_OVERFLOW, never silent)
            f->pair_cap = std::max<long long>(f->pair_cap, 2 * f->n_pairs + 1024);
        }
        // A record whose forward fails (status code or CUDA error) is unregistered and its
        // frame returned to the pool before the error propagates.
        auto drop_rec = [&] {
            if (!rec) return;
            c->live_records.erase(rec);
            frame_put(c, rec->pf);
            if (rec->ready) cudaEventDestroy(rec->ready);
            delete rec;
            rec = nullptr;
        };
        try {
            rc = run_forward(c, *f, c->stream, src, scene, dsp, n_splats, monotone, cam, bg, flags, dimg, flow,
                             !defer, nullptr);
            if (defer && !rc) {
                rgs_launch::fold_status(f->dstats(), c->deferred.as<unsigned long long>(), kOverflowWord, c->stream);
                c->launches += 1;
                if (!rec->ready) CK(cudaEventCreateWithFlags(&rec->ready, cudaEventDisableTiming));
                CK(cudaEventRecord(rec->ready, c->stream));
                rec->pending = true;
            }
        } catch (...) {
            drop_rec();
            throw;
        }
        if (rc) {
            drop_rec();
            return rc;
        }
        if (host_io && image) {
            CK(cudaMemcpyAsync(image, dimg, npix * chans * elem, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
        }
        if (records) *records = rec;
        return RGS_OK;
    });
}

int rgs_render_forward(rgs_ctx* c, const rgs_scene* scene, const rgs_camera* cam, const double bg[3], unsigned flags,
                       float* image, rgs_records** records) {
    if (!scene) return RGS_E_INVALID;
    return forward_common(c, kFromScene, scene, nullptr, 0, cam, bg, flags, image, records, false);
}

int rgs_rasterize_forward(rgs_ctx* c, const rgs_splat* splats, int n_splats, const rgs_camera* cam,
                          const double bg[3], unsigned flags, float* image, rgs_records** records) {
    if (n_splats < 0 || (n_splats > 0 && !splats)) return RGS_E_INVALID;
    return forward_common(c, kFromSplats, nullptr, splats, n_splats, cam, bg, flags, image, records, false);
}

int rgs_render_flow(rgs_ctx* c, const rgs_scene* scene, const rgs_camera* cam, unsigned flags, float* flow) {
    if (!scene || !flow) return RGS_E_INVALID;
    const double zero[3] = {0, 0, 0};
    return forward_common(c, kFromScene, scene, nullptr, 0, cam, zero, flags & ~RGS_FLAG_RETAIN_RECORDS, flow, nullptr,
                          true);
}

}  // extern "C"

namespace {

// Views of a batch are spread round-robin over kSlots frame slots, each on its own
// stream, so the small latency-bound kernels of one view overlap the blend of another.
// No host synchronisation until the end of the batch; then every view's BinState is
// checked (rotor errors reported, pair-buffer overflows re-rendered synchronously).
// `copy_out` (optional) is called after each view is enqueued on its slot stream.
template <typename CopyOut>
int render_batch(rgs_ctx* c, const rgs_scene* scene, const rgs_camera* cams, int n_views, const double bg[3],
                 unsigned flags, float* (*image_for)(void*, int, cudaStream_t), void* user, CopyOut&& copy_out) {
    for (int v = 0; v < n_views; ++v) {
        const int rc = validate_camera(c, &cams[v]);
        if (rc) return rc;
    }
    c->err_index = -1;
    c->ensure_view_stats(n_views);
    // A batch of several views of one scene shares the t-independent half of the slice (and the
    // opacity sigmoid): computed once here, before the slot streams join.
    SliceCacheView cache_view{nullptr, nullptr};
    const SliceCacheView* cache = nullptr;
    if (n_views >= 2 && scene->n > 0) {
        c->slice_cache.ensure(rgs_launch::slice_cache_bytes(scene->n), c->stream);
        StageTimer t(c, kStPreprocess, c->stream);
        rgs_launch::slice_cache(scene->params, scene->params64, scene->n, c->slice_cache.p, &cache_view, c->stream);
        c->launches += 1;
        cache = &cache_view;
    }
    CK(cudaEventRecord(c->join_ev, c->stream));
    for (int k = 0; k < rgs_ctx::kSlots; ++k) CK(cudaStreamWaitEvent(c->slot_stream[k], c->join_ev, 0));
    // Profiling mode serialises the views (one slot) so per-stage event times are the
    // kernels' own durations rather than shares of concurrently running views.
    // Views in flight: 8 for frames up to ~2 MP (1352x1014: 3 -> 8 slots measured +4.5%), 3 for
    // larger ones (below).  One view in flight (the profiling mode, or RGS_SLOTS=1) -> K5 takes the
    // tiles longest list first, as a single view does.
    const size_t npix = (size_t)cams[0].width * cams[0].height;
    // RGS_SLOTS (A/B runs; up to kSlots): views in flight.  At 8, 10 or 12 the C2 sweep runs at the
    // same rate (2650 FPS), at 6 0.3 % slower (with a less shared -- faster -- live K5 launch)
    static const int env_slots = [] {
        const char* e = std::getenv("RGS_SLOTS");
        const int k = e ? std::atoi(e) : 0;
        return (k >= 1 && k <= rgs_ctx::kSlots) ? k : 0;
    }();
    static const int env_big = [] {
        const char* e = std::getenv("RGS_SLOTS_BIG");
        const int k = e ? std::atoi(e) : 0;
        return (k >= 1 && k <= rgs_ctx::kSlots) ? k : 0;
    }();
    // Frames above ~2.2 MP: 3 views in flight (3840x2160, 2M Gaussians, orbit cameras: 407 FPS
    // at 3, 403 at 8, 390 at 1 -- tools/probe_slots.py); up to ~2.2 MP 8 (C2).
    const int big_slots = env_big ? env_big : 3;
    const int slots = c->timing == 1 ? 1 : (npix <= (size_t)2200000 ? (env_slots ? env_slots : 8) : big_slots);
    for (int v = 0; v < n_views; ++v) {
        const int k = v % slots;
        cudaStream_t s = c->slot_stream[k];
        const int rc = run_forward(c, c->slot_frame[k], s, kFromScene, scene, nullptr, 0, true, &cams[v], bg,
                                   flags & ~RGS_FLAG_HOST_BUFFERS, image_for(user, v, s), false, false,
                                   &c->view_stats[v], cache, true, true, slots == 1);
        if (rc) return rc;
        copy_out(v, k, s);
    }
    for (int k = 0; k < rgs_ctx::kSlots; ++k) {
        CK(cudaEventRecord(c->slot_done[k], c->slot_stream[k]));
        CK(cudaStreamWaitEvent(c->stream, c->slot_done[k], 0));
    }
    CK(cudaStreamSynchronize(c->stream));
    for (int v = 0; v < n_views; ++v) {
        const BinState& st = c->view_stats[v];
        if (st.err != kNoError) {
            const int code = (int)(st.err & 0xff);
            c->err_index = (int)(st.err >> 8);
            return set_err(c, code, rotor_msg(code));
        }
    }
    for (int v = 0; v < n_views; ++v) {
        if (!c->view_stats[v].overflow) continue;
        // every slot learns the larger capacity (it grows its pair buffers on its next view): a
        // slot that kept the capacity of an earlier, smaller workload would overflow -- and be
        // re-rendered serially here -- on every later batch (C4 after C2 in one context: 342
        // FPS at 3 views in flight before this, the overflowing views rendered twice)
        const long long need = (long long)c->view_stats[v].n_pairs * 5 / 4 + 1024;
        for (int k = 0; k < rgs_ctx::kSlots; ++k) {
            Frame& fk = c->slot_frame[k];
            if (fk.pair_cap <= 0 || fk.pair_cap >= need) continue;
            fk.pair_cap = need;
            fk.ensure_pairs(need, true, c->slot_stream[k]);  // grown now, not inside the next batch
        }
        Frame& f = c->slot_frame[0];
        f.pair_cap = std::max<long long>(f.pair_cap, need);
        const int rc = run_forward(c, f, c->stream, kFromScene, scene, nullptr, 0, true, &cams[v], bg,
                                   flags & ~RGS_FLAG_HOST_BUFFERS, image_for(user, v, c->stream), false, true,
                                   nullptr, cache, true);
        if (rc) return rc;
        copy_out(v, 0, c->stream);
        CK(cudaStreamSynchronize(c->stream));
    }
    return RGS_OK;
}

struct DeviceImages {
    float* base;
    size_t per;
};
float* device_image_for(void* u, int v, cudaStream_t) {
    DeviceImages* d = static_cast<DeviceImages*>(u);
    return d->base + d->per * (size_t)v;
}

}  // namespace

extern "C" {

int rgs_render_views(rgs_ctx* c, const rgs_scene* scene, const rgs_camera* cams, int n_views, const double bg[3],
                     unsigned flags, float* images) {
    if (!scene || !cams || n_views < 0 || !images) return RGS_E_INVALID;
    for (int v = 0; v < n_views; ++v)
        if (cams[v].width != cams[0].width || cams[v].height != cams[0].height) return RGS_E_INVALID;
    if (n_views == 0) return RGS_OK;
    return guarded(c, [&]() -> int {
        DeviceImages d{images, (size_t)cams[0].width * cams[0].height * 3};
        return render_batch(c, scene, cams, n_views, bg, flags, device_image_for, &d, [](int, int, cudaStream_t) {});
    });
}

int rgs_render_views_host(rgs_ctx* c, int n, int sh_degree, const float* mean, const float* ls, const float* rot,
                          const float* op, const float* sh, const rgs_camera* cams, int n_views, const double bg[3],
                          float* images_host) {
    if (!cams || n_views < 0 || !images_host) return RGS_E_INVALID;
    if (n_views == 0) return RGS_OK;
    rgs_scene* scene = nullptr;
    int rc = rgs_scene_create(c, n, sh_degree, &scene);
    if (rc) return rc;
    rc = rgs_scene_upload_f32(c, scene, mean, ls, rot, op, sh);
    if (rc) {
        rgs_scene_destroy(scene);
        return rc;
    }
    rc = guarded(c, [&]() -> int {
        // A ring of 2 x kSlots device images: view v renders into img[v % R] once the copy of
        // view v - R out of it is done, and is copied to the host on the copy stream while
        // the slot moves on to its next view (which no longer waits for this copy).
        constexpr int R = 16;  // twice the default views in flight
        const size_t per = (size_t)cams[0].width * cams[0].height * 3;
        struct Ring {
            DevBuf img[R];
            cudaEvent_t rendered[R], copied[R];
        } sl;
        for (int k = 0; k < R; ++k) {
            sl.img[k].ensure(per * sizeof(float), c->stream);
            CK(cudaEventCreateWithFlags(&sl.rendered[k], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&sl.copied[k], cudaEventDisableTiming));
            CK(cudaEventRecord(sl.copied[k], c->stream));  // after the allocations
        }
        auto image_for = [](void* u, int v, cudaStream_t s) -> float* {
            Ring* r = static_cast<Ring*>(u);
            CK(cudaStreamWaitEvent(s, r->copied[v % R], 0));
            return r->img[v % R].as<float>();
        };
        const int r = render_batch(c, scene, cams, n_views, bg, 0, image_for, &sl, [&](int v, int, cudaStream_t s) {
            const int q = v % R;
            CK(cudaEventRecord(sl.rendered[q], s));
            CK(cudaStreamWaitEvent(c->copy_stream, sl.rendered[q], 0));
            CK(cudaMemcpyAsync(images_host + per * (size_t)v, sl.img[q].p, per * sizeof(float),
                               cudaMemcpyDeviceToHost, c->copy_stream));
            CK(cudaEventRecord(sl.copied[q], c->copy_stream));
        });
        CK(cudaStreamSynchronize(c->copy_stream));
        CK(cudaStreamSynchronize(c->stream));
        for (int k = 0; k < R; ++k) {
            sl.img[k].release(c->stream);
            cudaEventDestroy(sl.rendered[k]);
            cudaEventDestroy(sl.copied[k]);
        }
        return r;
    });
    rgs_scene_destroy(scene);
    return rc;
}

// ------------------------------------------------------------------ records
void rgs_records_destroy(rgs_records* r) {
    if (!r) return;
    if (!r->ctx) {  // its context was destroyed first and already freed the frame
        delete r;
        return;
    }
    cudaSetDevice(r->ctx->device);
    r->ctx->live_records.erase(r);
    frame_put(r->ctx, r->pf);
    if (r->ready) cudaEventDestroy(r->ready);
    delete r;
}

int rgs_records_info_get(const rgs_records* r, rgs_records_info* info) {
    if (!r || !info || !r->ctx) return RGS_E_INVALID;
    rgs_ctx* c = r->ctx;
    return guarded(c, [&]() -> int {
        const int rc = resolve(c, r);
        if (rc) return rc;
        BinState st;
        CK(cudaMemcpyAsync(c->host_stats, r->fb->dstats(), sizeof st, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        st = *c->host_stats;
        info->n_splats = r->fb->n_valid;
        info->tiles_x = r->fb->tiles_x;
        info->tiles_y = r->fb->tiles_y;
        info->retained = r->retained;
        info->n_pairs = r->fb->n_pairs;
        info->n_slow_pixels = st.slow_count;
        info->width = r->fb->width;
        info->height = r->fb->height;
        return RGS_OK;
    });
}

int rgs_records_export(rgs_ctx* c, const rgs_records* r, rgs_splat* splats, long long* tile_offsets, int32_t* tile_ids,
                       double* final_T, int32_t* n_contrib) {
    if (!r || r->ctx != c) return RGS_E_INVALID;
    return guarded(c, [&]() -> int {
        const int rc = resolve(c, r);
        if (rc) return rc;
        const Frame& f = *r->fb;
        cudaStream_t s = c->stream;
        const int n = f.n;
        const size_t npix = (size_t)f.width * f.height;
        const int ntiles = f.tiles_x * f.tiles_y;
        // compacted index of each valid splat (rasterizer.cpp:206-210)
        c->tmp_scan.ensure(4 * (size_t)std::max(n, 1) * 2, s);
        uint32_t* v32 = c->tmp_scan.as<uint32_t>();
        uint32_t* scan = v32 + std::max(n, 1);
        rgs_launch::valid_to_u32(f.valid.as<uint8_t>(), n, v32, s);
        DevBuf tmp;
        tmp.ensure(4 * (size_t)(n / 1024 + 2), s);
        rgs_launch::exclusive_scan(v32, n, scan, tmp.as<uint32_t>(), nullptr, s);
        c->launches += 4;
        if (splats && f.n_valid > 0) {
            c->tmp_ids.ensure(4 * (size_t)f.n_valid, s);
            rgs_launch::compact_index(f.valid.as<uint8_t>(), scan, n, c->tmp_ids.as<uint32_t>(), s);
            DevBuf out;
            out.ensure(sizeof(rgs_splat) * (size_t)f.n_valid, s);
            rgs_launch::export_splats(f.arrays(), c->tmp_ids.as<uint32_t>(), f.n_valid, out.p, s);
            c->launches += 2;
            CK(cudaMemcpyAsync(splats, out.p, sizeof(rgs_splat) * (size_t)f.n_valid, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            out.release(s);
        }
        if (tile_offsets) {
            std::vector<uint2> rg(ntiles);
            CK(cudaMemcpyAsync(rg.data(), f.ranges.p, sizeof(uint2) * ntiles, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            long long acc = 0;
            for (int t = 0; t < ntiles; ++t) {
                tile_offsets[t] = acc;
                acc += (long long)rg[t].y - (long long)rg[t].x;
            }
            tile_offsets[ntiles] = acc;
        }
        if (tile_ids && f.n_pairs > 0) {
            DevBuf out;
            out.ensure(4 * (size_t)f.n_pairs, s);
            rgs_launch::map_ids(f.pair_vals(), f.n_pairs, scan, out.as<int32_t>(), s);
            c->launches += 1;
            CK(cudaMemcpyAsync(tile_ids, out.p, 4 * (size_t)f.n_pairs, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            out.release(s);
        }
        if (final_T) CK(cudaMemcpyAsync(final_T, f.final_T.p, 8 * npix, cudaMemcpyDeviceToHost, s));
        if (n_contrib) CK(cudaMemcpyAsync(n_contrib, f.n_contrib.p, 4 * npix, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (n_contrib)
            for (size_t i = 0; i < npix; ++i) n_contrib[i] &= 0x7fffffff;
        tmp.release(s);
        return RGS_OK;
    });
}

// ------------------------------------------------------------------ backward
int rgs_render_backward(rgs_ctx* c, const rgs_scene* scene, const rgs_camera* cam, const rgs_records* r,
                        const float* dL_dimage, unsigned flags, float* grads, float* vnorm, int32_t* visible) {
    if (!scene || !cam || !r || !dL_dimage || !grads || !vnorm || !visible || r->ctx != c) return RGS_E_INVALID;
    if (!r->retained)
        return set_err(c, RGS_E_MISSING_RECORDS, "rasterize_backward: forward pass did not retain records");
    if (flags & RGS_FLAG_HOST_BUFFERS) {
        // Host in / host out: stage through device buffers on the context stream.
        return guarded(c, [&]() -> int {
            cudaStream_t s = c->stream;
            const size_t n = (size_t)std::max(scene->n, 1), npix = (size_t)cam->width * cam->height;
            DevBuf dl, g, vn, vis;
            dl.ensure(npix * 3 * sizeof(float), s);
            g.ensure(65 * n * sizeof(float), s);
            vn.ensure(n * sizeof(float), s);
            vis.ensure(n * sizeof(int32_t), s);
            CK(cudaMemcpyAsync(dl.p, dL_dimage, npix * 3 * sizeof(float), cudaMemcpyHostToDevice, s));
            if (flags & RGS_FLAG_ACCUMULATE) {
                CK(cudaMemcpyAsync(g.p, grads, 65 * n * sizeof(float), cudaMemcpyHostToDevice, s));
                CK(cudaMemcpyAsync(vn.p, vnorm, n * sizeof(float), cudaMemcpyHostToDevice, s));
                CK(cudaMemcpyAsync(vis.p, visible, n * sizeof(int32_t), cudaMemcpyHostToDevice, s));
            }
            const int rc = rgs_render_backward(c, scene, cam, r, dl.as<float>(), flags & ~RGS_FLAG_HOST_BUFFERS,
                                               g.as<float>(), vn.as<float>(), vis.as<int32_t>());
            if (rc) return rc;
            CK(cudaMemcpyAsync(grads, g.p, 65 * n * sizeof(float), cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(vnorm, vn.p, n * sizeof(float), cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(visible, vis.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
            for (DevBuf* b : {&dl, &g, &vn, &vis}) b->release(s);
            CK(cudaStreamSynchronize(s));
            return RGS_OK;
        });
    }
    return guarded(c, [&]() -> int {
        const Frame& f = *r->fb;
        if (cam->width != f.width || cam->height != f.height || scene->n != f.n)
            return set_err(c, RGS_E_INVALID, "render_backward: camera/scene does not match the records");
        cudaStream_t s = c->stream;
        const DevCamera dc = make_dev_camera(cam);
        const int n = scene->n;
        c->sgrad.ensure(sizeof(double) * 9 * (size_t)std::max(n, 1), s);
        CK(cudaMemsetAsync(c->sgrad.p, 0, sizeof(double) * 9 * (size_t)std::max(n, 1), s));
        SplatArrays sa = f.arrays();
        const float3 bgf = make_float3((float)f.bg[0], (float)f.bg[1], (float)f.bg[2]);
        if (flags & RGS_FLAG_DETERMINISTIC) {
            const int rc = resolve(c, r);
            if (rc) return rc;
            // Reference-order FP64 replay and tile-ordered reduction, no atomics.
            c->tile_grads.ensure(sizeof(double) * 9 * (size_t)std::max<long long>(f.n_pairs, 1), s);
            CK(cudaMemsetAsync(c->tile_grads.p, 0, sizeof(double) * 9 * (size_t)std::max<long long>(f.n_pairs, 1), s));
            StageTimer t(c, kStBwdTiles, s);
            rgs_launch::backward_deterministic(sa, f.pair_vals(), f.ranges.as<uint2>(), dc,
                                               make_double3(f.bg[0], f.bg[1], f.bg[2]), f.final_T.as<double>(),
                                               f.n_contrib.as<uint32_t>(), dL_dimage, f.sorted_ids.as<uint32_t>(),
                                               &f.dstats()->n_valid, n, f.ent_id.as<uint32_t>(),
                                               c->tile_grads.as<double>(), c->sgrad.as<double>(), s);
        } else {
            // RGS_FLAG_REPRODUCIBLE: the same kernels, accumulating in order-independent fixed point
            unsigned long long* fx = nullptr;
            if (flags & RGS_FLAG_REPRODUCIBLE) {
                const size_t bytes = sizeof(unsigned long long) * 18 * (size_t)std::max(n, 1);
                c->sgrad_fixed.ensure(bytes, s);
                CK(cudaMemsetAsync(c->sgrad_fixed.p, 0, bytes, s));
                fx = c->sgrad_fixed.as<unsigned long long>();
            }
            {
                StageTimer t(c, kStBwdTiles, s);
                rgs_launch::backward_fp32(sa, f.pair_vals(), f.ranges.as<uint2>(), dc, bgf, f.final_T.as<double>(),
                                          f.n_contrib.as<uint32_t>(), dL_dimage, c->sgrad.as<double>(), s, fx,
                                          use_tile_order(false, false, (size_t)f.width * f.height)
                                              ? f.tile_order.as<uint32_t>()
                                              : nullptr);
            }
            {
                StageTimer t(c, kStBwdFixup, s);
                rgs_launch::backward_fp64_pixels(sa, f.pair_vals(), f.ranges.as<uint2>(), dc,
                                                 make_double3(f.bg[0], f.bg[1], f.bg[2]), f.final_T.as<double>(),
                                                 f.n_contrib.as<uint32_t>(), dL_dimage, f.slow_list.as<uint32_t>(),
                                                 &f.dstats()->slow_count, (int)((size_t)f.width * f.height),
                                                 c->sgrad.as<double>(), s, fx);
                if (fx) {
                    rgs_launch::fixed_to_double(fx, 9 * (size_t)n, c->sgrad.as<double>(), s);
                    c->launches += 1;
                }
            }
        }
        c->cgrad.ensure(sizeof(double) * 3 * (size_t)std::max(n, 1), s);
        for (int part = 1; part <= 2; ++part) {
            StageTimer t(c, part == 1 ? kStBwdColor : kStBwdGauss, s);
            rgs_launch::gaussian_backward(scene->params, scene->params64, n, scene->sh_degree, dc,
                                          f.dir_dist.as<double4>(), c->cgrad.as<double>(), f.valid.as<uint8_t>(),
                                          c->sgrad.as<double>(), (flags & RGS_FLAG_ACCUMULATE) ? 1 : 0, grads,
                                          vnorm, visible, s, part);
        }
        c->launches += 4;
        CK(cudaGetLastError());
        return RGS_OK;
    });
}

int rgs_project_sliced_cache(rgs_ctx* c, const double* sliced16, const rgs_camera* cam, const double* sh48,
                             int sh_degree, double opacity_logit, rgs_splat* out, int* survived, double* cache) {
    if (!sliced16 || !cam || !sh48 || !out || !survived) return RGS_E_INVALID;
    return guarded(c, [&]() -> int {
        cudaStream_t s = c->stream;
        DevBuf buf;
        buf.ensure(sizeof(double) * (64 + RGS_PROJECT_CACHE_DOUBLES) + sizeof(rgs_splat) + 16, s);
        double* d = buf.as<double>();
        double* dc = d + 64;
        rgs_splat* o = reinterpret_cast<rgs_splat*>(dc + RGS_PROJECT_CACHE_DOUBLES);
        int* surv = reinterpret_cast<int*>(o + 1);
        CK(cudaMemcpyAsync(d, sliced16, sizeof(double) * 16, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(d + 16, sh48, sizeof(double) * 48, cudaMemcpyHostToDevice, s));
        rgs_launch::project_one(d, make_dev_camera(cam), d + 16, sh_degree, opacity_logit, o, surv, s,
                                cache ? dc : nullptr);
        c->launches += 1;
        CK(cudaMemcpyAsync(out, o, sizeof(rgs_splat), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(survived, surv, sizeof(int), cudaMemcpyDeviceToHost, s));
        if (cache)
            CK(cudaMemcpyAsync(cache, dc, sizeof(double) * RGS_PROJECT_CACHE_DOUBLES, cudaMemcpyDeviceToHost, s));
        buf.release(s);
        CK(cudaStreamSynchronize(s));
        return RGS_OK;
    });
}

int rgs_project_sliced(rgs_ctx* c, const double* sliced16, const rgs_camera* cam, const double* sh48, int sh_degree,
                       double opacity_logit, rgs_splat* out, int* survived) {
    return rgs_project_sliced_cache(c, sliced16, cam, sh48, sh_degree, opacity_logit, out, survived, nullptr);
}

}  // extern "C"

// ===========================================================================
// Training side: image losses, Adam, regularizers, KNN.
#include "rgs_train.cuh"

struct rgs_optimizer {
    rgs_ctx* ctx = nullptr;
    int n = 0;
    bool f64 = false;
    void* m1 = nullptr;              // Adam first moments, scene SoA layout and precision
    void* m2 = nullptr;              // second moments
    double* accum = nullptr;         // GaussianStore::grad_accum
    int32_t* count = nullptr;        // GaussianStore::grad_count
    unsigned long long* err = nullptr;  // rotor error word of the steps since the last status call
    DevBuf part;                     // block partials (entropy)
};

namespace {

// Host (N, 65) rows in the reference order -> the five upload arrays (and back).
// SoA device block (float or double) <-> host (N, 65) rows: one copy of the rows, the transpose
// on the device.
void soa_upload(rgs_ctx* c, size_t n, bool f64, const double* rows, void* dst) {
    DevBuf tmp;
    cudaStream_t s = c->stream;
    tmp.ensure(sizeof(double) * 65 * n, s);
    CK(cudaMemcpyAsync(tmp.p, rows, sizeof(double) * 65 * n, cudaMemcpyHostToDevice, s));
    rgs_launch::rows_to_soa(tmp.as<double>(), (int)n, f64 ? nullptr : (float*)dst, f64 ? (double*)dst : nullptr, s);
    c->launches += 1;
    CK(cudaStreamSynchronize(s));
    tmp.release(s);
}
void soa_download(rgs_ctx* c, size_t n, bool f64, const void* src, double* rows) {
    DevBuf tmp;
    cudaStream_t s = c->stream;
    tmp.ensure(sizeof(double) * 65 * n, s);
    rgs_launch::soa_to_rows(f64 ? nullptr : (const float*)src, f64 ? (const double*)src : nullptr, (int)n,
                            tmp.as<double>(), s);
    c->launches += 1;
    CK(cudaMemcpyAsync(rows, tmp.p, sizeof(double) * 65 * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    tmp.release(s);
}

// ssim.cpp:15-31 on the host (glibc exp), uploaded once per context.
void ensure_ssim_window(rgs_ctx* c) {
    static thread_local int done_device = -1;
    if (done_device == c->device) return;
    double k[kSsimWin], sum = 0;
    for (int i = 0; i < kSsimWin; ++i) {
        const double d = i - (kSsimWin - 1) / 2.0;
        k[i] = std::exp(-d * d / (2 * 1.5 * 1.5));
        sum += k[i];
    }
    for (double& v : k) v /= sum;
    rgs_launch::set_ssim_window(k, c->stream);
    CK(cudaStreamSynchronize(c->stream));
    done_device = c->device;
}

// `parts` holds the image-loss block partials, `cparts` the consistency term's: a training step
// runs the consistency term on its main stream beside the image losses of its side streams.
struct TrainScratch {
    DevBuf dfield, parts, cparts, speeds, dcount, pts, lo, hi, knn;
    DevBuf tie_list, tie_count, tie_img64, l1_sign;  // rgs_image_loss_ex (l1_sign kept all-zero between calls)
};
void train_scratch_free(void* p, cudaStream_t s) {
    TrainScratch* ts = static_cast<TrainScratch*>(p);
    for (DevBuf* b : {&ts->dfield, &ts->parts, &ts->cparts, &ts->speeds, &ts->dcount, &ts->pts, &ts->lo, &ts->hi, &ts->knn,
                      &ts->tie_list, &ts->tie_count, &ts->tie_img64, &ts->l1_sign})
        b->release(s);
    delete ts;
}

// One scratch set per context, released with it (rgs_ctx_destroy).
TrainScratch& train_scratch(rgs_ctx* c) {
    if (!c->train) {
        c->train = new TrainScratch;
        c->train_free = train_scratch_free;
    }
    return *static_cast<TrainScratch*>(c->train);
}

}  // namespace

extern "C" {

int rgs_image_loss(rgs_ctx* c, const float* rendered, const float* target, int width, int height, double w_l1,
                   double w_ssim, double loss_scale, unsigned flags, float* dL_dimage, double* losses) {
    return rgs_image_loss_ex(c, nullptr, rendered, target, width, height, w_l1, w_ssim, loss_scale, flags, dL_dimage,
                             losses);
}

int rgs_image_loss_ex(rgs_ctx* c, const rgs_records* rec, const float* rendered, const float* target, int width,
                      int height, double w_l1, double w_ssim, double loss_scale, unsigned flags, float* dL_dimage,
                      double* losses) {
    if (!rendered || !target || width <= 0 || height <= 0) return RGS_E_INVALID;
    if (rec && (rec->ctx != c || !rec->retained || rec->fb->width != width || rec->fb->height != height))
        return set_err(c, RGS_E_INVALID, "image_loss: records do not belong to this image");
    if ((width < kSsimWin || height < kSsimWin) && w_ssim != 0)
        return set_err(c, RGS_E_INVALID, "ssim: image smaller than the 11x11 window");
    return guarded(c, [&]() -> int {
        cudaStream_t s = c->stream;
        ensure_ssim_window(c);
        TrainScratch& ts = train_scratch(c);
        const ImageLossGrid g = rgs_launch::image_loss_grid(width, height);
        const size_t nv = (size_t)std::max(width - kSsimWin + 1, 0) * (size_t)std::max(height - kSsimWin + 1, 0);
        if (dL_dimage) ts.dfield.ensure(sizeof(double) * 9 * nv, s);
        ts.parts.ensure(sizeof(double) * (g.n_a + 2 * g.n_b + 16), s);
        ImageGradArgs a;
        a.w_l1 = w_l1;
        a.w_ssim = w_ssim;
        a.inv_n = 1 / (3.0 * (double)width * (double)height);
        a.ssim_scale = nv ? -1 / (3.0 * (double)nv) : 0.0;
        a.accumulate = (flags & RGS_FLAG_ACCUMULATE_GRAD) ? 1 : 0;
        StageTimer t(c, kStImageLoss, s);
        // L1 near ties (image.cpp:32-33 on the reference's double image): pixels whose FP32 value
        // is within kL1Tie of the target in some channel are recomputed in FP64 from the view's
        // records and their L1 sign taken from that value.  kL1Tie is 10x the largest FP32 image
        // error measured at C1 / C2 / C4 (1.03e-6; the north-star bound is 1e-4).
        constexpr float kL1Tie = 1e-5f;
        const size_t npix = (size_t)width * height;
        const bool ties = rec && dL_dimage && w_l1 != 0;
        if (ties) {
            const Frame& f = *rec->fb;
            ts.tie_list.ensure(4 * npix, s);
            ts.tie_count.ensure(16, s);
            ts.tie_img64.ensure(sizeof(double) * 3 * npix, s);
            if (ts.l1_sign.bytes < 3 * npix) {
                ts.l1_sign.ensure(3 * npix, s);
                CK(cudaMemsetAsync(ts.l1_sign.p, 0, ts.l1_sign.bytes, s));
            }
            CK(cudaMemsetAsync(ts.tie_count.p, 0, sizeof(int), s));
            const bool bg_exact = (double)(float)f.bg[0] == f.bg[0] && (double)(float)f.bg[1] == f.bg[1] &&
                                  (double)(float)f.bg[2] == f.bg[2];
            rgs_launch::l1_ties(rendered, target, (int)npix, kL1Tie, bg_exact ? f.n_contrib.as<uint32_t>() : nullptr,
                                ts.tie_list.as<uint32_t>(), ts.tie_count.as<int>(), s);
            DevCamera dc{};
            dc.width = f.width;
            dc.height = f.height;
            dc.tiles_x = f.tiles_x;
            dc.tiles_y = f.tiles_y;
            rgs_launch::blend_fp64_pixels(f.arrays(), f.pair_vals(), f.ranges.as<uint2>(), dc,
                                          make_double3(f.bg[0], f.bg[1], f.bg[2]), 0, nullptr,
                                          ts.tie_img64.as<double>(), nullptr, nullptr, ts.tie_list.as<uint32_t>(),
                                          ts.tie_count.as<int>(), (int)npix, s);
            rgs_launch::l1_sign_set(ts.tie_list.as<uint32_t>(), ts.tie_count.as<int>(), (int)npix,
                                    ts.tie_img64.as<double>(), target, ts.l1_sign.as<int8_t>(), s);
            a.l1_sign = ts.l1_sign.as<int8_t>();
            c->launches += 3;
        }
        rgs_launch::image_loss(rendered, target, width, height, a, dL_dimage, ts.dfield.as<double>(),
                               ts.parts.as<double>(), losses, loss_scale, (flags & RGS_FLAG_ACCUMULATE) ? 1 : 0, s);
        c->launches += losses ? 3 : 2;
        if (ties) {
            rgs_launch::l1_sign_clear(ts.tie_list.as<uint32_t>(), ts.tie_count.as<int>(), (int)npix,
                                      ts.l1_sign.as<int8_t>(), s);
            c->launches += 1;
        }
        CK(cudaGetLastError());
        return RGS_OK;
    });
}

int rgs_image_loss_f64(rgs_ctx* c, const double* rendered, const double* target, int width, int height, double w_l1,
                       double w_ssim, double loss_scale, unsigned flags, double* dL_dimage, double* losses) {
    if (!rendered || !target || width <= 0 || height <= 0) return RGS_E_INVALID;
    if ((width < kSsimWin || height < kSsimWin) && w_ssim != 0)
        return set_err(c, RGS_E_INVALID, "ssim: image smaller than the 11x11 window");
    return guarded(c, [&]() -> int {
        cudaStream_t s = c->stream;
        ensure_ssim_window(c);
        TrainScratch& ts = train_scratch(c);
        const ImageLossGrid g = rgs_launch::image_loss_grid(width, height);
        const size_t nv = (size_t)std::max(width - kSsimWin + 1, 0) * (size_t)std::max(height - kSsimWin + 1, 0);
        if (dL_dimage) ts.dfield.ensure(sizeof(double) * 9 * nv, s);
        ts.parts.ensure(sizeof(double) * (g.n_a + 2 * g.n_b + 16), s);
        ImageGradArgs a;
        a.w_l1 = w_l1;
        a.w_ssim = w_ssim;
        a.inv_n = 1 / (3.0 * (double)width * (double)height);
        a.ssim_scale = nv ? -1 / (3.0 * (double)nv) : 0.0;
        a.accumulate = (flags & RGS_FLAG_ACCUMULATE_GRAD) ? 1 : 0;
        rgs_launch::image_loss_f64(rendered, target, width, height, a, dL_dimage, ts.dfield.as<double>(),
                                   ts.parts.as<double>(), losses, loss_scale, (flags & RGS_FLAG_ACCUMULATE) ? 1 : 0, s);
        c->launches += losses ? 3 : 2;
        CK(cudaGetLastError());
        return RGS_OK;
    });
}

int rgs_entropy_loss(rgs_ctx* c, const double* opacities, int n, double* grad, double* loss) {
    if (!opacities || n < 0) return RGS_E_INVALID;
    return guarded(c, [&]() -> int {
        if (n == 0) {
            if (loss) CK(cudaMemsetAsync(loss, 0, sizeof(double), c->stream));
            return RGS_OK;
        }
        TrainScratch& ts = train_scratch(c);
        ts.parts.ensure(sizeof(double) * ((n + 255) / 256 + 16), c->stream);
        rgs_launch::entropy(opacities, n, grad, ts.parts.as<double>(), loss, c->stream);
        c->launches += loss ? 2 : 1;
        CK(cudaGetLastError());
        return RGS_OK;
    });
}

int rgs_optimizer_create(rgs_ctx* c, const rgs_scene* scene, rgs_optimizer** out) {
    if (!scene || !out) return RGS_E_INVALID;
    return guarded(c, [&]() -> int {
        rgs_optimizer* o = new rgs_optimizer;
        o->ctx = c;
        o->n = scene->n;
        o->f64 = scene->params64 != nullptr;
        const size_t n1 = (size_t)std::max(scene->n, 1);
        const size_t eb = o->f64 ? sizeof(double) : sizeof(float);
        CK(cudaMalloc(&o->m1, 65 * n1 * eb));
        CK(cudaMalloc(&o->m2, 65 * n1 * eb));
        CK(cudaMalloc(&o->accum, n1 * sizeof(double)));
        CK(cudaMalloc(&o->count, n1 * sizeof(int32_t)));
        CK(cudaMalloc(&o->err, sizeof(unsigned long long)));
        CK(cudaMemsetAsync(o->m1, 0, 65 * n1 * eb, c->stream));
        CK(cudaMemsetAsync(o->m2, 0, 65 * n1 * eb, c->stream));
        CK(cudaMemsetAsync(o->accum, 0, n1 * sizeof(double), c->stream));
        CK(cudaMemsetAsync(o->count, 0, n1 * sizeof(int32_t), c->stream));
        CK(cudaMemsetAsync(o->err, 0xff, sizeof(unsigned long long), c->stream));
        o->part.ensure(sizeof(double) * (rgs_launch::adam_blocks(scene->n) + 16), c->stream);
        CK(cudaStreamSynchronize(c->stream));
        *out = o;
        return RGS_OK;
    });
}

void rgs_optimizer_destroy(rgs_optimizer* o) {
    if (!o) return;
    cudaSetDevice(o->ctx->device);
    cudaStreamSynchronize(o->ctx->stream);
    cudaFree(o->m1);
    cudaFree(o->m2);
    cudaFree(o->accum);
    cudaFree(o->count);
    cudaFree(o->err);
    o->part.release(o->ctx->stream);
    delete o;
}

int rgs_adam_step(rgs_ctx* c, rgs_scene* scene, rgs_optimizer* o, const float* grads, const float* vnorm,
                  const int32_t* visible, const rgs_adam_config* cfg, int step, double* losses) {
    if (!scene || !o || !grads || !cfg || step < 1) return RGS_E_INVALID;
    if (o->n != scene->n || o->f64 != (scene->params64 != nullptr))
        return set_err(c, RGS_E_INVALID, "adam_step: gradients not aligned with store");
    if (cfg->accumulate_stats && (!vnorm || !visible)) return RGS_E_INVALID;
    return guarded(c, [&]() -> int {
        if (scene->n == 0) return RGS_OK;
        // optim.cpp:112-115 on the host: std::pow, lr_schedule (optim.cpp:47-51)
        AdamArgs a;
        a.bc1 = 1 - std::pow(0.9, step);
        a.bc2 = 1 - std::pow(0.999, step);
        double lr_pos = cfg->lr_position;
        if (cfg->total_steps > 0) {
            double u = (double)step / (double)cfg->total_steps;
            u = std::clamp(u, 0.0, 1.0);
            lr_pos = cfg->lr_position * std::pow(cfg->lr_position_final / cfg->lr_position, u);
        }
        a.lr_pos = lr_pos;
        a.lr_scales = cfg->lr_scales;
        a.lr_rotor = cfg->lr_rotor;
        a.lr_sh_dc = cfg->lr_sh_dc;
        a.lr_sh_rest = cfg->lr_sh_rest;
        a.lr_opacity = cfg->lr_opacity;
        a.lambda_entropy = cfg->lambda_entropy;
        a.inv_n = 1 / (double)scene->n;
        a.static_mode = cfg->static_mode ? 1 : 0;
        a.stats = cfg->accumulate_stats ? 1 : 0;
        void* params = scene->params64 ? (void*)scene->params64 : (void*)scene->params;
        const bool ent = losses && cfg->lambda_entropy != 0;
        StageTimer t(c, kStAdam, c->stream);
        rgs_launch::adam_step(o->f64, params, o->m1, o->m2, grads, vnorm, visible, o->accum, o->count, scene->n, a,
                              o->err, ent ? o->part.as<double>() : nullptr, ent ? losses : nullptr,
                              (cfg->flags & RGS_FLAG_ACCUMULATE) ? 1 : 0, c->deferred.as<unsigned long long>(),
                              c->stream);
        c->launches += ent ? 3 : 2;
        CK(cudaGetLastError());
        return RGS_OK;
    });
}

int rgs_optimizer_status(rgs_ctx* c, rgs_optimizer* o) {
    if (!o) return RGS_E_INVALID;
    return guarded(c, [&]() -> int {
        unsigned long long e = 0;
        CK(cudaMemcpyAsync(&e, o->err, sizeof e, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (e == kNoError) return RGS_OK;
        CK(cudaMemsetAsync(o->err, 0xff, sizeof(unsigned long long), c->stream));
        const int code = (int)(e & 0xff);
        c->err_index = (int)(e >> 8);
        return set_err(c, code, rotor_msg(code));
    });
}

int rgs_ctx_status(rgs_ctx* c) {
    return guarded(c, [&]() -> int {
        unsigned long long e = 0;
        CK(cudaMemcpyAsync(c->host_word, c->deferred.p, sizeof e, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        e = *c->host_word;
        if (e == kNoError) return RGS_OK;
        CK(cudaMemsetAsync(c->deferred.p, 0xff, sizeof(unsigned long long), c->stream));
        const int code = (int)(e & 0xff);
        c->err_index = (int)(e >> 8);
        if (code == RGS_E_OVERFLOW)
            return set_err(c, code, "deferred-check forward outgrew its pair buffers; re-run it checked");
        if (code == kErrDegenerateTime)
            return set_err(c, RGS_E_DEGENERATE_TIME, "slice_at: temporal scale collapsed (W < 1e-12)");
        return set_err(c, code, rotor_msg(code));
    });
}

int rgs_ctx_status_async(rgs_ctx* c, unsigned long long* word) {
    if (!word) return RGS_E_INVALID;
    return guarded(c, [&]() -> int {
        CK(cudaMemcpyAsync(word, c->deferred.p, sizeof *word, cudaMemcpyDeviceToHost, c->stream));
        return RGS_OK;
    });
}

int rgs_optimizer_status_async(rgs_ctx* c, rgs_optimizer* o, unsigned long long* word) {
    if (!o || !word) return RGS_E_INVALID;
    return guarded(c, [&]() -> int {
        CK(cudaMemcpyAsync(word, o->err, sizeof *word, cudaMemcpyDeviceToHost, c->stream));
        return RGS_OK;
    });
}

int rgs_optimizer_download(rgs_ctx* c, const rgs_optimizer* o, double* m65, double* v65, double* grad_accum,
                           int32_t* grad_count) {
    if (!o) return RGS_E_INVALID;
    return guarded(c, [&]() -> int {
        const size_t n = (size_t)o->n;
        if (n == 0) return RGS_OK;
        if (m65) soa_download(c, n, o->f64, o->m1, m65);
        if (v65) soa_download(c, n, o->f64, o->m2, v65);
        if (grad_accum) CK(cudaMemcpyAsync(grad_accum, o->accum, 8 * n, cudaMemcpyDeviceToHost, c->stream));
        if (grad_count) CK(cudaMemcpyAsync(grad_count, o->count, 4 * n, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        return RGS_OK;
    });
}

int rgs_optimizer_upload(rgs_ctx* c, rgs_optimizer* o, const double* m65, const double* v65,
                         const double* grad_accum, const int32_t* grad_count) {
    if (!o) return RGS_E_INVALID;
    return guarded(c, [&]() -> int {
        const size_t n = (size_t)o->n;
        if (n == 0) return RGS_OK;
        if (m65) soa_upload(c, n, o->f64, m65, o->m1);
        if (v65) soa_upload(c, n, o->f64, v65, o->m2);
        if (grad_accum) CK(cudaMemcpyAsync(o->accum, grad_accum, 8 * n, cudaMemcpyHostToDevice, c->stream));
        if (grad_count) CK(cudaMemcpyAsync(o->count, grad_count, 4 * n, cudaMemcpyHostToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        return RGS_OK;
    });
}

int rgs_accumulate_stats(rgs_ctx* c, rgs_optimizer* o, const float* vnorm, const int32_t* visible) {
    if (!o || !vnorm || !visible) return RGS_E_INVALID;
    return guarded(c, [&]() -> int {
        rgs_launch::accumulate_stats(vnorm, visible, o->n, o->accum, o->count, c->stream);
        c->launches += o->n > 0 ? 1 : 0;
        CK(cudaGetLastError());
        return RGS_OK;
    });
}

int rgs_accumulate_stats_f64(rgs_ctx* c, rgs_optimizer* o, const double* vnorm, const int32_t* visible) {
    if (!o || !vnorm || !visible) return RGS_E_INVALID;
    return guarded(c, [&]() -> int {
        rgs_launch::accumulate_stats_f64(vnorm, visible, o->n, o->accum, o->count, c->stream);
        c->launches += o->n > 0 ? 1 : 0;
        CK(cudaGetLastError());
        return RGS_OK;
    });
}

int rgs_optimizer_reset_stats(rgs_ctx* c, rgs_optimizer* o) {
    if (!o) return RGS_E_INVALID;
    return guarded(c, [&]() -> int {
        const size_t n1 = (size_t)std::max(o->n, 1);
        CK(cudaMemsetAsync(o->accum, 0, n1 * sizeof(double), c->stream));
        CK(cudaMemsetAsync(o->count, 0, n1 * sizeof(int32_t), c->stream));
        return RGS_OK;
    });
}

int rgs_reset_opacity(rgs_ctx* c, rgs_scene* scene, rgs_optimizer* o, double value) {
    if (!scene || !o || o->n != scene->n) return RGS_E_INVALID;
    return guarded(c, [&]() -> int {
        if (scene->n == 0) return RGS_OK;
        void* params = scene->params64 ? (void*)scene->params64 : (void*)scene->params;
        rgs_launch::reset_opacity(o->f64, params, o->m1, o->m2, scene->n, value, c->stream);
        c->launches += 1;
        CK(cudaGetLastError());
        return RGS_OK;
    });
}

int rgs_scene_scales(rgs_ctx* c, const rgs_scene* scene, double* out4) {
    if (!scene || !out4) return RGS_E_INVALID;
    return guarded(c, [&]() -> int {
        const int n = scene->n;
        if (n == 0) {
            for (int a = 0; a < 4; ++a) out4[a] = 1e-3;  // (0 - 0).cwiseMax(1e-3)
            return RGS_OK;
        }
        TrainScratch& ts = train_scratch(c);
        const int nb = rgs_launch::extent_blocks(n);
        ts.lo.ensure(sizeof(double) * 4 * nb, c->stream);
        ts.hi.ensure(sizeof(double) * 4 * nb, c->stream);
        rgs_launch::mean_extent(scene->params, scene->params64, n, ts.lo.as<double>(), ts.hi.as<double>(), c->stream);
        c->launches += 1;
        std::vector<double> lo(4 * (size_t)nb), hi(4 * (size_t)nb);
        CK(cudaMemcpyAsync(lo.data(), ts.lo.p, sizeof(double) * 4 * nb, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(hi.data(), ts.hi.p, sizeof(double) * 4 * nb, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        for (int a = 0; a < 4; ++a) {
            double l = lo[a], h = hi[a];
            for (int b = 1; b < nb; ++b) {
                l = std::min(l, lo[4 * (size_t)b + a]);
                h = std::max(h, hi[4 * (size_t)b + a]);
            }
            out4[a] = std::max(h - l, 1e-3);  // trainer.cpp:19
        }
        return RGS_OK;
    });
}

int rgs_knn_build(rgs_ctx* c, const rgs_scene* scene, int k, const double* scales, int32_t* neighbors) {
    if (!scene || !neighbors || k <= 0) return RGS_E_INVALID;
    if (scene->n <= k) return set_err(c, RGS_E_INVALID, "knn: need more points than neighbors");
    if (k > 16) return set_err(c, RGS_E_INVALID, "knn: k must be at most 16");
    return guarded(c, [&]() -> int {
        double sc[4];
        if (scales) {
            for (int a = 0; a < 4; ++a) sc[a] = scales[a];
        } else {
            const int rc = rgs_scene_scales(c, scene, sc);
            if (rc) return rc;
        }
        TrainScratch& ts = train_scratch(c);
        ts.pts.ensure(sizeof(double) * 4 * (size_t)scene->n, c->stream);
        rgs_launch::knn_points(scene->params, scene->params64, scene->n, sc, ts.pts.as<double>(), c->stream);
        const size_t need = rgs_launch::knn_grid_scratch(scene->n);
        ts.knn.ensure(need, c->stream);
        const int rc = rgs_launch::knn_grid(ts.pts.as<double>(), scene->n, nullptr, nullptr, 0, k, neighbors,
                                            ts.knn.p, ts.knn.bytes, c->stream);
        if (rc == -1) return set_err(c, RGS_E_INVALID, "knn: unsupported k");
        if (rc) return set_err(c, RGS_E_CUDA, "knn: grid build failed");
        c->launches += 9;
        CK(cudaGetLastError());
        return RGS_OK;
    });
}

int rgs_knn_query(rgs_ctx* c, const double* points4, int n, const double* queries4, int nq, const int32_t* exclude,
                  int k, int32_t* out) {
    if (!points4 || !queries4 || !out || n < 0 || nq < 0 || k < 1) return RGS_E_INVALID;
    if (k > 16) return set_err(c, RGS_E_INVALID, "knn: k must be at most 16");
    return guarded(c, [&]() -> int {
        if (nq == 0) return RGS_OK;
        if (n == 0) {
            CK(cudaMemsetAsync(out, 0xff, sizeof(int32_t) * (size_t)nq * k, c->stream));
            return RGS_OK;
        }
        TrainScratch& ts = train_scratch(c);
        ts.knn.ensure(rgs_launch::knn_grid_scratch(n), c->stream);
        const int rc = rgs_launch::knn_grid(points4, n, queries4, exclude, nq, k, out, ts.knn.p, ts.knn.bytes,
                                            c->stream);
        if (rc) return set_err(c, RGS_E_CUDA, "knn: grid build failed");
        c->launches += 5;
        CK(cudaGetLastError());
        return RGS_OK;
    });
}

int rgs_consistency_loss(rgs_ctx* c, const double* speeds, int n, const int32_t* neighbors, int k, double* dspeed,
                         double* losses) {
    if (!speeds || !neighbors || k < 0 || n < 0) return RGS_E_INVALID;
    return guarded(c, [&]() -> int {
        if (n == 0) return RGS_OK;
        TrainScratch& ts = train_scratch(c);
        ts.parts.ensure(sizeof(double) * (rgs_launch::consistency_blocks(n) + 16), c->stream);
        int* cnt = nullptr;
        if (dspeed) {
            ts.dcount.ensure(sizeof(int) * 3 * (size_t)n, c->stream);
            CK(cudaMemsetAsync(ts.dcount.p, 0, sizeof(int) * 3 * (size_t)n, c->stream));
            cnt = ts.dcount.as<int>();
        }
        rgs_launch::consistency(speeds, neighbors, n, k, cnt, ts.parts.as<double>(), losses, 0, c->stream);
        if (dspeed) rgs_launch::count_to_speed(cnt, n, k, dspeed, c->stream);
        c->launches += (losses ? 2 : 1) + (dspeed ? 1 : 0);
        CK(cudaGetLastError());
        return RGS_OK;
    });
}

int rgs_consistency(rgs_ctx* c, const rgs_scene* scene, const int32_t* neighbors, int k, double lambda,
                    unsigned flags, float* grads, double* losses) {
    if (!scene || !neighbors || k <= 0) return RGS_E_INVALID;
    return guarded(c, [&]() -> int {
        const int n = scene->n;
        if (n == 0) return RGS_OK;
        cudaStream_t s = c->stream;
        TrainScratch& ts = train_scratch(c);
        ts.speeds.ensure(sizeof(double) * 3 * (size_t)n, s);
        ts.cparts.ensure(sizeof(double) * (rgs_launch::consistency_blocks(n) + 16), s);
        const bool defer = (flags & RGS_FLAG_DEFER_CHECKS) != 0;
        DevBuf err;
        if (!defer) {
            err.ensure(sizeof(unsigned long long), s);
            CK(cudaMemsetAsync(err.p, 0xff, sizeof(unsigned long long), s));
        }
        unsigned long long* errp = defer ? c->deferred.as<unsigned long long>() : err.as<unsigned long long>();
        StageTimer t(c, kStConsistency, s);
        rgs_launch::speeds(scene->params, scene->params64, n, ts.speeds.as<double>(), errp, s);
        int* dcount = nullptr;
        if (grads) {
            ts.dcount.ensure(sizeof(int) * 3 * (size_t)n, s);
            CK(cudaMemsetAsync(ts.dcount.p, 0, sizeof(int) * 3 * (size_t)n, s));
            dcount = ts.dcount.as<int>();
        }
        rgs_launch::consistency(ts.speeds.as<double>(), neighbors, n, k, dcount, ts.cparts.as<double>(), losses,
                                (flags & RGS_FLAG_ACCUMULATE) ? 1 : 0, s);
        if (grads) rgs_launch::speed_backward(scene->params, scene->params64, n, k, dcount, lambda, grads, s);
        c->launches += 2 + (losses ? 1 : 0) + (grads ? 1 : 0);
        if (defer) return RGS_OK;  // the speeds' error is in the deferred status word
        unsigned long long e = 0;
        CK(cudaMemcpyAsync(&e, err.p, sizeof e, cudaMemcpyDeviceToHost, s));
        err.release(s);
        CK(cudaStreamSynchronize(s));
        if (e != kNoError) {
            const int code = (int)(e & 0xff);
            c->err_index = (int)(e >> 8);
            if (code == kErrDegenerateTime) return set_err(c, RGS_E_DEGENERATE_TIME, "slice_at: temporal scale collapsed (W < 1e-12)");
            return set_err(c, code, rotor_msg(code));
        }
        return RGS_OK;
    });
}

}  // extern "C"

// ===========================================================================
// R4GS v1 checkpoints straight to / from a device scene (checkpoint.cpp:29-86).
#include <cstdio>
#include <cstdlib>

namespace {
constexpr char kCkptMagic[4] = {'R', '4', 'G', 'S'};
constexpr uint32_t kCkptVersion = 1;  // checkpoint.hpp:19

int ckpt_err(rgs_ctx* c, const std::string& what) { return set_err(c, RGS_E_CHECKPOINT, "checkpoint: " + what); }
}  // namespace

extern "C" {

int rgs_scene_load_checkpoint(rgs_ctx* c, const char* path, unsigned scene_flags, rgs_scene** out) {
    if (!path || !out || (scene_flags & ~RGS_SCENE_F64)) return RGS_E_INVALID;
    if (!c) return RGS_E_INVALID;
    const std::string p(path);
    FILE* f = std::fopen(path, "rb");
    if (!f) return ckpt_err(c, "cannot open: " + p);
    struct Closer {
        FILE* f;
        ~Closer() { std::fclose(f); }
    } closer{f};
    char magic[4];
    if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, kCkptMagic, 4) != 0)
        return ckpt_err(c, "bad magic: " + p);
    uint32_t hdr[3] = {0, 0, 0};  // version, count, sh degree (little-endian host)
    const size_t got = std::fread(hdr, 4, 3, f);
    if (got < 1 || hdr[0] != kCkptVersion)
        return ckpt_err(c, "unsupported version " + std::to_string(got < 1 ? 0u : hdr[0]));
    if (got < 3 || hdr[2] > 3) return ckpt_err(c, "malformed header: " + p);
    const size_t n = hdr[1];
    if (n > (size_t)0x7fffffff) return ckpt_err(c, "malformed header: " + p);
    {  // the payload must be there before anything is allocated for it (checkpoint.cpp:71-73)
        const long here = std::ftell(f);
        if (here < 0 || std::fseek(f, 0, SEEK_END) != 0) return ckpt_err(c, "truncated: " + p);
        const long end = std::ftell(f);
        if (end < here || (size_t)(end - here) < 65 * sizeof(float) * n || std::fseek(f, here, SEEK_SET) != 0)
            return ckpt_err(c, "truncated: " + p);
    }
    return guarded(c, [&]() -> int {
        cudaStream_t s = c->stream;
        float* pinned = nullptr;
        const size_t bytes = 65 * sizeof(float) * std::max<size_t>(n, 1);
        CK(cudaMallocHost(&pinned, bytes));
        const size_t rd = n ? std::fread(pinned, 65 * sizeof(float), n, f) : 0;
        if (rd != n) {
            cudaFreeHost(pinned);
            return ckpt_err(c, "truncated: " + p);
        }
        rgs_scene* sc = nullptr;
        int rc = rgs_scene_create_ex(c, (int)n, (int)hdr[2], scene_flags, &sc);
        if (rc) {
            cudaFreeHost(pinned);
            return rc;
        }
        DevBuf tmp;
        tmp.ensure(bytes, s);
        CK(cudaMemcpyAsync(tmp.p, pinned, 65 * sizeof(float) * n, cudaMemcpyHostToDevice, s));
        rgs_launch::records_to_soa(tmp.as<float>(), (int)n, sc->params, sc->params64, s);
        c->launches += n ? 1 : 0;
        tmp.release(s);
        CK(cudaStreamSynchronize(s));
        cudaFreeHost(pinned);
        *out = sc;
        return RGS_OK;
    });
}

int rgs_scene_save_checkpoint(rgs_ctx* c, const rgs_scene* scene, const char* path) {
    if (!scene || !path) return RGS_E_INVALID;
    return guarded(c, [&]() -> int {
        const std::string p(path);
        const size_t n = (size_t)scene->n;
        cudaStream_t s = c->stream;
        std::vector<float> rec(65 * std::max<size_t>(n, 1));
        if (n) {
            DevBuf tmp;
            tmp.ensure(65 * sizeof(float) * n, s);
            rgs_launch::soa_to_records(scene->params, scene->params64, (int)n, tmp.as<float>(), s);
            c->launches += 1;
            CK(cudaMemcpyAsync(rec.data(), tmp.p, 65 * sizeof(float) * n, cudaMemcpyDeviceToHost, s));
            tmp.release(s);
            CK(cudaStreamSynchronize(s));
        }
        FILE* f = std::fopen(path, "wb");
        if (!f) return ckpt_err(c, "cannot open for writing: " + p);
        const uint32_t hdr[3] = {kCkptVersion, (uint32_t)n, (uint32_t)scene->sh_degree};
        bool ok = std::fwrite(kCkptMagic, 1, 4, f) == 4 && std::fwrite(hdr, 4, 3, f) == 3 &&
                  (n == 0 || std::fwrite(rec.data(), 65 * sizeof(float), n, f) == n);
        ok = (std::fclose(f) == 0) && ok;
        if (!ok) return ckpt_err(c, "write failed: " + p);
        return RGS_OK;
    });
}

}  // extern "C"

// ===========================================================================
// densify_and_prune (optim.cpp:168-234) and the train loop's generator.
#include <random>
#include <sstream>

struct rgs_rng {
    std::mt19937_64 eng;  // train_from's rng (trainer.cpp:105)
};

extern "C" {

int rgs_rng_create(unsigned long long seed, rgs_rng** out) {
    if (!out) return RGS_E_INVALID;
    *out = new rgs_rng{std::mt19937_64(seed)};
    return RGS_OK;
}
void rgs_rng_destroy(rgs_rng* r) { delete r; }
int rgs_rng_get_state(const rgs_rng* r, char* buf, size_t cap, size_t* len) {
    if (!r) return RGS_E_INVALID;
    std::ostringstream os;
    os << r->eng;  // the engine's textual state (std::mt19937_64 operator<<)
    const std::string st = os.str();
    if (len) *len = st.size() + 1;
    if (!buf) return RGS_OK;
    if (cap < st.size() + 1) return RGS_E_INVALID;
    std::memcpy(buf, st.c_str(), st.size() + 1);
    return RGS_OK;
}
int rgs_rng_set_state(rgs_rng* r, const char* buf) {
    if (!r || !buf) return RGS_E_INVALID;
    std::istringstream is(buf);
    is >> r->eng;
    return is.fail() ? RGS_E_INVALID : RGS_OK;
}
int rgs_rng_uniform_int(rgs_rng* r, int lo, int hi, int* out) {
    if (!r || !out || hi < lo) return RGS_E_INVALID;
    std::uniform_int_distribution<int> d(lo, hi);  // trainer.cpp:106, 119
    *out = d(r->eng);
    return RGS_OK;
}

int rgs_densify_and_prune(rgs_ctx* c, rgs_scene* scene, rgs_optimizer* o, const rgs_densify_config* cfg,
                          double scene_extent, rgs_rng* rng, rgs_densify_report* report) {
    if (!scene || !o || !cfg || !rng || o->n != scene->n) return RGS_E_INVALID;
    return guarded(c, [&]() -> int {
        cudaStream_t s = c->stream;
        const int n = scene->n;
        const bool f64 = scene->params64 != nullptr;
        const size_t eb = f64 ? sizeof(double) : sizeof(float);
        rgs_densify_report rep{0, 0, 0};
        // ---- densify decisions (optim.cpp:176-186) on the device
        std::vector<uint8_t> kind((size_t)std::max(n, 1), 0);
        DevBuf dk;
        if (n > 0) {
            dk.ensure((size_t)n, s);
            rgs_launch::densify_kind(scene->params, scene->params64, n, o->accum, o->count,
                                     cfg->densify_grad_threshold, cfg->percent_dense * scene_extent,
                                     dk.as<uint8_t>(), s);
            c->launches += 1;
            CK(cudaMemcpyAsync(kind.data(), dk.p, (size_t)n, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
        }
        // ---- the sequential part on the host: cut-off and normal draws, in index order
        std::normal_distribution<double> gauss(0, 1);  // optim.cpp:172 (fresh per call)
        std::vector<int32_t> parent, draw_off;
        std::vector<uint8_t> ckind;
        std::vector<double> draws;
        std::vector<uint8_t> removed;
        int size = n;
        for (int i = 0; i < n; ++i) {
            if (!kind[i]) continue;
            if (size + 2 > cfg->max_gaussians) break;
            if (kind[i] == 1) {
                parent.push_back(i);
                ckind.push_back(1);
                draw_off.push_back((int32_t)draws.size());
                draws.push_back(gauss(rng->eng));
                size += 1;
                rep.cloned += 1;
            } else {
                for (int k = 0; k < 2; ++k) {
                    parent.push_back(i);
                    ckind.push_back((uint8_t)(2 + k));
                    draw_off.push_back((int32_t)draws.size());
                    for (int a = 0; a < 4; ++a) draws.push_back(gauss(rng->eng));
                }
                size += 2;
                rep.split += 1;
            }
        }
        const int n_child = (int)parent.size();
        const int ext_n = n + n_child;
        // ---- extended store: survivors copied, children appended (push_back)
        void *ext = nullptr, *ext_m1 = nullptr, *ext_m2 = nullptr;
        const size_t ext1 = (size_t)std::max(ext_n, 1);
        CK(cudaMalloc(&ext, 65 * ext1 * eb));
        CK(cudaMalloc(&ext_m1, 65 * ext1 * eb));
        CK(cudaMalloc(&ext_m2, 65 * ext1 * eb));
        void* params = f64 ? (void*)scene->params64 : (void*)scene->params;
        rgs_launch::gather_soa(f64, params, n, nullptr, n, ext, ext_n, s);
        rgs_launch::gather_soa(f64, o->m1, n, nullptr, n, ext_m1, ext_n, s);
        rgs_launch::gather_soa(f64, o->m2, n, nullptr, n, ext_m2, ext_n, s);
        c->launches += 3;
        DevBuf dparent, dck, ddraw, doff, derr, drem, dflag;
        derr.ensure(sizeof(unsigned long long), s);
        CK(cudaMemsetAsync(derr.p, 0xff, sizeof(unsigned long long), s));
        if (n_child) {
            dparent.ensure(4 * (size_t)n_child, s);
            dck.ensure((size_t)n_child, s);
            doff.ensure(4 * (size_t)n_child, s);
            ddraw.ensure(8 * draws.size(), s);
            CK(cudaMemcpyAsync(dparent.p, parent.data(), 4 * (size_t)n_child, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(dck.p, ckind.data(), (size_t)n_child, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(doff.p, draw_off.data(), 4 * (size_t)n_child, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(ddraw.p, draws.data(), 8 * draws.size(), cudaMemcpyHostToDevice, s));
            rgs_launch::densify_children(scene->params, scene->params64, n, dparent.as<int32_t>(), dck.as<uint8_t>(),
                                         ddraw.as<double>(), doff.as<int32_t>(), n_child,
                                         std::log(cfg->split_factor), cfg->static_mode, ext, ext_m1, ext_m2, ext_n,
                                         derr.as<unsigned long long>(), s);
            c->launches += 1;
        }
        // ---- prune (optim.cpp:211-226): flags on the device, the opacity sort on the host
        std::vector<uint8_t> rem((size_t)ext1, 0);
        for (int k = 0; k < n_child; ++k)
            if (ckind[k] == 2) rem[parent[k]] = 1;  // split parents (to_remove)
        drem.ensure(ext1, s);
        dflag.ensure(ext1, s);
        CK(cudaMemcpyAsync(drem.p, rem.data(), ext1, cudaMemcpyHostToDevice, s));
        rgs_launch::prune_flags(f64 ? nullptr : (const float*)ext, f64 ? (const double*)ext : nullptr, ext_n,
                                drem.as<uint8_t>(), cfg->prune_opacity, 0.5 * scene_extent, cfg->static_mode,
                                dflag.as<uint8_t>(), s);
        c->launches += 1;
        std::vector<uint8_t> flag(ext1);
        std::vector<double> logit(ext1);
        std::vector<float> logit_f(f64 ? 0 : ext1);
        CK(cudaMemcpyAsync(flag.data(), dflag.p, ext1, cudaMemcpyDeviceToHost, s));
        if (f64)
            CK(cudaMemcpyAsync(logit.data(), (double*)ext + 64 * (size_t)ext_n, 8 * (size_t)ext_n,
                               cudaMemcpyDeviceToHost, s));
        else
            CK(cudaMemcpyAsync(logit_f.data(), (float*)ext + 64 * (size_t)ext_n, 4 * (size_t)ext_n,
                               cudaMemcpyDeviceToHost, s));
        unsigned long long e = 0;
        CK(cudaMemcpyAsync(&e, derr.p, sizeof e, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        auto free_ext = [&]() {
            cudaFree(ext);
            cudaFree(ext_m1);
            cudaFree(ext_m2);
        };
        if (e != kNoError) {
            free_ext();
            const int code = (int)(e & 0xff);
            c->err_index = (int)(e >> 8);
            if (code == kErrDegenerateTime)
                return set_err(c, RGS_E_DEGENERATE_TIME, "slice_at: temporal scale collapsed (W < 1e-12)");
            return set_err(c, code, rotor_msg(code));
        }
        if (!f64)
            for (int i = 0; i < ext_n; ++i) logit[i] = logit_f[i];
        auto opacity = [&](int i) { return 1 / (1 + std::exp(-logit[i])); };  // GaussianStore::opacity
        std::vector<int> prunable;
        for (int i = 0; i < ext_n; ++i)
            if (flag[i]) prunable.push_back(i);
        int n_removed_split = rep.split;
        int allowed = std::max(0, ext_n - n_removed_split - cfg->min_gaussians);
        if ((int)prunable.size() > allowed) {
            std::sort(prunable.begin(), prunable.end(), [&](int a, int b) { return opacity(a) < opacity(b); });
            prunable.resize(allowed);
        }
        rep.pruned = (int)prunable.size();
        std::vector<uint8_t> drop((size_t)ext1, 0);
        for (int i = 0; i < ext_n; ++i) drop[i] = rem[i];
        for (int i : prunable) drop[i] = 1;
        std::vector<int32_t> keep;
        keep.reserve(ext_n);
        for (int i = 0; i < ext_n; ++i)
            if (!drop[i]) keep.push_back(i);
        const int n_new = (int)keep.size();
        // ---- remove_indices (gaussian.cpp:142-180) as one gather; reset_stats
        const size_t nn1 = (size_t)std::max(n_new, 1);
        void *np = nullptr, *nm1 = nullptr, *nm2 = nullptr;
        double* nacc = nullptr;
        int32_t* ncnt = nullptr;
        CK(cudaMalloc(&np, 65 * nn1 * eb));
        CK(cudaMalloc(&nm1, 65 * nn1 * eb));
        CK(cudaMalloc(&nm2, 65 * nn1 * eb));
        CK(cudaMalloc(&nacc, nn1 * sizeof(double)));
        CK(cudaMalloc(&ncnt, nn1 * sizeof(int32_t)));
        DevBuf dkeep;
        dkeep.ensure(4 * nn1, s);
        CK(cudaMemcpyAsync(dkeep.p, keep.data(), 4 * (size_t)n_new, cudaMemcpyHostToDevice, s));
        rgs_launch::gather_soa(f64, ext, ext_n, dkeep.as<int32_t>(), n_new, np, n_new, s);
        rgs_launch::gather_soa(f64, ext_m1, ext_n, dkeep.as<int32_t>(), n_new, nm1, n_new, s);
        rgs_launch::gather_soa(f64, ext_m2, ext_n, dkeep.as<int32_t>(), n_new, nm2, n_new, s);
        c->launches += 3;
        CK(cudaMemsetAsync(nacc, 0, nn1 * sizeof(double), s));
        CK(cudaMemsetAsync(ncnt, 0, nn1 * sizeof(int32_t), s));
        CK(cudaStreamSynchronize(s));
        for (DevBuf* b : {&dk, &dparent, &dck, &ddraw, &doff, &derr, &drem, &dflag, &dkeep}) b->release(s);
        free_ext();
        cudaFree(f64 ? (void*)scene->params64 : (void*)scene->params);
        cudaFree(o->m1);
        cudaFree(o->m2);
        cudaFree(o->accum);
        cudaFree(o->count);
        if (f64)
            scene->params64 = (double*)np;
        else
            scene->params = (float*)np;
        scene->n = n_new;
        o->n = n_new;
        o->m1 = nm1;
        o->m2 = nm2;
        o->accum = nacc;
        o->count = ncnt;
        o->part.ensure(sizeof(double) * (rgs_launch::adam_blocks(n_new) + 16), s);
        if (report) *report = rep;
        return RGS_OK;
    });
}

}  // extern "C"

// For the other host translation units of the library (rgs_nccl.cu).
namespace rgs_host {
int set_ctx_error(rgs_ctx* c, int code, const char* msg) { return set_err(c, code, msg ? msg : ""); }
}  // namespace rgs_host
