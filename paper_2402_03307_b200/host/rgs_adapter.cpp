// Drop-in C++ implementation of the reference's render entry points over the C ABI.
//
// A maintainer of /root/reference/proj compiles this file INSTEAD OF src/rasterizer.cpp
// and links librgs_cuda.so: every declaration of include/rgs/rasterizer.hpp keeps its
// signature, argument meaning and exceptions:
//   project            rasterizer.hpp:52-54   -> rgs_project_sliced_cache (device, FP64)
//   render_forward     rasterizer.hpp:82-83   -> rgs_render_forward + rgs_records_export
//   rasterize_forward  rasterizer.hpp:87-89   -> rgs_rasterize_forward
//   render_backward    rasterizer.hpp:93-95   -> rgs_render_backward
//   render_flow        rasterizer.hpp:99      -> rgs_render_flow
// Behaviour differences: `threads` is ignored; project() fills ProjectCache (computed on the
// device) but RenderRecords::caches are not filled (the device backward recomputes what it
// needs); rotor errors always throw.
// Device-side caching: the device copy of a store is kept and reused while
// the store's contents (a 64-bit hash of every parameter array), size and SH degree are
// unchanged, and the device records of the last render_forward stay alive so that the
// render_backward of the same view (evaluate_loss, trainer.cpp:35-52) uses them instead of
// re-rendering; a backward whose records were not the last forward's (or whose pixel records
// were changed) re-renders the view from the store, as before.
// Environment: RGS_DEVICE selects the CUDA device (default 0).  RGS_KAT_MODE=1 selects the
// reference-KAT precision mode: FP64 blending with double images, and the deterministic
// FP64 backward (reference summation order, bitwise reproducible).
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "rgs/rasterizer.hpp"
#include "rgs_cuda.h"
#include "rgs_dropin_common.hpp"

namespace rgs {
namespace {

rgs_ctx* context() { return dropin::context(); }

bool kat_mode() {
    const char* v = std::getenv("RGS_KAT_MODE");
    return v && v[0] == '1';
}

[[noreturn]] void raise(int rc) {
    const std::string msg = rgs_ctx_last_error(context());
    switch (rc) {
        case RGS_E_CAMERA: throw std::runtime_error(msg);
        case RGS_E_MISSING_RECORDS: throw MissingRecordsError();
        case RGS_E_ZERO_ROTOR: throw ZeroRotorError();
        case RGS_E_NONFINITE_ROTOR: throw NonFiniteRotorError();
        default: throw std::runtime_error("rgs_b200: " + msg);
    }
}

void check(int rc) {
    if (rc != RGS_OK) raise(rc);
}

rgs_camera to_c(const Camera& cam) {
    rgs_camera c;
    std::memset(&c, 0, sizeof c);  // (compared bytewise by the records reuse)
    c.width = cam.width;
    c.height = cam.height;
    c.fx = cam.fx;
    c.fy = cam.fy;
    c.cx = cam.cx;
    c.cy = cam.cy;
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) c.world_to_camera[4 * i + j] = cam.world_to_camera(i, j);
    c.time = cam.time;
    return c;
}

Splat2D from_c(const rgs_splat& s) {
    Splat2D o;
    o.mean2 = Vec2(s.mean2[0], s.mean2[1]);
    o.conic = Vec3(s.conic[0], s.conic[1], s.conic[2]);
    o.depth = s.depth;
    o.color = Vec3(s.color[0], s.color[1], s.color[2]);
    o.alpha_base = s.alpha_base;
    o.flow2 = Vec2(s.flow2[0], s.flow2[1]);
    o.radius = s.radius;
    o.source_index = s.source_index;
    return o;
}

rgs_splat to_c(const Splat2D& s) {
    rgs_splat o;
    std::memset(&o, 0, sizeof o);
    o.mean2[0] = s.mean2[0];
    o.mean2[1] = s.mean2[1];
    for (int k = 0; k < 3; ++k) o.conic[k] = s.conic[k];
    o.depth = s.depth;
    for (int k = 0; k < 3; ++k) o.color[k] = s.color[k];
    o.alpha_base = s.alpha_base;
    o.flow2[0] = s.flow2[0];
    o.flow2[1] = s.flow2[1];
    o.radius = s.radius;
    o.source_index = s.source_index;
    return o;
}

using dropin::hash_vec;

// GaussianStore (gaussian.hpp:79-103) -> the cached device scene (FP64 storage: the store's
// double values reach the kernels unrounded).  Re-uploaded only when the contents change.
struct SceneCache {
    rgs_scene* s = nullptr;
    int n = -1, sh = -1;
    uint64_t hash = 0;
    long long uploads = 0, hits = 0, d2d = 0;
};
SceneCache& scene_cache() {
    static SceneCache c;
    return c;
}

rgs_scene* device_scene(const GaussianStore& store, uint64_t* key = nullptr) {
    SceneCache& c = scene_cache();
    const int n = store.size();
    const uint64_t h = dropin::params_hash(store);
    if (key) *key = h;
    if (c.s && c.n == n && c.sh == store.active_sh_degree && c.hash == h) {
        ++c.hits;
        return c.s;
    }
    if (c.s && c.n != n) {
        rgs_scene_destroy(c.s);
        c.s = nullptr;
    }
    if (!c.s) check(rgs_scene_create_ex(context(), n, store.active_sh_degree, RGS_SCENE_F64, &c.s));
    rgs_scene_set_sh_degree(c.s, store.active_sh_degree);
    // the training side just wrote exactly these parameters on the device: copy them over
    if (const double* src = dropin::published_params(h, n, store.active_sh_degree)) {
        c.n = -1;
        if (n) check(rgs_memcpy(context(), rgs_scene_params_f64(c.s), src, sizeof(double) * 65 * (size_t)n));
        c.n = n;
        c.sh = store.active_sh_degree;
        c.hash = h;
        ++c.d2d;
        return c.s;
    }
    double* mean = dropin::scratch<double>(0, 4 * (size_t)n).data();
    double* ls = dropin::scratch<double>(1, 4 * (size_t)n).data();
    double* rot = dropin::scratch<double>(2, 8 * (size_t)n).data();
    double* op = dropin::scratch<double>(3, (size_t)n).data();
    double* sh = dropin::scratch<double>(4, 48 * (size_t)n).data();
    dropin::parallel_for((size_t)n, [&](size_t i0, size_t i1) {
        for (size_t i = i0; i < i1; ++i) {
            for (int a = 0; a < 4; ++a) mean[4 * i + a] = store.mean[i][a];
            for (int a = 0; a < 4; ++a) ls[4 * i + a] = store.log_scales[i][a];
            const Vec8 cf = store.rotor[i].coeffs();
            for (int a = 0; a < 8; ++a) rot[8 * i + a] = cf[a];
            op[i] = store.opacity_logit[i];
            for (int ch = 0; ch < 3; ++ch)
                for (int k = 0; k < 16; ++k) sh[48 * i + ch * 16 + k] = store.sh[i](ch, k);
        }
    });
    c.n = -1;  // invalid until the upload succeeded
    check(rgs_scene_upload_f64(context(), c.s, mean, ls, rot, op, sh, nullptr));
    c.n = n;
    c.sh = store.active_sh_degree;
    c.hash = h;
    ++c.uploads;
    return c.s;
}

struct RecordsHandle {
    rgs_records* r = nullptr;
    ~RecordsHandle() { rgs_records_destroy(r); }
};

// The device records of the last render_forward, for its render_backward.
struct LastForward {
    rgs_records* r = nullptr;
    uint64_t scene_key = 0, nc_hash = 0;
    rgs_camera cam{};
    double bg[3] = {0, 0, 0};
    const int* nc_data = nullptr;
    size_t nc_size = 0;
    long long reused = 0;
    void reset(rgs_records* nr) {
        if (r) rgs_records_destroy(r);
        r = nr;
    }
};
LastForward& last_forward() {
    static LastForward lf;
    return lf;
}

unsigned image_flags() { return RGS_FLAG_HOST_BUFFERS | (kat_mode() ? RGS_FLAG_IMAGE_F64 : 0u); }

// Renders into a reference Image (double, interleaved); FP32 device images are widened.
template <typename Fn>
void render_image(Image* image, int w, int h, int channels, Fn&& fn) {
    *image = Image(w, h, channels);
    if (kat_mode()) {
        fn(reinterpret_cast<float*>(image->data.data()));
    } else {
        const size_t cnt = (size_t)w * h * channels;
        float* tmp = dropin::scratch<float>(3, cnt).data();
        fn(tmp);
        dropin::parallel_for(cnt, [&](size_t i0, size_t i1) {
            for (size_t i = i0; i < i1; ++i) image->data[i] = tmp[i];
        });
    }
}

void export_records(const RecordsHandle& h, RenderRecords* rec, const Vec3& background) {
    rgs_records_info info;
    check(rgs_records_info_get(h.r, &info));
    const size_t ns = (size_t)info.n_splats, npix = (size_t)info.width * info.height;
    const rgs_splat* sp = dropin::scratch<rgs_splat>(0, ns).data();
    const int nt = info.tiles_x * info.tiles_y;
    const long long* off = dropin::scratch<long long>(0, (size_t)nt + 1).data();
    const int32_t* ids = dropin::scratch<int32_t>(2, (size_t)std::max<long long>(info.n_pairs, 1)).data();
    const int32_t* nc = dropin::scratch<int32_t>(1, npix).data();
    rec->final_T.resize(npix);
    check(rgs_records_export(context(), h.r, const_cast<rgs_splat*>(sp), const_cast<long long*>(off),
                             const_cast<int32_t*>(ids), rec->final_T.data(), const_cast<int32_t*>(nc)));
    rec->splats.resize(ns);
    dropin::parallel_for(ns, [&](size_t i0, size_t i1) {
        for (size_t i = i0; i < i1; ++i) rec->splats[i] = from_c(sp[i]);
    });
    rec->tile_splats.resize(nt);
    for (int t = 0; t < nt; ++t) rec->tile_splats[t].assign(ids + off[t], ids + off[t + 1]);
    rec->n_contrib.assign(nc, nc + npix);
    rec->tiles_x = info.tiles_x;
    rec->tiles_y = info.tiles_y;
    rec->background = background;
}

}  // namespace

std::optional<Splat2D> project(const SlicedGaussian3D& s, const Camera& cam, const ShCoeffs& sh, int sh_degree,
                               Scalar opacity_logit, ProjectCache* cache) {
    double sliced[16];
    for (int a = 0; a < 3; ++a) sliced[a] = s.mean[a];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) sliced[3 + 3 * i + j] = s.cov(i, j);
    sliced[12] = s.decay;
    for (int a = 0; a < 3; ++a) sliced[13 + a] = s.speed[a];
    double sh48[48];
    for (int ch = 0; ch < 3; ++ch)
        for (int k = 0; k < 16; ++k) sh48[ch * 16 + k] = sh(ch, k);
    const rgs_camera c = to_c(cam);
    rgs_splat out;
    int survived = 0;
    double pc[RGS_PROJECT_CACHE_DOUBLES];
    check(rgs_project_sliced_cache(context(), sliced, &c, sh48, sh_degree, opacity_logit, &out, &survived,
                                   cache ? pc : nullptr));
    if (!survived) return std::nullopt;
    if (cache) {  // rasterizer.cpp:261-275
        cache->cov3 = s.cov;
        cache->mean3 = s.mean;
        cache->speed = s.speed;
        cache->decay = s.decay;
        cache->p_cam = Vec3(pc[0], pc[1], pc[2]);
        for (int r = 0; r < 2; ++r)
            for (int k = 0; k < 3; ++k) cache->T(r, k) = pc[3 + 3 * r + k];
        for (int r = 0; r < 2; ++r)
            for (int k = 0; k < 2; ++k) cache->cov2(r, k) = pc[9 + 2 * r + k];
        cache->dir = Vec3(pc[13], pc[14], pc[15]);
        cache->view_dist = pc[16];
        for (int k = 0; k < 16; ++k) cache->basis[k] = pc[17 + k];
        for (int k = 0; k < 16; ++k)
            for (int j = 0; j < 3; ++j) cache->basis_grad(k, j) = pc[33 + 3 * k + j];
        for (int ch = 0; ch < 3; ++ch) cache->clamped[ch] = pc[81 + ch] != 0.0;
        cache->opacity = pc[84];
    }
    return from_c(out);
}

void rasterize_forward(const std::vector<Splat2D>& splats, const Camera& cam, const Vec3& background,
                       int /*threads*/, Image* image, RenderRecords* records) {
    std::vector<rgs_splat> sp(splats.size());
    for (size_t i = 0; i < splats.size(); ++i) sp[i] = to_c(splats[i]);
    const rgs_camera c = to_c(cam);
    const double bg[3] = {background[0], background[1], background[2]};
    RecordsHandle h;
    render_image(image, cam.width, cam.height, 3, [&](float* img) {
        check(rgs_rasterize_forward(context(), sp.data(), (int)sp.size(), &c, bg, image_flags(), img, &h.r));
    });
    if (records) {
        export_records(h, records, background);
        records->splats = splats;
    }
}

RenderOutput render_forward(const GaussianStore& store, const Camera& cam, const RenderOptions& opts) {
    cam.validate();
    uint64_t key = 0;
    rgs_scene* scene = device_scene(store, &key);
    const rgs_camera c = to_c(cam);
    const double bg[3] = {opts.background[0], opts.background[1], opts.background[2]};
    RenderOutput out;
    RecordsHandle h;
    render_image(&out.image, cam.width, cam.height, 3, [&](float* img) {
        check(rgs_render_forward(context(), scene, &c, bg, image_flags() | RGS_FLAG_RETAIN_RECORDS, img, &h.r));
    });
    export_records(h, &out.records, opts.background);
    out.records.retained = opts.retain_records;
    if (opts.retain_records) {  // kept for the render_backward of this view
        LastForward& lf = last_forward();
        lf.reset(h.r);
        h.r = nullptr;
        lf.scene_key = key;
        lf.cam = c;
        for (int k = 0; k < 3; ++k) lf.bg[k] = bg[k];
        lf.nc_data = out.records.n_contrib.data();
        lf.nc_size = out.records.n_contrib.size();
        lf.nc_hash = hash_vec(out.records.n_contrib, 7);
    }
    return out;
}

StoreGrads render_backward(const GaussianStore& store, const Camera& cam, const RenderRecords& rec,
                           const Image& dL_dimage, int /*threads*/) {
    if (!rec.retained) throw MissingRecordsError();
    uint64_t key = 0;
    rgs_scene* scene = device_scene(store, &key);
    const rgs_camera c = to_c(cam);
    const double bg[3] = {rec.background[0], rec.background[1], rec.background[2]};
    // The device records of this view: the last forward's when `rec` came from it (same store
    // contents, camera, background, and the very pixel records it returned), else rebuilt by
    // re-rendering (deterministic: the same decisions as `rec`).
    RecordsHandle h;
    rgs_records* dev_rec = nullptr;
    LastForward& lf = last_forward();
    if (lf.r && lf.scene_key == key && std::memcmp(&lf.cam, &c, sizeof c) == 0 && lf.bg[0] == bg[0] &&
        lf.bg[1] == bg[1] && lf.bg[2] == bg[2] && lf.nc_data == rec.n_contrib.data() &&
        lf.nc_size == rec.n_contrib.size() && lf.nc_hash == hash_vec(rec.n_contrib, 7)) {
        dev_rec = lf.r;
        ++lf.reused;
    } else {
        std::vector<double> img64((size_t)cam.width * cam.height * 3);
        check(rgs_render_forward(context(), scene, &c, bg, image_flags() | RGS_FLAG_RETAIN_RECORDS,
                                 reinterpret_cast<float*>(img64.data()), &h.r));
        dev_rec = h.r;
    }
    const int n = store.size();
    const size_t ndl = dL_dimage.data.size(), n1 = (size_t)std::max(n, 1);
    float* dl = dropin::scratch<float>(2, ndl).data();
    dropin::parallel_for(ndl, [&](size_t i0, size_t i1) {
        for (size_t i = i0; i < i1; ++i) dl[i] = (float)dL_dimage.data[i];
    });
    const float* g = dropin::scratch<float>(0, 65 * n1).data();
    const float* vn = dropin::scratch<float>(1, n1).data();
    const int32_t* vis = dropin::scratch<int32_t>(0, n1).data();
    // thread-count invariant like the reference's fixed-order reduction (rasterizer.cpp:372-384):
    // the FP64 replay in KAT mode, the fixed-point accumulation otherwise
    const unsigned flags = RGS_FLAG_HOST_BUFFERS | (kat_mode() ? RGS_FLAG_DETERMINISTIC : RGS_FLAG_REPRODUCIBLE);
    check(rgs_render_backward(context(), scene, &c, dev_rec, dl, flags, const_cast<float*>(g), const_cast<float*>(vn),
                              const_cast<int32_t*>(vis)));
    // device SoA (rgs_scene_params layout) -> per-Gaussian gradients
    StoreGrads out;
    out.resize(n);
    const size_t N = (size_t)n;
    dropin::parallel_for(N, [&](size_t i0, size_t i1) {
        for (size_t i = i0; i < i1; ++i) {
            GaussianParamGrad& p = out.g[i];
            for (int a = 0; a < 4; ++a) p.d_mean[a] = g[4 * i + a];
            for (int a = 0; a < 4; ++a) p.d_log_scales[a] = g[4 * N + 4 * i + a];
            Vec8 r;
            for (int a = 0; a < 4; ++a) r[a] = g[8 * N + 4 * i + a];
            for (int a = 0; a < 4; ++a) r[4 + a] = g[12 * N + 4 * i + a];
            p.d_rotor = r;
            p.d_opacity_logit = g[64 * N + i];
            for (int j = 0; j < 48; ++j) p.d_sh(j % 3, j / 3) = g[(16 + 4 * (size_t)(j / 4)) * N + 4 * i + (j % 4)];
            out.viewspace_norm[i] = vn[i];
            out.visible[i] = vis[i] > 0 ? 1 : 0;
        }
    });
    return out;
}

Image render_flow(const GaussianStore& store, const Camera& cam, int /*threads*/) {
    cam.validate();
    rgs_scene* scene = device_scene(store);
    const rgs_camera c = to_c(cam);
    Image flow;
    render_image(&flow, cam.width, cam.height, 2, [&](float* img) {
        check(rgs_render_flow(context(), scene, &c, image_flags() | (kat_mode() ? RGS_FLAG_BLEND_FP64 : 0u), img));
    });
    return flow;
}

}  // namespace rgs

// Adapter statistics (tests / bench of the drop-in path): device-scene uploads, cache hits and
// backward passes that reused the forward's device records.
extern "C" void rgs_adapter_stats(long long* uploads, long long* hits, long long* records_reused) {
    if (uploads) *uploads = rgs::scene_cache().uploads;
    if (hits) *hits = rgs::scene_cache().hits;
    if (records_reused) *records_reused = rgs::last_forward().reused;
}
