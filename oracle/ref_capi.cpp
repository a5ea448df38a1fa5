// C wrapper around the UNMODIFIED reference render path, for oracle/_ref only.
//
// TEST INFRASTRUCTURE — never linked into the product.  The reference sources
// (/root/reference/proj/src/{rotor,gaussian,sh,rasterizer,image}.cpp and
// tests/reference.hpp) are compiled in place by oracle/Makefile against the
// Eigen subset in include/eigen_subset; this file only marshals plain arrays
// into the reference's own types and calls its public API:
//   render_forward     rasterizer.hpp:82-83   (rasterizer.cpp:308-318)
//   rasterize_forward  rasterizer.hpp:87-89   (rasterizer.cpp:278-306)
//   render_backward    rasterizer.hpp:93-95   (rasterizer.cpp:320-397)
//   render_flow        rasterizer.hpp:99      (rasterizer.cpp:399-425)
//   project / slice_at / normalize / to_matrix (rasterizer.hpp:52-54,
//   gaussian.hpp:64, rotor.hpp:41-52)
//   naive_render / random_scene (tests/reference.hpp:27-116)
//
// Scene arrays (per Gaussian, row-major): mean[4], log_scales[4],
// rotor[8] (s,b01,b02,b03,b12,b13,b23,p), opacity_logit[1], sh[48] channel-major
// (sh[ch*16+k] = ShCoeffs(ch,k)).  Camera: ref_camera below.  Errors are returned
// as the same integer codes as include/rgs_cuda.h (RGS_E_*).
#include <cstdint>
#include <cstring>
#include <exception>
#include <vector>

#include "reference.hpp"
#include "rgs/rasterizer.hpp"

using namespace rgs;

extern "C" {

typedef struct {
    int width, height;
    double fx, fy, cx, cy;
    double world_to_camera[16];  // row-major
    double time;
} ref_camera;

// 13 doubles + source index (112 bytes), same as rgs_splat in include/rgs_cuda.h.
typedef struct {
    double mean2[2];
    double conic[3];
    double depth;
    double color[3];
    double alpha_base;
    double flow2[2];
    double radius;
    int32_t source_index;
    int32_t pad;
} ref_splat;

enum { RGS_OK = 0, RGS_E_CAMERA = 1, RGS_E_MISSING_RECORDS = 2, RGS_E_ZERO_ROTOR = 3,
       RGS_E_NONFINITE_ROTOR = 4, RGS_E_CUDA = 5, RGS_E_INVALID = 6, RGS_E_DEGENERATE_TIME = 7,
       RGS_E_OTHER = 99 };

}  // extern "C"

namespace {

thread_local char g_err[512];

Camera to_cam(const ref_camera* c) {
    Camera cam;
    cam.width = c->width;
    cam.height = c->height;
    cam.fx = c->fx;
    cam.fy = c->fy;
    cam.cx = c->cx;
    cam.cy = c->cy;
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) cam.world_to_camera(i, j) = c->world_to_camera[4 * i + j];
    cam.time = c->time;
    return cam;
}

GaussianStore to_store(int n, const double* mean, const double* ls, const double* rot,
                       const double* op, const double* sh, int deg) {
    GaussianStore s;
    s.active_sh_degree = deg;
    for (int i = 0; i < n; ++i) {
        Gaussian4D g;
        for (int a = 0; a < 4; ++a) g.mean[a] = mean[4 * i + a];
        for (int a = 0; a < 4; ++a) g.log_scales[a] = ls[4 * i + a];
        Vec8 c;
        for (int a = 0; a < 8; ++a) c[a] = rot[8 * i + a];
        g.rotor = Rotor4::from_coeffs(c);
        g.opacity_logit = op[i];
        for (int ch = 0; ch < 3; ++ch)
            for (int k = 0; k < 16; ++k) g.sh(ch, k) = sh[48 * i + ch * 16 + k];
        s.push_back(g);
    }
    return s;
}

void from_splat(const Splat2D& s, ref_splat* o) {
    o->mean2[0] = s.mean2[0];
    o->mean2[1] = s.mean2[1];
    for (int k = 0; k < 3; ++k) o->conic[k] = s.conic[k];
    o->depth = s.depth;
    for (int k = 0; k < 3; ++k) o->color[k] = s.color[k];
    o->alpha_base = s.alpha_base;
    o->flow2[0] = s.flow2[0];
    o->flow2[1] = s.flow2[1];
    o->radius = s.radius;
    o->source_index = s.source_index;
    o->pad = 0;
}

Splat2D to_splat(const ref_splat& o) {
    Splat2D s;
    s.mean2 = Vec2(o.mean2[0], o.mean2[1]);
    s.conic = Vec3(o.conic[0], o.conic[1], o.conic[2]);
    s.depth = o.depth;
    s.color = Vec3(o.color[0], o.color[1], o.color[2]);
    s.alpha_base = o.alpha_base;
    s.flow2 = Vec2(o.flow2[0], o.flow2[1]);
    s.radius = o.radius;
    s.source_index = o.source_index;
    return s;
}

int map_exception() {
    try {
        throw;
    } catch (const MissingRecordsError& e) {
        std::snprintf(g_err, sizeof g_err, "%s", e.what());
        return RGS_E_MISSING_RECORDS;
    } catch (const ZeroRotorError& e) {
        std::snprintf(g_err, sizeof g_err, "%s", e.what());
        return RGS_E_ZERO_ROTOR;
    } catch (const NonFiniteRotorError& e) {
        std::snprintf(g_err, sizeof g_err, "%s", e.what());
        return RGS_E_NONFINITE_ROTOR;
    } catch (const DegenerateTimeError& e) {
        std::snprintf(g_err, sizeof g_err, "%s", e.what());
        return RGS_E_DEGENERATE_TIME;
    } catch (const std::runtime_error& e) {
        std::snprintf(g_err, sizeof g_err, "%s", e.what());
        // Camera::validate throws plain runtime_error (camera.hpp:21-26).
        return std::strncmp(e.what(), "camera:", 7) == 0 ? RGS_E_CAMERA : RGS_E_OTHER;
    } catch (const std::exception& e) {
        std::snprintf(g_err, sizeof g_err, "%s", e.what());
        return RGS_E_OTHER;
    }
}

}  // namespace

struct ref_records {
    RenderRecords rec;
    int width = 0, height = 0;
};

extern "C" {

const char* ref_last_error(void) { return g_err; }

int ref_render_forward(int n, const double* mean, const double* ls, const double* rot,
                       const double* op, const double* sh, int sh_degree, const ref_camera* c,
                       const double* bg, int threads, int retain, double* image_out,
                       ref_records** rec_out) {
    try {
        GaussianStore store = to_store(n, mean, ls, rot, op, sh, sh_degree);
        Camera cam = to_cam(c);
        RenderOptions opts;
        opts.background = Vec3(bg[0], bg[1], bg[2]);
        opts.threads = threads;
        opts.retain_records = retain != 0;
        RenderOutput out = render_forward(store, cam, opts);
        std::memcpy(image_out, out.image.data.data(), out.image.data.size() * sizeof(double));
        if (rec_out) {
            auto* r = new ref_records;
            r->rec = std::move(out.records);
            r->width = cam.width;
            r->height = cam.height;
            *rec_out = r;
        }
        return RGS_OK;
    } catch (...) {
        return map_exception();
    }
}

int ref_rasterize_forward(int n_splats, const ref_splat* splats, const ref_camera* c,
                          const double* bg, int threads, double* image_out,
                          ref_records** rec_out) {
    try {
        std::vector<Splat2D> sp(n_splats);
        for (int i = 0; i < n_splats; ++i) sp[i] = to_splat(splats[i]);
        Camera cam = to_cam(c);
        Image img;
        auto* r = new ref_records;
        rasterize_forward(sp, cam, Vec3(bg[0], bg[1], bg[2]), threads, &img, &r->rec);
        r->rec.splats = sp;
        r->width = cam.width;
        r->height = cam.height;
        std::memcpy(image_out, img.data.data(), img.data.size() * sizeof(double));
        if (rec_out)
            *rec_out = r;
        else
            delete r;
        return RGS_OK;
    } catch (...) {
        return map_exception();
    }
}

void ref_records_free(ref_records* r) { delete r; }
int ref_records_num_splats(const ref_records* r) { return (int)r->rec.splats.size(); }
int ref_records_num_tiles(const ref_records* r) { return r->rec.tiles_x * r->rec.tiles_y; }
int ref_records_retained(const ref_records* r) { return r->rec.retained ? 1 : 0; }
long long ref_records_num_pairs(const ref_records* r) {
    long long p = 0;
    for (const auto& t : r->rec.tile_splats) p += (long long)t.size();
    return p;
}
void ref_records_splats(const ref_records* r, ref_splat* out) {
    for (size_t i = 0; i < r->rec.splats.size(); ++i) from_splat(r->rec.splats[i], &out[i]);
}
// offsets: num_tiles + 1 entries; ids: num_pairs entries.
void ref_records_tiles(const ref_records* r, long long* offsets, int32_t* ids) {
    long long p = 0;
    size_t t = 0;
    for (; t < r->rec.tile_splats.size(); ++t) {
        offsets[t] = p;
        for (int id : r->rec.tile_splats[t]) ids[p++] = id;
    }
    offsets[t] = p;
}
void ref_records_pixels(const ref_records* r, double* final_T, int32_t* n_contrib) {
    size_t npix = r->rec.final_T.size();
    if (final_T) std::memcpy(final_T, r->rec.final_T.data(), npix * sizeof(double));
    if (n_contrib)
        for (size_t i = 0; i < npix; ++i) n_contrib[i] = r->rec.n_contrib[i];
}

// grads: per Gaussian 65 doubles in scene order (mean4, ls4, rotor8, opacity, sh48
// channel-major); vnorm: N; visible: N.
int ref_render_backward(int n, const double* mean, const double* ls, const double* rot,
                        const double* op, const double* sh, int sh_degree, const ref_camera* c,
                        const ref_records* rec, const double* dL_dimage, int threads,
                        double* grads, double* vnorm, uint8_t* visible) {
    try {
        GaussianStore store = to_store(n, mean, ls, rot, op, sh, sh_degree);
        Camera cam = to_cam(c);
        Image dl(cam.width, cam.height, 3);
        std::memcpy(dl.data.data(), dL_dimage, dl.data.size() * sizeof(double));
        StoreGrads g = render_backward(store, cam, rec->rec, dl, threads);
        for (int i = 0; i < n; ++i) {
            double* o = grads + 65 * (size_t)i;
            const GaussianParamGrad& gi = g.g[i];
            for (int a = 0; a < 4; ++a) o[a] = gi.d_mean[a];
            for (int a = 0; a < 4; ++a) o[4 + a] = gi.d_log_scales[a];
            for (int a = 0; a < 8; ++a) o[8 + a] = gi.d_rotor[a];
            o[16] = gi.d_opacity_logit;
            for (int ch = 0; ch < 3; ++ch)
                for (int k = 0; k < 16; ++k) o[17 + ch * 16 + k] = gi.d_sh(ch, k);
            vnorm[i] = g.viewspace_norm[i];
            visible[i] = g.visible[i];
        }
        return RGS_OK;
    } catch (...) {
        return map_exception();
    }
}

int ref_render_flow(int n, const double* mean, const double* ls, const double* rot,
                    const double* op, const double* sh, int sh_degree, const ref_camera* c,
                    int threads, double* flow_out) {
    try {
        GaussianStore store = to_store(n, mean, ls, rot, op, sh, sh_degree);
        Image f = render_flow(store, to_cam(c), threads);
        std::memcpy(flow_out, f.data.data(), f.data.size() * sizeof(double));
        return RGS_OK;
    } catch (...) {
        return map_exception();
    }
}

// tests/reference.hpp:77-116 (naive per-pixel renderer in global depth order).
int ref_naive_render(int n, const double* mean, const double* ls, const double* rot,
                     const double* op, const double* sh, int sh_degree, const ref_camera* c,
                     const double* bg, double* image_out, double* weight_sum, double* final_T) {
    try {
        GaussianStore store = to_store(n, mean, ls, rot, op, sh, sh_degree);
        refimpl::NaiveResult r = refimpl::naive_render(store, to_cam(c), Vec3(bg[0], bg[1], bg[2]));
        std::memcpy(image_out, r.image.data.data(), r.image.data.size() * sizeof(double));
        if (weight_sum) std::memcpy(weight_sum, r.weight_sum.data(), r.weight_sum.size() * sizeof(double));
        if (final_T) std::memcpy(final_T, r.final_T.data(), r.final_T.size() * sizeof(double));
        return RGS_OK;
    } catch (...) {
        return map_exception();
    }
}

// tests/oracles.hpp:93-101 global RNG: reseed to 20240817 (the reference's seed).
void ref_rng_reseed(unsigned long long seed) { oracle::rng().seed(seed); }
double ref_rng_uniform(double lo, double hi) { return oracle::uniform(lo, hi); }

// tests/reference.hpp:27-46, drawing from the global RNG.
void ref_random_scene(int n, int sh_degree, double* mean, double* ls, double* rot, double* op,
                      double* sh) {
    GaussianStore s = refimpl::random_scene(n, sh_degree);
    for (int i = 0; i < n; ++i) {
        Gaussian4D g = s.get(i);
        for (int a = 0; a < 4; ++a) mean[4 * i + a] = g.mean[a];
        for (int a = 0; a < 4; ++a) ls[4 * i + a] = g.log_scales[a];
        Vec8 c = g.rotor.coeffs();
        for (int a = 0; a < 8; ++a) rot[8 * i + a] = c[a];
        op[i] = g.opacity_logit;
        for (int ch = 0; ch < 3; ++ch)
            for (int k = 0; k < 16; ++k) sh[48 * i + ch * 16 + k] = g.sh(ch, k);
    }
}

// Single-Gaussian slice (gaussian.cpp:32-47).  out: mean3, cov9 (row-major),
// decay, speed3, lambda  -> 17 doubles.
int ref_slice_at(const double* mean, const double* ls, const double* rot, double t, double* out) {
    try {
        Gaussian4D g;
        for (int a = 0; a < 4; ++a) g.mean[a] = mean[a];
        for (int a = 0; a < 4; ++a) g.log_scales[a] = ls[a];
        Vec8 c;
        for (int a = 0; a < 8; ++a) c[a] = rot[a];
        g.rotor = Rotor4::from_coeffs(c);
        SlicedGaussian3D s = slice_at(g, t);
        for (int a = 0; a < 3; ++a) out[a] = s.mean[a];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) out[3 + 3 * i + j] = s.cov(i, j);
        out[12] = s.decay;
        for (int a = 0; a < 3; ++a) out[13 + a] = s.speed[a];
        out[16] = s.lambda;
        return RGS_OK;
    } catch (...) {
        return map_exception();
    }
}

// rotor.cpp:117-136 and :170-181.
int ref_normalize(const double* rot, double* out) {
    try {
        Vec8 c;
        for (int a = 0; a < 8; ++a) c[a] = rot[a];
        Vec8 n = normalize(Rotor4::from_coeffs(c)).coeffs();
        for (int a = 0; a < 8; ++a) out[a] = n[a];
        return RGS_OK;
    } catch (...) {
        return map_exception();
    }
}
int ref_to_matrix(const double* rot, double* out16) {
    try {
        Vec8 c;
        for (int a = 0; a < 8; ++a) c[a] = rot[a];
        Mat4 m = to_matrix(Rotor4::from_coeffs(c));
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j) out16[4 * i + j] = m(i, j);
        return RGS_OK;
    } catch (...) {
        return map_exception();
    }
}

// Single projection of an already-sliced Gaussian (rasterizer.cpp:215-276).
// sliced: mean3, cov9 row-major, decay, speed3 (16 doubles).  Returns 1 and fills
// *out when the splat survives, 0 when culled, <0 on error.
// The same with project()'s ProjectCache flattened as rgs_project_sliced_cache's layout
// (include/rgs_cuda.h): p_cam, T, cov2, dir, view_dist, basis, basis_grad, clamped, opacity.
int ref_project_cache(const double* sliced, const ref_camera* c, const double* sh48, int sh_degree,
                      double opacity_logit, ref_splat* out, double* pc) {
    try {
        SlicedGaussian3D s;
        s.mean = Vec3(sliced[0], sliced[1], sliced[2]);
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) s.cov(i, j) = sliced[3 + 3 * i + j];
        s.decay = sliced[12];
        s.speed = Vec3(sliced[13], sliced[14], sliced[15]);
        ShCoeffs sh;
        for (int ch = 0; ch < 3; ++ch)
            for (int k = 0; k < 16; ++k) sh(ch, k) = sh48[ch * 16 + k];
        ProjectCache cache;
        auto sp = project(s, to_cam(c), sh, sh_degree, opacity_logit, &cache);
        if (!sp) return 0;
        from_splat(*sp, out);
        for (int k = 0; k < 3; ++k) pc[k] = cache.p_cam[k];
        for (int r = 0; r < 2; ++r)
            for (int k = 0; k < 3; ++k) pc[3 + 3 * r + k] = cache.T(r, k);
        for (int r = 0; r < 2; ++r)
            for (int k = 0; k < 2; ++k) pc[9 + 2 * r + k] = cache.cov2(r, k);
        for (int k = 0; k < 3; ++k) pc[13 + k] = cache.dir[k];
        pc[16] = cache.view_dist;
        for (int k = 0; k < 16; ++k) pc[17 + k] = cache.basis[k];
        for (int k = 0; k < 16; ++k)
            for (int j = 0; j < 3; ++j) pc[33 + 3 * k + j] = cache.basis_grad(k, j);
        for (int ch = 0; ch < 3; ++ch) pc[81 + ch] = cache.clamped[ch] ? 1.0 : 0.0;
        pc[84] = cache.opacity;
        return 1;
    } catch (...) {
        return -map_exception();
    }
}

int ref_project(const double* sliced, const ref_camera* c, const double* sh48, int sh_degree,
                double opacity_logit, ref_splat* out) {
    try {
        SlicedGaussian3D s;
        s.mean = Vec3(sliced[0], sliced[1], sliced[2]);
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) s.cov(i, j) = sliced[3 + 3 * i + j];
        s.decay = sliced[12];
        s.speed = Vec3(sliced[13], sliced[14], sliced[15]);
        ShCoeffs sh;
        for (int ch = 0; ch < 3; ++ch)
            for (int k = 0; k < 16; ++k) sh(ch, k) = sh48[ch * 16 + k];
        auto sp = project(s, to_cam(c), sh, sh_degree, opacity_logit);
        if (!sp) return 0;
        from_splat(*sp, out);
        return 1;
    } catch (...) {
        return -map_exception();
    }
}

}  // extern "C"
