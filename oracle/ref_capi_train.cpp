// C wrapper around the UNMODIFIED reference training-side sources, for oracle/_ref only.
//
// TEST INFRASTRUCTURE — never linked into the product.  Compiled in place by
// oracle/Makefile together with ref_capi.cpp.  Covers the SURVEY.md §8(e)/(f) rows that
// sit either side of the render path:
//   l1_loss / l1_loss_backward / psnr       image.cpp:7-36
//   ssim_loss_with_grad                     ssim.cpp:62-142
//   entropy_loss_with_grad                  loss.cpp:16-31
//   consistency_loss + build_knn4d          loss.cpp:33-58, knn.cpp:101-116
//   scene_scales / evaluate_loss            trainer.cpp:12-84
//   adam_step / accumulate_stats            optim.cpp:110-166
//   reset_opacity                           optim.cpp:236-243
//   save_checkpoint / load_checkpoint       checkpoint.cpp:29-86
//
// Array layouts: scene arrays as ref_capi.cpp; per-Gaussian 65-vectors (gradients, Adam
// moments) in the order mean4, log_scales4, rotor8, opacity_logit, sh48 channel-major;
// images row-major, channel-interleaved (image.hpp:15-28).
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "rgs/checkpoint.hpp"
#include "rgs/knn.hpp"
#include "rgs/loss.hpp"
#include "rgs/optim.hpp"
#include "rgs/ssim.hpp"
#include "rgs/trainer.hpp"

using namespace rgs;

// trainer.cpp's train_from references Dataset::camera_for (dataset.cpp, which needs JSON
// and PNG libraries absent here).  The oracle never calls train_from; this definition
// only satisfies the linker.
Camera Dataset::camera_for(int) const { throw std::runtime_error("oracle/_ref: dataset I/O not built"); }

extern "C" {
typedef struct {
    int width, height;
    double fx, fy, cx, cy;
    double world_to_camera[16];
    double time;
} ref_camera_t;

// TrainConfig subset used by adam_step (optim.hpp:17-63).
typedef struct {
    double lr_position, lr_position_final, lr_scales, lr_rotor, lr_sh_dc, lr_sh_rest, lr_opacity;
    int total_steps;
    int static_mode;
} ref_adam_config;

// LossWeights (loss.hpp:11-16).
typedef struct {
    double lambda_ssim, lambda_entropy, lambda_consistency;
    int k_neighbors;
} ref_loss_weights;
}

namespace {

thread_local char g_err2[512];

int fail(const std::exception& e) {
    std::snprintf(g_err2, sizeof g_err2, "%s", e.what());
    return 99;
}

Image to_image(int w, int h, const double* d) {
    Image im(w, h, 3);
    std::memcpy(im.data.data(), d, im.data.size() * sizeof(double));
    return im;
}

Camera to_cam2(const ref_camera_t* c) {
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

GaussianStore to_store2(int n, const double* mean, const double* ls, const double* rot, const double* op,
                        const double* sh, int deg) {
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

void from_store(const GaussianStore& s, double* mean, double* ls, double* rot, double* op, double* sh) {
    for (int i = 0; i < s.size(); ++i) {
        for (int a = 0; a < 4; ++a) mean[4 * i + a] = s.mean[i][a];
        for (int a = 0; a < 4; ++a) ls[4 * i + a] = s.log_scales[i][a];
        Vec8 c = s.rotor[i].coeffs();
        for (int a = 0; a < 8; ++a) rot[8 * i + a] = c[a];
        op[i] = s.opacity_logit[i];
        for (int ch = 0; ch < 3; ++ch)
            for (int k = 0; k < 16; ++k) sh[48 * i + ch * 16 + k] = s.sh[i](ch, k);
    }
}

void grads_out(const StoreGrads& g, double* grads, double* vnorm, uint8_t* visible) {
    for (int i = 0; i < g.size(); ++i) {
        double* o = grads + 65 * (size_t)i;
        const GaussianParamGrad& gi = g.g[i];
        for (int a = 0; a < 4; ++a) o[a] = gi.d_mean[a];
        for (int a = 0; a < 4; ++a) o[4 + a] = gi.d_log_scales[a];
        for (int a = 0; a < 8; ++a) o[8 + a] = gi.d_rotor[a];
        o[16] = gi.d_opacity_logit;
        for (int ch = 0; ch < 3; ++ch)
            for (int k = 0; k < 16; ++k) o[17 + ch * 16 + k] = gi.d_sh(ch, k);
        if (vnorm) vnorm[i] = g.viewspace_norm[i];
        if (visible) visible[i] = g.visible[i];
    }
}

StoreGrads grads_in(int n, const double* grads, const double* vnorm, const uint8_t* visible) {
    StoreGrads g;
    g.resize(n);
    for (int i = 0; i < n; ++i) {
        const double* o = grads + 65 * (size_t)i;
        GaussianParamGrad& gi = g.g[i];
        for (int a = 0; a < 4; ++a) gi.d_mean[a] = o[a];
        for (int a = 0; a < 4; ++a) gi.d_log_scales[a] = o[4 + a];
        for (int a = 0; a < 8; ++a) gi.d_rotor[a] = o[8 + a];
        gi.d_opacity_logit = o[16];
        for (int ch = 0; ch < 3; ++ch)
            for (int k = 0; k < 16; ++k) gi.d_sh(ch, k) = o[17 + ch * 16 + k];
        if (vnorm) g.viewspace_norm[i] = vnorm[i];
        if (visible) g.visible[i] = visible[i];
    }
    return g;
}

// Moments: 65-vectors in the gradient order.
void moments_in(GaussianStore& s, const double* m, const double* v) {
    for (int i = 0; i < s.size(); ++i) {
        const double* a = m + 65 * (size_t)i;
        const double* b = v + 65 * (size_t)i;
        for (int k = 0; k < 4; ++k) s.m_mean[i][k] = a[k], s.v_mean[i][k] = b[k];
        for (int k = 0; k < 4; ++k) s.m_ls[i][k] = a[4 + k], s.v_ls[i][k] = b[4 + k];
        for (int k = 0; k < 8; ++k) s.m_rot[i][k] = a[8 + k], s.v_rot[i][k] = b[8 + k];
        s.m_op[i] = a[16];
        s.v_op[i] = b[16];
        for (int ch = 0; ch < 3; ++ch)
            for (int k = 0; k < 16; ++k) {
                s.m_sh[i](ch, k) = a[17 + ch * 16 + k];
                s.v_sh[i](ch, k) = b[17 + ch * 16 + k];
            }
    }
}
void moments_out(const GaussianStore& s, double* m, double* v) {
    for (int i = 0; i < s.size(); ++i) {
        double* a = m + 65 * (size_t)i;
        double* b = v + 65 * (size_t)i;
        for (int k = 0; k < 4; ++k) a[k] = s.m_mean[i][k], b[k] = s.v_mean[i][k];
        for (int k = 0; k < 4; ++k) a[4 + k] = s.m_ls[i][k], b[4 + k] = s.v_ls[i][k];
        for (int k = 0; k < 8; ++k) a[8 + k] = s.m_rot[i][k], b[8 + k] = s.v_rot[i][k];
        a[16] = s.m_op[i];
        b[16] = s.v_op[i];
        for (int ch = 0; ch < 3; ++ch)
            for (int k = 0; k < 16; ++k) {
                a[17 + ch * 16 + k] = s.m_sh[i](ch, k);
                b[17 + ch * 16 + k] = s.v_sh[i](ch, k);
            }
    }
}

TrainConfig to_config(const ref_adam_config* c) {
    TrainConfig t;
    t.lr_position = c->lr_position;
    t.lr_position_final = c->lr_position_final;
    t.lr_scales = c->lr_scales;
    t.lr_rotor = c->lr_rotor;
    t.lr_sh_dc = c->lr_sh_dc;
    t.lr_sh_rest = c->lr_sh_rest;
    t.lr_opacity = c->lr_opacity;
    t.total_steps = c->total_steps;
    t.static_mode = c->static_mode != 0;
    return t;
}

Knn4DIndex to_knn(int n, int k, const int32_t* nbrs) {
    Knn4DIndex idx;
    idx.k = k;
    idx.store_size = n;
    idx.neighbors.resize(n);
    for (int i = 0; i < n; ++i) idx.neighbors[i].assign(nbrs + (size_t)k * i, nbrs + (size_t)k * (i + 1));
    return idx;
}

}  // namespace

extern "C" {

const char* ref_train_last_error(void) { return g_err2; }

// image.cpp:7-36.  grad (may be NULL) = l1_loss_backward.
int ref_l1_loss(int w, int h, const double* rendered, const double* target, double* loss, double* grad) {
    try {
        Image a = to_image(w, h, rendered), b = to_image(w, h, target);
        *loss = l1_loss(a, b);
        if (grad) {
            Image g = l1_loss_backward(a, b);
            std::memcpy(grad, g.data.data(), g.data.size() * sizeof(double));
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

double ref_psnr(int w, int h, const double* a, const double* b) {
    return psnr(to_image(w, h, a), to_image(w, h, b));
}

// ssim.cpp: 1 - mean SSIM and (grad != NULL) its gradient w.r.t. `rendered`.
int ref_ssim_loss(int w, int h, const double* rendered, const double* target, double* loss, double* grad) {
    try {
        Image a = to_image(w, h, rendered), b = to_image(w, h, target);
        if (grad) {
            Image g;
            *loss = ssim_loss_with_grad(a, b, &g);
            std::memcpy(grad, g.data.data(), g.data.size() * sizeof(double));
        } else {
            *loss = ssim_loss(a, b);
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// loss.cpp:16-31.
double ref_entropy_loss(int n, const double* opacities, double* grad) {
    std::vector<double> o(opacities, opacities + n), g;
    double v = entropy_loss_with_grad(o, grad ? &g : nullptr);
    if (grad)
        for (int i = 0; i < n; ++i) grad[i] = g[i];
    return v;
}

// trainer.cpp:12-20 -> out[4].
void ref_scene_scales(int n, const double* mean, void* out4) {
    GaussianStore s;
    for (int i = 0; i < n; ++i) {
        Gaussian4D g;
        for (int a = 0; a < 4; ++a) g.mean[a] = mean[4 * i + a];
        s.push_back(g);
    }
    Vec4 v = scene_scales(s);
    for (int a = 0; a < 4; ++a) static_cast<double*>(out4)[a] = v[a];
}

// knn.cpp:101-116: neighbors[n*k], distance-ascending, ties by index.
int ref_build_knn4d(int n, const double* mean, int k, const double* scales, int threads, int32_t* nbrs) {
    try {
        GaussianStore s;
        for (int i = 0; i < n; ++i) {
            Gaussian4D g;
            for (int a = 0; a < 4; ++a) g.mean[a] = mean[4 * i + a];
            s.push_back(g);
        }
        Knn4DIndex idx = build_knn4d(s, k, Vec4(scales[0], scales[1], scales[2], scales[3]), threads);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < k; ++j) nbrs[(size_t)k * i + j] = idx.neighbors[i][j];
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// loss.cpp:33-58.  speeds[n*3]; dspeed[n*3] may be NULL.
double ref_consistency_loss(int n, const double* speeds, int k, const int32_t* nbrs, double* dspeed) {
    std::vector<Vec3> s(n), g;
    for (int i = 0; i < n; ++i) s[i] = Vec3(speeds[3 * i], speeds[3 * i + 1], speeds[3 * i + 2]);
    Knn4DIndex idx = to_knn(n, k, nbrs);
    double v = consistency_loss(s, idx, dspeed ? &g : nullptr);
    if (dspeed)
        for (int i = 0; i < n; ++i)
            for (int a = 0; a < 3; ++a) dspeed[3 * i + a] = g[i][a];
    return v;
}

// gaussian.cpp gaussian_speed: speeds[n*3].
int ref_gaussian_speeds(int n, const double* mean, const double* ls, const double* rot, double* speeds) {
    try {
        std::vector<double> op(n, 0.0), sh(48 * (size_t)n, 0.0);
        GaussianStore s = to_store2(n, mean, ls, rot, op.data(), sh.data(), 0);
        for (int i = 0; i < n; ++i) {
            Vec3 v = gaussian_speed(s.get(i));
            for (int a = 0; a < 3; ++a) speeds[3 * i + a] = v[a];
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// trainer.cpp:22-84.  targets: n_frames images (H*W*3 each, same size as the cameras).
// nbrs may be NULL (consistency skipped, as knn == nullptr).  losses[5] = l1, ssim,
// entropy, consistency, total.  grads / vnorm / visible may be NULL (no gradients).
int ref_evaluate_loss(int n, const double* mean, const double* ls, const double* rot, const double* op,
                      const double* sh, int sh_degree, int n_frames, const ref_camera_t* cams,
                      const double* targets, const ref_loss_weights* w, const double* bg, const int32_t* nbrs,
                      int threads, double* losses, double* grads, double* vnorm, uint8_t* visible) {
    try {
        GaussianStore store = to_store2(n, mean, ls, rot, op, sh, sh_degree);
        std::vector<Image> imgs;
        std::vector<TrainFrame> frames(n_frames);
        imgs.reserve(n_frames);
        size_t off = 0;
        for (int f = 0; f < n_frames; ++f) {
            frames[f].cam = to_cam2(&cams[f]);
            imgs.push_back(to_image(cams[f].width, cams[f].height, targets + off));
            off += (size_t)cams[f].width * cams[f].height * 3;
        }
        for (int f = 0; f < n_frames; ++f) frames[f].target = &imgs[f];
        LossWeights lw;
        lw.lambda_ssim = w->lambda_ssim;
        lw.lambda_entropy = w->lambda_entropy;
        lw.lambda_consistency = w->lambda_consistency;
        lw.k_neighbors = w->k_neighbors;
        Knn4DIndex knn;
        if (nbrs) knn = to_knn(n, w->k_neighbors, nbrs);
        StoreGrads g;
        LossBreakdown lb = evaluate_loss(store, frames, lw, Vec3(bg[0], bg[1], bg[2]), nbrs ? &knn : nullptr,
                                         threads, grads ? &g : nullptr);
        losses[0] = lb.l1;
        losses[1] = lb.ssim;
        losses[2] = lb.entropy;
        losses[3] = lb.consistency;
        losses[4] = lb.total;
        if (grads) grads_out(g, grads, vnorm, visible);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// optim.cpp:159-166 on raw arrays (accum / count updated in place).
void ref_accumulate_stats(int n, const double* vnorm, const uint8_t* visible, double* accum, int32_t* count) {
    GaussianStore s;
    for (int i = 0; i < n; ++i) s.push_back(Gaussian4D{});
    for (int i = 0; i < n; ++i) {
        s.grad_accum[i] = accum[i];
        s.grad_count[i] = count[i];
    }
    StoreGrads g;
    g.resize(n);
    for (int i = 0; i < n; ++i) {
        g.viewspace_norm[i] = vnorm[i];
        g.visible[i] = visible[i];
    }
    accumulate_stats(s, g);
    for (int i = 0; i < n; ++i) {
        accum[i] = s.grad_accum[i];
        count[i] = s.grad_count[i];
    }
}

// optim.cpp:110-157: one Adam step (1-based `step`), in place on the scene arrays and
// the moments m[n*65], v[n*65].
int ref_adam_step(int n, double* mean, double* ls, double* rot, double* op, double* sh, double* m, double* v,
                  const double* grads, const ref_adam_config* cfg, int step) {
    try {
        GaussianStore s = to_store2(n, mean, ls, rot, op, sh, 0);
        moments_in(s, m, v);
        StoreGrads g = grads_in(n, grads, nullptr, nullptr);
        adam_step(s, g, to_config(cfg), step);
        from_store(s, mean, ls, rot, op, sh);
        moments_out(s, m, v);
        return 0;
    } catch (const ZeroRotorError& e) {
        std::snprintf(g_err2, sizeof g_err2, "%s", e.what());
        return 3;
    } catch (const NonFiniteRotorError& e) {
        std::snprintf(g_err2, sizeof g_err2, "%s", e.what());
        return 4;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// optim.cpp:lr_schedule
double ref_lr_schedule(int step, int total, double lr_init, double lr_final) {
    return lr_schedule(step, total, lr_init, lr_final);
}

// optim.cpp reset_opacity on raw arrays (m_op / v_op zeroed).
void ref_reset_opacity(int n, double* op, double* m_op, double* v_op, double value) {
    GaussianStore s;
    for (int i = 0; i < n; ++i) {
        Gaussian4D g;
        g.opacity_logit = op[i];
        s.push_back(g);
    }
    reset_opacity(s, value);
    for (int i = 0; i < n; ++i) {
        op[i] = s.opacity_logit[i];
        m_op[i] = s.m_op[i];
        v_op[i] = s.v_op[i];
    }
}

// checkpoint.cpp:29-86.
int ref_save_checkpoint(const char* path, int n, const double* mean, const double* ls, const double* rot,
                        const double* op, const double* sh, int sh_degree) {
    try {
        save_checkpoint(path, to_store2(n, mean, ls, rot, op, sh, sh_degree));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}
// Returns the Gaussian count (or -1); arrays may be NULL to query the size.
int ref_load_checkpoint(const char* path, double* mean, double* ls, double* rot, double* op, double* sh,
                        int* sh_degree) {
    try {
        GaussianStore s = load_checkpoint(path);
        if (sh_degree) *sh_degree = s.active_sh_degree;
        if (mean) from_store(s, mean, ls, rot, op, sh);
        return s.size();
    } catch (const std::exception& e) {
        fail(e);
        return -1;
    }
}

}  // extern "C"

extern "C" {
typedef struct {
    double densify_grad_threshold, percent_dense, split_factor, prune_opacity;
    int min_gaussians, max_gaussians;
    int static_mode;
} ref_densify_config;

// optim.cpp:168-234 with a std::mt19937_64(seed) as the train loop's generator.  Inputs are
// the store (+ moments m/v as 65-rows, grad_accum, grad_count); outputs go to arrays of
// capacity `cap` Gaussians.  Returns the new size (or -1); report3 = cloned, split, pruned.
int ref_densify_and_prune(int n, const double* mean, const double* ls, const double* rot, const double* op,
                          const double* sh, const double* m, const double* v, const double* accum,
                          const int32_t* count, const ref_densify_config* cfg, double extent,
                          unsigned long long seed, int* report3, int cap, double* mean_o, double* ls_o,
                          double* rot_o, double* op_o, double* sh_o, double* m_o, double* v_o, double* accum_o,
                          int32_t* count_o) {
    try {
        GaussianStore s = to_store2(n, mean, ls, rot, op, sh, 0);
        moments_in(s, m, v);
        for (int i = 0; i < n; ++i) {
            s.grad_accum[i] = accum[i];
            s.grad_count[i] = count[i];
        }
        TrainConfig t;
        t.densify_grad_threshold = cfg->densify_grad_threshold;
        t.percent_dense = cfg->percent_dense;
        t.split_factor = cfg->split_factor;
        t.prune_opacity = cfg->prune_opacity;
        t.min_gaussians = cfg->min_gaussians;
        t.max_gaussians = cfg->max_gaussians;
        t.static_mode = cfg->static_mode != 0;
        std::mt19937_64 rng(seed);
        DensifyReport r = densify_and_prune(s, t, extent, rng);
        report3[0] = r.cloned;
        report3[1] = r.split;
        report3[2] = r.pruned;
        if (s.size() > cap) return -1;
        from_store(s, mean_o, ls_o, rot_o, op_o, sh_o);
        moments_out(s, m_o, v_o);
        for (int i = 0; i < s.size(); ++i) {
            accum_o[i] = s.grad_accum[i];
            count_o[i] = s.grad_count[i];
        }
        return s.size();
    } catch (const std::exception& e) {
        fail(e);
        return -1;
    }
}
}
