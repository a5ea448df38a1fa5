// The reference's own training step -- trainer.cpp's evaluate_loss, then accumulate_stats and
// adam_step in train_from's order (trainer.cpp:134-150) -- compiled unmodified against the two
// drop-ins (paper_2402_03307_b200/host/rgs_adapter.cpp for rasterizer.hpp,
// host/rgs_train_adapter.cpp for image / ssim / loss / knn / optim), so every render, image loss
// and optimizer call runs on the device through the C ABI while the store stays the
// reference's host GaussianStore.  bench.py's drop-in leg times it.  Test / bench
// infrastructure (tests/cpp/Makefile -> _build/librgs_ref_dropin.so).
#include <chrono>
#include <cstring>
#include <vector>

#include <stdexcept>

#include "rgs/dataset.hpp"
#include "rgs/optim.hpp"
#include "rgs/trainer.hpp"

using namespace rgs;

// trainer.cpp's train_from references Dataset::camera_for (dataset.cpp: JSON / PNG I/O, outside
// this path); the step below never calls train_from.
Camera Dataset::camera_for(int) const { throw std::runtime_error("drop-in harness: dataset I/O not built"); }

extern "C" {

typedef struct {
    int width, height;
    double fx, fy, cx, cy;
    double world_to_camera[16];  // row-major
    double time;
} dropin_camera;

// Store arrays in the reference's memory order (gaussian.hpp:79-85): mean/ls 4, rotor 8,
// opacity 1, sh 48 (channel-major 3 x 16) doubles per Gaussian.  targets: n_frames images of
// H*W*3 doubles.  nbrs (n * k) may be NULL (no consistency term).  Runs `steps` training steps
// from step `first_step`; losses[5] = the last step's l1, ssim, entropy, consistency, total;
// seconds[steps] = wall time of each step.
int dropin_train_steps(int n, const double* mean, const double* ls, const double* rot, const double* op,
                       const double* sh, int sh_degree, int n_frames, const dropin_camera* cams,
                       const double* targets, const int32_t* nbrs, int k, int first_step, int total_steps, int steps,
                       double* losses, double* seconds) {
    try {
        GaussianStore store;
        for (int i = 0; i < n; ++i) {
            Gaussian4D g;
            g.mean = Vec4(mean[4 * i], mean[4 * i + 1], mean[4 * i + 2], mean[4 * i + 3]);
            g.log_scales = Vec4(ls[4 * i], ls[4 * i + 1], ls[4 * i + 2], ls[4 * i + 3]);
            Vec8 r;
            for (int a = 0; a < 8; ++a) r[a] = rot[8 * i + a];
            g.rotor = Rotor4::from_coeffs(r);
            g.opacity_logit = op[i];
            for (int ch = 0; ch < 3; ++ch)
                for (int q = 0; q < 16; ++q) g.sh(ch, q) = sh[48 * i + 16 * ch + q];
            store.push_back(g);
        }
        store.active_sh_degree = sh_degree;
        std::vector<Image> imgs;
        std::vector<TrainFrame> frames(n_frames);
        size_t off = 0;
        for (int f = 0; f < n_frames; ++f) {
            Camera& c = frames[f].cam;
            c.width = cams[f].width;
            c.height = cams[f].height;
            c.fx = cams[f].fx;
            c.fy = cams[f].fy;
            c.cx = cams[f].cx;
            c.cy = cams[f].cy;
            for (int i = 0; i < 4; ++i)
                for (int j = 0; j < 4; ++j) c.world_to_camera(i, j) = cams[f].world_to_camera[4 * i + j];
            c.time = cams[f].time;
            Image im(c.width, c.height, 3);
            const size_t cnt = (size_t)c.width * c.height * 3;
            std::memcpy(im.data.data(), targets + off, cnt * sizeof(double));
            off += cnt;
            imgs.push_back(std::move(im));
        }
        for (int f = 0; f < n_frames; ++f) frames[f].target = &imgs[f];
        TrainConfig cfg;
        cfg.total_steps = total_steps;
        cfg.batch = n_frames;
        Knn4DIndex knn;
        if (nbrs) {
            knn.k = k;
            knn.store_size = n;
            knn.scene_scales = scene_scales(store);
            knn.neighbors.assign(n, std::vector<int>(k));
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < k; ++j) knn.neighbors[i][j] = nbrs[(size_t)k * i + j];
        }
        for (int s = 0; s < steps; ++s) {
            const auto t0 = std::chrono::steady_clock::now();
            StoreGrads grads;
            const LossBreakdown lb = evaluate_loss(store, frames, cfg.loss, cfg.background, nbrs ? &knn : nullptr,
                                                   1, &grads);
            accumulate_stats(store, grads);
            adam_step(store, grads, cfg, first_step + s);
            seconds[s] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            losses[0] = lb.l1;
            losses[1] = lb.ssim;
            losses[2] = lb.entropy;
            losses[3] = lb.consistency;
            losses[4] = lb.total;
        }
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

}  // extern "C"

// The same step with each part timed (seconds[10]): evaluate_loss's pieces in its order --
// [0] render_forward x views, [1] l1_loss + l1_loss_backward, [2] ssim_loss_with_grad,
// [3] dL/dimage assembly, [4] render_backward, [5] StoreGrads::add, [6] entropy (host loop +
// entropy_loss_with_grad), [7] consistency (host gaussian_speed / slice_backward loops of
// trainer.cpp + consistency_loss), [8] accumulate_stats, [9] adam_step.
#include "rgs/loss.hpp"
#include "rgs/ssim.hpp"

extern "C" int dropin_profile_step(int n, const double* mean, const double* ls, const double* rot, const double* op,
                                   const double* sh, int sh_degree, int n_frames, const dropin_camera* cams,
                                   const double* targets, const int32_t* nbrs, int k, int step, double* seconds) {
    using clk = std::chrono::steady_clock;
    auto sec = [](clk::time_point a) { return std::chrono::duration<double>(clk::now() - a).count(); };
    try {
        GaussianStore store;
        for (int i = 0; i < n; ++i) {
            Gaussian4D g;
            g.mean = Vec4(mean[4 * i], mean[4 * i + 1], mean[4 * i + 2], mean[4 * i + 3]);
            g.log_scales = Vec4(ls[4 * i], ls[4 * i + 1], ls[4 * i + 2], ls[4 * i + 3]);
            Vec8 r;
            for (int a = 0; a < 8; ++a) r[a] = rot[8 * i + a];
            g.rotor = Rotor4::from_coeffs(r);
            g.opacity_logit = op[i];
            for (int ch = 0; ch < 3; ++ch)
                for (int q = 0; q < 16; ++q) g.sh(ch, q) = sh[48 * i + 16 * ch + q];
            store.push_back(g);
        }
        store.active_sh_degree = sh_degree;
        std::vector<Image> imgs;
        std::vector<Camera> cm(n_frames);
        size_t off = 0;
        for (int f = 0; f < n_frames; ++f) {
            Camera& c = cm[f];
            c.width = cams[f].width;
            c.height = cams[f].height;
            c.fx = cams[f].fx;
            c.fy = cams[f].fy;
            c.cx = cams[f].cx;
            c.cy = cams[f].cy;
            for (int i = 0; i < 4; ++i)
                for (int j = 0; j < 4; ++j) c.world_to_camera(i, j) = cams[f].world_to_camera[4 * i + j];
            c.time = cams[f].time;
            Image im(c.width, c.height, 3);
            const size_t cnt = (size_t)c.width * c.height * 3;
            std::memcpy(im.data.data(), targets + off, cnt * sizeof(double));
            off += cnt;
            imgs.push_back(std::move(im));
        }
        TrainConfig cfg;
        // two steps on the same store: the timings are the second's (device mirrors warm, as in
        // the timed steps of dropin_train_steps)
        for (int rep = 0; rep < 2; ++rep) {
            for (int q = 0; q < 10; ++q) seconds[q] = 0;
            const LossWeights& w = cfg.loss;
            RenderOptions opts;
            opts.retain_records = true;
            StoreGrads grads;
            grads.resize(n);
            const double inv_b = 1.0 / n_frames;
            for (int f = 0; f < n_frames; ++f) {
                auto t = clk::now();
                RenderOutput ro = render_forward(store, cm[f], opts);
                seconds[0] += sec(t);
                t = clk::now();
                Image g_l1 = l1_loss_backward(ro.image, imgs[f]);
                volatile double l1 = l1_loss(ro.image, imgs[f]) * inv_b;
                (void)l1;
                seconds[1] += sec(t);
                t = clk::now();
                Image g_ssim;
                volatile double ss = ssim_loss_with_grad(ro.image, imgs[f], &g_ssim);
                (void)ss;
                seconds[2] += sec(t);
                t = clk::now();
                Image dl(ro.image.width, ro.image.height, 3);
                for (size_t i = 0; i < dl.data.size(); ++i)
                    dl.data[i] = (1 - w.lambda_ssim) * inv_b * g_l1.data[i] + w.lambda_ssim * inv_b * g_ssim.data[i];
                seconds[3] += sec(t);
                t = clk::now();
                StoreGrads fg = render_backward(store, cm[f], ro.records, dl, 1);
                seconds[4] += sec(t);
                t = clk::now();
                grads.add(fg);
                seconds[5] += sec(t);
            }
            auto t = clk::now();
            std::vector<Scalar> ops(n), g_op;
            for (int i = 0; i < n; ++i) ops[i] = store.opacity(i);
            entropy_loss_with_grad(ops, &g_op);
            for (int i = 0; i < n; ++i) grads.g[i].d_opacity_logit += w.lambda_entropy * g_op[i] * ops[i] * (1 - ops[i]);
            seconds[6] = sec(t);
            if (nbrs) {
                t = clk::now();
                Knn4DIndex knn;
                knn.k = k;
                knn.store_size = n;
                knn.neighbors.assign(n, std::vector<int>(k));
                for (int i = 0; i < n; ++i)
                    for (int j = 0; j < k; ++j) knn.neighbors[i][j] = nbrs[(size_t)k * i + j];
                std::vector<Vec3> speeds(n);
                std::vector<SliceCache> caches(n);
                for (int i = 0; i < n; ++i) speeds[i] = gaussian_speed(store.get(i), &caches[i]);
                std::vector<Vec3> g_speed;
                consistency_loss(speeds, knn, &g_speed);
                for (int i = 0; i < n; ++i)
                    slice_backward(store.get(i), caches[i], Mat3::Zero(), Vec3::Zero(), 0,
                                   w.lambda_consistency * g_speed[i], &grads.g[i]);
                seconds[7] = sec(t);
            }
            t = clk::now();
            accumulate_stats(store, grads);
            seconds[8] = sec(t);
            t = clk::now();
            adam_step(store, grads, cfg, step + rep);
            seconds[9] = sec(t);
        }
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}
