// Shared declarations of the training-side kernels (k_train.cu) and the C-ABI host code.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "rgs_internal.cuh"

namespace rgs_dev {

constexpr int kSsimWin = 11;  // ssim.cpp:12
constexpr int kSsimTX = 32;   // tile of valid positions / pixels per block (x)
constexpr int kSsimTY = 8;    // (y); 256 threads (K8b)
constexpr int kSsimATY = 16;  // K8a tile height; 512 threads
constexpr int kSsimAThreads = kSsimTX * kSsimATY;
constexpr int kErrDegenerateTime = 7;

// dL/dimage assembly (trainer.cpp:41-50): w_l1 * l1_grad + w_ssim * ssim_grad.
struct ImageGradArgs {
    double w_l1, w_ssim;
    double inv_n;       // 1 / (3 W H)               (image.cpp:31)
    double ssim_scale;  // -1 / (3 (W-10) (H-10))    (ssim.cpp:131-134)
    int accumulate;     // dL/dimage += instead of =
    // L1 signs decided in FP64 (rgs_image_loss_ex): per pixel and channel 0 = none, else
    // sign(rendered64 - target) + 2; NULL: every sign from the FP32 image
    const int8_t* l1_sign = nullptr;
};

struct ImageLossGrid {
    int a_x, a_y, b_x, b_y, n_a, n_b;
};

// One Adam step (optim.cpp:110-157); learning rate and bias corrections computed on the
// host with the reference's std::pow.
struct AdamArgs {
    double lr_pos, lr_scales, lr_rotor, lr_sh_dc, lr_sh_rest, lr_opacity;
    double bc1, bc2;
    double lambda_entropy, inv_n;
    int static_mode;
    int stats;
};

}  // namespace rgs_dev

namespace rgs_launch {
using namespace rgs_dev;
void set_ssim_window(const double* k11, cudaStream_t s);
ImageLossGrid image_loss_grid(int W, int H);
void image_loss(const float* img, const float* tgt, int W, int H, const ImageGradArgs& a, float* dl,
                double* dfield, double* parts, double* losses, double loss_scale, int accumulate, cudaStream_t s);
void adam_step(bool f64, void* params, void* m1, void* m2, const float* grads, const float* vnorm,
               const int32_t* visible, double* accum, int32_t* count, int n, const AdamArgs& a,
               unsigned long long* err, double* part_entropy, double* losses_entropy, int accumulate,
               const unsigned long long* skip, cudaStream_t s);
int adam_blocks(int n);
// L1 near-tie re-decision (rgs_image_loss_ex): pixels with |rendered - target| <= eps in some
// channel -> list; after their FP64 recompute (blend_fp64_pixels into img64), the FP64 signs.
void l1_ties(const float* img, const float* tgt, int npix, float eps, const uint32_t* n_contrib, uint32_t* list,
             int* count, cudaStream_t s);
void l1_sign_set(const uint32_t* list, const int* count, int max_items, const double* img64, const float* tgt,
                 int8_t* sign, cudaStream_t s);
void l1_sign_clear(const uint32_t* list, const int* count, int max_items, int8_t* sign, cudaStream_t s);
void image_loss_f64(const double* img, const double* tgt, int W, int H, const ImageGradArgs& a, double* dl,
                    double* dfield, double* parts, double* losses, double loss_scale, int accumulate, cudaStream_t s);
void entropy(const double* op, int n, double* grad, double* parts, double* loss, cudaStream_t s);
void accumulate_stats(const float* vnorm, const int32_t* visible, int n, double* accum, int32_t* count,
                      cudaStream_t s);
void accumulate_stats_f64(const double* vnorm, const int32_t* visible, int n, double* accum, int32_t* count,
                          cudaStream_t s);
void reset_opacity(bool f64, void* params, void* m1, void* m2, int n, double value, cudaStream_t s);
void speeds(const float* params, const double* params64, int n, double* out, unsigned long long* err,
            cudaStream_t s);
// dL/dspeed as integer counts of consistency_unit(n, k) = inv_n inv_k (3 int per Gaussian, zeroed by
// the caller); count_to_speed turns them into doubles.
void consistency(const double* speeds, const int32_t* nbrs, int n, int k, int* dcount, double* parts,
                 double* losses_slot, int accumulate, cudaStream_t s);
double consistency_unit(int n, int k);
void count_to_speed(const int* dcount, int n, int k, double* dspeed, cudaStream_t s);
int consistency_blocks(int n);
void speed_backward(const float* params, const double* params64, int n, int k, const int* dcount, double lambda,
                    float* grads, cudaStream_t s);
void knn_points(const float* params, const double* params64, int n, const double* scales, double* pts4,
                cudaStream_t s);
int knn_grid(const double* pts4, int n, const double* queries4, const int32_t* qexcl, int nq, int k, int32_t* out,
             void* scratch, size_t scratch_bytes, cudaStream_t s);
size_t knn_grid_scratch(int n);
int extent_blocks(int n);
void mean_extent(const float* params, const double* params64, int n, double* part_lo, double* part_hi,
                 cudaStream_t s);
void densify_kind(const float* params, const double* params64, int n, const double* accum, const int32_t* count,
                  double thr, double clone_limit, uint8_t* kind, cudaStream_t s);
void densify_children(const float* params, const double* params64, int n, const int32_t* parent,
                      const uint8_t* ckind, const double* draws, const int32_t* draw_off, int n_child,
                      double log_split, int static_mode, void* ext, void* ext_m1, void* ext_m2, int ext_n,
                      unsigned long long* err, cudaStream_t s);
void gather_soa(bool f64, const void* src, int n_src, const int32_t* map, int n_map, void* dst, int n_dst,
                cudaStream_t s);
void prune_flags(const float* params, const double* params64, int n, const uint8_t* removed, double prune_opacity,
                 double big_scale, int static_mode, uint8_t* flag, cudaStream_t s);
}  // namespace rgs_launch
