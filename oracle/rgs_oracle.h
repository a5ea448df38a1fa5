/* CPU oracle for the 4D-rotor slicing + splatting hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library, and only as the
 * checker or the timed CPU baseline — never as the product path.
 *
 * A plain-C restatement (double precision, same expression order, no FMA) of
 * the reference's render path in /root/reference/proj:
 *   rotor.cpp:113-194, gaussian.cpp:9-101, sh.cpp:16-97,
 *   rasterizer.cpp:14-425, tests/reference.hpp:49-116.
 * Pinned bit-for-bit against oracle/_ref (the reference's own sources compiled
 * in place) by tests/test_oracle_vs_ref.py and the committed fixtures in
 * tests/golden/ (generated from oracle/_ref by tests/golden/make_golden.py).
 *
 * Array conventions match include/rgs_cuda.h "host scene" layout:
 *   mean[N*4], log_scales[N*4], rotor[N*8] (s,b01,b02,b03,b12,b13,b23,p),
 *   opacity_logit[N], sh[N*48] channel-major (sh[ch*16+k]).
 * Images are row-major, channel-interleaved doubles.
 */
#ifndef RGS_ORACLE_H
#define RGS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int width, height;
    double fx, fy, cx, cy;
    double world_to_camera[16]; /* row-major */
    double time;
} orc_camera;

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
} orc_splat;

typedef struct orc_records orc_records;

/* Error codes: identical to include/rgs_cuda.h. */
enum {
    ORC_OK = 0,
    ORC_E_CAMERA = 1,
    ORC_E_MISSING_RECORDS = 2,
    ORC_E_ZERO_ROTOR = 3,
    ORC_E_NONFINITE_ROTOR = 4,
    ORC_E_INVALID = 6,
    ORC_E_DEGENERATE_TIME = 7
};

const char* orc_last_error(void);

int orc_render_forward(int n, const double* mean, const double* ls, const double* rot,
                       const double* op, const double* sh, int sh_degree, const orc_camera* cam,
                       const double* bg, int threads, int retain, double* image_out,
                       orc_records** rec_out);
int orc_rasterize_forward(int n_splats, const orc_splat* splats, const orc_camera* cam,
                          const double* bg, int threads, double* image_out, orc_records** rec_out);
int orc_render_backward(int n, const double* mean, const double* ls, const double* rot,
                        const double* op, const double* sh, int sh_degree, const orc_camera* cam,
                        const orc_records* rec, const double* dL_dimage, int threads,
                        double* grads, double* vnorm, uint8_t* visible);
int orc_render_flow(int n, const double* mean, const double* ls, const double* rot,
                    const double* op, const double* sh, int sh_degree, const orc_camera* cam,
                    int threads, double* flow_out);
int orc_naive_render(int n, const double* mean, const double* ls, const double* rot,
                     const double* op, const double* sh, int sh_degree, const orc_camera* cam,
                     const double* bg, double* image_out, double* weight_sum, double* final_T);

void orc_records_free(orc_records* r);
int orc_records_num_splats(const orc_records* r);
int orc_records_num_tiles(const orc_records* r);
int orc_records_retained(const orc_records* r);
long long orc_records_num_pairs(const orc_records* r);
void orc_records_splats(const orc_records* r, orc_splat* out);
void orc_records_tiles(const orc_records* r, long long* offsets, int32_t* ids);
void orc_records_pixels(const orc_records* r, double* final_T, int32_t* n_contrib);

/* Single-Gaussian pieces. */
int orc_normalize(const double* rot, double* out);
int orc_to_matrix(const double* rot, double* out16);
int orc_slice_at(const double* mean, const double* ls, const double* rot, double t, double* out17);
int orc_project(const double* sliced16, const orc_camera* cam, const double* sh48, int sh_degree,
                double opacity_logit, orc_splat* out);

/* ---- training side; image.cpp, ssim.cpp, loss.cpp, knn.cpp,
 * optim.cpp, trainer.cpp.  65-vectors (gradients, Adam moments) are ordered mean4,
 * log_scales4, rotor8, opacity_logit, sh48 channel-major. */
typedef struct {
    double lr_position, lr_position_final, lr_scales, lr_rotor, lr_sh_dc, lr_sh_rest, lr_opacity;
    int total_steps;
    int static_mode;
} orc_adam_config; /* TrainConfig subset, optim.hpp:17-63 */

typedef struct {
    double lambda_ssim, lambda_entropy, lambda_consistency;
    int k_neighbors;
} orc_loss_weights; /* LossWeights, loss.hpp:11-16 */

double orc_psnr(long long n_values, const double* a, const double* b);
double orc_l1_loss(long long n_values, const double* rendered, const double* target, double* grad);
void orc_ssim_window(double* k11);
int orc_ssim_loss(int w, int h, const double* rendered, const double* target, double* loss, double* grad);
double orc_entropy_loss(int n, const double* opacities, double* grad);
double orc_consistency_loss(int n, const double* speeds, int k, const int32_t* nbrs, double* dspeed);
void orc_scene_scales(int n, const double* mean, double* out4);
int orc_knn4d(int n, const double* mean, int k, const double* scales, int threads, int32_t* nbrs);
int orc_gaussian_speeds(int n, const double* mean, const double* ls, const double* rot, double* speeds);
double orc_lr_schedule(int step, int total, double lr_init, double lr_final);
int orc_adam_step(int n, double* mean, double* ls, double* rot, double* op, double* sh, double* m, double* v,
                  const double* grads, const orc_adam_config* cfg, int step);
void orc_accumulate_stats(int n, const double* vnorm, const uint8_t* visible, double* accum, int32_t* count);
void orc_reset_opacity(int n, double* op, double* m_op, double* v_op, double value);
int orc_evaluate_loss(int n, const double* mean, const double* ls, const double* rot, const double* op,
                      const double* sh, int sh_degree, int n_frames, const orc_camera* cams,
                      const double* targets, const orc_loss_weights* w, const double* bg, const int32_t* nbrs,
                      int threads, double* losses, double* grads, double* vnorm, uint8_t* visible);

#ifdef __cplusplus
}
#endif
#endif
