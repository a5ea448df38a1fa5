/* rgs_cuda.h — C ABI of the B200-native 4D-rotor Gaussian slicing + splatting path.
 *
 * Drop-in boundary for the reference renderer API in /root/reference/proj/include/rgs:
 *   render_forward     rasterizer.hpp:82-83   -> rgs_render_forward / rgs_render_views
 *   rasterize_forward  rasterizer.hpp:87-89   -> rgs_rasterize_forward
 *   render_backward    rasterizer.hpp:93-95   -> rgs_render_backward
 *   render_flow        rasterizer.hpp:99      -> rgs_render_flow
 *   RenderRecords      rasterizer.hpp:61-70   -> rgs_records (opaque; rgs_records_export)
 *   GaussianStore      gaussian.hpp:79-103    -> rgs_scene   (device-resident FP32 SoA)
 *   StoreGrads         gaussian.hpp:106-119   -> grads / viewspace_norm / visible buffers
 *   Camera             camera.hpp:11-27       -> rgs_camera
 * The C++ drop-ins (paper_2402_03307_b200/host/rgs_adapter.cpp for rasterizer.hpp,
 * host/rgs_train_adapter.cpp for image / ssim / loss / knn / optim) and the Python
 * mirror (paper_2402_03307_b200/rgs.py, train.py) sit on top of exactly these symbols.
 *
 * Plain C: pointers and sizes only, no CUDA or torch types in signatures (streams
 * are passed as void*).  Every entry point returns an rgs_status; on failure
 * rgs_ctx_last_error() gives the reference's exception message.
 *
 * Precision contract:
 *   * slicing / projection / SH / culls / tile rectangles / depth keys: FP64 with
 *     the reference's expression order and no FMA contraction -> tile lists and
 *     per-tile order match the CPU reference bit for bit;
 *   * blending: FP32 with a per-evaluation error bound; any pixel whose gate
 *     decision falls inside the bound is recomputed in FP64 ("slow pixel"),
 *     so gate decisions match FP64 and the image is within 1e-4;
 *     RGS_FLAG_BLEND_FP64 forces the FP64 path for every pixel.
 */
#ifndef RGS_CUDA_H
#define RGS_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RGS_ABI_VERSION 1

typedef enum {
    RGS_OK = 0,
    RGS_E_CAMERA = 1,          /* std::runtime_error from Camera::validate (camera.hpp:21-26) */
    RGS_E_MISSING_RECORDS = 2, /* MissingRecordsError (rasterizer.hpp:78-80) */
    RGS_E_ZERO_ROTOR = 3,      /* ZeroRotorError (rotor.hpp:56-58, rotor.cpp:121) */
    RGS_E_NONFINITE_ROTOR = 4, /* NonFiniteRotorError (rotor.hpp:59-61, rotor.cpp:119,132-134) */
    RGS_E_CUDA = 5,            /* CUDA runtime failure */
    RGS_E_INVALID = 6,         /* bad argument (null pointer, size mismatch, ...) */
    RGS_E_DEGENERATE_TIME = 7, /* DegenerateTimeError escaping gaussian_speed (gaussian.hpp:31-33) */
    RGS_E_NO_DEVICE = 8,       /* no CUDA device: the product has no CPU fallback */
    RGS_E_CHECKPOINT = 9,      /* CheckpointError (checkpoint.hpp:10-12) */
    RGS_E_OVERFLOW = 10        /* a deferred-check forward outgrew its pair buffers (re-run it checked) */
} rgs_status;

/* Render flags. */
#define RGS_FLAG_RETAIN_RECORDS 1u /* RenderOptions::retain_records (rasterizer.hpp:56-60) */
#define RGS_FLAG_BLEND_FP64 2u     /* blend every pixel in FP64 (reference-KAT mode) */
#define RGS_FLAG_ACCUMULATE 4u     /* backward: add into grads (StoreGrads::add, gaussian.cpp:199) */
#define RGS_FLAG_HOST_BUFFERS 8u   /* image / splat pointers are host memory */
#define RGS_FLAG_IMAGE_F64 16u     /* image is double* (implies RGS_FLAG_BLEND_FP64): the reference's Image */
#define RGS_FLAG_DETERMINISTIC 32u /* backward: FP64, reference summation order, no atomics (bitwise reproducible) */
#define RGS_FLAG_ACCUMULATE_GRAD 64u /* rgs_image_loss: dL_dimage += instead of = */
#define RGS_FLAG_DEFER_CHECKS 128u  /* rgs_render_forward / rgs_consistency: no host synchronisation;
                                       rotor / degenerate-time errors and pair-buffer overflow are
                                       folded into the context's deferred status word
                                       (rgs_ctx_status / rgs_ctx_status_async) */
#define RGS_FLAG_REPRODUCIBLE 256u  /* backward (production FP32 path): the screen-space gradients are
                                       summed in order-independent 2 x 64-bit fixed point instead of
                                       FP64 atomics -- bitwise identical results run to run (the
                                       reference's thread invariance, rasterizer.cpp:372-384) */

typedef struct rgs_ctx rgs_ctx;
typedef struct rgs_scene rgs_scene;
typedef struct rgs_records rgs_records;

/* camera.hpp:11-27.  world_to_camera is row-major 4x4, +z forward. */
typedef struct {
    int width, height;
    double fx, fy, cx, cy;
    double world_to_camera[16];
    double time;
} rgs_camera;

/* Splat2D (rasterizer.hpp:21-30), 112 bytes. */
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
} rgs_splat;

typedef struct {
    int n_splats;      /* RenderRecords::splats.size() */
    int tiles_x, tiles_y;
    int retained;      /* RenderRecords::retained */
    long long n_pairs; /* sum over tiles of tile_splats[t].size() */
    int n_slow_pixels; /* pixels recomputed in FP64 by the guard band */
    int width, height;
} rgs_records_info;

/* ---------------------------------------------------------------- context */
int rgs_abi_version(void);
int rgs_device_count(void);
int rgs_ctx_create(int device, rgs_ctx** out);
void rgs_ctx_destroy(rgs_ctx* ctx);
/* Use `stream` (a cudaStream_t) for all subsequent work; NULL = the context's own stream. */
int rgs_ctx_set_stream(rgs_ctx* ctx, void* stream);
void* rgs_ctx_stream(rgs_ctx* ctx);
const char* rgs_ctx_last_error(const rgs_ctx* ctx);
/* Gaussian index of the last rotor error (ZeroRotor / NonFiniteRotor), -1 if none. */
int rgs_ctx_error_index(const rgs_ctx* ctx);
/* Block until the context's stream is idle. */
int rgs_ctx_synchronize(rgs_ctx* ctx);
/* Count of kernels this context launched since creation (bench evidence). */
long long rgs_ctx_kernel_launches(const rgs_ctx* ctx);

/* ---------------------------------------------------------------- binning */
/* How a view's (tile, splat) pairs are put into per-tile (depth, index) order -- the result is
 * identical (bin_and_sort, rasterizer.cpp:57-74), the cost profile differs:
 *   RGS_BINNING_RADIX:   pairs emitted in depth-rank order, then stable LSD byte passes by tile;
 *   RGS_BINNING_SCATTER: per-chunk tile counts, then every pair written at its final position
 *                        (images up to 256 x 256 and 8192 tiles; larger ones use the radix passes);
 *   RGS_BINNING_AUTO:    the scatter for single views (shorter critical path: training, drop-in),
 *                        the radix passes for the views of rgs_render_views / rgs_render_batch
 *                        (several views in flight: they overlap the other views' blends better).
 * The default comes from the environment variable RGS_BINNING=auto|radix|scatter (auto if unset). */
#define RGS_BINNING_AUTO 0
#define RGS_BINNING_RADIX 1
#define RGS_BINNING_SCATTER 2
int rgs_ctx_set_binning(rgs_ctx* ctx, int mode);

/* ---------------------------------------------------------------- profiling */
/* Per-stage CUDA-event timing on the launching stream and counting of evaluated / blended
 * (pixel, splat) pairs in the FP32 blend (count_evals != 0; the E and B of the blend roofline).
 * timing == 1: every stage, views serialised (each stage's own duration);
 * timing == 2: live -- only the FP32 blend (K5), on its stream, views still pipelined (its
 * duration inside a normal run, sharing the GPU). */
int rgs_profile_num_stages(void);
const char* rgs_profile_stage_name(int stage);
int rgs_ctx_set_profiling(rgs_ctx* ctx, int timing, int count_evals);
int rgs_ctx_profile_reset(rgs_ctx* ctx);
/* stage_ms[rgs_profile_num_stages()], stage_launches[...], evals[3] = {E, B, E_kernel}; any may be
 * NULL.  E: (pixel, splat) evaluations of the reference algorithm (every tile-list entry up
 * to each pixel's termination), B: blended pairs, E_kernel: pairs the kernel evaluated
 * after its per-warp culling. */
int rgs_ctx_profile_read(rgs_ctx* ctx, double* stage_ms, long long* stage_launches,
                         unsigned long long* evals);
/* With count_evals: the FP32 blend's slow-pixel decisions by reason since the last reset --
 * out4 = {power > 0 gate, alpha >= 1/255 gate, backward clamp gate, T(1 - alpha) < 1e-4 gate}. */
int rgs_ctx_profile_slow_reasons(rgs_ctx* ctx, unsigned long long* out4);
/* With count_evals: the FP32 blend's warp visits since the last reset -- out2 = {survivor
 * entries walked by a warp, of those the ones where at least one lane blended}. */
int rgs_ctx_profile_blend_visits(rgs_ctx* ctx, unsigned long long* out2);
/* FP32 FMA-pipe throughput of this device (FFMA probe, best of 5), TFLOP/s with FMA = 2. */
int rgs_measure_fp32_tflops(rgs_ctx* ctx, double* tflops);
/* FP64 FMA-pipe throughput of this device (DFMA probe, best of 5), TFLOP/s with FMA = 2: the
 * denominator of the FP64-bound kernels' roofline (K1 / K7b / K8). */
int rgs_measure_fp64_tflops(rgs_ctx* ctx, double* tflops);

/* ---------------------------------------------------------------- scene */
/* Device scene (GaussianStore replacement).  Host layout of the upload arrays
 * (the reference's Eigen memory order, gaussian.hpp:79-85):
 *   mean[N*4] (x,y,z,t), log_scales[N*4], rotor[N*8] (s,b01,b02,b03,b12,b13,b23,p),
 *   opacity_logit[N], sh[N*48] channel-major (sh[i*48 + ch*16 + k] = ShCoeffs(ch,k)).
 * Device storage is FP32 SoA (65 floats per Gaussian, see rgs_scene_params). */
int rgs_scene_create(rgs_ctx* ctx, int n, int sh_degree, rgs_scene** out);
/* Scene storage flags for rgs_scene_create_ex. */
#define RGS_SCENE_F64 1u /* store parameters as float64 (exact for any GaussianStore) */
/* As rgs_scene_create; RGS_SCENE_F64 keeps the 65 parameters per Gaussian in
 * float64 (same element layout, rgs_scene_params_f64) so the preprocess and the
 * parameter backward read the reference's double values unrounded. */
int rgs_scene_create_ex(rgs_ctx* ctx, int n, int sh_degree, unsigned scene_flags, rgs_scene** out);
void rgs_scene_destroy(rgs_scene* scene);
int rgs_scene_size(const rgs_scene* scene);
int rgs_scene_set_sh_degree(rgs_scene* scene, int sh_degree);
/* Host float64 arrays.  FP32 scenes round to float32 (exact for checkpoint-loaded
 * stores, checkpoint.cpp:75-82) and *n_inexact (may be NULL) receives the number of
 * coefficients that were not float32-representable; RGS_SCENE_F64 scenes store the
 * values exactly (*n_inexact = 0). */
int rgs_scene_upload_f64(rgs_ctx* ctx, rgs_scene* scene, const double* mean, const double* log_scales,
                         const double* rotor, const double* opacity_logit, const double* sh,
                         long long* n_inexact);
/* float32 arrays in the same layout; host or device pointers (cudaMemcpyDefault). */
int rgs_scene_upload_f32(rgs_ctx* ctx, rgs_scene* scene, const float* mean, const float* log_scales,
                         const float* rotor, const float* opacity_logit, const float* sh);
/* Device pointer of the SoA parameter block (65*N floats):
 *   [0,4N) mean float4, [4N,8N) log_scales float4, [8N,12N) rotor(s,b01,b02,b03) float4,
 *   [12N,16N) rotor(b12,b13,b23,p) float4, [16N,64N) sh: 12 float4 blocks, block m
 *   holding coefficients j=4m..4m+3 with j = k*3+ch, [64N,65N) opacity_logit. */
float* rgs_scene_params(rgs_scene* scene);      /* NULL for RGS_SCENE_F64 scenes */
double* rgs_scene_params_f64(rgs_scene* scene); /* NULL for FP32 scenes */
/* Copy the device scene back to host arrays in the upload layout (float64). */
int rgs_scene_download_f64(rgs_ctx* ctx, const rgs_scene* scene, double* mean, double* log_scales,
                           double* rotor, double* opacity_logit, double* sh);

/* ---------------------------------------------------------------- forward */
/* render_forward (rasterizer.cpp:308-318).  image: H*W*3 floats, row-major,
 * channel-interleaved (device memory unless RGS_FLAG_HOST_BUFFERS).
 * records may be NULL; otherwise *records receives a new handle. */
int rgs_render_forward(rgs_ctx* ctx, const rgs_scene* scene, const rgs_camera* cam,
                       const double background[3], unsigned flags, float* image,
                       rgs_records** records);
/* A batch of views (camera x timestamp sweep): images[v] = render_forward(cams[v]).
 * images: n_views*H*W*3 floats; all cameras must share width/height. */
int rgs_render_views(rgs_ctx* ctx, const rgs_scene* scene, const rgs_camera* cams, int n_views,
                     const double background[3], unsigned flags, float* images);
/* End-to-end host path: uploads the host scene (upload layout, float32), renders
 * every view, copies the images back into host memory (pinned for best speed).
 * Timed region of bench.py's "e2e" figure. */
int rgs_render_views_host(rgs_ctx* ctx, int n, int sh_degree, const float* mean,
                          const float* log_scales, const float* rotor, const float* opacity_logit,
                          const float* sh, const rgs_camera* cams, int n_views,
                          const double background[3], float* images_host);
/* rasterize_forward (rasterizer.cpp:278-306) on already-projected splats. */
int rgs_rasterize_forward(rgs_ctx* ctx, const rgs_splat* splats, int n_splats, const rgs_camera* cam,
                          const double background[3], unsigned flags, float* image,
                          rgs_records** records);
/* render_flow (rasterizer.cpp:399-425).  flow: H*W*2 floats. */
int rgs_render_flow(rgs_ctx* ctx, const rgs_scene* scene, const rgs_camera* cam, unsigned flags,
                    float* flow);

/* ---------------------------------------------------------------- records */
void rgs_records_destroy(rgs_records* rec);
int rgs_records_info_get(const rgs_records* rec, rgs_records_info* info);
/* Materialise the reference's RenderRecords on the host.  Any pointer may be NULL.
 *   splats[n_splats]          compacted splats in Gaussian-index order (rasterizer.cpp:206-210)
 *   tile_offsets[tiles+1]     CSR offsets into tile_ids
 *   tile_ids[n_pairs]         per-tile depth-sorted indices into splats (rasterizer.cpp:57-74)
 *   final_T[H*W], n_contrib[H*W]. */
int rgs_records_export(rgs_ctx* ctx, const rgs_records* rec, rgs_splat* splats,
                       long long* tile_offsets, int32_t* tile_ids, double* final_T,
                       int32_t* n_contrib);

/* ---------------------------------------------------------------- backward */
/* render_backward (rasterizer.cpp:320-397).  dL_dimage: H*W*3 floats (device; host with
 * RGS_FLAG_HOST_BUFFERS, in which case grads / viewspace_norm / visible are host too).
 * grads: 65*N floats in the rgs_scene_params layout; viewspace_norm: N floats;
 * visible: N int32 (0/1, or a count with RGS_FLAG_ACCUMULATE, so visible>0
 * reproduces StoreGrads::add's OR).  Without RGS_FLAG_ACCUMULATE the outputs are
 * overwritten; with it they are added to. */
int rgs_render_backward(rgs_ctx* ctx, const rgs_scene* scene, const rgs_camera* cam,
                        const rgs_records* records, const float* dL_dimage, unsigned flags,
                        float* grads, float* viewspace_norm, int32_t* visible);

/* project() of one already-sliced Gaussian (rasterizer.hpp:52-54, rasterizer.cpp:215-276),
 * evaluated on the device with the same FP64 code as the render path.  Host pointers:
 * sliced = mean[3], cov[9] row-major, decay, speed[3]; sh48 channel-major.  *survived = 1 and
 * *out filled (source_index = -1) when the splat passes the culls, 0 when culled. */
int rgs_project_sliced(rgs_ctx* ctx, const double* sliced16, const rgs_camera* cam, const double* sh48,
                       int sh_degree, double opacity_logit, rgs_splat* out, int* survived);
/* The same, also returning project()'s ProjectCache (rasterizer.hpp:33-48, filled as
 * rasterizer.cpp:261-275 does) when the splat survives: cache = RGS_PROJECT_CACHE_DOUBLES doubles,
 *   [0, 3) p_cam, [3, 9) T = J R_wc (2 x 3 row-major), [9, 13) cov2 (dilated, 2 x 2 row-major),
 *   [13, 16) dir, [16] view_dist, [17, 33) SH basis, [33, 81) basis gradient (16 x 3 row-major,
 *   d basis_k / d dir_j), [81, 84) clamped (1 / 0 per channel), [84] opacity (sigmoid).
 * cov3, mean3, speed and decay are the sliced input.  cache may be NULL. */
#define RGS_PROJECT_CACHE_DOUBLES 85
int rgs_project_sliced_cache(rgs_ctx* ctx, const double* sliced16, const rgs_camera* cam, const double* sh48,
                             int sh_degree, double opacity_logit, rgs_splat* out, int* survived, double* cache);

/* ---------------------------------------------------------------- utilities */
/* Device memory for FFI callers without the CUDA runtime (the C++ drop-ins use these):
 * rgs_malloc returns NULL on failure; rgs_memcpy copies in any direction (cudaMemcpyDefault)
 * on the context stream and synchronises. */
void* rgs_malloc(rgs_ctx* ctx, size_t bytes);
void rgs_free(rgs_ctx* ctx, void* ptr);
int rgs_memcpy(rgs_ctx* ctx, void* dst, const void* src, size_t bytes);
/* Camera::validate (camera.hpp:21-26) on the host; RGS_E_CAMERA with the
 * reference's message on failure. */
int rgs_camera_validate(rgs_ctx* ctx, const rgs_camera* cam);

/* ---------------------------------------------------------------- training side
 * The callers and data formats either side of the render path:
 * evaluate_loss's image gradient (trainer.cpp:22-84), adam_step + accumulate_stats
 * (optim.cpp:110-166), the entropy and consistency regularizers (loss.cpp:16-58) with
 * their 4D KNN (knn.cpp:101-116), reset_opacity (optim.cpp:236-243) and scene_scales
 * (trainer.cpp:12-20).  All device pointers; stream-ordered on the context stream. */

/* Image losses and dL/dimage (image.cpp:20-36, ssim.cpp, trainer.cpp:41-50).
 * rendered / target: H*W*3 floats.  dL_dimage (may be NULL: losses only) =
 * w_l1 * d l1_loss/d rendered + w_ssim * d ssim_loss/d rendered (FP64 arithmetic in the
 * reference's summation order, stored as float).  losses (may be NULL): [0] l1_loss,
 * [1] ssim_loss = 1 - mean SSIM, [2] MSE (psnr = min(100, 10 log10(1/MSE)), image.cpp:7-18),
 * each multiplied by loss_scale.  RGS_FLAG_ACCUMULATE adds into losses, RGS_FLAG_ACCUMULATE_GRAD
 * into dL_dimage.  Images smaller than the 11x11 window have no SSIM: losses[1] is NaN and
 * w_ssim must be 0 (else the reference's "ssim: image smaller than the 11x11 window"). */
int rgs_image_loss(rgs_ctx* ctx, const float* rendered, const float* target, int width, int height,
                   double w_l1, double w_ssim, double loss_scale, unsigned flags, float* dL_dimage,
                   double* losses);
/* rgs_image_loss with the retained records of the forward that rendered `rendered` (NULL: as
 * rgs_image_loss): the L1 gradient's sign (image.cpp:32-33, on the reference's double image) is
 * re-decided in FP64 wherever the FP32 image is within 1e-5 of the target in some channel --
 * those pixels are recomputed from the records by the FP64 blend. */
int rgs_image_loss_ex(rgs_ctx* ctx, const rgs_records* records, const float* rendered, const float* target,
                      int width, int height, double w_l1, double w_ssim, double loss_scale, unsigned flags,
                      float* dL_dimage, double* losses);

/* As rgs_image_loss on float64 images (the reference's Image type) with a float64 dL_dimage: the
 * gradient is bit-identical to the reference's l1_loss_backward / ssim_loss_with_grad mix. */
int rgs_image_loss_f64(rgs_ctx* ctx, const double* rendered, const double* target, int width, int height,
                       double w_l1, double w_ssim, double loss_scale, unsigned flags, double* dL_dimage,
                       double* losses);
/* entropy_loss_with_grad (loss.cpp:16-31) on a device array of opacities: grad (may be NULL,
 * n doubles) = dL/dopacity; loss (may be NULL, device double). */
int rgs_entropy_loss(rgs_ctx* ctx, const double* opacities, int n, double* grad, double* loss);

/* TrainConfig subset of one optimizer step (optim.hpp:17-63) + the entropy weight
 * (LossWeights::lambda_entropy, loss.hpp:12), folded into the step as trainer.cpp:55-64 does. */
typedef struct {
    double lr_position, lr_position_final, lr_scales, lr_rotor, lr_sh_dc, lr_sh_rest, lr_opacity;
    int total_steps;
    int static_mode;
    double lambda_entropy;   /* 0: no entropy term */
    int accumulate_stats;    /* 1: also accumulate_stats(vnorm, visible) (optim.cpp:159-166) */
    unsigned flags;          /* RGS_FLAG_ACCUMULATE: losses[0] += entropy instead of = */
} rgs_adam_config;

/* Adam moments and densification statistics of one scene (GaussianStore::m_*, v_*,
 * grad_accum, grad_count; gaussian.hpp:87-95), zero-initialised, in the scene's precision. */
typedef struct rgs_optimizer rgs_optimizer;
int rgs_optimizer_create(rgs_ctx* ctx, const rgs_scene* scene, rgs_optimizer** out);
void rgs_optimizer_destroy(rgs_optimizer* opt);
/* One bias-corrected Adam step (1-based `step`) over all 65 parameters, rotors
 * re-normalised, static-mode masks (optim.cpp:110-157).  grads: 65*N floats (rgs_scene_params
 * layout, e.g. rgs_render_backward with RGS_FLAG_ACCUMULATE over the batch); vnorm / visible as
 * rgs_render_backward (needed with accumulate_stats).  losses (may be NULL): [0] = entropy_loss.
 * Rotor errors are reported by rgs_optimizer_status (no host sync here).  While the context's
 * deferred status word holds an error (a RGS_FLAG_DEFER_CHECKS forward or consistency term of
 * this step failed, or outgrew its pair buffers) the step is skipped on the device: scene and
 * moments stay as they were, as when the reference throws before adam_step. */
int rgs_adam_step(rgs_ctx* ctx, rgs_scene* scene, rgs_optimizer* opt, const float* grads, const float* vnorm,
                  const int32_t* visible, const rgs_adam_config* cfg, int step, double* losses);
/* ---------------------------------------------------------------- multi-GPU
 * The batch reduction of evaluate_loss (trainer.cpp:33-53: grads and viewspace norms summed,
 * visible OR-ed, gaussian.cpp:199-209) across the ranks of a replicated-scene training job, over
 * NCCL.  NCCL is resolved at run time (the process's libnccl, else libnccl.so.2): no link
 * dependency; rgs_nccl_available() says whether it was found.  A communicator is an ncclComm_t
 * passed as void* -- made by the caller's own NCCL, or by rgs_nccl_comm_create from a 128-byte
 * ncclUniqueId that rank 0 made with rgs_nccl_unique_id and shared out of band. */
int rgs_nccl_available(void);
int rgs_nccl_unique_id(unsigned char* id128);
int rgs_nccl_comm_create(rgs_ctx* ctx, int nranks, int rank, const unsigned char* id128, void** comm);
void rgs_nccl_comm_destroy(void* comm);
/* One NCCL group (a single fused launch) on the context's stream: all-reduce(sum) in place of
 * grads_vnorm (n_floats floats: the [65 N grads | N viewspace norms] block of the accumulated
 * backward), visible (n_visible int32 counts: > 0 is the reference's OR) and losses (n_losses
 * doubles: the image-loss sums).  Any pointer may be NULL when its count is 0. */
int rgs_allreduce_grads(rgs_ctx* ctx, void* nccl_comm, float* grads_vnorm, size_t n_floats, int32_t* visible,
                        size_t n_visible, double* losses, int n_losses);

/* The context's deferred status word (RGS_FLAG_DEFER_CHECKS calls): rgs_ctx_status synchronises
 * and returns (then clears) the first error, with its index in rgs_ctx_error_index;
 * rgs_ctx_status_async queues a copy of the raw word ((index << 8) | code, ~0 when clean; an
 * overflow reports code RGS_E_OVERFLOW) into pinned host memory without synchronising. */
int rgs_ctx_status(rgs_ctx* ctx);
int rgs_ctx_status_async(rgs_ctx* ctx, unsigned long long* word);
/* Synchronises; returns the ZeroRotor / NonFiniteRotor error of the steps since the last call. */
int rgs_optimizer_status(rgs_ctx* ctx, rgs_optimizer* opt);
/* Queues (no host sync) a copy of the optimizer's error word into *word (pinned host memory):
 * ~0 when no rotor error occurred since the last rgs_optimizer_status, else (index << 8) | code.
 * Lets a training loop read step k's status while step k+1 runs; rgs_optimizer_status then
 * raises and clears a reported error. */
int rgs_optimizer_status_async(rgs_ctx* ctx, rgs_optimizer* opt, unsigned long long* word);
/* Host arrays: m65 / v65 (N, 65) rows in the order mean4, log_scales4, rotor8, opacity_logit,
 * sh48 channel-major; grad_accum N doubles; grad_count N ints.  Any may be NULL. */
int rgs_optimizer_download(rgs_ctx* ctx, const rgs_optimizer* opt, double* m65, double* v65,
                           double* grad_accum, int32_t* grad_count);
int rgs_optimizer_upload(rgs_ctx* ctx, rgs_optimizer* opt, const double* m65, const double* v65,
                         const double* grad_accum, const int32_t* grad_count);
/* accumulate_stats (optim.cpp:159-166) on its own: accum += vnorm, count += 1 where visible > 0. */
int rgs_accumulate_stats(rgs_ctx* ctx, rgs_optimizer* opt, const float* vnorm, const int32_t* visible);
/* As rgs_accumulate_stats with float64 view-space norms (the reference's StoreGrads). */
int rgs_accumulate_stats_f64(rgs_ctx* ctx, rgs_optimizer* opt, const double* vnorm, const int32_t* visible);
/* GaussianStore::reset_stats (gaussian.cpp:186-189). */
int rgs_optimizer_reset_stats(rgs_ctx* ctx, rgs_optimizer* opt);
/* reset_opacity (optim.cpp:236-243): opacity -> min(opacity, value), its moments zeroed. */
int rgs_reset_opacity(rgs_ctx* ctx, rgs_scene* scene, rgs_optimizer* opt, double value);

/* R4GS v1 checkpoint (checkpoint.hpp:14-23) straight into a new device scene: header checks
 * and error messages as load_checkpoint (checkpoint.cpp:54-86); the 65-float records are
 * staged through pinned memory and transposed to the SoA on the device.  scene_flags:
 * RGS_SCENE_F64 for FP64 storage (the values are float32 either way). */
int rgs_scene_load_checkpoint(rgs_ctx* ctx, const char* path, unsigned scene_flags, rgs_scene** out);
/* save_checkpoint (checkpoint.cpp:29-52): float32 records, byte-identical to the reference. */
int rgs_scene_save_checkpoint(rgs_ctx* ctx, const rgs_scene* scene, const char* path);

/* The train loop's generator (std::mt19937_64 seeded with TrainConfig::seed, trainer.cpp:105):
 * the batch picks (std::uniform_int_distribution<int>, trainer.cpp:106,119) and the normal
 * draws of densify_and_prune come from the same engine, as in the reference. */
typedef struct rgs_rng rgs_rng;
int rgs_rng_create(unsigned long long seed, rgs_rng** out);
void rgs_rng_destroy(rgs_rng* rng);
int rgs_rng_uniform_int(rgs_rng* rng, int lo, int hi, int* out);
/* The engine's state as text (std::mt19937_64 operator<< / >>), so a caller's own engine can be
 * handed to rgs_densify_and_prune and taken back.  get: *len = bytes needed incl. the NUL. */
int rgs_rng_get_state(const rgs_rng* rng, char* buf, size_t cap, size_t* len);
int rgs_rng_set_state(rgs_rng* rng, const char* buf);

/* TrainConfig's adaptive density control fields (optim.hpp:31-42). */
typedef struct {
    double densify_grad_threshold, percent_dense, split_factor, prune_opacity;
    int min_gaussians, max_gaussians;
    int static_mode;
} rgs_densify_config;
typedef struct {
    int cloned, split, pruned;
} rgs_densify_report; /* DensifyReport (optim.hpp:94-96) */
/* densify_and_prune (optim.cpp:168-234) on the device scene and its optimizer state: clone /
 * split decisions from the accumulated statistics, children appended in index order with the
 * generator's normal draws, prune by opacity / size / temporal extent (lowest opacities first
 * when bounded by min_gaussians), compaction, reset_stats.  The scene and optimizer are resized
 * (rgs_scene_params pointers change).  Synchronises. */
int rgs_densify_and_prune(rgs_ctx* ctx, rgs_scene* scene, rgs_optimizer* opt, const rgs_densify_config* cfg,
                          double scene_extent, rgs_rng* rng, rgs_densify_report* report);

/* scene_scales (trainer.cpp:12-20) -> host out4.  Synchronises. */
int rgs_scene_scales(rgs_ctx* ctx, const rgs_scene* scene, double* out4);
/* build_knn4d (knn.cpp:101-116): neighbors[N*k] (device int32), exact, ordered by (distance,
 * index) on mean / scales; scales = NULL uses rgs_scene_scales.  1 <= k <= 16. */
int rgs_knn_build(rgs_ctx* ctx, const rgs_scene* scene, int k, const double* scales, int32_t* neighbors);
/* KdTree4::knn (knn.cpp:60-99) for a batch of query points: the k (<= 16) nearest data points
 * of each query, ordered by (squared distance, index), skipping exclude[q] (may be NULL);
 * out[nq*k] (device), -1 where fewer than k data points exist.  points4 / queries4: device
 * arrays of 4 doubles per point. */
int rgs_knn_query(rgs_ctx* ctx, const double* points4, int n, const double* queries4, int nq, const int32_t* exclude,
                  int k, int32_t* out);
/* consistency_loss (loss.cpp:33-58) on given speeds (device, 3 doubles each) and a neighbour
 * table (device, n*k): dspeed (may be NULL, n*3) = dL/dspeed; losses (may be NULL): [0] = loss. */
int rgs_consistency_loss(rgs_ctx* ctx, const double* speeds, int n, const int32_t* neighbors, int k, double* dspeed,
                         double* losses);
/* consistency_loss (loss.cpp:33-58) over gaussian_speed (gaussian.cpp:103-110) and its
 * gradient through slice_backward (trainer.cpp:66-77): grads (may be NULL) += lambda *
 * dL/dparams; losses (may be NULL): [0] = consistency_loss (+= with RGS_FLAG_ACCUMULATE).
 * Synchronises (DegenerateTimeError / rotor errors are reported). */
int rgs_consistency(rgs_ctx* ctx, const rgs_scene* scene, const int32_t* neighbors, int k, double lambda,
                    unsigned flags, float* grads, double* losses);

#ifdef __cplusplus
}
#endif
#endif /* RGS_CUDA_H */
