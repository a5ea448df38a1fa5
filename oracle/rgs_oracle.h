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

#ifdef __cplusplus
}
#endif
#endif
