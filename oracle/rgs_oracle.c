/* CPU oracle: plain-C restatement of the reference render path.
 *
 * TEST INFRASTRUCTURE ONLY — see rgs_oracle.h.  Only tests/, smoke() and the
 * bench CPU-baseline legs may load this; the product path never does.
 *
 * Every function follows the cited reference lines with the same double
 * precision expression order as the reference compiled against
 * include/eigen_subset (sequential-k products, no FMA: built -ffp-contract=off).
 * Pinned against oracle/_ref (the reference's own sources) bit for bit in
 * tests/test_oracle_vs_ref.py and via tests/golden/.
 */
#define _GNU_SOURCE
#include "rgs_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ errors */

static _Thread_local char g_err[256];
const char* orc_last_error(void) { return g_err; }
static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

/* ------------------------------------------------------------ constants */
/* rasterizer.hpp:13-18, gaussian.hpp:57-59, rotor.cpp:71 */
#define TILE 16
static const double kNearPlane = 0.2;
static const double kAlphaClamp = 0.99;
static const double kMinAlpha = 1.0 / 255.0;
static const double kStopT = 1e-4;
static const double kCovDilation = 0.3;
static const double kCov3Eps = 1e-9;
static const double kTemporalFloor = 1e-12;
static const double kVisibility = 16;
static const double kEpsBranch = 1e-12;

/* std::max / std::min semantics (returns first argument on ties / NaN). */
static inline double smax(double a, double b) { return (a < b) ? b : a; }
static inline double smin(double a, double b) { return (b < a) ? b : a; }

/* x86-64 cvttsd2si: out-of-range or NaN -> INT_MIN (the reference's
 * (int)std::floor(..) at rasterizer.cpp:32-35 compiles to it). */
static inline int x86_double_to_int(double v) {
    if (!(v >= -2147483648.0 && v < 2147483648.0)) return (int)0x80000000u;
    return (int)v;
}

/* ------------------------------------------------------------ thread pool */
/* parallel.hpp:24-45: static block partition, results thread-count independent. */
typedef void (*body_fn)(int i, void* ctx);
typedef struct {
    int lo, hi;
    body_fn fn;
    void* ctx;
} pf_task;
static void* pf_run(void* p) {
    pf_task* t = (pf_task*)p;
    for (int i = t->lo; i < t->hi; ++i) t->fn(i, t->ctx);
    return NULL;
}
static void parallel_for(int begin, int end, int threads, body_fn fn, void* ctx) {
    int n = end - begin;
    if (n <= 0) return;
    if (threads > n) threads = n;
    if (threads < 1) threads = 1;
    if (threads == 1) {
        for (int i = begin; i < end; ++i) fn(i, ctx);
        return;
    }
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
    pf_task* tasks = (pf_task*)malloc(sizeof(pf_task) * threads);
    int chunk = (n + threads - 1) / threads, used = 0;
    for (int w = 0; w < threads; ++w) {
        int lo = begin + w * chunk, hi = lo + chunk < end ? lo + chunk : end;
        if (lo >= hi) break;
        tasks[w] = (pf_task){lo, hi, fn, ctx};
        pthread_create(&th[w], NULL, pf_run, &tasks[w]);
        ++used;
    }
    for (int w = 0; w < used; ++w) pthread_join(th[w], NULL);
    free(th);
    free(tasks);
}

/* ------------------------------------------------------------ rotor */
/* rotor.cpp:18-51 — R4D entries as quadratic forms, row-major entry order. */
typedef struct {
    int a, b;
    double c;
} qterm;
/* ------------------------------------------------------------------ fixed-size sums
 * Reduction order of the fixed-size dot products / norms / small matrix products on the
 * forward path (the sensitivity study of tests/test_eigen_order.py builds this file three
 * ways):
 *   ORC_SUM_ORDER 0: sequential, left to right -- the Eigen subset the reference is built
 *                    against here (include/eigen_subset), and the default;
 *   ORC_SUM_ORDER 1: Eigen 3.4's completely unrolled scalar redux (redux_novec_unroller):
 *                    recursive halving, a0 + (a1 + a2), (a0 + a1) + (a2 + a3), ...;
 *   ORC_SUM_ORDER 2: Eigen 3.4's SSE2 packet redux for doubles (packets of 2): the packets
 *                    summed by halving, then the two lanes; an odd tail added last. */
#ifndef ORC_SUM_ORDER
#define ORC_SUM_ORDER 0
#endif
static double sum_halving(const double* t, int n) {
    if (n == 1) return t[0];
    const int h = n / 2;
    return sum_halving(t, h) + sum_halving(t + h, n - h);
}
static double sum_packets(const double* t, int npk, int lane) { /* lane `lane` of packets [0, npk) */
    if (npk == 1) return t[lane];
    const int h = npk / 2;
    return sum_packets(t, h, lane) + sum_packets(t + 2 * h, npk - h, lane);
}
static double sumn(const double* t, int n) {
#if ORC_SUM_ORDER == 0
    double s = t[0];
    for (int i = 1; i < n; ++i) s += t[i];
    return s;
#elif ORC_SUM_ORDER == 1
    return sum_halving(t, n);
#else
    if (n < 2) return t[0];
    const int npk = n / 2;
    double s = sum_packets(t, npk, 0) + sum_packets(t, npk, 1);
    if (n & 1) s = s + t[n - 1];
    return s;
#endif
}
static inline double dot3(double a0, double b0, double a1, double b1, double a2, double b2) {
    const double t[3] = {a0 * b0, a1 * b1, a2 * b2};
    return sumn(t, 3);
}

static const qterm kMapTerms[16][8] = {
    {{0, 0, 1}, {1, 1, -1}, {2, 2, -1}, {3, 3, -1}, {4, 4, 1}, {5, 5, 1}, {6, 6, 1}, {7, 7, -1}},
    {{1, 0, 2}, {2, 4, -2}, {3, 5, -2}, {6, 7, 2}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}},
    {{1, 4, 2}, {2, 0, 2}, {3, 6, -2}, {5, 7, -2}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}},
    {{1, 5, 2}, {2, 6, 2}, {3, 0, 2}, {4, 7, 2}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}},
    {{1, 0, -2}, {2, 4, -2}, {3, 5, -2}, {6, 7, -2}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}},
    {{0, 0, 1}, {1, 1, -1}, {2, 2, 1}, {3, 3, 1}, {4, 4, -1}, {5, 5, -1}, {6, 6, 1}, {7, 7, -1}},
    {{1, 2, -2}, {3, 7, 2}, {4, 0, 2}, {5, 6, -2}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}},
    {{1, 3, -2}, {2, 7, -2}, {4, 6, 2}, {5, 0, 2}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}},
    {{1, 4, 2}, {2, 0, -2}, {3, 6, -2}, {5, 7, 2}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}},
    {{1, 2, -2}, {3, 7, -2}, {4, 0, -2}, {5, 6, -2}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}},
    {{0, 0, 1}, {1, 1, 1}, {2, 2, -1}, {3, 3, 1}, {4, 4, -1}, {5, 5, 1}, {6, 6, -1}, {7, 7, -1}},
    {{1, 7, 2}, {2, 3, -2}, {4, 5, -2}, {6, 0, 2}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}},
    {{1, 5, 2}, {2, 6, 2}, {3, 0, -2}, {4, 7, -2}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}},
    {{1, 3, -2}, {2, 7, 2}, {4, 6, 2}, {5, 0, -2}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}},
    {{1, 7, -2}, {2, 3, -2}, {4, 5, -2}, {6, 0, -2}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}},
    {{0, 0, 1}, {1, 1, 1}, {2, 2, 1}, {3, 3, -1}, {4, 4, 1}, {5, 5, -1}, {6, 6, -1}, {7, 7, -1}},
};

/* rotor.cpp:113-115 */
static double rotor_epsilon(const double* v) {
    return v[7] * v[0] - v[1] * v[6] + v[2] * v[5] - v[3] * v[4];
}
/* rotor.cpp:54-58 */
static void epsilon_gradient(const double* v, double* g) {
    g[0] = v[7];
    g[1] = -v[6];
    g[2] = v[5];
    g[3] = -v[4];
    g[4] = -v[3];
    g[5] = v[2];
    g[6] = -v[1];
    g[7] = v[0];
}
static double sqnorm8(const double* v) {
    double t[8];
    for (int i = 0; i < 8; ++i) t[i] = v[i] * v[i];
    return sumn(t, 8);
}

/* rotor.cpp:117-136.  Returns ORC_OK or an error code. */
static int rotor_normalize(const double* in, double* v) {
    for (int i = 0; i < 8; ++i) {
        v[i] = in[i];
        if (!isfinite(v[i])) return ORC_E_NONFINITE_ROTOR;
    }
    double l2 = sqnorm8(v);
    if (!(l2 > 1e-20)) return ORC_E_ZERO_ROTOR;
    double eps = rotor_epsilon(v);
    if (fabs(eps) >= kEpsBranch) {
        double rad = smax(l2 * l2 - 4 * eps * eps, 0.0);
        double delta = -2 * eps / (l2 + sqrt(rad));
        double g[8];
        epsilon_gradient(v, g);
        for (int i = 0; i < 8; ++i) v[i] = v[i] + delta * g[i];
    }
    double nrm = sqrt(sqnorm8(v));
    for (int i = 0; i < 8; ++i) v[i] = v[i] / nrm;
    for (int i = 0; i < 8; ++i)
        if (!isfinite(v[i])) return ORC_E_NONFINITE_ROTOR;
    if (fabs(rotor_epsilon(v)) > 1e-9 || fabs(sqnorm8(v) - 1) > 1e-9) return ORC_E_NONFINITE_ROTOR;
    return ORC_OK;
}

/* rotor.cpp:170-181 (the NotNormalized guard is unreachable after normalize). */
static void rotor_to_matrix(const double* v, double* m /* 4x4 row-major */) {
    for (int e = 0; e < 16; ++e) {
        double val = 0;
        for (int t = 0; t < 8; ++t) {
            const qterm* q = &kMapTerms[e][t];
            val += q->c * v[q->a] * v[q->b];
        }
        m[e] = val;
    }
}

/* rotor.cpp:183-194, 16x8 row-major. */
static void to_matrix_jacobian(const double* v, double* j) {
    memset(j, 0, sizeof(double) * 128);
    for (int e = 0; e < 16; ++e)
        for (int t = 0; t < 8; ++t) {
            const qterm* q = &kMapTerms[e][t];
            if (q->c == 0) continue;
            j[e * 8 + q->a] += q->c * v[q->b];
            j[e * 8 + q->b] += q->c * v[q->a];
        }
}

/* rotor.cpp:138-168, 8x8 row-major (Jn = j2 * j1). */
static void normalize_jacobian(const double* v, double* out) {
    double l2 = sqnorm8(v);
    double eps = rotor_epsilon(v);
    double grad[8], j1[64], updated[8];
    epsilon_gradient(v, grad);
    for (int i = 0; i < 8; ++i) updated[i] = v[i];
    if (fabs(eps) >= kEpsBranch) {
        double rad = smax(l2 * l2 - 4 * eps * eps, 0.0);
        double sq = smax(sqrt(rad), 1e-30);
        double den = l2 + sq;
        double delta = -2 * eps / den;
        double ddelta_deps = -2 / den - 8 * eps * eps / (sq * den * den);
        double ddelta_dl2 = 2 * eps * (1 + l2 / sq) / (den * den);
        double ddr[8];
        for (int i = 0; i < 8; ++i) ddr[i] = ddelta_deps * grad[i] + ddelta_dl2 * 2 * v[i];
        for (int i = 0; i < 8; ++i) updated[i] = v[i] + delta * grad[i];
        /* epsilon_hessian, rotor.cpp:62-69 */
        double h[64];
        memset(h, 0, sizeof h);
        h[0 * 8 + 7] = h[7 * 8 + 0] = 1;
        h[1 * 8 + 6] = h[6 * 8 + 1] = -1;
        h[2 * 8 + 5] = h[5 * 8 + 2] = 1;
        h[3 * 8 + 4] = h[4 * 8 + 3] = -1;
        for (int i = 0; i < 8; ++i)
            for (int k = 0; k < 8; ++k)
                j1[i * 8 + k] = ((i == k ? 1.0 : 0.0) + grad[i] * ddr[k]) + delta * h[i * 8 + k];
    } else {
        for (int i = 0; i < 8; ++i)
            for (int k = 0; k < 8; ++k)
                j1[i * 8 + k] = (i == k ? 1.0 : 0.0) - (grad[i] * grad[k]) / l2;
    }
    double len = sqrt(sqnorm8(updated));
    double u[8], j2[64];
    for (int i = 0; i < 8; ++i) u[i] = updated[i] / len;
    for (int i = 0; i < 8; ++i)
        for (int k = 0; k < 8; ++k) j2[i * 8 + k] = ((i == k ? 1.0 : 0.0) - u[i] * u[k]) / len;
    for (int i = 0; i < 8; ++i)
        for (int k = 0; k < 8; ++k) {
            double s = j2[i * 8 + 0] * j1[0 * 8 + k];
            for (int m = 1; m < 8; ++m) s += j2[i * 8 + m] * j1[m * 8 + k];
            out[i * 8 + k] = s;
        }
}

/* ------------------------------------------------------------ slicing */
/* gaussian.hpp:36-45 SliceCache */
typedef struct {
    double normalized[8];
    double R[16];
    double q[4];
    double U[9];
    double V[3];
    double W;
    double dt;
    double decay;
} slice_cache;

typedef struct {
    double mean[3];
    double cov[9];
    double decay;
    double speed[3];
    double lambda;
} sliced3;

/* gaussian.cpp:9-17 */
static int assemble_cache(const double* ls, const double* rot, slice_cache* c) {
    int rc = rotor_normalize(rot, c->normalized);
    if (rc) return rc;
    rotor_to_matrix(c->normalized, c->R);
    for (int k = 0; k < 4; ++k) c->q[k] = exp(2 * ls[k]);
    /* sigma = (R * diag(q)) * R^T, sequential k */
    double m1[16], sig[16];
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) m1[i * 4 + j] = c->R[i * 4 + j] * c->q[j];
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
            double t[4];
            for (int k = 0; k < 4; ++k) t[k] = m1[i * 4 + k] * c->R[j * 4 + k];
            sig[i * 4 + j] = sumn(t, 4);
        }
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) c->U[i * 3 + j] = sig[i * 4 + j];
    for (int i = 0; i < 3; ++i) c->V[i] = sig[i * 4 + 3];
    c->W = sig[15];
    return ORC_OK;
}

/* gaussian.cpp:32-47 */
static int slice_at(const double* mean, const double* ls, const double* rot, double t, sliced3* out,
                    slice_cache* c) {
    int rc = assemble_cache(ls, rot, c);
    if (rc) return rc;
    if (c->W < kTemporalFloor) return ORC_E_DEGENERATE_TIME;
    c->dt = t - mean[3];
    out->lambda = 1 / c->W;
    for (int i = 0; i < 3; ++i) out->speed[i] = c->V[i] / c->W;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double b = (c->V[i] * c->V[j]) / c->W;
            double d = kCov3Eps * (i == j ? 1.0 : 0.0);
            out->cov[i * 3 + j] = (c->U[i * 3 + j] - b) + d;
        }
    for (int i = 0; i < 3; ++i) out->mean[i] = mean[i] + c->dt * out->speed[i];
    out->decay = exp(-0.5 * out->lambda * c->dt * c->dt);
    c->decay = out->decay;
    return ORC_OK;
}

/* ------------------------------------------------------------ SH */
/* sh.cpp:6-12 */
static const double C0 = 0.28209479177387814;
static const double C1 = 0.4886025119029199;
static const double C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                             -1.0925484305920792, 0.5462742152960396};
static const double C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                             0.3731763325901154,  -0.4570457994644658, 1.445305721320277,
                             -0.5900435899266435};

/* sh.cpp:16-85; grad is 16x3 row-major (may be NULL). */
static void sh_basis(const double* dir, int degree, double* b, double* grad) {
    const double x = dir[0], y = dir[1], z = dir[2];
    memset(b, 0, sizeof(double) * 16);
    if (grad) memset(grad, 0, sizeof(double) * 48);
#define G(k, a) grad[(k) * 3 + (a)]
    b[0] = C0;
    if (degree >= 1) {
        b[1] = -C1 * y;
        b[2] = C1 * z;
        b[3] = -C1 * x;
        if (grad) {
            G(1, 1) = -C1;
            G(2, 2) = C1;
            G(3, 0) = -C1;
        }
    }
    if (degree >= 2) {
        const double xx = x * x, yy = y * y, zz = z * z;
        b[4] = C2[0] * x * y;
        b[5] = C2[1] * y * z;
        b[6] = C2[2] * (2 * zz - xx - yy);
        b[7] = C2[3] * x * z;
        b[8] = C2[4] * (xx - yy);
        if (grad) {
            G(4, 0) = C2[0] * y;
            G(4, 1) = C2[0] * x;
            G(5, 1) = C2[1] * z;
            G(5, 2) = C2[1] * y;
            G(6, 0) = C2[2] * -2 * x;
            G(6, 1) = C2[2] * -2 * y;
            G(6, 2) = C2[2] * 4 * z;
            G(7, 0) = C2[3] * z;
            G(7, 2) = C2[3] * x;
            G(8, 0) = C2[4] * 2 * x;
            G(8, 1) = C2[4] * -2 * y;
        }
    }
    if (degree >= 3) {
        const double xx = x * x, yy = y * y, zz = z * z;
        b[9] = C3[0] * y * (3 * xx - yy);
        b[10] = C3[1] * x * y * z;
        b[11] = C3[2] * y * (4 * zz - xx - yy);
        b[12] = C3[3] * z * (2 * zz - 3 * xx - 3 * yy);
        b[13] = C3[4] * x * (4 * zz - xx - yy);
        b[14] = C3[5] * z * (xx - yy);
        b[15] = C3[6] * x * (xx - 3 * yy);
        if (grad) {
            G(9, 0) = C3[0] * 6 * x * y;
            G(9, 1) = C3[0] * (3 * xx - 3 * yy);
            G(10, 0) = C3[1] * y * z;
            G(10, 1) = C3[1] * x * z;
            G(10, 2) = C3[1] * x * y;
            G(11, 0) = C3[2] * -2 * x * y;
            G(11, 1) = C3[2] * (4 * zz - xx - 3 * yy);
            G(11, 2) = C3[2] * 8 * y * z;
            G(12, 0) = C3[3] * -6 * x * z;
            G(12, 1) = C3[3] * -6 * y * z;
            G(12, 2) = C3[3] * (6 * zz - 3 * xx - 3 * yy);
            G(13, 0) = C3[4] * (4 * zz - 3 * xx - yy);
            G(13, 1) = C3[4] * -2 * x * y;
            G(13, 2) = C3[4] * 8 * x * z;
            G(14, 0) = C3[5] * 2 * x * z;
            G(14, 1) = C3[5] * -2 * y * z;
            G(14, 2) = C3[5] * (xx - yy);
            G(15, 0) = C3[6] * (3 * xx - 3 * yy);
            G(15, 1) = C3[6] * -6 * x * y;
        }
    }
#undef G
}

/* ------------------------------------------------------------ projection */
/* rasterizer.hpp:33-48 ProjectCache */
typedef struct {
    slice_cache slice;
    double cov3[9];
    double mean3[3];
    double speed[3];
    double decay;
    double p_cam[3];
    double T[6]; /* 2x3 row-major */
    double cov2[4];
    double dir[3];
    double view_dist;
    double basis[16];
    double basis_grad[48];
    int clamped[3];
    double opacity;
} project_cache;

static void cam_rotation(const orc_camera* cam, double* r) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r[i * 3 + j] = cam->world_to_camera[i * 4 + j];
}
static void cam_translation(const orc_camera* cam, double* t) {
    for (int i = 0; i < 3; ++i) t[i] = cam->world_to_camera[i * 4 + 3];
}
/* camera.hpp:17: center = -R^T t */
static void cam_center(const orc_camera* cam, double* c) {
    double r[9], t[3];
    cam_rotation(cam, r);
    cam_translation(cam, t);
    for (int i = 0; i < 3; ++i) c[i] = dot3(-r[0 * 3 + i], t[0], -r[1 * 3 + i], t[1], -r[2 * 3 + i], t[2]);
}
/* camera.hpp:19-24 */
static int cam_validate(const orc_camera* cam) {
    if (!(cam->fx > 0) || !(cam->fy > 0))
        return fail(ORC_E_CAMERA, "camera: focal lengths must be positive");
    double r[9], mx = 0;
    cam_rotation(cam, r);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = r[i * 3 + 0] * r[j * 3 + 0];
            s += r[i * 3 + 1] * r[j * 3 + 1];
            s += r[i * 3 + 2] * r[j * 3 + 2];
            double d = fabs(s - (i == j ? 1.0 : 0.0));
            if (i == 0 && j == 0)
                mx = d;
            else
                mx = smax(mx, d);
        }
    if (mx > 1e-6) return fail(ORC_E_CAMERA, "camera: rotation block not orthogonal");
    return ORC_OK;
}

/* rasterizer.cpp:14-20 */
static void projection_jacobian(const orc_camera* cam, const double* p, double* j) {
    const double z = p[2], z2 = z * z;
    j[0] = cam->fx / z;
    j[1] = 0;
    j[2] = -cam->fx * p[0] / z2;
    j[3] = 0;
    j[4] = cam->fy / z;
    j[5] = -cam->fy * p[1] / z2;
}

static double sigmoid(double x) { return 1 / (1 + exp(-x)); }

/* rasterizer.cpp:215-276.  Returns 1 if the splat survives, 0 if culled. */
static int project(const sliced3* s, const orc_camera* cam, const double* sh48, int sh_degree,
                   double opacity_logit, orc_splat* out, project_cache* cache) {
    double R[9], t[3];
    cam_rotation(cam, R);
    cam_translation(cam, t);
    double p[3];
    for (int i = 0; i < 3; ++i)
        p[i] = dot3(R[i * 3 + 0], s->mean[0], R[i * 3 + 1], s->mean[1], R[i * 3 + 2], s->mean[2]) + t[i];
    if (p[2] <= kNearPlane) return 0;

    memset(out, 0, sizeof *out);
    out->depth = p[2];
    out->mean2[0] = cam->fx * p[0] / p[2] + cam->cx;
    out->mean2[1] = cam->fy * p[1] / p[2] + cam->cy;

    double J[6], T[6];
    projection_jacobian(cam, p, J);
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j)
            T[i * 3 + j] = dot3(J[i * 3 + 0], R[0 * 3 + j], J[i * 3 + 1], R[1 * 3 + j], J[i * 3 + 2], R[2 * 3 + j]);
    double A[6], cov2[4];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j)
            A[i * 3 + j] = dot3(T[i * 3 + 0], s->cov[0 * 3 + j], T[i * 3 + 1], s->cov[1 * 3 + j], T[i * 3 + 2],
                                s->cov[2 * 3 + j]);
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j)
            cov2[i * 2 + j] = dot3(A[i * 3 + 0], T[j * 3 + 0], A[i * 3 + 1], T[j * 3 + 1], A[i * 3 + 2], T[j * 3 + 2]) +
                              kCovDilation * (i == j ? 1.0 : 0.0);
    double det = cov2[0] * cov2[3] - cov2[2] * cov2[1];
    if (det <= 0) return 0;
    double invdet = 1.0 / (cov2[0] * cov2[3] - cov2[2] * cov2[1]);
    out->conic[0] = cov2[3] * invdet;
    out->conic[1] = -cov2[1] * invdet;
    out->conic[2] = cov2[0] * invdet;

    double mid = 0.5 * (cov2[0] + cov2[3]);
    double max_eig = mid + sqrt(smax(0.01, mid * mid - det));
    out->radius = 3 * sqrt(max_eig);
    if (out->mean2[0] + out->radius < 0 || out->mean2[0] - out->radius > cam->width - 1 ||
        out->mean2[1] + out->radius < 0 || out->mean2[1] - out->radius > cam->height - 1)
        return 0;

    double opacity = sigmoid(opacity_logit);
    out->alpha_base = opacity * s->decay;
    if (out->alpha_base < kMinAlpha) return 0;

    double ctr[3], v[3];
    cam_center(cam, ctr);
    for (int i = 0; i < 3; ++i) v[i] = s->mean[i] - ctr[i];
    double dist = sqrt(dot3(v[0], v[0], v[1], v[1], v[2], v[2]));
    double dir[3];
    if (dist > 0) {
        for (int i = 0; i < 3; ++i) dir[i] = v[i] / dist;
    } else {
        dir[0] = 0;
        dir[1] = 0;
        dir[2] = 1;
    }
    double basis[16], bgrad[48];
    sh_basis(dir, sh_degree, basis, cache ? bgrad : NULL);
    int clamped[3];
    for (int ch = 0; ch < 3; ++ch) {
        const double* row = sh48 + ch * 16;
        double tt[16];
        for (int k = 0; k < 16; ++k) tt[k] = row[k] * basis[k];
        double col = sumn(tt, 16) + 0.5;
        clamped[ch] = col < 0;
        if (clamped[ch]) col = 0;
        out->color[ch] = col;
    }
    for (int i = 0; i < 2; ++i)
        out->flow2[i] = dot3(T[i * 3 + 0], s->speed[0], T[i * 3 + 1], s->speed[1], T[i * 3 + 2], s->speed[2]);
    if (cache) {
        memcpy(cache->cov3, s->cov, sizeof cache->cov3);
        memcpy(cache->mean3, s->mean, sizeof cache->mean3);
        memcpy(cache->speed, s->speed, sizeof cache->speed);
        cache->decay = s->decay;
        memcpy(cache->p_cam, p, sizeof p);
        memcpy(cache->T, T, sizeof T);
        memcpy(cache->cov2, cov2, sizeof cov2);
        memcpy(cache->dir, dir, sizeof dir);
        cache->view_dist = dist;
        memcpy(cache->basis, basis, sizeof basis);
        memcpy(cache->basis_grad, bgrad, sizeof bgrad);
        for (int ch = 0; ch < 3; ++ch) cache->clamped[ch] = clamped[ch];
        cache->opacity = opacity;
    }
    return 1;
}

/* ------------------------------------------------------------ build_splats */
typedef struct {
    int n, sh_degree;
    const double *mean, *ls, *rot, *op, *sh;
    const orc_camera* cam;
    orc_splat* tmp;
    unsigned char* ok;
    int* err; /* per Gaussian error code */
} build_ctx;

/* One Gaussian of rasterizer.cpp:189-204 (slice, visibility gate, project). */
static int slice_and_project(const build_ctx* b, int i, orc_splat* out, project_cache* pc) {
    sliced3 s;
    slice_cache local;
    slice_cache* sc = pc ? &pc->slice : &local;
    int rc = slice_at(b->mean + 4 * i, b->ls + 4 * i, b->rot + 8 * i, b->cam->time, &s, sc);
    if (rc == ORC_E_DEGENERATE_TIME) return 0; /* caught: skipped (rasterizer.cpp:194-198) */
    if (rc) return -rc;                        /* rotor errors propagate */
    double dt = b->cam->time - b->mean[4 * i + 3];
    if (s.lambda * dt * dt > kVisibility) return 0;
    if (!project(&s, b->cam, b->sh + 48 * i, b->sh_degree, b->op[i], out, pc)) return 0;
    out->source_index = i;
    return 1;
}

static void build_body(int i, void* p) {
    build_ctx* b = (build_ctx*)p;
    int r = slice_and_project(b, i, &b->tmp[i], NULL);
    b->ok[i] = r > 0;
    b->err[i] = r < 0 ? -r : 0;
}

/* rasterizer.cpp:184-211: parallel slice+project, compaction in index order. */
static int build_splats(const build_ctx* proto, int threads, orc_splat** splats_out, int* count) {
    build_ctx b = *proto;
    b.tmp = (orc_splat*)malloc(sizeof(orc_splat) * (b.n > 0 ? b.n : 1));
    b.ok = (unsigned char*)calloc(b.n > 0 ? b.n : 1, 1);
    b.err = (int*)calloc(b.n > 0 ? b.n : 1, sizeof(int));
    parallel_for(0, b.n, threads, build_body, &b);
    int rc = ORC_OK;
    for (int i = 0; i < b.n; ++i)
        if (b.err[i]) {
            rc = b.err[i];
            break;
        }
    int m = 0;
    for (int i = 0; i < b.n; ++i)
        if (b.ok[i]) b.tmp[m++] = b.tmp[i];
    free(b.ok);
    free(b.err);
    if (rc) {
        free(b.tmp);
        return fail(rc, rc == ORC_E_ZERO_ROTOR ? "normalize: zero rotor"
                                               : "normalize: result violates rotor invariants");
    }
    *splats_out = b.tmp;
    *count = m;
    return ORC_OK;
}

/* ------------------------------------------------------------ binning */
struct orc_records {
    orc_splat* splats;
    int n_splats;
    int tiles_x, tiles_y;
    long long* offsets; /* tiles + 1 */
    int32_t* ids;
    double* final_T;
    int32_t* n_contrib;
    int width, height;
    double background[3];
    int retained;
};

/* rasterizer.cpp:26-38 */
static int tile_range(const orc_splat* s, int tiles_x, int tiles_y, int* x0, int* x1, int* y0,
                      int* y1) {
    int a;
    a = x86_double_to_int(floor((s->mean2[0] - s->radius) / TILE));
    *x0 = a > 0 ? a : 0;
    a = x86_double_to_int(floor((s->mean2[0] + s->radius) / TILE));
    *x1 = a < tiles_x - 1 ? a : tiles_x - 1;
    a = x86_double_to_int(floor((s->mean2[1] - s->radius) / TILE));
    *y0 = a > 0 ? a : 0;
    a = x86_double_to_int(floor((s->mean2[1] + s->radius) / TILE));
    *y1 = a < tiles_y - 1 ? a : tiles_y - 1;
    return *x0 <= *x1 && *y0 <= *y1;
}

static const orc_splat* g_sort_splats; /* qsort context (per-call, guarded below) */
typedef struct {
    const orc_splat* splats;
    const long long* offsets;
    int32_t* ids;
} sort_ctx;

/* Depth, then source index (rasterizer.cpp:68-71); a strict total order, so the
 * result equals std::sort's. */
static void sort_tile(int32_t* a, long long n, const orc_splat* sp) {
    /* insertion-merge sort: stable and allocation-free for the small lists;
     * bottom-up merge for large ones. */
    if (n < 2) return;
    if (n <= 32) {
        for (long long i = 1; i < n; ++i) {
            int32_t v = a[i];
            long long j = i - 1;
            while (j >= 0) {
                const orc_splat *x = &sp[a[j]], *y = &sp[v];
                int gt = x->depth != y->depth ? x->depth > y->depth
                                               : x->source_index > y->source_index;
                if (!gt) break;
                a[j + 1] = a[j];
                --j;
            }
            a[j + 1] = v;
        }
        return;
    }
    int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * n);
    for (long long w = 1; w < n; w *= 2) {
        for (long long lo = 0; lo < n; lo += 2 * w) {
            long long mid = lo + w < n ? lo + w : n, hi = lo + 2 * w < n ? lo + 2 * w : n;
            long long i = lo, j = mid, k = lo;
            while (i < mid && j < hi) {
                const orc_splat *x = &sp[a[i]], *y = &sp[a[j]];
                int take_right = x->depth != y->depth ? y->depth < x->depth
                                                       : y->source_index < x->source_index;
                tmp[k++] = take_right ? a[j++] : a[i++];
            }
            while (i < mid) tmp[k++] = a[i++];
            while (j < hi) tmp[k++] = a[j++];
        }
        memcpy(a, tmp, sizeof(int32_t) * n);
    }
    free(tmp);
}
static void sort_body(int t, void* p) {
    sort_ctx* c = (sort_ctx*)p;
    sort_tile(c->ids + c->offsets[t], c->offsets[t + 1] - c->offsets[t], c->splats);
}

/* rasterizer.cpp:57-74: serial binning in splat order, per-tile depth sort. */
static void bin_and_sort(orc_records* r, int threads) {
    int ntiles = r->tiles_x * r->tiles_y;
    long long* counts = (long long*)calloc(ntiles + 1, sizeof(long long));
    for (int i = 0; i < r->n_splats; ++i) {
        int x0, x1, y0, y1;
        if (!tile_range(&r->splats[i], r->tiles_x, r->tiles_y, &x0, &x1, &y0, &y1)) continue;
        for (int ty = y0; ty <= y1; ++ty)
            for (int tx = x0; tx <= x1; ++tx) counts[(long long)ty * r->tiles_x + tx]++;
    }
    r->offsets = (long long*)malloc(sizeof(long long) * (ntiles + 1));
    long long acc = 0;
    for (int t = 0; t < ntiles; ++t) {
        r->offsets[t] = acc;
        acc += counts[t];
    }
    r->offsets[ntiles] = acc;
    r->ids = (int32_t*)malloc(sizeof(int32_t) * (acc > 0 ? acc : 1));
    for (int t = 0; t < ntiles; ++t) counts[t] = r->offsets[t];
    for (int i = 0; i < r->n_splats; ++i) {
        int x0, x1, y0, y1;
        if (!tile_range(&r->splats[i], r->tiles_x, r->tiles_y, &x0, &x1, &y0, &y1)) continue;
        for (int ty = y0; ty <= y1; ++ty)
            for (int tx = x0; tx <= x1; ++tx) r->ids[counts[(long long)ty * r->tiles_x + tx]++] = i;
    }
    free(counts);
    sort_ctx c = {r->splats, r->offsets, r->ids};
    parallel_for(0, ntiles, threads, sort_body, &c);
}

/* ------------------------------------------------------------ blending */
typedef struct {
    const orc_records* r;
    const double* payload; /* 3 per splat */
    double bg[3];
    int channels;
    double* image;
    double* final_T;
    int32_t* n_contrib;
} blend_ctx;

typedef struct {
    double mx, my, ca, cb, cc, alpha_base;
    double payload[3];
} tile_splat;

/* rasterizer.cpp:77-123 */
static void blend_tile(int t, void* p) {
    blend_ctx* c = (blend_ctx*)p;
    const orc_records* r = c->r;
    int tile_x = t % r->tiles_x, tile_y = t / r->tiles_x;
    int px0 = tile_x * TILE, py0 = tile_y * TILE;
    int px1 = px0 + TILE < r->width ? px0 + TILE : r->width;
    int py1 = py0 + TILE < r->height ? py0 + TILE : r->height;
    long long n = r->offsets[t + 1] - r->offsets[t];
    tile_splat* local = (tile_splat*)malloc(sizeof(tile_splat) * (n > 0 ? n : 1));
    for (long long k = 0; k < n; ++k) {
        int id = r->ids[r->offsets[t] + k];
        const orc_splat* s = &r->splats[id];
        local[k] = (tile_splat){s->mean2[0], s->mean2[1], s->conic[0], s->conic[1], s->conic[2],
                                s->alpha_base, {c->payload[3 * id], c->payload[3 * id + 1],
                                                c->payload[3 * id + 2]}};
    }
    for (int y = py0; y < py1; ++y)
        for (int x = px0; x < px1; ++x) {
            double T = 1, acc[3] = {0, 0, 0};
            int contrib = 0;
            for (long long pos = 0; pos < n; ++pos) {
                const tile_splat* s = &local[pos];
                double dx = x - s->mx, dy = y - s->my;
                double power = -0.5 * (s->ca * dx * dx + s->cc * dy * dy) - s->cb * dx * dy;
                if (power > 0) continue;
                double a = smin(kAlphaClamp, s->alpha_base * exp(power));
                if (a < kMinAlpha) continue;
                double test_T = T * (1 - a);
                if (test_T < kStopT) break;
                double w = a * T;
                for (int ch = 0; ch < 3; ++ch) acc[ch] = acc[ch] + s->payload[ch] * w;
                T = test_T;
                contrib = (int)pos + 1;
            }
            for (int ch = 0; ch < 3; ++ch) acc[ch] = acc[ch] + T * c->bg[ch];
            size_t pix = (size_t)y * r->width + x;
            for (int ch = 0; ch < c->channels; ++ch) c->image[pix * c->channels + ch] = acc[ch];
            if (c->final_T) c->final_T[pix] = T;
            if (c->n_contrib) c->n_contrib[pix] = contrib;
        }
    free(local);
}

static orc_records* records_new(const orc_camera* cam) {
    orc_records* r = (orc_records*)calloc(1, sizeof(orc_records));
    r->width = cam->width;
    r->height = cam->height;
    r->tiles_x = (cam->width + TILE - 1) / TILE;
    r->tiles_y = (cam->height + TILE - 1) / TILE;
    return r;
}

void orc_records_free(orc_records* r) {
    if (!r) return;
    free(r->splats);
    free(r->offsets);
    free(r->ids);
    free(r->final_T);
    free(r->n_contrib);
    free(r);
}

/* rasterizer.cpp:278-306 (records always filled: final_T = 1, n_contrib = 0 init). */
static void rasterize_into(orc_records* r, const double* bg, int threads, double* image) {
    bin_and_sort(r, threads);
    size_t npix = (size_t)r->width * r->height;
    double* payload = (double*)malloc(sizeof(double) * 3 * (r->n_splats > 0 ? r->n_splats : 1));
    for (int i = 0; i < r->n_splats; ++i)
        for (int ch = 0; ch < 3; ++ch) payload[3 * i + ch] = r->splats[i].color[ch];
    r->final_T = (double*)malloc(sizeof(double) * npix);
    r->n_contrib = (int32_t*)calloc(npix, sizeof(int32_t));
    for (size_t i = 0; i < npix; ++i) r->final_T[i] = 1;
    memset(image, 0, sizeof(double) * npix * 3);
    for (int ch = 0; ch < 3; ++ch) r->background[ch] = bg[ch];
    blend_ctx c = {r, payload, {bg[0], bg[1], bg[2]}, 3, image, r->final_T, r->n_contrib};
    parallel_for(0, r->tiles_x * r->tiles_y, threads, blend_tile, &c);
    free(payload);
}

int orc_rasterize_forward(int n_splats, const orc_splat* splats, const orc_camera* cam,
                          const double* bg, int threads, double* image_out, orc_records** rec_out) {
    orc_records* r = records_new(cam);
    r->n_splats = n_splats;
    r->splats = (orc_splat*)malloc(sizeof(orc_splat) * (n_splats > 0 ? n_splats : 1));
    memcpy(r->splats, splats, sizeof(orc_splat) * n_splats);
    rasterize_into(r, bg, threads, image_out);
    if (rec_out)
        *rec_out = r;
    else
        orc_records_free(r);
    return ORC_OK;
}

/* rasterizer.cpp:308-318 */
int orc_render_forward(int n, const double* mean, const double* ls, const double* rot,
                       const double* op, const double* sh, int sh_degree, const orc_camera* cam,
                       const double* bg, int threads, int retain, double* image_out,
                       orc_records** rec_out) {
    int rc = cam_validate(cam);
    if (rc) return rc;
    build_ctx b = {n, sh_degree, mean, ls, rot, op, sh, cam, NULL, NULL, NULL};
    orc_records* r = records_new(cam);
    rc = build_splats(&b, threads, &r->splats, &r->n_splats);
    if (rc) {
        orc_records_free(r);
        return rc;
    }
    rasterize_into(r, bg, threads, image_out);
    r->retained = retain != 0;
    if (rec_out)
        *rec_out = r;
    else
        orc_records_free(r);
    return ORC_OK;
}

int orc_records_num_splats(const orc_records* r) { return r->n_splats; }
int orc_records_num_tiles(const orc_records* r) { return r->tiles_x * r->tiles_y; }
int orc_records_retained(const orc_records* r) { return r->retained; }
long long orc_records_num_pairs(const orc_records* r) { return r->offsets[r->tiles_x * r->tiles_y]; }
void orc_records_splats(const orc_records* r, orc_splat* out) {
    memcpy(out, r->splats, sizeof(orc_splat) * r->n_splats);
}
void orc_records_tiles(const orc_records* r, long long* offsets, int32_t* ids) {
    int nt = r->tiles_x * r->tiles_y;
    memcpy(offsets, r->offsets, sizeof(long long) * (nt + 1));
    memcpy(ids, r->ids, sizeof(int32_t) * r->offsets[nt]);
}
void orc_records_pixels(const orc_records* r, double* final_T, int32_t* n_contrib) {
    size_t npix = (size_t)r->width * r->height;
    if (final_T) memcpy(final_T, r->final_T, sizeof(double) * npix);
    if (n_contrib) memcpy(n_contrib, r->n_contrib, sizeof(int32_t) * npix);
}

/* ------------------------------------------------------------ backward */
typedef struct {
    double d_color[3];
    double d_conic[3];
    double d_mean2[2];
    double d_alpha_base;
} splat_grad;

/* rasterizer.cpp:42-55 */
static int splat_alpha(const orc_splat* s, double px, double py, double* alpha, double* raw,
                       double* d) {
    double d0 = px - s->mean2[0], d1 = py - s->mean2[1];
    double power = -0.5 * (s->conic[0] * d0 * d0 + s->conic[2] * d1 * d1) - s->conic[1] * d0 * d1;
    if (power > 0) return 0;
    double rr = s->alpha_base * exp(power);
    double a = smin(kAlphaClamp, rr);
    if (a < kMinAlpha) return 0;
    *alpha = a;
    *raw = rr;
    d[0] = d0;
    d[1] = d1;
    return 1;
}

typedef struct {
    const orc_records* rec;
    const double* dL; /* image gradient, 3 per pixel */
    splat_grad** tile_grads;
} bwd_tile_ctx;

/* rasterizer.cpp:329-369: per-tile reverse replay. */
static void bwd_tile(int t, void* p) {
    bwd_tile_ctx* c = (bwd_tile_ctx*)p;
    const orc_records* rec = c->rec;
    long long n = rec->offsets[t + 1] - rec->offsets[t];
    if (n == 0) return;
    const int32_t* list = rec->ids + rec->offsets[t];
    splat_grad* grads = (splat_grad*)calloc(n, sizeof(splat_grad));
    c->tile_grads[t] = grads;
    int tile_x = t % rec->tiles_x, tile_y = t / rec->tiles_x;
    int px0 = tile_x * TILE, py0 = tile_y * TILE;
    int px1 = px0 + TILE < rec->width ? px0 + TILE : rec->width;
    int py1 = py0 + TILE < rec->height ? py0 + TILE : rec->height;
    for (int y = py0; y < py1; ++y)
        for (int x = px0; x < px1; ++x) {
            size_t pix = (size_t)y * rec->width + x;
            int contrib = rec->n_contrib[pix];
            if (contrib == 0) continue;
            const double* dLdC = c->dL + 3 * pix;
            double T_run = rec->final_T[pix];
            double suffix[3];
            for (int ch = 0; ch < 3; ++ch) suffix[ch] = rec->background[ch] * rec->final_T[pix];
            for (int pos = contrib - 1; pos >= 0; --pos) {
                const orc_splat* s = &rec->splats[list[pos]];
                double a, raw, d[2];
                if (!splat_alpha(s, (double)x, (double)y, &a, &raw, d)) continue;
                double T_before = T_run / (1 - a);
                double w = a * T_before;
                splat_grad* sg = &grads[pos];
                for (int ch = 0; ch < 3; ++ch) sg->d_color[ch] = sg->d_color[ch] + w * dLdC[ch];
                double v[3];
                for (int ch = 0; ch < 3; ++ch) v[ch] = s->color[ch] * T_before - suffix[ch] / (1 - a);
                double dL_da = dLdC[0] * v[0];
                dL_da += dLdC[1] * v[1];
                dL_da += dLdC[2] * v[2];
                if (raw <= kAlphaClamp) {
                    sg->d_alpha_base += dL_da * (a / s->alpha_base);
                    double dL_dpower = dL_da * a;
                    double g3[3] = {-0.5 * d[0] * d[0], -d[0] * d[1], -0.5 * d[1] * d[1]};
                    for (int k = 0; k < 3; ++k) sg->d_conic[k] = sg->d_conic[k] + dL_dpower * g3[k];
                    double cd[2] = {s->conic[0] * d[0] + s->conic[1] * d[1],
                                    s->conic[1] * d[0] + s->conic[2] * d[1]};
                    for (int k = 0; k < 2; ++k) sg->d_mean2[k] = sg->d_mean2[k] + dL_dpower * cd[k];
                }
                for (int ch = 0; ch < 3; ++ch) suffix[ch] = suffix[ch] + s->color[ch] * w;
                T_run = T_before;
            }
        }
}

/* gaussian.cpp:57-101.  out: 16 doubles (mean4, ls4, rotor8), accumulated. */
static void slice_backward(const double* rotor_raw, const slice_cache* c, const double* Gc,
                           const double* dL_dmean3, double dL_ddecay, const double* dL_dspeed,
                           double* out) {
    double* d_mean = out;
    double* d_ls = out + 4;
    double* d_rot = out + 8;
    const double W = c->W;
    const double lambda = 1 / W;
    double speed[3];
    for (int i = 0; i < 3; ++i) speed[i] = c->V[i] / W;

    double dL_dlambda = dL_ddecay * (-0.5 * c->dt * c->dt) * c->decay;
    d_mean[3] += dL_ddecay * lambda * c->dt * c->decay;

    for (int i = 0; i < 3; ++i) d_mean[i] += dL_dmean3[i];
    {
        double s = speed[0] * dL_dmean3[0];
        s += speed[1] * dL_dmean3[1];
        s += speed[2] * dL_dmean3[2];
        d_mean[3] += -s;
    }
    double dL_dV[3];
    for (int i = 0; i < 3; ++i) dL_dV[i] = (c->dt / W) * dL_dmean3[i] + dL_dspeed[i] / W;
    double vdm = c->V[0] * dL_dmean3[0];
    vdm += c->V[1] * dL_dmean3[1];
    vdm += c->V[2] * dL_dmean3[2];
    double vds = c->V[0] * dL_dspeed[0];
    vds += c->V[1] * dL_dspeed[1];
    vds += c->V[2] * dL_dspeed[2];
    double dL_dW = -(c->dt * vdm + vds) / (W * W);

    /* cov3 = U - V V^T / W (independent entries) */
    double S[9], SV[3], GV[3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) S[i * 3 + j] = Gc[i * 3 + j] + Gc[j * 3 + i];
    for (int i = 0; i < 3; ++i) {
        double s = S[i * 3 + 0] * c->V[0];
        s += S[i * 3 + 1] * c->V[1];
        s += S[i * 3 + 2] * c->V[2];
        SV[i] = s;
        double g = Gc[i * 3 + 0] * c->V[0];
        g += Gc[i * 3 + 1] * c->V[1];
        g += Gc[i * 3 + 2] * c->V[2];
        GV[i] = g;
    }
    for (int i = 0; i < 3; ++i) dL_dV[i] += (-SV[i]) / W;
    {
        double s = c->V[0] * GV[0];
        s += c->V[1] * GV[1];
        s += c->V[2] * GV[2];
        dL_dW += s / (W * W);
    }
    dL_dW += -dL_dlambda / (W * W);

    double G4[16];
    memset(G4, 0, sizeof G4);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) G4[i * 4 + j] = Gc[i * 3 + j];
    for (int i = 0; i < 3; ++i) G4[i * 4 + 3] = dL_dV[i];
    G4[15] = dL_dW;

    const double* R = c->R;
    double RtG[16], RtGR[16];
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
            double s = R[0 * 4 + i] * G4[0 * 4 + j];
            for (int k = 1; k < 4; ++k) s += R[k * 4 + i] * G4[k * 4 + j];
            RtG[i * 4 + j] = s;
        }
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
            double s = RtG[i * 4 + 0] * R[0 * 4 + j];
            for (int k = 1; k < 4; ++k) s += RtG[i * 4 + k] * R[k * 4 + j];
            RtGR[i * 4 + j] = s;
        }
    for (int k = 0; k < 4; ++k) d_ls[k] += 2 * c->q[k] * RtGR[k * 4 + k];

    double GG[16], GGR[16], dL_dR[16];
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) GG[i * 4 + j] = G4[i * 4 + j] + G4[j * 4 + i];
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
            double s = GG[i * 4 + 0] * R[0 * 4 + j];
            for (int k = 1; k < 4; ++k) s += GG[i * 4 + k] * R[k * 4 + j];
            GGR[i * 4 + j] = s;
        }
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) dL_dR[i * 4 + j] = GGR[i * 4 + j] * c->q[j];

    double mj[128];
    to_matrix_jacobian(c->normalized, mj);
    double dL_drn[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int e = 0; e < 16; ++e) {
        double w = dL_dR[e];
        if (w != 0)
            for (int k = 0; k < 8; ++k) dL_drn[k] += w * mj[e * 8 + k];
    }
    double Jn[64];
    normalize_jacobian(rotor_raw, Jn);
    for (int k = 0; k < 8; ++k) {
        double s = Jn[0 * 8 + k] * dL_drn[0];
        for (int i = 1; i < 8; ++i) s += Jn[i * 8 + k] * dL_drn[i];
        d_rot[k] += s;
    }
}

/* rasterizer.cpp:134-181.  out: 65 doubles (mean4, ls4, rot8, opacity, sh48 ch-major). */
static void project_backward(const double* rotor_raw, const double* sh48, const orc_camera* cam,
                             const project_cache* pc, const splat_grad* sg, double* out) {
    double* d_op = out + 16;
    double* d_sh = out + 17;
    double dL_ddir[3] = {0, 0, 0};
    for (int ch = 0; ch < 3; ++ch) {
        if (pc->clamped[ch]) continue;
        if (sg->d_color[ch] == 0) continue;
        for (int k = 0; k < 16; ++k) d_sh[ch * 16 + k] += sg->d_color[ch] * pc->basis[k];
        for (int a = 0; a < 3; ++a) {
            double s = pc->basis_grad[0 * 3 + a] * sh48[ch * 16 + 0];
            for (int k = 1; k < 16; ++k) s += pc->basis_grad[k * 3 + a] * sh48[ch * 16 + k];
            dL_ddir[a] += sg->d_color[ch] * s;
        }
    }
    double dL_dmean3[3] = {0, 0, 0};
    if (dL_ddir[0] != 0 || dL_ddir[1] != 0 || dL_ddir[2] != 0) {
        double M[9];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                M[i * 3 + j] = ((i == j ? 1.0 : 0.0) - pc->dir[i] * pc->dir[j]) / pc->view_dist;
        for (int i = 0; i < 3; ++i) {
            double s = M[i * 3 + 0] * dL_ddir[0];
            s += M[i * 3 + 1] * dL_ddir[1];
            s += M[i * 3 + 2] * dL_ddir[2];
            dL_dmean3[i] += s;
        }
    }
    double dL_ddecay = sg->d_alpha_base * pc->opacity;
    *d_op += sg->d_alpha_base * pc->decay * pc->opacity * (1 - pc->opacity);

    const double* c2 = pc->cov2;
    double invdet = 1.0 / (c2[0] * c2[3] - c2[2] * c2[1]);
    double con[4] = {c2[3] * invdet, -c2[1] * invdet, -c2[2] * invdet, c2[0] * invdet};
    double ghat[4] = {sg->d_conic[0], sg->d_conic[1] / 2, sg->d_conic[1] / 2, sg->d_conic[2]};
    double P1[4], H[4];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j)
            P1[i * 2 + j] = (-con[i * 2 + 0]) * ghat[0 * 2 + j] + (-con[i * 2 + 1]) * ghat[1 * 2 + j];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) H[i * 2 + j] = P1[i * 2 + 0] * con[0 * 2 + j] + P1[i * 2 + 1] * con[1 * 2 + j];

    const double* T = pc->T;
    double Q[6], dcov3[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 2; ++j) Q[i * 2 + j] = T[0 * 3 + i] * H[0 * 2 + j] + T[1 * 3 + i] * H[1 * 2 + j];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) dcov3[i * 3 + j] = Q[i * 2 + 0] * T[0 * 3 + j] + Q[i * 2 + 1] * T[1 * 3 + j];

    double HH[4], HT[6], dT[6];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) HH[i * 2 + j] = H[i * 2 + j] + H[j * 2 + i];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j) HT[i * 3 + j] = HH[i * 2 + 0] * T[0 * 3 + j] + HH[i * 2 + 1] * T[1 * 3 + j];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = HT[i * 3 + 0] * pc->cov3[0 * 3 + j];
            s += HT[i * 3 + 1] * pc->cov3[1 * 3 + j];
            s += HT[i * 3 + 2] * pc->cov3[2 * 3 + j];
            dT[i * 3 + j] = s;
        }

    double J[6];
    projection_jacobian(cam, pc->p_cam, J);
    double dpc[3];
    for (int i = 0; i < 3; ++i) dpc[i] = J[0 * 3 + i] * sg->d_mean2[0] + J[1 * 3 + i] * sg->d_mean2[1];

    double Rc[9], dJ[6];
    cam_rotation(cam, Rc);
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = dT[i * 3 + 0] * Rc[j * 3 + 0];
            s += dT[i * 3 + 1] * Rc[j * 3 + 1];
            s += dT[i * 3 + 2] * Rc[j * 3 + 2];
            dJ[i * 3 + j] = s;
        }
    const double z = pc->p_cam[2], z2 = z * z, z3 = z2 * z;
    const double px = pc->p_cam[0], py = pc->p_cam[1];
    dpc[0] += dJ[0 * 3 + 2] * (-cam->fx / z2);
    dpc[1] += dJ[1 * 3 + 2] * (-cam->fy / z2);
    dpc[2] += dJ[0 * 3 + 0] * (-cam->fx / z2) + dJ[0 * 3 + 2] * (2 * cam->fx * px / z3) +
              dJ[1 * 3 + 1] * (-cam->fy / z2) + dJ[1 * 3 + 2] * (2 * cam->fy * py / z3);
    for (int i = 0; i < 3; ++i) {
        double s = Rc[0 * 3 + i] * dpc[0];
        s += Rc[1 * 3 + i] * dpc[1];
        s += Rc[2 * 3 + i] * dpc[2];
        dL_dmean3[i] += s;
    }
    const double zero3[3] = {0, 0, 0};
    slice_backward(rotor_raw, &pc->slice, dcov3, dL_dmean3, dL_ddecay, zero3, out);
}

typedef struct {
    build_ctx b;
    const orc_records* rec;
    const splat_grad* sgrads;
    double* grads;
    double* vnorm;
    uint8_t* visible;
} bwd_splat_ctx;

static void bwd_splat(int i, void* p) {
    bwd_splat_ctx* c = (bwd_splat_ctx*)p;
    int src = c->rec->splats[i].source_index;
    project_cache pc;
    orc_splat tmp;
    memset(&pc, 0, sizeof pc);
    slice_and_project(&c->b, src, &tmp, &pc); /* recompute the forward cache */
    double* o = c->grads + 65 * (size_t)src;
    project_backward(c->b.rot + 8 * src, c->b.sh + 48 * src, c->b.cam, &pc, &c->sgrads[i], o);
    const double* dm = c->sgrads[i].d_mean2;
    c->vnorm[src] = sqrt(dm[0] * dm[0] + dm[1] * dm[1]);
    c->visible[src] = 1;
}

/* rasterizer.cpp:320-397 */
int orc_render_backward(int n, const double* mean, const double* ls, const double* rot,
                        const double* op, const double* sh, int sh_degree, const orc_camera* cam,
                        const orc_records* rec, const double* dL_dimage, int threads,
                        double* grads, double* vnorm, uint8_t* visible) {
    if (!rec->retained)
        return fail(ORC_E_MISSING_RECORDS, "rasterize_backward: forward pass did not retain records");
    int ntiles = rec->tiles_x * rec->tiles_y;
    splat_grad** tg = (splat_grad**)calloc(ntiles, sizeof(splat_grad*));
    bwd_tile_ctx tc = {rec, dL_dimage, tg};
    parallel_for(0, ntiles, threads, bwd_tile, &tc);
    splat_grad* sgr = (splat_grad*)calloc(rec->n_splats > 0 ? rec->n_splats : 1, sizeof(splat_grad));
    for (int t = 0; t < ntiles; ++t) {
        if (!tg[t]) continue;
        long long cnt = rec->offsets[t + 1] - rec->offsets[t];
        for (long long k = 0; k < cnt; ++k) {
            splat_grad* dst = &sgr[rec->ids[rec->offsets[t] + k]];
            const splat_grad* src = &tg[t][k];
            for (int a = 0; a < 3; ++a) dst->d_color[a] += src->d_color[a];
            for (int a = 0; a < 3; ++a) dst->d_conic[a] += src->d_conic[a];
            for (int a = 0; a < 2; ++a) dst->d_mean2[a] += src->d_mean2[a];
            dst->d_alpha_base += src->d_alpha_base;
        }
        free(tg[t]);
    }
    free(tg);
    memset(grads, 0, sizeof(double) * 65 * (size_t)n);
    memset(vnorm, 0, sizeof(double) * n);
    memset(visible, 0, n);
    bwd_splat_ctx sc = {{n, sh_degree, mean, ls, rot, op, sh, cam, NULL, NULL, NULL},
                        rec, sgr, grads, vnorm, visible};
    parallel_for(0, rec->n_splats, threads, bwd_splat, &sc);
    free(sgr);
    return ORC_OK;
}

/* rasterizer.cpp:399-425 */
int orc_render_flow(int n, const double* mean, const double* ls, const double* rot,
                    const double* op, const double* sh, int sh_degree, const orc_camera* cam,
                    int threads, double* flow_out) {
    int rc = cam_validate(cam);
    if (rc) return rc;
    build_ctx b = {n, sh_degree, mean, ls, rot, op, sh, cam, NULL, NULL, NULL};
    orc_records* r = records_new(cam);
    rc = build_splats(&b, threads, &r->splats, &r->n_splats);
    if (rc) {
        orc_records_free(r);
        return rc;
    }
    bin_and_sort(r, threads);
    size_t npix = (size_t)cam->width * cam->height;
    double* payload = (double*)malloc(sizeof(double) * 3 * (r->n_splats > 0 ? r->n_splats : 1));
    for (int i = 0; i < r->n_splats; ++i) {
        payload[3 * i] = r->splats[i].flow2[0];
        payload[3 * i + 1] = r->splats[i].flow2[1];
        payload[3 * i + 2] = 0;
    }
    double* rgb = (double*)calloc(npix * 3, sizeof(double));
    blend_ctx c = {r, payload, {0, 0, 0}, 3, rgb, NULL, NULL};
    parallel_for(0, r->tiles_x * r->tiles_y, threads, blend_tile, &c);
    for (size_t i = 0; i < npix; ++i) {
        flow_out[2 * i] = rgb[3 * i];
        flow_out[2 * i + 1] = rgb[3 * i + 1];
    }
    free(rgb);
    free(payload);
    orc_records_free(r);
    return ORC_OK;
}

/* tests/reference.hpp:77-116: naive per-pixel walk in global depth order. */
int orc_naive_render(int n, const double* mean, const double* ls, const double* rot,
                     const double* op, const double* sh, int sh_degree, const orc_camera* cam,
                     const double* bg, double* image_out, double* weight_sum, double* final_T) {
    build_ctx b = {n, sh_degree, mean, ls, rot, op, sh, cam, NULL, NULL, NULL};
    orc_splat* sp = NULL;
    int m = 0;
    int rc = build_splats(&b, 1, &sp, &m);
    if (rc) return rc;
    /* global order by (depth, source_index) */
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (m > 0 ? m : 1));
    for (int i = 0; i < m; ++i) order[i] = i;
    sort_tile(order, m, sp);
    for (int y = 0; y < cam->height; ++y)
        for (int x = 0; x < cam->width; ++x) {
            double T = 1, wsum = 0, acc[3] = {0, 0, 0};
            for (int k = 0; k < m; ++k) {
                const orc_splat* s = &sp[order[k]];
                int tx = x / TILE, ty = y / TILE;
                if (tx < floor((s->mean2[0] - s->radius) / TILE) ||
                    tx > floor((s->mean2[0] + s->radius) / TILE) ||
                    ty < floor((s->mean2[1] - s->radius) / TILE) ||
                    ty > floor((s->mean2[1] + s->radius) / TILE))
                    continue;
                double d0 = x - s->mean2[0], d1 = y - s->mean2[1];
                double power =
                    -0.5 * (s->conic[0] * d0 * d0 + s->conic[2] * d1 * d1) - s->conic[1] * d0 * d1;
                if (power > 0) continue;
                double a = smin(kAlphaClamp, s->alpha_base * exp(power));
                if (a < kMinAlpha) continue;
                if (T * (1 - a) < kStopT) break;
                for (int ch = 0; ch < 3; ++ch) acc[ch] = acc[ch] + s->color[ch] * (a * T);
                wsum += a * T;
                T *= 1 - a;
            }
            for (int ch = 0; ch < 3; ++ch) acc[ch] = acc[ch] + T * bg[ch];
            size_t pix = (size_t)y * cam->width + x;
            for (int ch = 0; ch < 3; ++ch) image_out[pix * 3 + ch] = acc[ch];
            if (weight_sum) weight_sum[pix] = wsum;
            if (final_T) final_T[pix] = T;
        }
    free(order);
    free(sp);
    return ORC_OK;
}

/* ------------------------------------------------------------ single pieces */
int orc_normalize(const double* rot, double* out) {
    int rc = rotor_normalize(rot, out);
    if (rc) return fail(rc, rc == ORC_E_ZERO_ROTOR ? "normalize: zero rotor"
                                                   : "normalize: result violates rotor invariants");
    return ORC_OK;
}
int orc_to_matrix(const double* rot, double* out16) {
    if (fabs(sqnorm8(rot) - 1) > 1e-6 || fabs(rotor_epsilon(rot)) > 1e-6)
        return fail(ORC_E_INVALID, "to_matrix: rotor not normalized");
    rotor_to_matrix(rot, out16);
    return ORC_OK;
}
int orc_slice_at(const double* mean, const double* ls, const double* rot, double t, double* out) {
    sliced3 s;
    slice_cache c;
    int rc = slice_at(mean, ls, rot, t, &s, &c);
    if (rc) return fail(rc, rc == ORC_E_DEGENERATE_TIME
                                ? "slice_at: temporal scale collapsed (W < 1e-12)"
                                : "normalize failed");
    memcpy(out, s.mean, 3 * sizeof(double));
    memcpy(out + 3, s.cov, 9 * sizeof(double));
    out[12] = s.decay;
    memcpy(out + 13, s.speed, 3 * sizeof(double));
    out[16] = s.lambda;
    return ORC_OK;
}
int orc_project(const double* sliced, const orc_camera* cam, const double* sh48, int sh_degree,
                double opacity_logit, orc_splat* out) {
    sliced3 s;
    memcpy(s.mean, sliced, 3 * sizeof(double));
    memcpy(s.cov, sliced + 3, 9 * sizeof(double));
    s.decay = sliced[12];
    memcpy(s.speed, sliced + 13, 3 * sizeof(double));
    s.lambda = 1;
    int r = project(&s, cam, sh48, sh_degree, opacity_logit, out, NULL);
    if (r) out->source_index = -1;
    return r;
}

/* ======================================================================
 * Training side: image losses, regularizers, the Adam
 * step and densification statistics, and evaluate_loss's batch reduction.
 * Pinned against oracle/_ref (image.cpp, ssim.cpp, loss.cpp, knn.cpp,
 * optim.cpp, trainer.cpp compiled in place) by tests/test_oracle_train.py.
 * ==================================================================== */

/* image.cpp:7-18 */
double orc_psnr(long long n_values, const double* a, const double* b) {
    double mse = 0;
    for (long long i = 0; i < n_values; ++i) {
        double d = a[i] - b[i];
        mse += d * d;
    }
    mse /= (double)n_values;
    if (mse <= 0) return 100;
    double v = 10 * log10(1 / mse);
    return v < 100 ? v : 100;
}

/* image.cpp:20-36.  grad (may be NULL) = l1_loss_backward. */
double orc_l1_loss(long long n_values, const double* rendered, const double* target, double* grad) {
    double sum = 0;
    for (long long i = 0; i < n_values; ++i) sum += fabs(rendered[i] - target[i]);
    if (grad) {
        double inv_n = 1 / (double)n_values;
        for (long long i = 0; i < n_values; ++i) {
            double d = rendered[i] - target[i];
            grad[i] = d > 0 ? inv_n : (d < 0 ? -inv_n : 0);
        }
    }
    return sum / (double)n_values;
}

/* ssim.cpp:15-31: normalised 11-tap Gaussian window, sigma 1.5. */
enum { kWin = 11 };
static void ssim_window(double* k) {
    const double sigma = 1.5;
    double sum = 0;
    for (int i = 0; i < kWin; ++i) {
        double d = i - (kWin - 1) / 2.0;
        k[i] = exp(-d * d / (2 * sigma * sigma));
        sum += k[i];
    }
    for (int i = 0; i < kWin; ++i) k[i] /= sum;
}
void orc_ssim_window(double* k11) { ssim_window(k11); }

/* ssim.cpp:42-58: valid-region separable convolution (rows, then columns). */
static void conv_valid(const double* k, const double* in, int w, int h, double* rows, double* out) {
    int rw = w - kWin + 1, oh = h - kWin + 1;
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < rw; ++x) {
            double s = 0;
            for (int i = 0; i < kWin; ++i) s += k[i] * in[(size_t)y * w + x + i];
            rows[(size_t)y * rw + x] = s;
        }
    for (int y = 0; y < oh; ++y)
        for (int x = 0; x < rw; ++x) {
            double s = 0;
            for (int i = 0; i < kWin; ++i) s += k[i] * rows[(size_t)(y + i) * rw + x];
            out[(size_t)y * rw + x] = s;
        }
}

/* ssim.cpp:61-72: adjoint of conv_valid (scatter back to the input support). */
static void conv_valid_adjoint(const double* k, const double* g, int gw, int gh, int in_w, int in_h,
                               double* cols, double* out) {
    memset(cols, 0, sizeof(double) * (size_t)gw * in_h);
    for (int y = 0; y < gh; ++y)
        for (int x = 0; x < gw; ++x)
            for (int i = 0; i < kWin; ++i) cols[(size_t)(y + i) * gw + x] += k[i] * g[(size_t)y * gw + x];
    memset(out, 0, sizeof(double) * (size_t)in_w * in_h);
    for (int y = 0; y < in_h; ++y)
        for (int x = 0; x < gw; ++x)
            for (int i = 0; i < kWin; ++i) out[(size_t)y * in_w + x + i] += k[i] * cols[(size_t)y * gw + x];
}

/* ssim.cpp:74-142: 1 - mean SSIM over the valid region, channels 0..2; grad (may be
 * NULL) = d loss / d rendered (zero outside the valid support). */
int orc_ssim_loss(int w, int h, const double* xi, const double* yi, double* loss, double* grad) {
    if (w < kWin || h < kWin) return fail(ORC_E_INVALID, "ssim: image smaller than the 11x11 window");
    const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
    double k[kWin];
    ssim_window(k);
    const size_t np = (size_t)w * h;
    const int vw = w - kWin + 1, vh = h - kWin + 1;
    const size_t nv = (size_t)vw * vh;
    double* f = (double*)malloc(sizeof(double) * np * 5);
    double* m = (double*)malloc(sizeof(double) * nv * 5);
    double* rows = (double*)malloc(sizeof(double) * (size_t)vw * h);
    double* d = (double*)malloc(sizeof(double) * nv * 3);
    double* adj = (double*)malloc(sizeof(double) * np * 3);
    double* cols = (double*)malloc(sizeof(double) * (size_t)vw * h);
    double total = 0;
    size_t count = 0;
    for (int ch = 0; ch < 3; ++ch) {
        double *x = f, *y = f + np, *xx = f + 2 * np, *yy = f + 3 * np, *xy = f + 4 * np;
        for (size_t p = 0; p < np; ++p) {
            double a = xi[p * 3 + ch], b = yi[p * 3 + ch];
            x[p] = a;
            y[p] = b;
            xx[p] = a * a;
            yy[p] = b * b;
            xy[p] = a * b;
        }
        for (int q = 0; q < 5; ++q) conv_valid(k, f + q * np, w, h, rows, m + q * nv);
        const double *mx = m, *my = m + nv, *sxx = m + 2 * nv, *syy = m + 3 * nv, *sxy = m + 4 * nv;
        for (size_t p = 0; p < nv; ++p) {
            double ux = mx[p], uy = my[p];
            double vx = sxx[p] - ux * ux;
            double vy = syy[p] - uy * uy;
            double vxy = sxy[p] - ux * uy;
            double a1 = 2 * ux * uy + C1, a2 = 2 * vxy + C2;
            double b1 = ux * ux + uy * uy + C1, b2 = vx + vy + C2;
            double s = (a1 * a2) / (b1 * b2);
            total += s;
            ++count;
            if (grad) {
                double d_ssim = 1;
                double d_a1 = d_ssim * a2 / (b1 * b2);
                double d_a2 = d_ssim * a1 / (b1 * b2);
                double d_b1 = -d_ssim * s / b1;
                double d_b2 = -d_ssim * s / b2;
                double d_ux = d_a1 * 2 * uy + d_b1 * 2 * ux;
                double d_vx = d_b2;
                double d_vxy = d_a2 * 2;
                d_ux += -2 * ux * d_vx - uy * d_vxy;
                d[p] = d_ux;
                d[nv + p] = d_vx;
                d[2 * nv + p] = d_vxy;
            }
        }
        if (grad) {
            for (int q = 0; q < 3; ++q) conv_valid_adjoint(k, d + q * nv, vw, vh, w, h, cols, adj + q * np);
            for (size_t p = 0; p < np; ++p)
                grad[p * 3 + ch] = adj[p] + 2 * x[p] * adj[np + p] + y[p] * adj[2 * np + p];
        }
    }
    double mean = total / (double)count;
    if (grad) {
        double fct = -1 / (double)count;
        for (size_t p = 0; p < np * 3; ++p) grad[p] *= fct;
    }
    *loss = 1 - mean;
    free(f);
    free(m);
    free(rows);
    free(d);
    free(adj);
    free(cols);
    return ORC_OK;
}

/* loss.cpp:16-31 */
double orc_entropy_loss(int n, const double* opacities, double* grad) {
    const double clampv = 1e-6;
    if (n == 0) return 0;
    double total = 0;
    const double inv_n = 1 / (double)n;
    for (int i = 0; i < n; ++i) {
        double o = opacities[i];
        o = o < clampv ? clampv : (1 - clampv < o ? 1 - clampv : o); /* std::clamp */
        total += -o * log(o);
        if (grad) grad[i] = (opacities[i] > clampv && opacities[i] < 1 - clampv) ? -(log(o) + 1) * inv_n : 0;
    }
    return total * inv_n;
}

/* loss.cpp:33-58.  dspeed (may be NULL) n*3, zeroed then accumulated. */
double orc_consistency_loss(int n, const double* speeds, int k, const int32_t* nbrs, double* dspeed) {
    if (dspeed) memset(dspeed, 0, sizeof(double) * 3 * (size_t)n);
    if (n == 0) return 0;
    const double inv_n = 1 / (double)n;
    double total = 0;
    for (int i = 0; i < n; ++i) {
        if (k <= 0) continue;
        const double inv_k = 1 / (double)k;
        double avg[3] = {0, 0, 0};
        for (int j = 0; j < k; ++j)
            for (int a = 0; a < 3; ++a) avg[a] += speeds[3 * (size_t)nbrs[(size_t)k * i + j] + a];
        for (int a = 0; a < 3; ++a) avg[a] *= inv_k;
        double diff[3], sgn[3];
        for (int a = 0; a < 3; ++a) {
            diff[a] = speeds[3 * (size_t)i + a] - avg[a];
            sgn[a] = (double)(diff[a] > 0) - (double)(diff[a] < 0);
        }
        double s = fabs(diff[0]);
        s += fabs(diff[1]);
        s += fabs(diff[2]);
        total += s;
        if (dspeed) {
            for (int a = 0; a < 3; ++a) dspeed[3 * (size_t)i + a] += inv_n * sgn[a];
            for (int j = 0; j < k; ++j)
                for (int a = 0; a < 3; ++a)
                    dspeed[3 * (size_t)nbrs[(size_t)k * i + j] + a] -= inv_n * inv_k * sgn[a];
        }
    }
    return total * inv_n;
}

/* trainer.cpp:12-20 */
void orc_scene_scales(int n, const double* mean, double* out4) {
    double lo[4] = {0, 0, 0, 0}, hi[4] = {0, 0, 0, 0};
    if (n > 0)
        for (int a = 0; a < 4; ++a) lo[a] = hi[a] = mean[a];
    for (int i = 0; i < n; ++i)
        for (int a = 0; a < 4; ++a) {
            double v = mean[4 * (size_t)i + a];
            lo[a] = v < lo[a] ? v : lo[a];
            hi[a] = hi[a] < v ? v : hi[a];
        }
    for (int a = 0; a < 4; ++a) {
        double e = hi[a] - lo[a];
        out4[a] = e < 1e-3 ? 1e-3 : e;
    }
}

/* knn.cpp:101-116: exact k nearest neighbours on mean / scales, excluding self, ordered by
 * (squared distance, index) -- KdTree4's contract (knn.hpp:18-20), as a brute-force scan. */
typedef struct {
    int n, k;
    const double* pts;
    int32_t* nbrs;
} knn_ctx;
static void knn_body(int i, void* p) {
    knn_ctx* c = (knn_ctx*)p;
    const int k = c->k;
    double bd[64];
    int bi[64];
    int cnt = 0;
    const double* q = c->pts + 4 * (size_t)i;
    for (int j = 0; j < c->n; ++j) {
        if (j == i) continue;
        const double* pj = c->pts + 4 * (size_t)j;
        double d0 = pj[0] - q[0], d1 = pj[1] - q[1], d2 = pj[2] - q[2], d3 = pj[3] - q[3];
        double dd = d0 * d0;
        dd += d1 * d1;
        dd += d2 * d2;
        dd += d3 * d3;
        if (cnt == k && !(dd < bd[k - 1] || (dd == bd[k - 1] && j < bi[k - 1]))) continue;
        int pos = cnt < k ? cnt++ : k - 1;
        while (pos > 0 && (dd < bd[pos - 1] || (dd == bd[pos - 1] && j < bi[pos - 1]))) {
            bd[pos] = bd[pos - 1];
            bi[pos] = bi[pos - 1];
            --pos;
        }
        bd[pos] = dd;
        bi[pos] = j;
    }
    for (int j = 0; j < k; ++j) c->nbrs[(size_t)k * i + j] = bi[j];
}
int orc_knn4d(int n, const double* mean, int k, const double* scales, int threads, int32_t* nbrs) {
    if (n <= k) return fail(ORC_E_INVALID, "knn: need more points than neighbors");
    if (k > 64) return fail(ORC_E_INVALID, "knn: k > 64 unsupported by the oracle");
    double* pts = (double*)malloc(sizeof(double) * 4 * (size_t)n);
    for (size_t i = 0; i < 4 * (size_t)n; ++i) pts[i] = mean[i] / scales[i % 4];
    knn_ctx c = {n, k, pts, nbrs};
    parallel_for(0, n, threads, knn_body, &c);
    free(pts);
    return ORC_OK;
}

/* gaussian.cpp:103-110 */
int orc_gaussian_speeds(int n, const double* mean, const double* ls, const double* rot, double* speeds) {
    (void)mean;
    for (int i = 0; i < n; ++i) {
        slice_cache c;
        int rc = assemble_cache(ls + 4 * (size_t)i, rot + 8 * (size_t)i, &c);
        if (rc) return rc;
        if (c.W < kTemporalFloor) return fail(ORC_E_DEGENERATE_TIME, "slice: degenerate temporal variance");
        for (int a = 0; a < 3; ++a) speeds[3 * (size_t)i + a] = c.V[a] / c.W;
    }
    return ORC_OK;
}

/* optim.cpp:47-51 */
double orc_lr_schedule(int step, int total, double lr_init, double lr_final) {
    if (total <= 0) return lr_init;
    double u = (double)step / (double)total;
    u = u < 0 ? 0 : (1 < u ? 1 : u);
    return lr_init * pow(lr_final / lr_init, u);
}

/* optim.cpp:19-23 (kAdamBeta1/2, kAdamEps: optim.hpp:70-72) */
static void adam_scalar(double* p, double* m, double* v, double g, double lr, double bc1, double bc2) {
    const double b1 = 0.9, b2 = 0.999, eps = 1e-15;
    *m = b1 * *m + (1 - b1) * g;
    *v = b2 * *v + (1 - b2) * g * g;
    *p -= lr * (*m / bc1) / (sqrt(*v / bc2) + eps);
}

/* optim.cpp:110-157.  m, v: n*65 in the gradient order; grads: n*65. */
int orc_adam_step(int n, double* mean, double* ls, double* rot, double* op, double* sh, double* m, double* v,
                  const double* grads, const orc_adam_config* cfg, int step) {
    const double bc1 = 1 - pow(0.9, step);
    const double bc2 = 1 - pow(0.999, step);
    const double lr_pos = orc_lr_schedule(step, cfg->total_steps, cfg->lr_position, cfg->lr_position_final);
    const int st = cfg->static_mode != 0;
    for (int i = 0; i < n; ++i) {
        const double* g = grads + 65 * (size_t)i;
        double* mi = m + 65 * (size_t)i;
        double* vi = v + 65 * (size_t)i;
        for (int a = 0; a < 4; ++a) {
            if (st && a == 3) continue;
            adam_scalar(&mean[4 * (size_t)i + a], &mi[a], &vi[a], g[a], lr_pos, bc1, bc2);
        }
        for (int a = 0; a < (st ? 3 : 4); ++a)
            adam_scalar(&ls[4 * (size_t)i + a], &mi[4 + a], &vi[4 + a], g[4 + a], cfg->lr_scales, bc1, bc2);
        double rc[8];
        for (int a = 0; a < 8; ++a) rc[a] = rot[8 * (size_t)i + a];
        for (int a = 0; a < 8; ++a) {
            if (st && (a == 3 || a == 5 || a == 6 || a == 7)) continue; /* kTemporalRotorIdx */
            adam_scalar(&rc[a], &mi[8 + a], &vi[8 + a], g[8 + a], cfg->lr_rotor, bc1, bc2);
        }
        double nr[8];
        int rcode = rotor_normalize(rc, nr);
        if (rcode) return rcode;
        if (st) nr[3] = nr[5] = nr[6] = nr[7] = 0;
        for (int a = 0; a < 8; ++a) rot[8 * (size_t)i + a] = nr[a];
        adam_scalar(&op[i], &mi[16], &vi[16], g[16], cfg->lr_opacity, bc1, bc2);
        for (int c = 0; c < 16; ++c) {
            double lr = c == 0 ? cfg->lr_sh_dc : cfg->lr_sh_rest;
            for (int ch = 0; ch < 3; ++ch) {
                int j = 17 + ch * 16 + c;
                adam_scalar(&sh[48 * (size_t)i + ch * 16 + c], &mi[j], &vi[j], g[j], lr, bc1, bc2);
            }
        }
    }
    return ORC_OK;
}

/* optim.cpp:159-166 */
void orc_accumulate_stats(int n, const double* vnorm, const uint8_t* visible, double* accum, int32_t* count) {
    for (int i = 0; i < n; ++i) {
        if (!visible[i]) continue;
        accum[i] += vnorm[i];
        count[i] += 1;
    }
}

/* optim.cpp:236-243 */
void orc_reset_opacity(int n, double* op, double* m_op, double* v_op, double value) {
    for (int i = 0; i < n; ++i) {
        double o = sigmoid(op[i]);
        o = (value < o) ? value : o;
        op[i] = log(o / (1 - o));
        m_op[i] = 0;
        v_op[i] = 0;
    }
}

/* trainer.cpp:22-84: batch losses and summed gradients.  targets: n_frames images of
 * H*W*3; nbrs (n*k) may be NULL (consistency skipped).  losses[5] = l1, ssim, entropy,
 * consistency, total.  grads (n*65) / vnorm / visible may be NULL (no gradients). */
int orc_evaluate_loss(int n, const double* mean, const double* ls, const double* rot, const double* op,
                      const double* sh, int sh_degree, int n_frames, const orc_camera* cams,
                      const double* targets, const orc_loss_weights* w, const double* bg, const int32_t* nbrs,
                      int threads, double* losses, double* grads, double* vnorm, uint8_t* visible) {
    double l1 = 0, ssim = 0, entropy = 0, consistency = 0;
    const int want = grads != NULL;
    if (want) {
        memset(grads, 0, sizeof(double) * 65 * (size_t)n);
        memset(vnorm, 0, sizeof(double) * (size_t)n);
        memset(visible, 0, (size_t)n);
    }
    const double inv_b = n_frames == 0 ? 0 : 1 / (double)n_frames;
    size_t off = 0;
    for (int f = 0; f < n_frames; ++f) {
        const orc_camera* cam = &cams[f];
        const size_t nv = (size_t)cam->width * cam->height * 3;
        const double* tgt = targets + off;
        off += nv;
        double* img = (double*)malloc(sizeof(double) * nv);
        orc_records* rec = NULL;
        int rc = orc_render_forward(n, mean, ls, rot, op, sh, sh_degree, cam, bg, threads, want, img, &rec);
        if (rc) {
            free(img);
            return rc;
        }
        double sl = 0;
        if (!want) {
            l1 += orc_l1_loss((long long)nv, img, tgt, NULL) * inv_b;
            rc = orc_ssim_loss(cam->width, cam->height, img, tgt, &sl, NULL);
            if (rc) return rc;
            ssim += sl * inv_b;
        } else {
            double* gl1 = (double*)malloc(sizeof(double) * nv);
            double* gss = (double*)malloc(sizeof(double) * nv);
            double lv = orc_l1_loss((long long)nv, img, tgt, gl1);
            l1 += lv * inv_b;
            rc = orc_ssim_loss(cam->width, cam->height, img, tgt, &sl, gss);
            if (rc) return rc;
            ssim += sl * inv_b;
            const double wl1 = (1 - w->lambda_ssim) * inv_b;
            const double wss = w->lambda_ssim * inv_b;
            for (size_t i = 0; i < nv; ++i) gl1[i] = wl1 * gl1[i] + wss * gss[i];
            double* fg = (double*)malloc(sizeof(double) * 65 * (size_t)n);
            double* fv = (double*)malloc(sizeof(double) * (size_t)n);
            uint8_t* fvis = (uint8_t*)malloc((size_t)n + 1);
            rc = orc_render_backward(n, mean, ls, rot, op, sh, sh_degree, cam, rec, gl1, threads, fg, fv, fvis);
            if (rc) return rc;
            for (size_t i = 0; i < 65 * (size_t)n; ++i) grads[i] += fg[i];
            for (int i = 0; i < n; ++i) {
                vnorm[i] += fv[i];
                visible[i] |= fvis[i];
            }
            free(fg);
            free(fv);
            free(fvis);
            free(gl1);
            free(gss);
        }
        orc_records_free(rec);
        free(img);
    }
    if (w->lambda_entropy != 0) {
        double* o = (double*)malloc(sizeof(double) * ((size_t)n + 1));
        double* g = (double*)malloc(sizeof(double) * ((size_t)n + 1));
        for (int i = 0; i < n; ++i) o[i] = sigmoid(op[i]);
        entropy = orc_entropy_loss(n, o, want ? g : NULL);
        if (want)
            for (int i = 0; i < n; ++i)
                grads[65 * (size_t)i + 16] += w->lambda_entropy * g[i] * o[i] * (1 - o[i]);
        free(o);
        free(g);
    }
    if (w->lambda_consistency != 0 && nbrs != NULL && n > 0) {
        double* sp = (double*)malloc(sizeof(double) * 3 * (size_t)n);
        double* gs = (double*)malloc(sizeof(double) * 3 * (size_t)n);
        int rc = orc_gaussian_speeds(n, mean, ls, rot, sp);
        if (rc) return rc;
        consistency = orc_consistency_loss(n, sp, w->k_neighbors, nbrs, want ? gs : NULL);
        if (want)
            for (int i = 0; i < n; ++i) {
                slice_cache c;
                assemble_cache(ls + 4 * (size_t)i, rot + 8 * (size_t)i, &c);
                c.dt = 0;
                c.decay = 1; /* SliceCache default (gaussian.hpp:44) */
                const double zero9[9] = {0}, zero3[3] = {0};
                double ds[3];
                for (int a = 0; a < 3; ++a) ds[a] = w->lambda_consistency * gs[3 * (size_t)i + a];
                slice_backward(rot + 8 * (size_t)i, &c, zero9, zero3, 0, ds, grads + 65 * (size_t)i);
            }
        free(sp);
        free(gs);
    }
    losses[0] = l1;
    losses[1] = ssim;
    losses[2] = entropy;
    losses[3] = consistency;
    losses[4] = (1 - w->lambda_ssim) * l1 + w->lambda_ssim * ssim + w->lambda_entropy * entropy +
                w->lambda_consistency * consistency;
    return ORC_OK;
}
