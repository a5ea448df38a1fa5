// FP64 device math of the per-Gaussian path: rotor normalisation, R4D, Schur slice,
// EWA projection and SH colour, plus their analytic backward.
//
// Parity contract: this header is only included from translation units compiled with
// -fmad=false, and every expression keeps the reference's operation order
// (products summed sequentially over k starting from the first term, exactly as
// the reference compiled against include/eigen_subset and oracle/rgs_oracle.c).
// Line citations are to /root/reference/proj.
#pragma once

#include "glibc_exp.h"
#include "rgs_internal.cuh"

namespace rgs_dev {

__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }

// x86-64 cvttsd2si semantics of (int)std::floor(..) (rasterizer.cpp:32-35).
__device__ __forceinline__ int x86_double_to_int(double v) {
    if (!(v >= -2147483648.0 && v < 2147483648.0)) return (int)0x80000000u;
    return (int)v;
}

// rotor.cpp:113-115
__device__ __forceinline__ double rotor_epsilon(const double* v) {
    return v[7] * v[0] - v[1] * v[6] + v[2] * v[5] - v[3] * v[4];
}
// rotor.cpp:54-58
__device__ __forceinline__ void epsilon_gradient(const double* v, double* g) {
    g[0] = v[7];
    g[1] = -v[6];
    g[2] = v[5];
    g[3] = -v[4];
    g[4] = -v[3];
    g[5] = v[2];
    g[6] = -v[1];
    g[7] = v[0];
}
__device__ __forceinline__ double sqnorm8(const double* v) {
    double s = v[0] * v[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) s += v[i] * v[i];
    return s;
}

// Error codes (rgs_status).
constexpr int kErrZeroRotor = 3;
constexpr int kErrNonFiniteRotor = 4;

// rotor.cpp:117-136.  Returns 0 or an error code.
__device__ __forceinline__ int d_normalize(const double* in, double* v) {
    bool finite = true;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        v[i] = in[i];
        finite = finite && isfinite(v[i]);
    }
    if (!finite) return kErrNonFiniteRotor;
    double l2 = sqnorm8(v);
    if (!(l2 > 1e-20)) return kErrZeroRotor;
    double eps = rotor_epsilon(v);
    if (fabs(eps) >= kEpsBranch) {
        double rad = smax(l2 * l2 - 4 * eps * eps, 0.0);
        double delta = -2 * eps / (l2 + sqrt(rad));
        double g[8];
        epsilon_gradient(v, g);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = v[i] + delta * g[i];
    }
    double nrm = sqrt(sqnorm8(v));
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        v[i] = v[i] / nrm;
        finite = finite && isfinite(v[i]);
    }
    if (!finite) return kErrNonFiniteRotor;
    if (fabs(rotor_epsilon(v)) > 1e-9 || fabs(sqnorm8(v) - 1) > 1e-9) return kErrNonFiniteRotor;
    return 0;
}

// rotor.cpp:18-51 / 170-181: one R4D entry as the reference's 8-term quadratic form
// (zero-coefficient slots included so signed zeros match).
#define RGS_QT(a, b, c) val += (c) * v[a] * v[b]
#define RGS_QZ val += 0.0 * v[0] * v[0]
// Four zero-coefficient terms: each adds 0.0 * v0 * v0 = +0 (v is finite after normalize), and
// adding +0 four times equals adding it once (it only turns -0 into +0).
#define RGS_QZ4 val += 0.0
__device__ __forceinline__ void d_to_matrix(const double* v, double* m) {
    double val;
    // R00
    val = 0; RGS_QT(0, 0, 1.0); RGS_QT(1, 1, -1.0); RGS_QT(2, 2, -1.0); RGS_QT(3, 3, -1.0);
    RGS_QT(4, 4, 1.0); RGS_QT(5, 5, 1.0); RGS_QT(6, 6, 1.0); RGS_QT(7, 7, -1.0); m[0] = val;
    // R01
    val = 0; RGS_QT(1, 0, 2.0); RGS_QT(2, 4, -2.0); RGS_QT(3, 5, -2.0); RGS_QT(6, 7, 2.0);
    RGS_QZ4; m[1] = val;
    // R02
    val = 0; RGS_QT(1, 4, 2.0); RGS_QT(2, 0, 2.0); RGS_QT(3, 6, -2.0); RGS_QT(5, 7, -2.0);
    RGS_QZ4; m[2] = val;
    // R03
    val = 0; RGS_QT(1, 5, 2.0); RGS_QT(2, 6, 2.0); RGS_QT(3, 0, 2.0); RGS_QT(4, 7, 2.0);
    RGS_QZ4; m[3] = val;
    // R10
    val = 0; RGS_QT(1, 0, -2.0); RGS_QT(2, 4, -2.0); RGS_QT(3, 5, -2.0); RGS_QT(6, 7, -2.0);
    RGS_QZ4; m[4] = val;
    // R11
    val = 0; RGS_QT(0, 0, 1.0); RGS_QT(1, 1, -1.0); RGS_QT(2, 2, 1.0); RGS_QT(3, 3, 1.0);
    RGS_QT(4, 4, -1.0); RGS_QT(5, 5, -1.0); RGS_QT(6, 6, 1.0); RGS_QT(7, 7, -1.0); m[5] = val;
    // R12
    val = 0; RGS_QT(1, 2, -2.0); RGS_QT(3, 7, 2.0); RGS_QT(4, 0, 2.0); RGS_QT(5, 6, -2.0);
    RGS_QZ4; m[6] = val;
    // R13
    val = 0; RGS_QT(1, 3, -2.0); RGS_QT(2, 7, -2.0); RGS_QT(4, 6, 2.0); RGS_QT(5, 0, 2.0);
    RGS_QZ4; m[7] = val;
    // R20
    val = 0; RGS_QT(1, 4, 2.0); RGS_QT(2, 0, -2.0); RGS_QT(3, 6, -2.0); RGS_QT(5, 7, 2.0);
    RGS_QZ4; m[8] = val;
    // R21
    val = 0; RGS_QT(1, 2, -2.0); RGS_QT(3, 7, -2.0); RGS_QT(4, 0, -2.0); RGS_QT(5, 6, -2.0);
    RGS_QZ4; m[9] = val;
    // R22
    val = 0; RGS_QT(0, 0, 1.0); RGS_QT(1, 1, 1.0); RGS_QT(2, 2, -1.0); RGS_QT(3, 3, 1.0);
    RGS_QT(4, 4, -1.0); RGS_QT(5, 5, 1.0); RGS_QT(6, 6, -1.0); RGS_QT(7, 7, -1.0); m[10] = val;
    // R23
    val = 0; RGS_QT(1, 7, 2.0); RGS_QT(2, 3, -2.0); RGS_QT(4, 5, -2.0); RGS_QT(6, 0, 2.0);
    RGS_QZ4; m[11] = val;
    // R30
    val = 0; RGS_QT(1, 5, 2.0); RGS_QT(2, 6, 2.0); RGS_QT(3, 0, -2.0); RGS_QT(4, 7, -2.0);
    RGS_QZ4; m[12] = val;
    // R31
    val = 0; RGS_QT(1, 3, -2.0); RGS_QT(2, 7, 2.0); RGS_QT(4, 6, 2.0); RGS_QT(5, 0, -2.0);
    RGS_QZ4; m[13] = val;
    // R32
    val = 0; RGS_QT(1, 7, -2.0); RGS_QT(2, 3, -2.0); RGS_QT(4, 5, -2.0); RGS_QT(6, 0, -2.0);
    RGS_QZ4; m[14] = val;
    // R33
    val = 0; RGS_QT(0, 0, 1.0); RGS_QT(1, 1, 1.0); RGS_QT(2, 2, 1.0); RGS_QT(3, 3, -1.0);
    RGS_QT(4, 4, 1.0); RGS_QT(5, 5, -1.0); RGS_QT(6, 6, -1.0); RGS_QT(7, 7, -1.0); m[15] = val;
}
#undef RGS_QT
#undef RGS_QZ
#undef RGS_QZ4

// SliceCache (gaussian.hpp:36-45) restricted to what the device needs.
struct SliceState {
    double nrm[8];
    double R[16];
    double q[4];
    double U[9];
    double V[3];
    double W;
    double dt;
    double decay;
    // outputs of slice_at (gaussian.cpp:32-47)
    double mean[3];
    double cov[9];
    double speed[3];
    double lambda;
};

// gaussian.cpp:9-17 + 32-40, the part of slice_at that does not depend on t: normalize,
// to_matrix, Sigma4 = R diag(q) R^T, the DegenerateTime check, lambda, speed and the Schur
// complement cov3.  Returns 0 (ok), an error code, or -1 for DegenerateTimeError (caught by
// build_splats -> Gaussian skipped).
__device__ __forceinline__ int d_slice_static(const double* ls, const double* rot, SliceState& s) {
    int rc = d_normalize(rot, s.nrm);
    if (rc) return rc;
    d_to_matrix(s.nrm, s.R);
#pragma unroll
    for (int k = 0; k < 4; ++k) s.q[k] = rgs_exp::glibc_exp(2 * ls[k]);
    // sigma = (R diag(q)) R^T, only the U, V, W entries are used.
    double m1[16];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) m1[i * 4 + j] = s.R[i * 4 + j] * s.q[j];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (i == 3 && j != 3) continue;
            double a = m1[i * 4 + 0] * s.R[j * 4 + 0];
#pragma unroll
            for (int k = 1; k < 4; ++k) a += m1[i * 4 + k] * s.R[j * 4 + k];
            if (i < 3 && j < 3) s.U[i * 3 + j] = a;
            else if (i < 3) s.V[i] = a;
            else s.W = a;
        }
    if (s.W < kTemporalFloor) return -1;
    s.lambda = 1 / s.W;
#pragma unroll
    for (int i = 0; i < 3; ++i) s.speed[i] = s.V[i] / s.W;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            double b = (s.V[i] * s.V[j]) / s.W;
            double d = kCov3Eps * (i == j ? 1.0 : 0.0);
            s.cov[i * 3 + j] = (s.U[i * 3 + j] - b) + d;
        }
    return 0;
}

// gaussian.cpp:41-44, the t-dependent rest: dt, the conditional mean and the temporal decay.
__device__ __forceinline__ void d_slice_time(const double* mean4, double t, SliceState& s) {
    s.dt = t - mean4[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) s.mean[i] = mean4[i] + s.dt * s.speed[i];
    s.decay = rgs_exp::glibc_exp(-0.5 * s.lambda * s.dt * s.dt);
}

// gaussian.cpp:9-17 + 32-47 (the same operations in the same order as the two halves above).
__device__ __forceinline__ int d_slice(const double* mean4, const double* ls, const double* rot, double t,
                                       SliceState& s) {
    const int rc = d_slice_static(ls, rot, s);
    if (rc) return rc;
    d_slice_time(mean4, t, s);
    return 0;
}

// sh.cpp:6-12
constexpr double kC0 = 0.28209479177387814;
constexpr double kC1 = 0.4886025119029199;
constexpr double kC2_0 = 1.0925484305920792, kC2_1 = -1.0925484305920792, kC2_2 = 0.31539156525252005,
                 kC2_3 = -1.0925484305920792, kC2_4 = 0.5462742152960396;
constexpr double kC3_0 = -0.5900435899266435, kC3_1 = 2.890611442640554, kC3_2 = -0.4570457994644658,
                 kC3_3 = 0.3731763325901154, kC3_4 = -0.4570457994644658, kC3_5 = 1.445305721320277,
                 kC3_6 = -0.5900435899266435;

// sh.cpp:16-85 (values).  Entries beyond the degree are zero.
__device__ __forceinline__ void d_sh_basis(const double* dir, int degree, double* b) {
    const double x = dir[0], y = dir[1], z = dir[2];
#pragma unroll
    for (int k = 0; k < 16; ++k) b[k] = 0;
    b[0] = kC0;
    if (degree >= 1) {
        b[1] = -kC1 * y;
        b[2] = kC1 * z;
        b[3] = -kC1 * x;
    }
    if (degree >= 2) {
        const double xx = x * x, yy = y * y, zz = z * z;
        b[4] = kC2_0 * x * y;
        b[5] = kC2_1 * y * z;
        b[6] = kC2_2 * (2 * zz - xx - yy);
        b[7] = kC2_3 * x * z;
        b[8] = kC2_4 * (xx - yy);
    }
    if (degree >= 3) {
        const double xx = x * x, yy = y * y, zz = z * z;
        b[9] = kC3_0 * y * (3 * xx - yy);
        b[10] = kC3_1 * x * y * z;
        b[11] = kC3_2 * y * (4 * zz - xx - yy);
        b[12] = kC3_3 * z * (2 * zz - 3 * xx - 3 * yy);
        b[13] = kC3_4 * x * (4 * zz - xx - yy);
        b[14] = kC3_5 * z * (xx - yy);
        b[15] = kC3_6 * x * (xx - 3 * yy);
    }
}

// Basis entry k of d_sh_basis (the same expression; k a compile-time constant in unrolled loops,
// so a caller can compute each entry where it is used instead of keeping all 16 live).
template <int K>
__device__ __forceinline__ double d_sh_basis_k(double x, double y, double z, double xx, double yy, double zz) {
    if constexpr (K == 0) return kC0;
    else if constexpr (K == 1) return -kC1 * y;
    else if constexpr (K == 2) return kC1 * z;
    else if constexpr (K == 3) return -kC1 * x;
    else if constexpr (K == 4) return kC2_0 * x * y;
    else if constexpr (K == 5) return kC2_1 * y * z;
    else if constexpr (K == 6) return kC2_2 * (2 * zz - xx - yy);
    else if constexpr (K == 7) return kC2_3 * x * z;
    else if constexpr (K == 8) return kC2_4 * (xx - yy);
    else if constexpr (K == 9) return kC3_0 * y * (3 * xx - yy);
    else if constexpr (K == 10) return kC3_1 * x * y * z;
    else if constexpr (K == 11) return kC3_2 * y * (4 * zz - xx - yy);
    else if constexpr (K == 12) return kC3_3 * z * (2 * zz - 3 * xx - 3 * yy);
    else if constexpr (K == 13) return kC3_4 * x * (4 * zz - xx - yy);
    else if constexpr (K == 14) return kC3_5 * z * (xx - yy);
    else return kC3_6 * x * (xx - 3 * yy);
}

__device__ __forceinline__ double d_sh_basis_at(int k, double x, double y, double z, double xx, double yy,
                                                double zz) {
    switch (k) {
        case 0: return d_sh_basis_k<0>(x, y, z, xx, yy, zz);
        case 1: return d_sh_basis_k<1>(x, y, z, xx, yy, zz);
        case 2: return d_sh_basis_k<2>(x, y, z, xx, yy, zz);
        case 3: return d_sh_basis_k<3>(x, y, z, xx, yy, zz);
        case 4: return d_sh_basis_k<4>(x, y, z, xx, yy, zz);
        case 5: return d_sh_basis_k<5>(x, y, z, xx, yy, zz);
        case 6: return d_sh_basis_k<6>(x, y, z, xx, yy, zz);
        case 7: return d_sh_basis_k<7>(x, y, z, xx, yy, zz);
        case 8: return d_sh_basis_k<8>(x, y, z, xx, yy, zz);
        case 9: return d_sh_basis_k<9>(x, y, z, xx, yy, zz);
        case 10: return d_sh_basis_k<10>(x, y, z, xx, yy, zz);
        case 11: return d_sh_basis_k<11>(x, y, z, xx, yy, zz);
        case 12: return d_sh_basis_k<12>(x, y, z, xx, yy, zz);
        case 13: return d_sh_basis_k<13>(x, y, z, xx, yy, zz);
        case 14: return d_sh_basis_k<14>(x, y, z, xx, yy, zz);
        default: return d_sh_basis_k<15>(x, y, z, xx, yy, zz);
    }
}

// sh.cpp:40-83 (direction gradient, 16x3 row-major; entries beyond degree zero).
__device__ __forceinline__ void d_sh_basis_grad(const double* dir, int degree, double* g) {
    const double x = dir[0], y = dir[1], z = dir[2];
#pragma unroll
    for (int k = 0; k < 48; ++k) g[k] = 0;
    if (degree >= 1) {
        g[1 * 3 + 1] = -kC1;
        g[2 * 3 + 2] = kC1;
        g[3 * 3 + 0] = -kC1;
    }
    if (degree >= 2) {
        g[4 * 3 + 0] = kC2_0 * y;
        g[4 * 3 + 1] = kC2_0 * x;
        g[5 * 3 + 1] = kC2_1 * z;
        g[5 * 3 + 2] = kC2_1 * y;
        g[6 * 3 + 0] = kC2_2 * -2 * x;
        g[6 * 3 + 1] = kC2_2 * -2 * y;
        g[6 * 3 + 2] = kC2_2 * 4 * z;
        g[7 * 3 + 0] = kC2_3 * z;
        g[7 * 3 + 2] = kC2_3 * x;
        g[8 * 3 + 0] = kC2_4 * 2 * x;
        g[8 * 3 + 1] = kC2_4 * -2 * y;
    }
    if (degree >= 3) {
        const double xx = x * x, yy = y * y, zz = z * z;
        g[9 * 3 + 0] = kC3_0 * 6 * x * y;
        g[9 * 3 + 1] = kC3_0 * (3 * xx - 3 * yy);
        g[10 * 3 + 0] = kC3_1 * y * z;
        g[10 * 3 + 1] = kC3_1 * x * z;
        g[10 * 3 + 2] = kC3_1 * x * y;
        g[11 * 3 + 0] = kC3_2 * -2 * x * y;
        g[11 * 3 + 1] = kC3_2 * (4 * zz - xx - 3 * yy);
        g[11 * 3 + 2] = kC3_2 * 8 * y * z;
        g[12 * 3 + 0] = kC3_3 * -6 * x * z;
        g[12 * 3 + 1] = kC3_3 * -6 * y * z;
        g[12 * 3 + 2] = kC3_3 * (6 * zz - 3 * xx - 3 * yy);
        g[13 * 3 + 0] = kC3_4 * (4 * zz - 3 * xx - yy);
        g[13 * 3 + 1] = kC3_4 * -2 * x * y;
        g[13 * 3 + 2] = kC3_4 * 8 * x * z;
        g[14 * 3 + 0] = kC3_5 * 2 * x * z;
        g[14 * 3 + 1] = kC3_5 * -2 * y * z;
        g[14 * 3 + 2] = kC3_5 * (xx - yy);
        g[15 * 3 + 0] = kC3_6 * (3 * xx - 3 * yy);
        g[15 * 3 + 1] = kC3_6 * -6 * x * y;
    }
}

// Row k of d_sh_basis_grad (the same expressions, so the same values), for loops that want
// one row at a time instead of the 48-entry array (K7a).
template <int K>
__device__ __forceinline__ void d_sh_basis_grad_row(double x, double y, double z, int degree, double* g) {
    g[0] = g[1] = g[2] = 0;
    if constexpr (K >= 1 && K <= 3) {
        if (degree >= 1) {
            if constexpr (K == 1) g[1] = -kC1;
            if constexpr (K == 2) g[2] = kC1;
            if constexpr (K == 3) g[0] = -kC1;
        }
    } else if constexpr (K >= 4 && K <= 8) {
        if (degree >= 2) {
            if constexpr (K == 4) {
                g[0] = kC2_0 * y;
                g[1] = kC2_0 * x;
            }
            if constexpr (K == 5) {
                g[1] = kC2_1 * z;
                g[2] = kC2_1 * y;
            }
            if constexpr (K == 6) {
                g[0] = kC2_2 * -2 * x;
                g[1] = kC2_2 * -2 * y;
                g[2] = kC2_2 * 4 * z;
            }
            if constexpr (K == 7) {
                g[0] = kC2_3 * z;
                g[2] = kC2_3 * x;
            }
            if constexpr (K == 8) {
                g[0] = kC2_4 * 2 * x;
                g[1] = kC2_4 * -2 * y;
            }
        }
    } else if constexpr (K >= 9) {
        if (degree >= 3) {
            const double xx = x * x, yy = y * y, zz = z * z;
            if constexpr (K == 9) {
                g[0] = kC3_0 * 6 * x * y;
                g[1] = kC3_0 * (3 * xx - 3 * yy);
            }
            if constexpr (K == 10) {
                g[0] = kC3_1 * y * z;
                g[1] = kC3_1 * x * z;
                g[2] = kC3_1 * x * y;
            }
            if constexpr (K == 11) {
                g[0] = kC3_2 * -2 * x * y;
                g[1] = kC3_2 * (4 * zz - xx - 3 * yy);
                g[2] = kC3_2 * 8 * y * z;
            }
            if constexpr (K == 12) {
                g[0] = kC3_3 * -6 * x * z;
                g[1] = kC3_3 * -6 * y * z;
                g[2] = kC3_3 * (6 * zz - 3 * xx - 3 * yy);
            }
            if constexpr (K == 13) {
                g[0] = kC3_4 * (4 * zz - 3 * xx - yy);
                g[1] = kC3_4 * -2 * x * y;
                g[2] = kC3_4 * 8 * x * z;
            }
            if constexpr (K == 14) {
                g[0] = kC3_5 * 2 * x * z;
                g[1] = kC3_5 * -2 * y * z;
                g[2] = kC3_5 * (xx - yy);
            }
            if constexpr (K == 15) {
                g[0] = kC3_6 * (3 * xx - 3 * yy);
                g[1] = kC3_6 * -6 * x * y;
            }
        }
    }
}

// ProjectCache subset (rasterizer.hpp:33-48) + the Splat2D outputs.
struct ProjState {
    double p[3];
    double T[6];  // J R, 2x3 row-major
    double cov2[4];
    double det;
    double mean2[2];
    double conic[3];
    double radius;
    double opacity;
    double alpha_base;
    double dir[3];
    double dist;
};

// rasterizer.cpp:215-243 geometric part (everything but SH colour / flow).
// Returns true when the splat survives the culls.
// `opacity_in`: the opacity logit, or (PRE_OPACITY) the opacity sigmoid(logit) already evaluated
// with the same expression (the per-scene slice cache of a batch).
template <bool PRE_OPACITY = false>
__device__ __forceinline__ bool d_project_geom(const SliceState& s, const DevCamera& cam, double opacity_in,
                                               ProjState& o) {
    const double opacity_logit = opacity_in;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        double a = cam.R[i * 3 + 0] * s.mean[0];
        a += cam.R[i * 3 + 1] * s.mean[1];
        a += cam.R[i * 3 + 2] * s.mean[2];
        o.p[i] = a + cam.t[i];
    }
    if (o.p[2] <= kNearPlane) return false;
    o.mean2[0] = cam.fx * o.p[0] / o.p[2] + cam.cx;
    o.mean2[1] = cam.fy * o.p[1] / o.p[2] + cam.cy;
    // projection_jacobian (rasterizer.cpp:14-20)
    const double z = o.p[2], z2 = z * z;
    double J[6];
    J[0] = cam.fx / z;
    J[1] = 0;
    J[2] = -cam.fx * o.p[0] / z2;
    J[3] = 0;
    J[4] = cam.fy / z;
    J[5] = -cam.fy * o.p[1] / z2;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            double a = J[i * 3 + 0] * cam.R[0 * 3 + j];
            a += J[i * 3 + 1] * cam.R[1 * 3 + j];
            a += J[i * 3 + 2] * cam.R[2 * 3 + j];
            o.T[i * 3 + j] = a;
        }
    double A[6];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            double a = o.T[i * 3 + 0] * s.cov[0 * 3 + j];
            a += o.T[i * 3 + 1] * s.cov[1 * 3 + j];
            a += o.T[i * 3 + 2] * s.cov[2 * 3 + j];
            A[i * 3 + j] = a;
        }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            double a = A[i * 3 + 0] * o.T[j * 3 + 0];
            a += A[i * 3 + 1] * o.T[j * 3 + 1];
            a += A[i * 3 + 2] * o.T[j * 3 + 2];
            o.cov2[i * 2 + j] = a + kCovDilation * (i == j ? 1.0 : 0.0);
        }
    o.det = o.cov2[0] * o.cov2[3] - o.cov2[2] * o.cov2[1];
    if (o.det <= 0) return false;
    const double invdet = 1.0 / o.det;
    o.conic[0] = o.cov2[3] * invdet;
    o.conic[1] = -o.cov2[1] * invdet;
    o.conic[2] = o.cov2[0] * invdet;
    const double mid = 0.5 * (o.cov2[0] + o.cov2[3]);
    const double max_eig = mid + sqrt(smax(0.01, mid * mid - o.det));
    o.radius = 3 * sqrt(max_eig);
    if (o.mean2[0] + o.radius < 0 || o.mean2[0] - o.radius > cam.width - 1 || o.mean2[1] + o.radius < 0 ||
        o.mean2[1] - o.radius > cam.height - 1)
        return false;
    o.opacity = PRE_OPACITY ? opacity_in : 1 / (1 + rgs_exp::glibc_exp(-opacity_logit));
    o.alpha_base = o.opacity * s.decay;
    if (o.alpha_base < kMinAlpha) return false;
    double v[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) v[i] = s.mean[i] - cam.center[i];
    o.dist = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    if (o.dist > 0) {
#pragma unroll
        for (int i = 0; i < 3; ++i) o.dir[i] = v[i] / o.dist;
    } else {
        o.dir[0] = 0;
        o.dir[1] = 0;
        o.dir[2] = 1;
    }
    return true;
}


// gaussian.cpp:84-100 + rotor.cpp:138-194: the tail of slice_backward shared by the
// render backward (K7) and the consistency regularizer -- from the 4x4 covariance
// gradient G4 to d log_scales (out[4..7]) and d rotor (out[8..15], w.r.t. the stored,
// pre-normalisation coefficients `rot`), accumulated.
__device__ __forceinline__ void d_g4_backward(const SliceState& s, const double* rot, const double* G4,
                                              double* out) {
    // d log_scales: 2 q_k (R^T G4 R)_kk
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        double acc = 0;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            double ga = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) ga += G4[a * 4 + b] * s.R[b * 4 + k];
            acc += s.R[a * 4 + k] * ga;
        }
        out[4 + k] += 2 * s.q[k] * acc;
    }
    // dL/dR = (G4 + G4^T) R diag(q)
    double dR[16];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            double a = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) a += (G4[r * 4 + k] + G4[k * 4 + r]) * s.R[k * 4 + c];
            dR[r * 4 + c] = a * s.q[c];
        }
    // through the quadratic forms (to_matrix_jacobian, rotor.cpp:183-194)
    const double* v = s.nrm;
    double drn[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define RGS_JT(e, a, b, c)               \
drn[a] += dR[e] * (c) * v[b];         \
drn[b] += dR[e] * (c) * v[a];
    RGS_JT(0, 0, 0, 1.0) RGS_JT(0, 1, 1, -1.0) RGS_JT(0, 2, 2, -1.0) RGS_JT(0, 3, 3, -1.0)
    RGS_JT(0, 4, 4, 1.0) RGS_JT(0, 5, 5, 1.0) RGS_JT(0, 6, 6, 1.0) RGS_JT(0, 7, 7, -1.0)
    RGS_JT(1, 1, 0, 2.0) RGS_JT(1, 2, 4, -2.0) RGS_JT(1, 3, 5, -2.0) RGS_JT(1, 6, 7, 2.0)
    RGS_JT(2, 1, 4, 2.0) RGS_JT(2, 2, 0, 2.0) RGS_JT(2, 3, 6, -2.0) RGS_JT(2, 5, 7, -2.0)
    RGS_JT(3, 1, 5, 2.0) RGS_JT(3, 2, 6, 2.0) RGS_JT(3, 3, 0, 2.0) RGS_JT(3, 4, 7, 2.0)
    RGS_JT(4, 1, 0, -2.0) RGS_JT(4, 2, 4, -2.0) RGS_JT(4, 3, 5, -2.0) RGS_JT(4, 6, 7, -2.0)
    RGS_JT(5, 0, 0, 1.0) RGS_JT(5, 1, 1, -1.0) RGS_JT(5, 2, 2, 1.0) RGS_JT(5, 3, 3, 1.0)
    RGS_JT(5, 4, 4, -1.0) RGS_JT(5, 5, 5, -1.0) RGS_JT(5, 6, 6, 1.0) RGS_JT(5, 7, 7, -1.0)
    RGS_JT(6, 1, 2, -2.0) RGS_JT(6, 3, 7, 2.0) RGS_JT(6, 4, 0, 2.0) RGS_JT(6, 5, 6, -2.0)
    RGS_JT(7, 1, 3, -2.0) RGS_JT(7, 2, 7, -2.0) RGS_JT(7, 4, 6, 2.0) RGS_JT(7, 5, 0, 2.0)
    RGS_JT(8, 1, 4, 2.0) RGS_JT(8, 2, 0, -2.0) RGS_JT(8, 3, 6, -2.0) RGS_JT(8, 5, 7, 2.0)
    RGS_JT(9, 1, 2, -2.0) RGS_JT(9, 3, 7, -2.0) RGS_JT(9, 4, 0, -2.0) RGS_JT(9, 5, 6, -2.0)
    RGS_JT(10, 0, 0, 1.0) RGS_JT(10, 1, 1, 1.0) RGS_JT(10, 2, 2, -1.0) RGS_JT(10, 3, 3, 1.0)
    RGS_JT(10, 4, 4, -1.0) RGS_JT(10, 5, 5, 1.0) RGS_JT(10, 6, 6, -1.0) RGS_JT(10, 7, 7, -1.0)
    RGS_JT(11, 1, 7, 2.0) RGS_JT(11, 2, 3, -2.0) RGS_JT(11, 4, 5, -2.0) RGS_JT(11, 6, 0, 2.0)
    RGS_JT(12, 1, 5, 2.0) RGS_JT(12, 2, 6, 2.0) RGS_JT(12, 3, 0, -2.0) RGS_JT(12, 4, 7, -2.0)
    RGS_JT(13, 1, 3, -2.0) RGS_JT(13, 2, 7, 2.0) RGS_JT(13, 4, 6, 2.0) RGS_JT(13, 5, 0, -2.0)
    RGS_JT(14, 1, 7, -2.0) RGS_JT(14, 2, 3, -2.0) RGS_JT(14, 4, 5, -2.0) RGS_JT(14, 6, 0, -2.0)
    RGS_JT(15, 0, 0, 1.0) RGS_JT(15, 1, 1, 1.0) RGS_JT(15, 2, 2, 1.0) RGS_JT(15, 3, 3, -1.0)
    RGS_JT(15, 4, 4, 1.0) RGS_JT(15, 5, 5, -1.0) RGS_JT(15, 6, 6, -1.0) RGS_JT(15, 7, 7, -1.0)
#undef RGS_JT
    // normalize_jacobian^T (rotor.cpp:138-168): Jn^T w = j1^T (j2^T w), j2 symmetric.
    double l2 = sqnorm8(rot);
    double eps = rotor_epsilon(rot);
    double grad[8], upd[8];
    epsilon_gradient(rot, grad);
#pragma unroll
    for (int k = 0; k < 8; ++k) upd[k] = rot[k];
    double delta = 0, ddr[8];
    const bool branch = fabs(eps) >= kEpsBranch;
    if (branch) {
        const double rad = smax(l2 * l2 - 4 * eps * eps, 0.0);
        const double sq = smax(sqrt(rad), 1e-30);
        const double den = l2 + sq;
        delta = -2 * eps / den;
        const double dde = -2 / den - 8 * eps * eps / (sq * den * den);
        const double ddl = 2 * eps * (1 + l2 / sq) / (den * den);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            ddr[k] = dde * grad[k] + ddl * 2 * rot[k];
            upd[k] = rot[k] + delta * grad[k];
        }
    }
    const double len = sqrt(sqnorm8(upd));
    double u[8], w2[8];
    double udot = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        u[k] = upd[k] / len;
        udot += u[k] * drn[k];
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) w2[k] = (drn[k] - u[k] * udot) / len;
    double gdot = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) gdot += grad[k] * w2[k];
    // epsilon Hessian pairs: (0,7)=+1, (1,6)=-1, (2,5)=+1, (3,4)=-1
    const double Hw[8] = {w2[7], -w2[6], w2[5], -w2[4], -w2[3], w2[2], -w2[1], w2[0]};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        double r;
        if (branch) r = w2[k] + ddr[k] * gdot + delta * Hw[k];
        else r = w2[k] - grad[k] * gdot / l2;
        out[8 + k] += r;
    }
}

}  // namespace rgs_dev
