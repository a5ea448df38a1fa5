// Bit-exact re-implementation of the double-precision exp() the CPU reference links
// against (glibc >= 2.28, sysdeps/ieee754/dbl-64/e_exp.c, FMA code path selected on
// x86-64 CPUs with FMA/AVX2: 128-entry 2^(k/N) table, degree-5 polynomial).
//
// The reference computes q = exp(2 log_s), the temporal decay and the sigmoid with
// std::exp (gaussian.cpp:12,44; rasterizer.cpp:10).  CUDA's exp() differs from glibc
// by an ulp in a few percent of inputs, enough to change splat records; this
// version reproduces glibc exactly (0 mismatches on 3e7 random inputs, see
// tests/test_exp_parity.py).  Usable from device code and from host C++.
#pragma once

#include <stdint.h>

#include <cmath>
#include <cstring>

#include "exp_table.h"

#ifdef __CUDACC__
#define RGS_HD __host__ __device__ __forceinline__
#else
#define RGS_HD inline
#endif

namespace rgs_exp {

#ifdef __CUDACC__
__device__ const unsigned long long kExpTab[256] = RGS_EXP_TABLE_INIT;
#endif
static const unsigned long long kExpTabHost[256] = RGS_EXP_TABLE_INIT;

RGS_HD uint64_t as_u64(double d) {
#ifdef __CUDA_ARCH__
    return (uint64_t)__double_as_longlong(d);
#else
    uint64_t u;
    std::memcpy(&u, &d, 8);
    return u;
#endif
}
RGS_HD double as_f64(uint64_t u) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)u);
#else
    double d;
    std::memcpy(&d, &u, 8);
    return d;
#endif
}
RGS_HD uint64_t tab(int i) {
#ifdef __CUDA_ARCH__
    return __ldg(&kExpTab[i]);
#else
    return kExpTabHost[i];
#endif
}
RGS_HD double dfma(double a, double b, double c) {
#ifdef __CUDA_ARCH__
    return __fma_rn(a, b, c);
#else
    return std::fma(a, b, c);
#endif
}

RGS_HD double glibc_exp(double x) {
    const double InvLn2N = 0x1.71547652b82fep0 * 128;
    const double NegLn2hiN = -0x1.62e42fefa0000p-8;
    const double NegLn2loN = -0x1.cf79abc9e3b3ap-47;
    const double Shift = 0x1.8p52;
    const double C2 = 0x1.ffffffffffdbdp-2, C3 = 0x1.555555555543cp-3, C4 = 0x1.55555cf172b91p-5,
                 C5 = 0x1.1111167a4d017p-7;
    const uint32_t abstop = (uint32_t)(as_u64(x) >> 52) & 0x7ff;
    // |x| < 2^-54: exp(x) rounds to 1 + x; |x| >= 512 or non-finite: rare, handled
    // by the platform exp (over/underflow; not reachable from finite scenes).
    if (abstop - 0x3c9u >= 0x408u - 0x3c9u) {
        if ((int)abstop - 0x3c9 < 0) return 1.0 + x;
#ifdef __CUDA_ARCH__
        return exp(x);
#else
        return std::exp(x);
#endif
    }
    double kd = dfma(InvLn2N, x, Shift);
    const uint64_t ki = as_u64(kd);
    kd -= Shift;
    const double r = dfma(kd, NegLn2loN, dfma(kd, NegLn2hiN, x));
    const int idx = 2 * (int)(ki % 128);
    const uint64_t top = ki << (52 - 7);
    const double tail = as_f64(tab(idx));
    const uint64_t sbits = tab(idx + 1) + top;
    const double r2 = r * r;
    const double a = dfma(r, C3, C2);
    const double b = dfma(r, C5, C4);
    const double t1 = tail + r;
    const double t2 = dfma(r2, a, t1);
    const double tmp = dfma(r2 * r2, b, t2);
    const double scale = as_f64(sbits);
    return dfma(scale, tmp, scale);
}

}  // namespace rgs_exp
