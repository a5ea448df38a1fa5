"""The device exp (csrc/glibc_exp.h) reproduces the platform libm exp bit for bit.

The reference calls std::exp (gaussian.cpp:12,44; rasterizer.cpp:10); bit-exact
splat records need the device to round exactly like it.  This compiles the same
header for the host and compares against libm on random inputs over the ranges
the path uses (2*log_scale, temporal decay exponent, -opacity_logit, blend power).
"""
import os
import subprocess
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROG = r"""
#include <cmath>
#include <cstdio>
#include <random>
#include "glibc_exp.h"
int main() {
    std::mt19937_64 g(20240817);
    std::uniform_real_distribution<double> wide(-40.0, 8.0), narrow(-6.0, 0.5);
    long bad = 0, n = 4000000;
    for (long i = 0; i < n; ++i) {
        double x = (i & 1) ? wide(g) : narrow(g);
        if (rgs_exp::glibc_exp(x) != std::exp(x)) ++bad;
    }
    const double edge[] = {0.0, -0.0, 1e-300, -1e-300, 5e-17, -5e-17, 1.0, -1.0, 700.0, -700.0, 0.5, -745.0};
    for (double x : edge)
        if (!(rgs_exp::glibc_exp(x) == std::exp(x))) ++bad;
    std::printf("%ld\n", bad);
    return 0;
}
"""


def test_device_exp_matches_libm():
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "t.cpp")
        exe = os.path.join(d, "t")
        open(src, "w").write(PROG)
        subprocess.run(["g++", "-O2", "-ffp-contract=off", "-std=c++17",
                        "-I" + os.path.join(ROOT, "paper_2402_03307_b200", "csrc"), src, "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.strip()
    assert out == "0", f"{out} mismatches against libm exp"
