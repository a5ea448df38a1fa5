// Training-side kernels either side of the render path:
//
//   K8a k_ssim_fields   SSIM forward on the valid region + the per-position adjoint
//                       seeds (ssim.cpp:74-125), block partial sums of SSIM
//   K8b k_image_grad    adjoint convolutions (ssim.cpp:61-72, as gathers in the
//                       reference's summation order) + L1 gradient (image.cpp:27-36)
//                       -> dL/dimage = w_l1 g_l1 + w_ssim g_ssim (trainer.cpp:41-50),
//                       block partial sums of |d| and d^2 (l1_loss, psnr)
//   K9  k_adam_step     optim.cpp:110-166 fused: entropy gradient (loss.cpp:16-31,
//                       trainer.cpp:55-64), accumulate_stats, Adam on all 65
//                       parameters, rotor re-normalisation, static-mode masks
//   K10 k_speeds / k_consistency / k_speed_backward
//                       consistency regularizer (loss.cpp:33-58, trainer.cpp:66-77)
//   K11 k_knn_grid      exact 4D k-nearest neighbours (knn.cpp:101-116) through a uniform grid
//       k_reset_opacity optim.cpp:236-243
//
// This TU is compiled with -fmad=false and keeps the reference's expression order, so
// on identical inputs the SSIM/L1 image gradient, the Adam update (FP64 scenes) and the
// neighbour lists are bit-identical to the reference; only block reductions of loss
// scalars (fixed-order trees) and libm log in the entropy term differ in the last ulps.
#include "fp64_math.cuh"
#include "rgs_train.cuh"

namespace rgs_dev {

__constant__ double c_win[kSsimWin];

// ---------------------------------------------------------------------------
// Deterministic block reduction of one double (256 threads).
__device__ __forceinline__ double block_sum(double v, double* red) {
    const int t = threadIdx.x;
    red[t] = v;
    __syncthreads();
#pragma unroll
    for (int s = 128; s > 0; s >>= 1) {
        if (t < s) red[t] = red[t] + red[t + s];
        __syncthreads();
    }
    const double r = red[0];
    __syncthreads();
    return r;
}

// ---------------------------------------------------------------------------
// Deterministic block reduction of one double over NT threads.
template <int NT>
__device__ __forceinline__ double block_sum_n(double v, double* red) {
    const int t = threadIdx.x;
    red[t] = v;
    __syncthreads();
#pragma unroll
    for (int s = NT / 2; s > 0; s >>= 1) {
        if (t < s) red[t] = red[t] + red[t + s];
        __syncthreads();
    }
    const double r = red[0];
    __syncthreads();
    return r;
}

// K8a: SSIM forward over one tile of valid positions and one channel.
// Tile: kSsimTX x kSsimATY valid positions (512 threads); input footprint (TX+10) x (TY+10).
// K8a dynamic shared memory (see the layout in the kernel).
template <typename TI>
constexpr size_t k8a_smem_bytes() {
    constexpr int IY = kSsimATY + kSsimWin - 1, IX = kSsimTX + kSsimWin - 1;
    return sizeof(double) * (5 * IY * kSsimTX + kSsimAThreads) + sizeof(TI) * 2 * IY * (IX + 1);
}

template <typename TI>
__global__ void __launch_bounds__(kSsimAThreads, 3) k_ssim_fields(const TI* __restrict__ img, const TI* __restrict__ tgt,
                                                     int W, int H, int want_grad, double* __restrict__ dfield,
                                                     double* __restrict__ part_ssim) {
    constexpr int TX = kSsimTX, TY = kSsimATY, IX = TX + kSsimWin - 1, IY = TY + kSsimWin - 1;
    // dynamic shared memory: rows[5][IY][TX] and red[] (double), then sa / sb [IY][IX + 1] (TI)
    // (the products a*a, b*b, a*b are formed per tap in registers: staging them in shared
    // memory as doubles measured 13% slower -- the taps are shared-memory bound, not FP64)
    extern __shared__ double k8a_smem[];
    auto rows = reinterpret_cast<double (*)[IY][TX]>(k8a_smem);
    double* red = k8a_smem + 5 * IY * TX;
    auto sa = reinterpret_cast<TI (*)[IX + 1]>(red + kSsimAThreads);
    auto sb = reinterpret_cast<TI (*)[IX + 1]>(reinterpret_cast<TI*>(red + kSsimAThreads) + IY * (IX + 1));
    const int vw = W - kSsimWin + 1, vh = H - kSsimWin + 1;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY, ch = blockIdx.z;
    const int t = threadIdx.x;
    for (int e = t; e < IY * IX; e += kSsimAThreads) {
        const int r = e / IX, c = e % IX;
        const int gx = x0 + c, gy = y0 + r;
        TI a = 0, b = 0;
        if (gx < W && gy < H) {
            const size_t p = ((size_t)gy * W + gx) * 3 + ch;
            a = img[p];
            b = tgt[p];
        }
        sa[r][c] = a;
        sb[r][c] = b;
    }
    __syncthreads();
    // Horizontal pass (ssim.cpp:44-49): rows(x, y) = sum_i k_i in(x + i, y), from 0.
    for (int e = t; e < IY * TX; e += kSsimAThreads) {
        const int r = e / TX, c = e % TX;
        double s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0;
#pragma unroll
        for (int i = 0; i < kSsimWin; ++i) {
            const double a = sa[r][c + i], b = sb[r][c + i];
            const double k = c_win[i];
            s0 += k * a;
            s1 += k * b;
            s2 += k * (a * a);
            s3 += k * (b * b);
            s4 += k * (a * b);
        }
        rows[0][r][c] = s0;
        rows[1][r][c] = s1;
        rows[2][r][c] = s2;
        rows[3][r][c] = s3;
        rows[4][r][c] = s4;
    }
    __syncthreads();
    const int c = t % TX, r = t / TX;
    const int vx = x0 + c, vy = y0 + r;
    double ssim = 0;
    if (vx < vw && vy < vh) {
        double m[5];
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            double s = 0;
#pragma unroll
            for (int i = 0; i < kSsimWin; ++i) s += c_win[i] * rows[q][r + i][c];
            m[q] = s;
        }
        const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
        const double ux = m[0], uy = m[1];
        const double vx2 = m[2] - ux * ux;
        const double vy2 = m[3] - uy * uy;
        const double vxy = m[4] - ux * uy;
        const double a1 = 2 * ux * uy + C1, a2 = 2 * vxy + C2;
        const double b1 = ux * ux + uy * uy + C1, b2 = vx2 + vy2 + C2;
        ssim = (a1 * a2) / (b1 * b2);
        if (want_grad) {
            // ssim.cpp:104-120
            const double d_ssim = 1;
            const double d_a1 = d_ssim * a2 / (b1 * b2);
            const double d_a2 = d_ssim * a1 / (b1 * b2);
            const double d_b1 = -d_ssim * ssim / b1;
            const double d_b2 = -d_ssim * ssim / b2;
            double d_ux = d_a1 * 2 * uy + d_b1 * 2 * ux;
            const double d_vx = d_b2;
            const double d_vxy = d_a2 * 2;
            d_ux += -2 * ux * d_vx - uy * d_vxy;
            const size_t nv = (size_t)vw * vh, p = (size_t)vy * vw + vx;
            double* base = dfield + (size_t)ch * 3 * nv;
            base[p] = d_ux;
            base[nv + p] = d_vx;
            base[2 * nv + p] = d_vxy;
        }
    }
    const double s = block_sum_n<kSsimAThreads>(ssim, red);
    if (t == 0)
        part_ssim[((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = s;
}

// K8b: per output pixel and channel: adjoint convolutions of the three seeds, the SSIM
// gradient, the L1 gradient and their weighted sum (FP32 dL/dimage for render_backward).
template <typename TI, typename TO>
__global__ void __launch_bounds__(kSsimAThreads) k_image_grad(const TI* __restrict__ img, const TI* __restrict__ tgt,
                                                    int W, int H, const double* __restrict__ dfield,
                                                    ImageGradArgs a, TO* __restrict__ dl,
                                                    double* __restrict__ part_l1, double* __restrict__ part_sq) {
    constexpr int TX = kSsimTX, TY = kSsimATY, DX = TX + kSsimWin - 1, DY = TY + kSsimWin - 1;
    __shared__ double sd[3][DY][DX];
    __shared__ double cols[3][TY][DX];
    __shared__ double red[kSsimAThreads];
    const int vw = W - kSsimWin + 1, vh = H - kSsimWin + 1;
    const int X0 = blockIdx.x * TX, Y0 = blockIdx.y * TY, ch = blockIdx.z;
    const int dx0 = X0 - (kSsimWin - 1), dy0 = Y0 - (kSsimWin - 1);
    const int t = threadIdx.x;
    const bool grad = dl != nullptr;
    if (grad && a.w_ssim != 0) {
        const size_t nv = (size_t)vw * vh;
        const double* base = dfield + (size_t)ch * 3 * nv;
        for (int e = t; e < 3 * DY * DX; e += kSsimAThreads) {
            const int q = e / (DY * DX), rem = e % (DY * DX), r = rem / DX, c = rem % DX;
            const int x = dx0 + c, y = dy0 + r;
            sd[q][r][c] = (x >= 0 && y >= 0 && x < vw && y < vh) ? base[q * nv + (size_t)y * vw + x] : 0.0;
        }
        __syncthreads();
        // cols(x, Y) = sum over y ascending of k[Y - y] g(x, y)   (ssim.cpp:64-67)
        for (int e = t; e < 3 * TY * DX; e += kSsimAThreads) {
            const int q = e / (TY * DX), rem = e % (TY * DX), r = rem / DX, c = rem % DX;
            // y = Y - 10 + i ascending; rows outside the valid region are zero in sd, so the
            // fixed 11 taps add +0 there and the sum equals the reference's clipped one
            double s = 0;
#pragma unroll
            for (int i = 0; i < kSsimWin; ++i) s += c_win[kSsimWin - 1 - i] * sd[q][r + i][c];
            cols[q][r][c] = s;
        }
        __syncthreads();
    }
    const int c = t % TX, r = t / TX;
    const int X = X0 + c, Y = Y0 + r;
    double l1 = 0, sq = 0;
    if (X < W && Y < H) {
        const size_t p = ((size_t)Y * W + X) * 3 + ch;
        const double xv = img[p], yv = tgt[p];
        const double d = xv - yv;
        l1 = fabs(d);
        sq = d * d;
        if (grad) {
            double g_ssim = 0;
            if (a.w_ssim != 0) {
                // out(X, y) = sum over x ascending of k[X - x] cols(x, y)   (ssim.cpp:68-71)
                // x = X - 10 + i ascending; columns outside the valid region are zero in cols
                double g[3];
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    double s = 0;
#pragma unroll
                    for (int i = 0; i < kSsimWin; ++i) s += c_win[kSsimWin - 1 - i] * cols[q][r][c + i];
                    g[q] = s;
                }
                g_ssim = g[0] + 2 * xv * g[1] + yv * g[2];  // ssim.cpp:124-125
                g_ssim *= a.ssim_scale;                     // -1 / count (ssim.cpp:131-134)
            }
            double g_l1 = d > 0 ? a.inv_n : (d < 0 ? -a.inv_n : 0);  // image.cpp:33
            if (a.l1_sign) {  // a near-tie pixel: the sign of the FP64 rendered value
                const int o = a.l1_sign[p];
                if (o) g_l1 = (double)(o - 2) * a.inv_n;
            }
            const double v = a.w_l1 * g_l1 + a.w_ssim * g_ssim;            // trainer.cpp:47-49
            dl[p] = a.accumulate ? (TO)((double)dl[p] + v) : (TO)v;
        }
    }
    const double s1 = block_sum_n<kSsimAThreads>(l1, red);
    const double s2 = block_sum_n<kSsimAThreads>(sq, red);
    if (t == 0) {
        const size_t b = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        part_l1[b] = s1;
        part_sq[b] = s2;
    }
}

// Fixed-order sum of block partials -> losses[slot] (+)= scale * sum / denom.
__global__ void __launch_bounds__(256) k_finalize(const double* __restrict__ parts, int n_parts, double denom,
                                                  double scale, int one_minus, int accumulate, double* out) {
    __shared__ double red[256];
    double s = 0;
    for (int i = threadIdx.x; i < n_parts; i += 256) s += parts[i];
    const double tot = block_sum(s, red);
    if (threadIdx.x == 0) {
        double v = tot / denom;
        if (one_minus) v = 1 - v;
        v = v * scale;
        *out = accumulate ? *out + v : v;
    }
}


// The image loss's three finalisations (L1, SSIM, squared error) in one launch, one block each.
struct FinalizeJob {
    const double* parts;
    int n_parts, one_minus, accumulate;
    double denom;
    double* out;
};
struct FinalizeJobs {
    FinalizeJob j[3];
};
__global__ void __launch_bounds__(256) k_finalize3(FinalizeJobs jobs, double scale) {
    const FinalizeJob& f = jobs.j[blockIdx.x];
    __shared__ double red[256];
    double s = 0;
    for (int i = threadIdx.x; i < f.n_parts; i += 256) s += f.parts[i];
    const double tot = block_sum(s, red);
    if (threadIdx.x == 0) {
        double v = tot / f.denom;
        if (f.one_minus) v = 1 - v;
        v = v * scale;
        *f.out = f.accumulate ? *f.out + v : v;
    }
}

// loss.cpp:16-31 on an opacity array (the standalone form of the term folded into K9).
__global__ void __launch_bounds__(256) k_entropy(const double* __restrict__ op, int n, double* __restrict__ grad,
                                                 double* part) {
    __shared__ double red[256];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double t = 0;
    if (i < n) {
        const double lo = 1e-6, hi = 1 - 1e-6, inv_n = 1 / (double)n;
        const double o0 = op[i];
        const double o = o0 < lo ? lo : (hi < o0 ? hi : o0);
        const double lg = log(o);
        t = -o * lg;
        if (grad) grad[i] = (o0 > lo && o0 < hi) ? -(lg + 1) * inv_n : 0;
    }
    const double s2 = block_sum(t, red);
    if (threadIdx.x == 0) part[blockIdx.x] = s2;
}

// optim.cpp:159-166 standalone.
template <typename TV>
__global__ void k_accumulate_stats(const TV* __restrict__ vnorm, const int32_t* __restrict__ visible, int n,
                                   double* __restrict__ accum, int32_t* __restrict__ count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !(visible[i] > 0)) return;
    accum[i] += (double)vnorm[i];
    count[i] += 1;
}

// ---------------------------------------------------------------------------
// K9: fused optimizer step, one thread per Gaussian (optim.cpp:110-166).
__device__ __forceinline__ void adam_scalar(double& p, double& m, double& v, double g, double lr, double bc1,
                                            double bc2) {
    // An all-zero (m, v, g) -- e.g. the SH coefficients above the active degree -- is a bitwise
    // no-op of the update below (m and v stay +0, p - 0 = p); skipping it avoids three IEEE
    // divisions and a square root of zero operands (their slow paths).
    if (g == 0 && m == 0 && v == 0) return;
    // optim.cpp:19-23 (kAdamBeta1 = 0.9, kAdamBeta2 = 0.999, kAdamEps = 1e-15)
    m = 0.9 * m + (1 - 0.9) * g;
    v = 0.999 * v + (1 - 0.999) * g * g;
    p -= lr * (m / bc1) / (sqrt(v / bc2) + 1e-15);
}

template <bool F64>
struct StoreT {
    using T = typename std::conditional<F64, double, float>::type;
};

template <bool F64>
__device__ __forceinline__ void ld4(const void* base, int n, int blk, int i, double* v) {
    if constexpr (F64) {
        const double2* p = reinterpret_cast<const double2*>(static_cast<const double*>(base) + 4 * (size_t)blk * n) +
                           2 * (size_t)i;
        const double2 a = p[0], b = p[1];
        v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    } else {
        const float4 f = reinterpret_cast<const float4*>(static_cast<const float*>(base) + 4 * (size_t)blk * n)[i];
        v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
    }
}
template <bool F64>
__device__ __forceinline__ void st4(void* base, int n, int blk, int i, const double* v) {
    if constexpr (F64) {
        double2* p = reinterpret_cast<double2*>(static_cast<double*>(base) + 4 * (size_t)blk * n) + 2 * (size_t)i;
        p[0] = make_double2(v[0], v[1]);
        p[1] = make_double2(v[2], v[3]);
    } else {
        reinterpret_cast<float4*>(static_cast<float*>(base) + 4 * (size_t)blk * n)[i] =
            make_float4((float)v[0], (float)v[1], (float)v[2], (float)v[3]);
    }
}
template <bool F64>
__device__ __forceinline__ double ld1(const void* base, size_t idx) {
    if constexpr (F64) return static_cast<const double*>(base)[idx];
    else return static_cast<const float*>(base)[idx];
}
template <bool F64>
__device__ __forceinline__ void st1(void* base, size_t idx, double v) {
    if constexpr (F64) static_cast<double*>(base)[idx] = v;
    else static_cast<float*>(base)[idx] = (float)v;
}

// One thread per (Gaussian, parameter group): blockIdx.y = 0 mean, 1 log scales, 2 rotor
// (both blocks + normalize), 3 opacity (+ entropy, + accumulate_stats), 4..15 SH blocks.
// Every group is independent, so the 16x wider grid hides the FP64 divide / sqrt latency.
// K9a: the plain Adam groups -- mean, log scales and the 12 SH blocks (14 of the 16 groups,
// 56 of the 65 parameters): four independent scalar updates per thread, few registers, so
// the FP64 divide / sqrt latency is hidden by occupancy.  Same arithmetic as k_adam_step.
template <bool F64>
__global__ void __launch_bounds__(128) k_adam_plain(void* params, void* mom1, void* mom2,
                                                    const float* __restrict__ grads, int n, AdamArgs a,
                                                    const unsigned long long* __restrict__ skip) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || (skip && *skip != ~0ull)) return;
    const int grp = blockIdx.y < 2 ? blockIdx.y : blockIdx.y + 2;
    double p[4], m[4], v[4], g[4];
    ld4<F64>(params, n, grp, i, p);
    ld4<F64>(mom1, n, grp, i, m);
    ld4<F64>(mom2, n, grp, i, v);
    ld4<false>(grads, n, grp, i, g);
    if (grp < 2) {
        // mean (lr_position schedule) / log scales; static mode freezes t
        const double lr = grp == 0 ? a.lr_pos : a.lr_scales;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (!(a.static_mode && k == 3)) adam_scalar(p[k], m[k], v[k], g[k], lr, a.bc1, a.bc2);
    } else {
        // SH block b = grp - 4 holds coefficients j = 4b..4b+3, j = k*3 + ch; DC is j < 3
        const int b = grp - 4;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const double lr = (4 * b + e) < 3 ? a.lr_sh_dc : a.lr_sh_rest;
            adam_scalar(p[e], m[e], v[e], g[e], lr, a.bc1, a.bc2);
        }
    }
    st4<F64>(params, n, grp, i, p);
    st4<F64>(mom1, n, grp, i, m);
    st4<F64>(mom2, n, grp, i, v);
}

template <bool F64>
__global__ void __launch_bounds__(128, 6) k_adam_step(void* params, void* mom1, void* mom2, const float* __restrict__ grads,
                                                   const float* __restrict__ vnorm, const int32_t* __restrict__ visible,
                                                   double* __restrict__ accum, int32_t* __restrict__ count, int n,
                                                   AdamArgs a, unsigned long long* err, double* part_entropy,
                                                   const unsigned long long* __restrict__ skip) {
    __shared__ double red[256];
    // A deferred forward of this step failed (rotor error, or a pair-buffer overflow that left
    // its gradients incomplete): the reference would have thrown before adam_step, so the
    // scene and moments are left untouched (block-uniform exit, before the barriers below).
    if (skip && *skip != ~0ull) return;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int grp = 2 + blockIdx.y;  // groups 2 (rotor) and 3 (opacity / stats); k_adam_plain does the rest
    double ent = 0;
    if (i < n) {
        if (grp == 2) {
            // rotor: Adam on the 8 stored coefficients, then normalize (rotor.cpp:117-136)
            double rc[8], rm[8], rv[8], rg[8];
            ld4<F64>(params, n, 2, i, rc);
            ld4<F64>(params, n, 3, i, rc + 4);
            ld4<F64>(mom1, n, 2, i, rm);
            ld4<F64>(mom1, n, 3, i, rm + 4);
            ld4<F64>(mom2, n, 2, i, rv);
            ld4<F64>(mom2, n, 3, i, rv + 4);
            ld4<false>(grads, n, 2, i, rg);
            ld4<false>(grads, n, 3, i, rg + 4);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const bool temporal = (k == 3 || k == 5 || k == 6 || k == 7);  // kTemporalRotorIdx
                if (!(a.static_mode && temporal)) adam_scalar(rc[k], rm[k], rv[k], rg[k], a.lr_rotor, a.bc1, a.bc2);
            }
            double nr[8];
            const int code = d_normalize(rc, nr);
            if (code) {
                atomicMin(err, ((unsigned long long)i << 8) | (unsigned long long)code);
            } else {
                if (a.static_mode) nr[3] = nr[5] = nr[6] = nr[7] = 0;
                st4<F64>(params, n, 2, i, nr);
                st4<F64>(params, n, 3, i, nr + 4);
            }
            st4<F64>(mom1, n, 2, i, rm);
            st4<F64>(mom1, n, 3, i, rm + 4);
            st4<F64>(mom2, n, 2, i, rv);
            st4<F64>(mom2, n, 3, i, rv + 4);
        } else if (grp == 3) {
            // accumulate_stats (optim.cpp:159-166) on the batch-summed view statistics
            if (a.stats && visible[i] > 0) {
                accum[i] += (double)vnorm[i];
                count[i] += 1;
            }
            // opacity (+ entropy regularizer, loss.cpp:16-31 folded as trainer.cpp:55-64)
            const size_t io = 64 * (size_t)n + i;
            double po = ld1<F64>(params, io), mo = ld1<F64>(mom1, io), vo = ld1<F64>(mom2, io);
            double go = grads[io];
            if (a.lambda_entropy != 0) {
                const double o = 1 / (1 + rgs_exp::glibc_exp(-po));  // GaussianStore::opacity
                const double lo = 1e-6, hi = 1 - 1e-6;
                const double oc = o < lo ? lo : (hi < o ? hi : o);
                const double lg = log(oc);
                ent = -oc * lg;
                const double ge = (o > lo && o < hi) ? -(lg + 1) * a.inv_n : 0;
                go = go + a.lambda_entropy * ge * o * (1 - o);
            }
            adam_scalar(po, mo, vo, go, a.lr_opacity, a.bc1, a.bc2);
            st1<F64>(params, io, po);
            st1<F64>(mom1, io, mo);
            st1<F64>(mom2, io, vo);
        }
    }
    if (part_entropy && grp == 3) {
        // 128-thread blocks: pad the reduction buffer.
        const int t = threadIdx.x;
        red[t] = ent;
        red[t + 128] = 0;
        __syncthreads();
        for (int s2 = 128; s2 > 0; s2 >>= 1) {
            if (t < s2) red[t] = red[t] + red[t + s2];
            __syncthreads();
        }
        if (t == 0) part_entropy[blockIdx.x] = red[0];
    }
}

// optim.cpp:236-243: opacity -> min(opacity, value) in probability space; its moments zeroed.
template <bool F64>
__global__ void k_reset_opacity(void* params, void* mom1, void* mom2, int n, double value) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const size_t io = 64 * (size_t)n + i;
    const double x = ld1<F64>(params, io);
    double o = 1 / (1 + rgs_exp::glibc_exp(-x));
    o = (value < o) ? value : o;  // std::min
    st1<F64>(params, io, log(o / (1 - o)));
    st1<F64>(mom1, io, 0.0);
    st1<F64>(mom2, io, 0.0);
}

// ---------------------------------------------------------------------------
// K10: consistency regularizer.
// gaussian_speed (gaussian.cpp:103-110): V / W of the normalised 4D covariance.
template <bool F64>
__global__ void __launch_bounds__(128) k_speeds(ParamView P, double* __restrict__ speeds,
                                                unsigned long long* err) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.n) return;
    double mean4[4], ls[4], rot[8];
    ld_block<F64>(P, 0, i, mean4);
    ld_block<F64>(P, 1, i, ls);
    ld_block<F64>(P, 2, i, rot);
    ld_block<F64>(P, 3, i, rot + 4);
    SliceState s;
    const int code = d_slice(mean4, ls, rot, 0.0, s);
    if (code > 0) {
        atomicMin(err, ((unsigned long long)i << 8) | (unsigned long long)code);
        return;
    }
    if (code < 0) {  // DegenerateTimeError escapes evaluate_loss in the reference
        atomicMin(err, ((unsigned long long)i << 8) | (unsigned long long)kErrDegenerateTime);
        return;
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) speeds[3 * (size_t)i + a] = s.V[a] / s.W;
}

// loss.cpp:33-58: loss partials and dL/dspeed.  Every term of dL/dspeed is +-inv_n (own) or
// -+inv_n inv_k (neighbour), so the gradient is accumulated exactly as an integer count of
// inv_n inv_k units (own sign x k, minus each neighbour's sign; integer atomics: the result is
// independent of their order) and scaled once where it is read (k_speed_backward /
// k_count_to_speed): bitwise reproducible, and no further from the exact sum than the
// reference's sequential FP64 accumulation.
__global__ void __launch_bounds__(256) k_consistency(const double* __restrict__ speeds,
                                                     const int32_t* __restrict__ nbrs, int n, int k,
                                                     int* __restrict__ dcount, double* part) {
    __shared__ double red[256];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double tot = 0;
    if (i < n && k > 0) {
        const double inv_n = 1 / (double)n, inv_k = 1 / (double)k;
        double avg[3] = {0, 0, 0};
        for (int j = 0; j < k; ++j) {
            const int q = nbrs[(size_t)k * i + j];
#pragma unroll
            for (int a = 0; a < 3; ++a) avg[a] += speeds[3 * (size_t)q + a];
        }
        double diff[3], sgn[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            avg[a] *= inv_k;
            diff[a] = speeds[3 * (size_t)i + a] - avg[a];
            sgn[a] = (double)(diff[a] > 0) - (double)(diff[a] < 0);
        }
        double s = fabs(diff[0]);
        s += fabs(diff[1]);
        s += fabs(diff[2]);
        tot = s;
        if (dcount) {
#pragma unroll
            for (int a = 0; a < 3; ++a)
                if (sgn[a] != 0) atomicAdd(&dcount[3 * (size_t)i + a], k * (int)sgn[a]);
            for (int j = 0; j < k; ++j) {
                const int q = nbrs[(size_t)k * i + j];
#pragma unroll
                for (int a = 0; a < 3; ++a)
                    if (sgn[a] != 0) atomicAdd(&dcount[3 * (size_t)q + a], -(int)sgn[a]);
            }
        }
    }
    const double s = block_sum(tot, red);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// slice_backward with only dL/dspeed (trainer.cpp:72-76): the speed gradient enters
// G4 through V and W; added into the FP32 gradient block (log scales, rotor).
template <bool F64>
__global__ void __launch_bounds__(128) k_speed_backward(ParamView P, const int* __restrict__ dcount, double unit,
                                                        double lambda, float* grads) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.n) return;
    double ds[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) ds[a] = lambda * (unit * (double)dcount[3 * (size_t)i + a]);
    if (ds[0] == 0 && ds[1] == 0 && ds[2] == 0) return;
    double mean4[4], ls[4], rot[8];
    ld_block<F64>(P, 0, i, mean4);
    ld_block<F64>(P, 1, i, ls);
    ld_block<F64>(P, 2, i, rot);
    ld_block<F64>(P, 3, i, rot + 4);
    SliceState s;
    if (d_slice(mean4, ls, rot, 0.0, s) != 0) return;
    const double W = s.W;
    double G4[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) G4[e] = 0;
    // gaussian.cpp:70-77 with dL_dmean3 = 0, dL_ddecay = 0, dL_dcov3 = 0
    double vds = s.V[0] * ds[0];
    vds += s.V[1] * ds[1];
    vds += s.V[2] * ds[2];
#pragma unroll
    for (int a = 0; a < 3; ++a) G4[a * 4 + 3] = ds[a] / W;
    G4[15] = -vds / (W * W);
    double out[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) out[e] = 0;
    d_g4_backward(s, rot, G4, out);
    const int n = P.n;
    float4* gl = reinterpret_cast<float4*>(grads + 4 * (size_t)n) + i;
    float4* g0 = reinterpret_cast<float4*>(grads + 8 * (size_t)n) + i;
    float4* g1 = reinterpret_cast<float4*>(grads + 12 * (size_t)n) + i;
    float4 t = *gl;
    *gl = make_float4((float)((double)t.x + out[4]), (float)((double)t.y + out[5]), (float)((double)t.z + out[6]),
                      (float)((double)t.w + out[7]));
    t = *g0;
    *g0 = make_float4((float)((double)t.x + out[8]), (float)((double)t.y + out[9]), (float)((double)t.z + out[10]),
                      (float)((double)t.w + out[11]));
    t = *g1;
    *g1 = make_float4((float)((double)t.x + out[12]), (float)((double)t.y + out[13]), (float)((double)t.z + out[14]),
                      (float)((double)t.w + out[15]));
}

// ---------------------------------------------------------------------------
// K11: exact KNN through a uniform 4D grid.  Points are counting-sorted by cell; a query
// scans the (2r+1)^4 block of cells around its own, shell by shell, until its k-th
// distance is below the distance to the unscanned region (with a relative safety margin
// for the rounding of that bound), or the block covers the grid.  The top-k insertion is
// lexicographic in (distance, index), so the result does not depend on the scan order and
// equals the brute-force / KdTree4 answer.
struct KnnGrid {
    double lo[4], cell[4];
    int G;  // cells per dimension
};

__device__ __forceinline__ int knn_cell_coord(double v, double lo, double cell, int G) {
    int c = (int)floor((v - lo) / cell);
    return c < 0 ? 0 : (c >= G ? G - 1 : c);
}
__device__ __forceinline__ int knn_cell_id(const double4& p, const KnnGrid& g) {
    const int a = knn_cell_coord(p.x, g.lo[0], g.cell[0], g.G), b = knn_cell_coord(p.y, g.lo[1], g.cell[1], g.G);
    const int c = knn_cell_coord(p.z, g.lo[2], g.cell[2], g.G), d = knn_cell_coord(p.w, g.lo[3], g.cell[3], g.G);
    return ((d * g.G + c) * g.G + b) * g.G + a;
}

__global__ void k_knn_bounds(const double4* __restrict__ pts, int n, double* part) {
    __shared__ double lo[4][256], hi[4][256];
    const int t = threadIdx.x;
    double l[4] = {INFINITY, INFINITY, INFINITY, INFINITY}, h[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    for (int i = blockIdx.x * 256 + t; i < n; i += gridDim.x * 256) {
        const double4 p = pts[i];
        const double v[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            l[a] = fmin(l[a], v[a]);
            h[a] = fmax(h[a], v[a]);
        }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        lo[a][t] = l[a];
        hi[a][t] = h[a];
    }
    __syncthreads();
    for (int s2 = 128; s2 > 0; s2 >>= 1) {
        if (t < s2)
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                lo[a][t] = fmin(lo[a][t], lo[a][t + s2]);
                hi[a][t] = fmax(hi[a][t], hi[a][t + s2]);
            }
        __syncthreads();
    }
    if (t < 4) {
        part[8 * blockIdx.x + t] = lo[t][0];
        part[8 * blockIdx.x + 4 + t] = hi[t][0];
    }
}

__global__ void k_knn_cells(const double4* __restrict__ pts, int n, KnnGrid g, uint32_t* __restrict__ cell,
                            uint32_t* __restrict__ count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t c = (uint32_t)knn_cell_id(pts[i], g);
    cell[i] = c;
    atomicAdd(&count[c], 1u);
}

__global__ void k_knn_scatter(const double4* __restrict__ pts, int n, const uint32_t* __restrict__ cell,
                              const uint32_t* __restrict__ start, uint32_t* __restrict__ cursor,
                              double4* __restrict__ spts, int32_t* __restrict__ sidx) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t c = cell[i];
    const uint32_t pos = start[c] + atomicAdd(&cursor[c], 1u);
    spts[pos] = pts[i];
    sidx[pos] = i;
}

template <int K>
__device__ __forceinline__ void topk_insert(double* bd, int* bi, double dd, int j) {
    if (!(dd < bd[K - 1] || (dd == bd[K - 1] && j < bi[K - 1]))) return;
    double cd = dd;
    int ci = j;
#pragma unroll
    for (int s = 0; s < K; ++s) {
        const bool less = cd < bd[s] || (cd == bd[s] && ci < bi[s]);
        const double td = bd[s];
        const int ti = bi[s];
        bd[s] = less ? cd : td;
        bi[s] = less ? ci : ti;
        cd = less ? td : cd;
        ci = less ? ti : ci;
    }
}

// Queries: qpts[t] (t < nq); result row qrow[t] (or t), excluded data index qexcl[t] (or -1);
// k_out <= K columns written, -1 where fewer than k_out candidates exist.
template <int K>
__global__ void __launch_bounds__(128) k_knn_grid(const double4* __restrict__ spts, const int32_t* __restrict__ sidx,
                                                  const uint32_t* __restrict__ start, KnnGrid g,
                                                  const double4* __restrict__ qpts, const int32_t* __restrict__ qrow,
                                                  const int32_t* __restrict__ qexcl, int nq, int k_out,
                                                  int32_t* __restrict__ out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nq) return;
    const double4 q = qpts[t];
    const int qi = qexcl ? qexcl[t] : -1;
    const int row = qrow ? qrow[t] : t;
    const int G = g.G;
    const int qc[4] = {knn_cell_coord(q.x, g.lo[0], g.cell[0], G), knn_cell_coord(q.y, g.lo[1], g.cell[1], G),
                       knn_cell_coord(q.z, g.lo[2], g.cell[2], G), knn_cell_coord(q.w, g.lo[3], g.cell[3], G)};
    const double qv[4] = {q.x, q.y, q.z, q.w};
    double bd[K];
    int bi[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
        bd[j] = INFINITY;
        bi[j] = 0x7fffffff;
    }
    for (int r = 0;; ++r) {
        int lo[4], hi[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            lo[a] = max(qc[a] - r, 0);
            hi[a] = min(qc[a] + r, G - 1);
        }
        for (int d = lo[3]; d <= hi[3]; ++d)
            for (int c = lo[2]; c <= hi[2]; ++c)
                for (int b = lo[1]; b <= hi[1]; ++b)
                    for (int a = lo[0]; a <= hi[0]; ++a) {
                        // only the shell at Chebyshev distance r from the query's cell
                        const int cheb = max(max(abs(a - qc[0]), abs(b - qc[1])), max(abs(c - qc[2]), abs(d - qc[3])));
                        if (cheb != r) continue;
                        const int cid = ((d * G + c) * G + b) * G + a;
                        const uint32_t e0 = start[cid], e1 = start[cid + 1];
                        for (uint32_t e = e0; e < e1; ++e) {
                            const int j = sidx[e];
                            if (j == qi) continue;
                            const double4 p = spts[e];
                            const double d0 = p.x - q.x, d1 = p.y - q.y, d2 = p.z - q.z, d3 = p.w - q.w;
                            double dd = d0 * d0;
                            dd += d1 * d1;
                            dd += d2 * d2;
                            dd += d3 * d3;
                            topk_insert<K>(bd, bi, dd, j);
                        }
                    }
        // distance from q to the unscanned region (sides at the grid edge are closed)
        double bound = INFINITY;
        bool all = true;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            if (qc[a] - r > 0) {
                bound = fmin(bound, qv[a] - (g.lo[a] + (double)(qc[a] - r) * g.cell[a]));
                all = false;
            }
            if (qc[a] + r < G - 1) {
                bound = fmin(bound, (g.lo[a] + (double)(qc[a] + r + 1) * g.cell[a]) - qv[a]);
                all = false;
            }
        }
        if (all) break;
        if (bi[K - 1] != 0x7fffffff && bound > 0 && bd[K - 1] < bound * bound * (1 - 1e-9)) break;
    }
    for (int j = 0; j < k_out; ++j) out[(size_t)k_out * row + j] = bi[j] == 0x7fffffff ? -1 : bi[j];
}

// Scaled 4D points (mean / scene scales, knn.cpp:106).
template <bool F64>
__global__ void k_knn_points(ParamView P, double4 scales, double4* pts) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.n) return;
    double m[4];
    ld_block<F64>(P, 0, i, m);
    pts[i] = make_double4(m[0] / scales.x, m[1] / scales.y, m[2] / scales.z, m[3] / scales.w);
}

// trainer.cpp:12-20: per-block min / max of the means (reduced on the host in order).
template <bool F64>
__global__ void __launch_bounds__(256) k_mean_extent(ParamView P, double* part_lo, double* part_hi) {
    __shared__ double lo[4][256], hi[4][256];
    const int i = blockIdx.x * blockDim.x + threadIdx.x, t = threadIdx.x;
    double m[4];
    if (i < P.n) {
        ld_block<F64>(P, 0, i, m);
    } else {
        ld_block<F64>(P, 0, blockIdx.x * blockDim.x, m);  // block's first Gaussian: neutral for min/max
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) lo[a][t] = hi[a][t] = m[a];
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (t < s)
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const double l = lo[a][t + s], h = hi[a][t + s];
                lo[a][t] = l < lo[a][t] ? l : lo[a][t];
                hi[a][t] = hi[a][t] < h ? h : hi[a][t];
            }
        __syncthreads();
    }
    if (t < 4) {
        part_lo[4 * (size_t)blockIdx.x + t] = lo[t][0];
        part_hi[4 * (size_t)blockIdx.x + t] = hi[t][0];
    }
}


// ---------------------------------------------------------------------------
// K12: densify_and_prune (optim.cpp:168-234).  The decisions run here, the sequential
// parts (the max_gaussians cut-off, the normal draws of the train loop's mt19937_64, the
// opacity sort of the prune set) on the host with the reference's own std:: types.
template <bool F64>
__global__ void k_densify_kind(ParamView P, const double* __restrict__ accum, const int32_t* __restrict__ count,
                               double thr, double clone_limit, uint8_t* __restrict__ kind) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.n) return;
    uint8_t k = 0;
    if (count[i] != 0) {
        const double avg = accum[i] / count[i];
        if (avg > thr) {
            double ls[4];
            ld_block<F64>(P, 1, i, ls);
            // log_scales.head<3>().array().exp().maxCoeff()
            double m = rgs_exp::glibc_exp(ls[0]);
            m = smax(m, rgs_exp::glibc_exp(ls[1]));
            m = smax(m, rgs_exp::glibc_exp(ls[2]));
            k = (m <= clone_limit) ? 1 : 2;
        }
    }
    kind[i] = k;
}

// Children of the processed candidates, appended at ext index n + c (moments zero,
// push_back gaussian.cpp:122-140).  kind: 1 clone, 2 / 3 first / second split child.
template <bool F64>
__global__ void k_densify_children(ParamView P, const int32_t* __restrict__ parent, const uint8_t* __restrict__ ckind,
                                   const double* __restrict__ draws, const int32_t* __restrict__ draw_off, int n_child,
                                   double log_split, int static_mode, void* ext, void* ext_m1, void* ext_m2,
                                   int ext_n, unsigned long long* err) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_child) return;
    const int p = parent[c], dst = P.n + c;
    double mean[4], ls[4], rot[8];
    ld_block<F64>(P, 0, p, mean);
    ld_block<F64>(P, 1, p, ls);
    ld_block<F64>(P, 2, p, rot);
    ld_block<F64>(P, 3, p, rot + 4);
    SliceState s;
    const int code = d_slice(mean, ls, rot, mean[3], s);  // slice_at(parent, parent.mean[3]) / gaussian_speed
    if (code != 0) {
        atomicMin(err, ((unsigned long long)p << 8) | (unsigned long long)(code < 0 ? kErrDegenerateTime : code));
        return;
    }
    const double* z = draws + draw_off[c];
    double cm[4] = {mean[0], mean[1], mean[2], mean[3]}, cl[4] = {ls[0], ls[1], ls[2], ls[3]};
    if (ckind[c] == 1) {
        // child.mean.head<3>() += gaussian_speed(parent) * (gauss(rng) * st)   (optim.cpp:189-191)
        const double st = rgs_exp::glibc_exp(ls[3]);
        const double f = z[0] * st;
#pragma unroll
        for (int a = 0; a < 3; ++a) cm[a] = mean[a] + (s.V[a] / s.W) * f;
    } else {
        // child.mean = parent.mean + (R * q.cwiseSqrt().asDiagonal()) * z   (optim.cpp:195-200)
        double sq[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) sq[j] = sqrt(s.q[j]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            double acc = (s.R[i * 4 + 0] * sq[0]) * z[0];
#pragma unroll
            for (int j = 1; j < 4; ++j) acc += (s.R[i * 4 + j] * sq[j]) * z[j];
            cm[i] = mean[i] + acc;
        }
        if (static_mode) cm[3] = mean[3];
#pragma unroll
        for (int a = 0; a < 4; ++a) cl[a] = ls[a] - log_split;
        if (static_mode) cl[3] = ls[3];
    }
    st4<F64>(ext, ext_n, 0, dst, cm);
    st4<F64>(ext, ext_n, 1, dst, cl);
    st4<F64>(ext, ext_n, 2, dst, rot);
    st4<F64>(ext, ext_n, 3, dst, rot + 4);
    double v[4];
#pragma unroll 1
    for (int b = 0; b < 12; ++b) {
        ld_block<F64>(P, 4 + b, p, v);
        st4<F64>(ext, ext_n, 4 + b, dst, v);
    }
    st1<F64>(ext, 64 * (size_t)ext_n + dst, ld_opacity<F64>(P, p));
    const double zero[4] = {0, 0, 0, 0};
#pragma unroll 1
    for (int b = 0; b < 16; ++b) {
        st4<F64>(ext_m1, ext_n, b, dst, zero);
        st4<F64>(ext_m2, ext_n, b, dst, zero);
    }
    st1<F64>(ext_m1, 64 * (size_t)ext_n + dst, 0.0);
    st1<F64>(ext_m2, 64 * (size_t)ext_n + dst, 0.0);
}

// Copy Gaussian map[j] of an SoA block of n_src Gaussians to slot j of one of n_dst.
template <typename T>
__global__ void k_gather_soa(const T* __restrict__ src, int n_src, const int32_t* __restrict__ map, int n_map,
                             T* __restrict__ dst, int n_dst) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n_map) return;
    const int i = map ? map[j] : j;
#pragma unroll 1
    for (int b = 0; b < 16; ++b) {
        const T* a = src + 4 * (size_t)b * n_src + 4 * (size_t)i;
        T* o = dst + 4 * (size_t)b * n_dst + 4 * (size_t)j;
        o[0] = a[0]; o[1] = a[1]; o[2] = a[2]; o[3] = a[3];
    }
    dst[64 * (size_t)n_dst + j] = src[64 * (size_t)n_src + i];
}

// Prune candidates (optim.cpp:212-221): flag, and the opacity logit for the host sort.
template <bool F64>
__global__ void k_prune_flags(ParamView P, const uint8_t* __restrict__ removed, double prune_opacity,
                              double big_scale, int static_mode, uint8_t* __restrict__ flag) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.n) return;
    if (removed[i]) {
        flag[i] = 0;
        return;
    }
    double ls[4];
    ld_block<F64>(P, 1, i, ls);
    double m = rgs_exp::glibc_exp(ls[0]);
    m = smax(m, rgs_exp::glibc_exp(ls[1]));
    m = smax(m, rgs_exp::glibc_exp(ls[2]));
    const double t_scale = rgs_exp::glibc_exp(ls[3]);
    const bool over_time = !static_mode && t_scale > 1.0;
    const double o = 1 / (1 + rgs_exp::glibc_exp(-ld_opacity<F64>(P, i)));
    flag[i] = (o < prune_opacity || m > big_scale || over_time) ? 1 : 0;
}

}  // namespace rgs_dev

// ---------------------------------------------------------------------------
namespace rgs_launch {
using namespace rgs_dev;

static inline int nblk(long long n, int t) { return (int)((n + t - 1) / t); }

void set_ssim_window(const double* k11, cudaStream_t s) {
    cudaMemcpyToSymbolAsync(c_win, k11, sizeof(double) * kSsimWin, 0, cudaMemcpyHostToDevice, s);
}

// Per-device kernel attributes (called from rgs_ctx_create on the context's device).
bool train_init() {
    const size_t s32 = k8a_smem_bytes<float>(), s64 = k8a_smem_bytes<double>();
    return cudaFuncSetAttribute(k_ssim_fields<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s32) ==
               cudaSuccess &&
           cudaFuncSetAttribute(k_ssim_fields<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s64) ==
               cudaSuccess;
}

ImageLossGrid image_loss_grid(int W, int H) {
    ImageLossGrid g;
    const int vw = W - kSsimWin + 1, vh = H - kSsimWin + 1;
    g.a_x = vw > 0 ? nblk(vw, kSsimTX) : 0;
    g.a_y = vh > 0 ? nblk(vh, kSsimATY) : 0;
    g.b_x = nblk(W, kSsimTX);
    g.b_y = nblk(H, kSsimATY);
    g.n_a = 3 * g.a_x * g.a_y;
    g.n_b = 3 * g.b_x * g.b_y;
    return g;
}

template <typename TI, typename TO>
void image_loss_t(const TI* img, const TI* tgt, int W, int H, const ImageGradArgs& a, TO* dl, double* dfield,
                  double* parts, double* losses, double loss_scale, int accumulate, cudaStream_t s) {
    const ImageLossGrid g = image_loss_grid(W, H);
    const double count = 3.0 * (double)(W - kSsimWin + 1) * (double)(H - kSsimWin + 1);
    const double nvals = 3.0 * (double)W * (double)H;
    double* pa = parts;
    double* pl1 = parts + g.n_a;
    double* psq = pl1 + g.n_b;
    // Images smaller than the window have no SSIM (the caller rejects w_ssim != 0 for them):
    // stage A is skipped and the SSIM slot is NaN.
    const bool has_ssim = W >= kSsimWin && H >= kSsimWin;
    const size_t smem = k8a_smem_bytes<TI>();
    if (has_ssim)
        k_ssim_fields<TI><<<dim3(g.a_x, g.a_y, 3), kSsimAThreads, smem, s>>>(img, tgt, W, H, dl != nullptr, dfield, pa);
    ImageGradArgs a2 = a;
    if (!has_ssim) a2.w_ssim = 0;
    k_image_grad<TI, TO><<<dim3(g.b_x, g.b_y, 3), kSsimAThreads, 0, s>>>(img, tgt, W, H, dfield, a2, dl, pl1, psq);
    if (losses) {
        FinalizeJobs jobs;
        jobs.j[0] = FinalizeJob{pl1, g.n_b, 0, accumulate, nvals, losses + 0};
        jobs.j[1] = has_ssim ? FinalizeJob{pa, g.n_a, 1, accumulate, count, losses + 1}
                             : FinalizeJob{pa, 0, 0, 0, 0.0, losses + 1};  // 0 / 0 = NaN
        jobs.j[2] = FinalizeJob{psq, g.n_b, 0, accumulate, nvals, losses + 2};
        k_finalize3<<<3, 256, 0, s>>>(jobs, loss_scale);
    }
}

void image_loss(const float* img, const float* tgt, int W, int H, const ImageGradArgs& a, float* dl,
                double* dfield, double* parts, double* losses, double loss_scale, int accumulate, cudaStream_t s) {
    image_loss_t<float, float>(img, tgt, W, H, a, dl, dfield, parts, losses, loss_scale, accumulate, s);
}
void image_loss_f64(const double* img, const double* tgt, int W, int H, const ImageGradArgs& a, double* dl,
                    double* dfield, double* parts, double* losses, double loss_scale, int accumulate, cudaStream_t s) {
    image_loss_t<double, double>(img, tgt, W, H, a, dl, dfield, parts, losses, loss_scale, accumulate, s);
}

void adam_step(bool f64, void* params, void* m1, void* m2, const float* grads, const float* vnorm,
               const int32_t* visible, double* accum, int32_t* count, int n, const AdamArgs& a,
               unsigned long long* err, double* part_entropy, double* losses_entropy, int accumulate,
               const unsigned long long* skip, cudaStream_t s) {
    const int nb = nblk(n, 128);
    if (f64) {
        k_adam_plain<true><<<dim3(nb, 14), 128, 0, s>>>(params, m1, m2, grads, n, a, skip);
        k_adam_step<true><<<dim3(nb, 2), 128, 0, s>>>(params, m1, m2, grads, vnorm, visible, accum, count, n, a, err,
                                                      part_entropy, skip);
    } else {
        k_adam_plain<false><<<dim3(nb, 14), 128, 0, s>>>(params, m1, m2, grads, n, a, skip);
        k_adam_step<false><<<dim3(nb, 2), 128, 0, s>>>(params, m1, m2, grads, vnorm, visible, accum, count, n, a,
                                                       err, part_entropy, skip);
    }
    if (part_entropy && losses_entropy)
        k_finalize<<<1, 256, 0, s>>>(part_entropy, nb, (double)n, 1.0, 0, accumulate, losses_entropy);
}

int adam_blocks(int n) { return nblk(n, 128); }

}  // namespace rgs_launch
namespace rgs_dev {
__global__ void k_l1_ties(const float* __restrict__ img, const float* __restrict__ tgt, int npix, float eps,
                          const uint32_t* __restrict__ n_contrib, uint32_t* list, int* count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npix) return;
    // a pixel no splat reached is the background in both precisions (n_contrib = 0, not slow;
    // n_contrib is NULL when the background is not float32-exact): nothing to re-decide
    if (n_contrib && n_contrib[i] == 0u) return;
    bool tie = false;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) tie |= fabsf(img[3 * (size_t)i + ch] - tgt[3 * (size_t)i + ch]) <= eps;
    if (tie) list[atomicAdd(count, 1)] = (uint32_t)i;
}
__global__ void k_l1_sign_set(const uint32_t* __restrict__ list, const int* __restrict__ count,
                              const double* __restrict__ img64, const float* __restrict__ tgt, int8_t* sign) {
    const int n = *count;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 3 * n; e += gridDim.x * blockDim.x) {
        const size_t p = 3 * (size_t)list[e / 3] + e % 3;
        const double d = img64[p] - (double)tgt[p];  // image.cpp:32 on the reference's double image
        sign[p] = (int8_t)(d > 0 ? 3 : (d < 0 ? 1 : 2));
    }
}
__global__ void k_l1_sign_clear(const uint32_t* __restrict__ list, const int* __restrict__ count, int8_t* sign) {
    const int n = *count;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 3 * n; e += gridDim.x * blockDim.x)
        sign[3 * (size_t)list[e / 3] + e % 3] = 0;
}
}  // namespace rgs_dev
namespace rgs_launch {
void l1_ties(const float* img, const float* tgt, int npix, float eps, const uint32_t* n_contrib, uint32_t* list,
             int* count, cudaStream_t s) {
    if (npix > 0) k_l1_ties<<<nblk(npix, 256), 256, 0, s>>>(img, tgt, npix, eps, n_contrib, list, count);
}
void l1_sign_set(const uint32_t* list, const int* count, int max_items, const double* img64, const float* tgt,
                 int8_t* sign, cudaStream_t s) {
    k_l1_sign_set<<<std::max(1, std::min(nblk(3 * max_items, 256), 148 * 4)), 256, 0, s>>>(list, count, img64, tgt,
                                                                                         sign);
}
void l1_sign_clear(const uint32_t* list, const int* count, int max_items, int8_t* sign, cudaStream_t s) {
    k_l1_sign_clear<<<std::max(1, std::min(nblk(3 * max_items, 256), 148 * 4)), 256, 0, s>>>(list, count, sign);
}

void entropy(const double* op, int n, double* grad, double* parts, double* loss, cudaStream_t s) {
    const int nb = nblk(n, 256);
    k_entropy<<<nb, 256, 0, s>>>(op, n, grad, parts);
    if (loss) k_finalize<<<1, 256, 0, s>>>(parts, nb, (double)n, 1.0, 0, 0, loss);
}

void accumulate_stats(const float* vnorm, const int32_t* visible, int n, double* accum, int32_t* count,
                      cudaStream_t s) {
    if (n > 0) k_accumulate_stats<float><<<nblk(n, 256), 256, 0, s>>>(vnorm, visible, n, accum, count);
}
void accumulate_stats_f64(const double* vnorm, const int32_t* visible, int n, double* accum, int32_t* count,
                          cudaStream_t s) {
    if (n > 0) k_accumulate_stats<double><<<nblk(n, 256), 256, 0, s>>>(vnorm, visible, n, accum, count);
}

void reset_opacity(bool f64, void* params, void* m1, void* m2, int n, double value, cudaStream_t s) {
    if (f64)
        k_reset_opacity<true><<<nblk(n, 256), 256, 0, s>>>(params, m1, m2, n, value);
    else
        k_reset_opacity<false><<<nblk(n, 256), 256, 0, s>>>(params, m1, m2, n, value);
}

void speeds(const float* params, const double* params64, int n, double* out, unsigned long long* err,
            cudaStream_t s) {
    ParamView P{params, n, params64};
    if (params64)
        k_speeds<true><<<nblk(n, 128), 128, 0, s>>>(P, out, err);
    else
        k_speeds<false><<<nblk(n, 128), 128, 0, s>>>(P, out, err);
}

void consistency(const double* speeds, const int32_t* nbrs, int n, int k, int* dcount, double* parts,
                 double* losses_slot, int accumulate, cudaStream_t s) {
    const int nb = nblk(n, 256);
    k_consistency<<<nb, 256, 0, s>>>(speeds, nbrs, n, k, dcount, parts);
    if (losses_slot) k_finalize<<<1, 256, 0, s>>>(parts, nb, (double)n, 1.0, 0, accumulate, losses_slot);
}

}  // namespace rgs_launch
namespace rgs_dev {
__global__ void k_count_to_speed(const int* __restrict__ dcount, size_t m, double unit, double* __restrict__ dspeed) {
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < m; e += (size_t)gridDim.x * blockDim.x)
        dspeed[e] = unit * (double)dcount[e];
}
}  // namespace rgs_dev
namespace rgs_launch {
double consistency_unit(int n, int k) { return (n > 0 && k > 0) ? (1 / (double)n) * (1 / (double)k) : 0.0; }

void count_to_speed(const int* dcount, int n, int k, double* dspeed, cudaStream_t s) {
    const size_t m = 3 * (size_t)n;
    if (m) k_count_to_speed<<<std::max(1, std::min(nblk((long long)m, 256), 148 * 8)), 256, 0, s>>>(
        dcount, m, consistency_unit(n, k), dspeed);
}

int consistency_blocks(int n) { return nblk(n, 256); }

void speed_backward(const float* params, const double* params64, int n, int k, const int* dcount, double lambda,
                    float* grads, cudaStream_t s) {
    ParamView P{params, n, params64};
    const double unit = consistency_unit(n, k);
    if (params64)
        k_speed_backward<true><<<nblk(n, 128), 128, 0, s>>>(P, dcount, unit, lambda, grads);
    else
        k_speed_backward<false><<<nblk(n, 128), 128, 0, s>>>(P, dcount, unit, lambda, grads);
}

void knn_points(const float* params, const double* params64, int n, const double* scales, double* pts4,
                cudaStream_t s) {
    ParamView P{params, n, params64};
    const double4 sc = make_double4(scales[0], scales[1], scales[2], scales[3]);
    if (params64)
        k_knn_points<true><<<nblk(n, 256), 256, 0, s>>>(P, sc, reinterpret_cast<double4*>(pts4));
    else
        k_knn_points<false><<<nblk(n, 256), 256, 0, s>>>(P, sc, reinterpret_cast<double4*>(pts4));
}

// Grid build over the data points + query launch.  queries4 == NULL: the data points are the
// queries (self excluded, rows in data order) -- build_knn4d.
int knn_grid(const double* pts4, int n, const double* queries4, const int32_t* qexcl, int nq, int k, int32_t* out,
             void* scratch, size_t scratch_bytes, cudaStream_t s) {
    const double4* p = reinterpret_cast<const double4*>(pts4);
    int G = (int)floor(pow(n / 2.0, 0.25));
    G = G < 1 ? 1 : (G > 48 ? 48 : G);
    const size_t ncell = (size_t)G * G * G * G;
    char* base = static_cast<char*>(scratch);
    auto take = [&](size_t bytes) {
        char* r = base;
        base += (bytes + 255) & ~size_t(255);
        return r;
    };
    double* part = (double*)take(8 * 64 * sizeof(double));
    uint32_t* cell = (uint32_t*)take(4 * (size_t)n);
    uint32_t* count = (uint32_t*)take(4 * (ncell + 1));
    uint32_t* start = (uint32_t*)take(4 * (ncell + 1));
    uint32_t* cursor = (uint32_t*)take(4 * ncell);
    uint32_t* tmp = (uint32_t*)take(4 * (ncell / 1024 + 4096));
    double4* spts = (double4*)take(32 * (size_t)n);
    int32_t* sidx = (int32_t*)take(4 * (size_t)n);
    if ((size_t)(base - static_cast<char*>(scratch)) > scratch_bytes) return -2;
    k_knn_bounds<<<64, 256, 0, s>>>(p, n, part);
    double hp[8 * 64];
    cudaMemcpyAsync(hp, part, sizeof hp, cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return -3;
    KnnGrid g;
    g.G = G;
    for (int a = 0; a < 4; ++a) {
        double lo = INFINITY, hi = -INFINITY;
        for (int b = 0; b < 64; ++b) {
            lo = fmin(lo, hp[8 * b + a]);
            hi = fmax(hi, hp[8 * b + 4 + a]);
        }
        g.lo[a] = lo;
        g.cell[a] = (hi > lo && isfinite(hi - lo)) ? (hi - lo) / G : 1.0;
    }
    cudaMemsetAsync(count, 0, 4 * (ncell + 1), s);
    cudaMemsetAsync(cursor, 0, 4 * ncell, s);
    k_knn_cells<<<nblk(n, 256), 256, 0, s>>>(p, n, g, cell, count);
    exclusive_scan(count, (int)ncell + 1, start, tmp, nullptr, s);
    k_knn_scatter<<<nblk(n, 256), 256, 0, s>>>(p, n, cell, start, cursor, spts, sidx);
    const double4* qp = queries4 ? reinterpret_cast<const double4*>(queries4) : spts;
    const int32_t* qrow = queries4 ? nullptr : sidx;
    const int32_t* qx = queries4 ? qexcl : sidx;
    const int nqq = queries4 ? nq : n;
    const int nb = nblk(nqq, 128);
    const int K = k <= 1 ? 1 : (k <= 2 ? 2 : (k <= 4 ? 4 : (k <= 8 ? 8 : 16)));
    if (k < 1 || k > 16) return -1;
    switch (K) {
        case 1: k_knn_grid<1><<<nb, 128, 0, s>>>(spts, sidx, start, g, qp, qrow, qx, nqq, k, out); break;
        case 2: k_knn_grid<2><<<nb, 128, 0, s>>>(spts, sidx, start, g, qp, qrow, qx, nqq, k, out); break;
        case 4: k_knn_grid<4><<<nb, 128, 0, s>>>(spts, sidx, start, g, qp, qrow, qx, nqq, k, out); break;
        case 8: k_knn_grid<8><<<nb, 128, 0, s>>>(spts, sidx, start, g, qp, qrow, qx, nqq, k, out); break;
        default: k_knn_grid<16><<<nb, 128, 0, s>>>(spts, sidx, start, g, qp, qrow, qx, nqq, k, out); break;
    }
    return 0;
}

size_t knn_grid_scratch(int n) {
    int G = (int)floor(pow(n / 2.0, 0.25));
    G = G < 1 ? 1 : (G > 48 ? 48 : G);
    const size_t ncell = (size_t)G * G * G * G;
    return 8 * 64 * 8 + 4 * (size_t)n + 3 * 4 * (ncell + 1) + 4 * (ncell / 1024 + 4096) + 36 * (size_t)n + 8 * 256;
}

int extent_blocks(int n) { return nblk(n, 256); }

void densify_kind(const float* params, const double* params64, int n, const double* accum, const int32_t* count,
                  double thr, double clone_limit, uint8_t* kind, cudaStream_t s) {
    ParamView P{params, n, params64};
    if (params64)
        k_densify_kind<true><<<nblk(n, 256), 256, 0, s>>>(P, accum, count, thr, clone_limit, kind);
    else
        k_densify_kind<false><<<nblk(n, 256), 256, 0, s>>>(P, accum, count, thr, clone_limit, kind);
}

void densify_children(const float* params, const double* params64, int n, const int32_t* parent,
                      const uint8_t* ckind, const double* draws, const int32_t* draw_off, int n_child,
                      double log_split, int static_mode, void* ext, void* ext_m1, void* ext_m2, int ext_n,
                      unsigned long long* err, cudaStream_t s) {
    if (n_child <= 0) return;
    ParamView P{params, n, params64};
    if (params64)
        k_densify_children<true><<<nblk(n_child, 128), 128, 0, s>>>(P, parent, ckind, draws, draw_off, n_child,
                                                                   log_split, static_mode, ext, ext_m1, ext_m2,
                                                                   ext_n, err);
    else
        k_densify_children<false><<<nblk(n_child, 128), 128, 0, s>>>(P, parent, ckind, draws, draw_off, n_child,
                                                                    log_split, static_mode, ext, ext_m1, ext_m2,
                                                                    ext_n, err);
}

void gather_soa(bool f64, const void* src, int n_src, const int32_t* map, int n_map, void* dst, int n_dst,
                cudaStream_t s) {
    if (n_map <= 0) return;
    if (f64)
        k_gather_soa<double><<<nblk(n_map, 256), 256, 0, s>>>((const double*)src, n_src, map, n_map, (double*)dst,
                                                              n_dst);
    else
        k_gather_soa<float><<<nblk(n_map, 256), 256, 0, s>>>((const float*)src, n_src, map, n_map, (float*)dst,
                                                             n_dst);
}

void prune_flags(const float* params, const double* params64, int n, const uint8_t* removed, double prune_opacity,
                 double big_scale, int static_mode, uint8_t* flag, cudaStream_t s) {
    ParamView P{params, n, params64};
    if (params64)
        k_prune_flags<true><<<nblk(n, 256), 256, 0, s>>>(P, removed, prune_opacity, big_scale, static_mode, flag);
    else
        k_prune_flags<false><<<nblk(n, 256), 256, 0, s>>>(P, removed, prune_opacity, big_scale, static_mode, flag);
}

void mean_extent(const float* params, const double* params64, int n, double* part_lo, double* part_hi,
                 cudaStream_t s) {
    ParamView P{params, n, params64};
    if (params64)
        k_mean_extent<true><<<nblk(n, 256), 256, 0, s>>>(P, part_lo, part_hi);
    else
        k_mean_extent<false><<<nblk(n, 256), 256, 0, s>>>(P, part_lo, part_hi);
}

}  // namespace rgs_launch
