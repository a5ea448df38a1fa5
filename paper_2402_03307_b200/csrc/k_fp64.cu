// FP64 kernels: per-Gaussian slice+project+SH (K1), FP64 pixel blend (guard-band
// fix-up / reference mode), FP64 backward replay of those pixels, and the
// per-Gaussian backward chain (K7).
//
// Compiled with -fmad=false: the FP64 expression order is the reference's
// (see fp64_math.cuh), which is what makes tile rectangles, depths and culls
// bit-identical to the CPU oracle.
#include "fp64_math.cuh"
#include <algorithm>
#include <type_traits>

#include "rgs_internal.cuh"

namespace rgs_dev {

__device__ __forceinline__ unsigned long long order_key(double d) {
    unsigned long long b = (unsigned long long)__double_as_longlong(d);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// rasterizer.cpp:26-38
__device__ __forceinline__ uint32_t d_tile_rect(double mx, double my, double r, int tiles_x, int tiles_y,
                                                ushort4* rect) {
    int a;
    a = x86_double_to_int(floor((mx - r) / kTile));
    int x0 = a > 0 ? a : 0;
    a = x86_double_to_int(floor((mx + r) / kTile));
    int x1 = a < tiles_x - 1 ? a : tiles_x - 1;
    a = x86_double_to_int(floor((my - r) / kTile));
    int y0 = a > 0 ? a : 0;
    a = x86_double_to_int(floor((my + r) / kTile));
    int y1 = a < tiles_y - 1 ? a : tiles_y - 1;
    if (!(x0 <= x1 && y0 <= y1)) {
        *rect = make_ushort4(0, 0, 0, 0);
        return 0;
    }
    *rect = make_ushort4((unsigned short)x0, (unsigned short)x1, (unsigned short)y0, (unsigned short)y1);
    return (uint32_t)(x1 - x0 + 1) * (uint32_t)(y1 - y0 + 1);
}

// FP32 blend record of one splat.
// Everything is in log2 units so the blend evaluates p2 = log2(e) * power and
// alpha = alpha_base * 2^p2 with one MUFU.EX2:
//   conic_f = (ca2, cb2, cc2, ab),  p2 = ca2 dx^2 + cc2 dy^2 + cb2 dx dy
//   color_f = (r, g, b, pa2),        pa2 = log2(1/(255 ab))   alpha gate: p2 < pa2
//   guard_f = (cs2n, pc2, R, lmax),  pc2 = log2(0.99 / ab)    clamp gate: p2 <= pc2
//   ext_f   = (ex, ey, gx2, gy2)     bbox half-extents of the alpha ellipse (per-warp
//                                    culling) and max |dp2/dx|, |dp2/dy| inside it.
// cs2n * q (q = ca2 dx^2 + cc2 dy^2 <= 0) bounds the FP32 rounding error of p2.
constexpr double kLog2e = 1.4426950408889634;

__device__ __forceinline__ void d_blend_record(const SplatArrays& out, int i, double ca, double cb, double cc,
                                               double ab, double r, double g, double b, double s00, double s11) {
    const double pa = log(kMinAlpha / ab);  // natural-log alpha threshold (<= 0)
    const double kappa = fabs(cb) / sqrt(ca * cc);
    // FP32 p2 = fma(v, dy, fma(t, dx, u dy)) with rounded coefficients carries <= ~5 u
    // (u = 2^-24) relative error on each of |ca2 dx^2|, |cc2 dy^2|, |cb2 dx dy| <= kappa |q| / 2,
    // i.e. <= 3.0e-7 (1 + kappa / 2) |q|; 6e-7 (1 + kappa) / (1 - kappa) keeps a 2x margin.
    double cs = (kappa < 0.999) ? 6e-7 * (1 + kappa) / (1 - kappa) : 1e30;
    if (!(ca > 0) || !(cc > 0)) cs = 1e30;
    const double L = fabs(pa) * 2;
    const double ex = sqrt(L * fmax(s00, 0.0)) * (1 + 1e-3) + 1e-2;
    const double ey = sqrt(L * fmax(s11, 0.0)) * (1 + 1e-3) + 1e-2;
    const double gx = kLog2e * sqrt(L * fmax(ca, 0.0));
    const double gy = kLog2e * sqrt(L * fmax(cc, 0.0));
    const float4 cf = make_float4((float)(-0.5 * kLog2e * ca), (float)(-kLog2e * cb), (float)(-0.5 * kLog2e * cc),
                                  (float)ab);
    out.conic_f[i] = cf;
    out.color_f[i] = make_float4((float)r, (float)g, (float)b, (float)(kLog2e * pa));
    // The blend kernels' per-splat constants, once per splat here instead of once per (tile, splat)
    // staging: R >= ln2 / (1 - min(0.99, ab)) (the T-gate's error growth per blend, rounded up) and
    // lmax >= the largest eigenvalue of the log2-power form (the radial cull), both from the FP32
    // conic K5 / K6 evaluate.
    const float am = fminf(0.99f, cf.w);
    const float R = __fmul_ru(__fdiv_ru(1.f, __fsub_rd(1.f, am)), 0.6931472f * 1.000001f);
    const float h = 0.5f * (cf.x + cf.z), dd = 0.5f * (cf.x - cf.z), o = 0.5f * cf.y;
    const float lm = h + sqrtf(fmaf(dd, dd, o * o));
    const float lmax = lm + 1e-5f * (fabsf(cf.x) + fabsf(cf.z) + fabsf(cf.y));
    out.guard_f[i] = make_float4((float)(-2.0 * cs), (float)log2(kAlphaClamp / ab), R, lmax);
    out.ext_f[i] = make_float4(isfinite(ex) ? (float)ex : 3e38f, isfinite(ey) ? (float)ey : 3e38f, (float)gx,
                               (float)gy);
}

__device__ __forceinline__ void store_splat(const SplatArrays& out, int i, double mx, double my, double ca,
                                            double cb, double cc, double ab, double r, double g, double b,
                                            double depth, double fx, double fy, double radius, int tiles_x,
                                            int tiles_y, uint32_t* ntiles, double s00, double s11) {
    out.mean2[i] = make_double2(mx, my);
    out.conic_ab[i] = make_double4(ca, cb, cc, ab);
    out.color_depth[i] = make_double4(r, g, b, depth);
    if (out.flow_radius) out.flow_radius[i] = make_double4(fx, fy, radius, 0.0);  // NULL: render-only batch
    ushort4 rect;
    *ntiles = d_tile_rect(mx, my, radius, tiles_x, tiles_y, &rect);
    out.rect[i] = rect;
    d_blend_record(out, i, ca, cb, cc, ab, r, g, b, s00, s11);
}

// Warp-aggregated: count of valid splats and min / max depth key (bucket range).
__device__ __forceinline__ void count_valid(bool ok, unsigned long long key, BinState* st) {
    const unsigned m = __ballot_sync(0xffffffffu, ok);
    if (!m) return;
    unsigned long long lo = ok ? key : ~0ull, hi = ok ? key : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, lo, o), b = __shfl_xor_sync(0xffffffffu, hi, o);
        lo = a < lo ? a : lo;
        hi = b > hi ? b : hi;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&st->n_valid, __popc(m));
        atomicMin(&st->key_min, lo);
        atomicMax(&st->key_max, hi);
    }
}

// Slice cache of a view batch: per Gaussian, the t-independent part of slice_at
// (d_slice_static: normalize, to_matrix, Sigma4, lambda, speed, cov3) and sigmoid(opacity), so
// the K1 of every view of a timestamp sweep only does the t-dependent rest.  The cached values
// are the outputs of the same FP64 operations, so every splat record stays bit-identical.
// SoA of double2 blocks: (cov00, cov01) (cov02, cov10) (cov11, cov12) (cov20, cov21)
// (cov22, lambda) (speed0, speed1) (speed2, opacity); status: 0 ok, -1 degenerate time (the
// Gaussian is skipped), > 0 rotor error code.
constexpr int kSliceCacheBlocks = 7;

template <bool F64>
__global__ void __launch_bounds__(128) k_slice_cache(ParamView P, SliceCacheView C) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.n) return;
    double ls[4], rot[8];
    ld_block<F64>(P, 1, i, ls);
    ld_block<F64>(P, 2, i, rot);
    ld_block<F64>(P, 3, i, rot + 4);
    SliceState s;
    const int rc = d_slice_static(ls, rot, s);
    C.status[i] = (int8_t)rc;
    if (rc != 0) return;
    const double op = 1 / (1 + rgs_exp::glibc_exp(-ld_opacity<F64>(P, i)));
    const size_t n = (size_t)P.n;
    C.blk[0 * n + i] = make_double2(s.cov[0], s.cov[1]);
    C.blk[1 * n + i] = make_double2(s.cov[2], s.cov[3]);
    C.blk[2 * n + i] = make_double2(s.cov[4], s.cov[5]);
    C.blk[3 * n + i] = make_double2(s.cov[6], s.cov[7]);
    C.blk[4 * n + i] = make_double2(s.cov[8], s.lambda);
    C.blk[5 * n + i] = make_double2(s.speed[0], s.speed[1]);
    C.blk[6 * n + i] = make_double2(s.speed[2], op);
}

// K1: slice + visibility gate + project + SH colour, one thread per Gaussian
// (rasterizer.cpp:189-204, gaussian.cpp:32-47, rasterizer.cpp:215-276, sh.cpp:16-97).
// CACHED: the t-independent half of the slice and the opacity come from the batch's slice cache.
template <bool F64, bool CACHED>
__global__ void __launch_bounds__(128, CACHED ? 8 : 1) k_preprocess(ParamView P, int sh_degree, DevCamera cam, SplatArrays out,
                                                    BinState* st, SliceCacheView C) {
    using ShT = typename std::conditional<F64, double, float>::type;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    bool ok = false;
    uint32_t ntiles = 0;
    unsigned long long key = ~0ull;
    if (i < P.n) {
        if (CACHED) {
            // The SH blocks are read only after the projection (by the splats that survive it):
            // start them towards L1 now, so their latency overlaps the FP64 chain.
            const int deg = sh_degree < 0 ? 0 : (sh_degree > 3 ? 3 : sh_degree);
            const int nblk = (3 * (deg + 1) * (deg + 1) + 3) / 4;
#pragma unroll
            for (int b = 0; b < 12; ++b) {
                if (b >= nblk) break;
                const void* a = F64 ? (const void*)(P.base64 + 4 * ((size_t)(4 + b) * P.n + i))
                                    : (const void*)(P.base + 4 * ((size_t)(4 + b) * P.n + i));
                asm volatile("prefetch.global.L1 [%0];" ::"l"(a));
            }
        }
        double mean4[4];
        ld_block<F64>(P, 0, i, mean4);
        SliceState s;
        int rc;
        double op;
        if (CACHED) {
            rc = C.status[i];
            if (rc == 0) {
                const size_t n = (size_t)P.n;
                double2 v;
                v = C.blk[0 * n + i]; s.cov[0] = v.x; s.cov[1] = v.y;
                v = C.blk[1 * n + i]; s.cov[2] = v.x; s.cov[3] = v.y;
                v = C.blk[2 * n + i]; s.cov[4] = v.x; s.cov[5] = v.y;
                v = C.blk[3 * n + i]; s.cov[6] = v.x; s.cov[7] = v.y;
                v = C.blk[4 * n + i]; s.cov[8] = v.x; s.lambda = v.y;
                v = C.blk[5 * n + i]; s.speed[0] = v.x; s.speed[1] = v.y;
                v = C.blk[6 * n + i]; s.speed[2] = v.x; op = v.y;
                d_slice_time(mean4, cam.time, s);
            }
        } else {
            double ls[4], rot[8];
            ld_block<F64>(P, 1, i, ls);
            ld_block<F64>(P, 2, i, rot);
            ld_block<F64>(P, 3, i, rot + 4);
            op = ld_opacity<F64>(P, i);
            rc = d_slice(mean4, ls, rot, cam.time, s);
        }
        if (rc > 0) {
            atomicMin(&st->err, ((unsigned long long)i << 8) | (unsigned long long)rc);
        } else if (rc == 0) {
            const double dt = cam.time - mean4[3];
            ProjState o;
            if (!(s.lambda * dt * dt > kVisibility) && d_project_geom<CACHED>(s, cam, op, o)) {
                ok = true;
                const int deg = sh_degree < 0 ? 0 : (sh_degree > 3 ? 3 : sh_degree);
                const int K = (deg + 1) * (deg + 1);
                const int nblk = (3 * K + 3) / 4;
                // colour = sh . basis + 0.5 per channel (rasterizer.cpp:245-257): the SH blocks are
                // streamed (coefficient j = 3k + ch), each channel still summed in increasing k, and
                // each basis entry (sh.cpp:16-85's expression) computed where it is used
                const double x = o.dir[0], y = o.dir[1], z = o.dir[2];
                const double xx = x * x, yy = y * y, zz = z * z;
                double col[3];
#pragma unroll
                for (int b = 0; b < 12; ++b) {
                    if (b < nblk) {
                        ShT v[4];
                        ld_block<F64>(P, 4 + b, i, v);
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int j = 4 * b + e, k = j / 3, ch = j % 3;
                            if (k == 0) col[ch] = (double)v[e] * kC0;
                            else if (k < K) col[ch] += (double)v[e] * d_sh_basis_at(k, x, y, z, xx, yy, zz);
                        }
                    }
                }
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    const double c = col[ch] + 0.5;
                    col[ch] = c < 0 ? 0.0 : c;
                }
                double flow[2];
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    double a = o.T[r * 3 + 0] * s.speed[0];
                    a += o.T[r * 3 + 1] * s.speed[1];
                    a += o.T[r * 3 + 2] * s.speed[2];
                    flow[r] = a;
                }
                store_splat(out, i, o.mean2[0], o.mean2[1], o.conic[0], o.conic[1], o.conic[2], o.alpha_base,
                            col[0], col[1], col[2], o.p[2], flow[0], flow[1], o.radius, cam.tiles_x, cam.tiles_y,
                            &ntiles, o.cov2[0], o.cov2[3]);
                key = order_key(o.p[2]);
                if (out.dir_dist) out.dir_dist[i] = make_double4(o.dir[0], o.dir[1], o.dir[2], o.dist);
            }
        }
        out.valid[i] = ok ? 1 : 0;
        out.tiles[i] = ntiles;
        out.depth_key[i] = key;
    }
    count_valid(ok, key, st);
}

// Host-provided splats (rasterize_forward, rasterizer.cpp:278-306).
struct HostSplat {
    double mean2[2];
    double conic[3];
    double depth;
    double color[3];
    double alpha_base;
    double flow2[2];
    double radius;
    int32_t source_index;
    int32_t pad;
};

__global__ void k_splats_from_host(const HostSplat* sp, int n, DevCamera cam, SplatArrays out, BinState* st) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long key = 0;
    if (i < n) {
        const HostSplat s = sp[i];
        uint32_t ntiles = 0;
        // screen covariance = conic^-1 (only its diagonal feeds the culling extents)
        const double det = s.conic[0] * s.conic[2] - s.conic[1] * s.conic[1];
        const double s00 = det > 0 ? s.conic[2] / det : 1e300, s11 = det > 0 ? s.conic[0] / det : 1e300;
        store_splat(out, i, s.mean2[0], s.mean2[1], s.conic[0], s.conic[1], s.conic[2], s.alpha_base, s.color[0],
                    s.color[1], s.color[2], s.depth, s.flow2[0], s.flow2[1], s.radius, cam.tiles_x, cam.tiles_y,
                    &ntiles, s00, s11);
        out.valid[i] = 1;
        out.tiles[i] = ntiles;
        key = order_key(s.depth);
        out.depth_key[i] = key;
        out.source_index[i] = s.source_index;
    }
    count_valid(i < n, key, st);
}

// ---------------------------------------------------------------------------
// FP64 pixel blend, one warp per listed pixel (rasterizer.cpp:97-122 exactly).
// Lanes evaluate 32 consecutive splats of the tile list in parallel; the
// sequential transmittance walk is then replayed identically by every lane.
__global__ void __launch_bounds__(256) k_blend_fp64(SplatArrays sp, const uint32_t* __restrict__ vals,
                                                    const uint2* __restrict__ ranges, DevCamera cam, double3 bg,
                                                    int flow_mode, float* image, double* image64, double* final_T,
                                                    uint32_t* n_contrib, const uint32_t* __restrict__ list,
                                                    const int* __restrict__ count) {
    const int lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int total = *count;
    for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < total; w += nwarps) {
        const uint32_t pix = list[w];
        const int x = pix % cam.width, y = pix / cam.width;
        const int tile = (y / kTile) * cam.tiles_x + (x / kTile);
        const uint2 rg = ranges[tile];
        double T = 1, acc0 = 0, acc1 = 0, acc2 = 0;
        int contrib = 0;
        bool done = false;
        // Software pipeline over the 32-entry batches: the splat ids run two batches ahead and
        // the records one batch ahead, so their dependent L2 round trips overlap the current
        // batch's exp and transmittance walk instead of starting it.
        const double4* __restrict__ colrec = flow_mode ? sp.flow_radius : sp.color_depth;
        uint32_t id1 = 0, id2 = 0;  // ids of the next batch and the one after
        if (rg.x + lane < rg.y) id1 = vals[rg.x + lane];
        if (rg.x + 32 + lane < rg.y) id2 = vals[rg.x + 32 + lane];
        double2 mN = make_double2(0, 0);
        double4 cabN = make_double4(0, 0, 0, 0), colN = make_double4(0, 0, 0, 0);
        if (rg.x + lane < rg.y) {
            mN = sp.mean2[id1];
            cabN = sp.conic_ab[id1];
            colN = colrec[id1];
        }
        for (uint32_t base = rg.x; base < rg.y && !done; base += 32) {
            const uint32_t j = base + lane;
            const double2 m = mN;
            const double4 cab = cabN, col = colN;
            // prefetch: records of batch base + 32 (ids already here), ids of batch base + 64
            if (j + 32 < rg.y) {
                mN = sp.mean2[id2];
                cabN = sp.conic_ab[id2];
                colN = colrec[id2];
            }
            if (j + 64 < rg.y) id2 = vals[j + 64];
            bool accept = false;
            double a = 0, c0 = 0, c1 = 0, c2 = 0;
            if (j < rg.y) {
                const double dx = x - m.x, dy = y - m.y;
                const double power = -0.5 * (cab.x * dx * dx + cab.z * dy * dy) - cab.y * dx * dy;
                if (!(power > 0)) {
                    a = smin(kAlphaClamp, cab.w * rgs_exp::glibc_exp(power));
                    accept = !(a < kMinAlpha);
                }
                if (accept) {
                    c0 = col.x;
                    c1 = col.y;
                    c2 = flow_mode ? 0.0 : col.z;
                }
            }
            // The transmittance walk (the only sequential part) is replayed by every lane with
            // one shuffle per accepted entry; each lane keeps the T in front of its own entry
            // and adds its colour contribution itself (summed over the warp at the end).
            unsigned mask = __ballot_sync(0xffffffffu, accept);
            double myT = 0;
            int stop_lane = 32;
            while (mask) {
                const int l = __ffs(mask) - 1;
                mask &= mask - 1;
                const double al = __shfl_sync(0xffffffffu, a, l);
                const double test_T = T * (1 - al);
                if (test_T < kStopT) {
                    done = true;
                    stop_lane = l;
                    break;
                }
                if (lane == l) myT = T;
                T = test_T;
                contrib = (int)(base + l - rg.x) + 1;
            }
            if (accept && lane < stop_lane) {
                const double wgt = a * myT;
                acc0 = acc0 + c0 * wgt;
                acc1 = acc1 + c1 * wgt;
                acc2 = acc2 + c2 * wgt;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            acc0 += __shfl_xor_sync(0xffffffffu, acc0, o);
            acc1 += __shfl_xor_sync(0xffffffffu, acc1, o);
            acc2 += __shfl_xor_sync(0xffffffffu, acc2, o);
        }
        if (lane == 0) {
            acc0 = acc0 + T * bg.x;
            acc1 = acc1 + T * bg.y;
            acc2 = acc2 + T * bg.z;
            const int ch = flow_mode ? 2 : 3;
            if (image64) {  // RGS_FLAG_IMAGE_F64: the reference's double image, unrounded
                image64[(size_t)pix * ch + 0] = acc0;
                image64[(size_t)pix * ch + 1] = acc1;
                if (!flow_mode) image64[(size_t)pix * 3 + 2] = acc2;
            } else {
                image[(size_t)pix * ch + 0] = (float)acc0;
                image[(size_t)pix * ch + 1] = (float)acc1;
                if (!flow_mode) image[(size_t)pix * 3 + 2] = (float)acc2;
            }
            if (!flow_mode) {
                if (final_T) final_T[pix] = T;
                if (n_contrib) n_contrib[pix] = (uint32_t)contrib | kSlowBit;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Deterministic backward (RGS_FLAG_DETERMINISTIC, the reference-KAT mode): the
// reference's own order, FP64 throughout, no atomics.
//   tiles:  one thread per tile replays its pixels row-major, positions descending,
//           into per-(tile, position) accumulators (rasterizer.cpp:428-468);
//   reduce: one thread per splat sums its accumulators over its tiles in increasing
//           tile order (rasterizer.cpp:471-483), locating itself in each tile list by
//           binary search on the depth rank.

__global__ void k_inverse_rank(const uint32_t* __restrict__ sorted_ids, const int* __restrict__ n_valid,
                               uint32_t* rank) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < *n_valid) rank[sorted_ids[r]] = (uint32_t)r;
}

__global__ void k_backward_det_tiles(SplatArrays sp, const uint32_t* __restrict__ vals,
                                     const uint2* __restrict__ ranges, DevCamera cam, double3 bg,
                                     const double* __restrict__ final_T, const uint32_t* __restrict__ n_contrib,
                                     const float* __restrict__ dL, double* tile_grads) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= cam.tiles_x * cam.tiles_y) return;
    const uint2 rg = ranges[t];
    const int px0 = (t % cam.tiles_x) * kTile, py0 = (t / cam.tiles_x) * kTile;
    const int px1 = min(px0 + kTile, cam.width), py1 = min(py0 + kTile, cam.height);
    for (int y = py0; y < py1; ++y)
        for (int x = px0; x < px1; ++x) {
            const size_t pix = (size_t)y * cam.width + x;
            const int contrib = (int)(n_contrib[pix] & ~kSlowBit);
            if (contrib == 0) continue;
            const double g0 = dL[pix * 3 + 0], g1 = dL[pix * 3 + 1], g2 = dL[pix * 3 + 2];
            double T_run = final_T[pix];
            double s0 = bg.x * final_T[pix], s1 = bg.y * final_T[pix], s2 = bg.z * final_T[pix];
            for (int pos = contrib - 1; pos >= 0; --pos) {
                const uint32_t id = vals[rg.x + pos];
                const double2 m = sp.mean2[id];
                const double4 cab = sp.conic_ab[id];
                const double dx = (double)x - m.x, dy = (double)y - m.y;
                const double power = -0.5 * (cab.x * dx * dx + cab.z * dy * dy) - cab.y * dx * dy;
                if (power > 0) continue;
                const double raw = cab.w * rgs_exp::glibc_exp(power);
                const double a = smin(kAlphaClamp, raw);
                if (a < kMinAlpha) continue;
                const double T_before = T_run / (1 - a);
                const double w = a * T_before;
                double* o = tile_grads + (size_t)(rg.x + pos) * 9;
                o[0] = o[0] + w * g0;
                o[1] = o[1] + w * g1;
                o[2] = o[2] + w * g2;
                const double4 c = sp.color_depth[id];
                double dL_da = g0 * (c.x * T_before - s0 / (1 - a));
                dL_da += g1 * (c.y * T_before - s1 / (1 - a));
                dL_da += g2 * (c.z * T_before - s2 / (1 - a));
                if (raw <= kAlphaClamp) {
                    o[8] += dL_da * (a / cab.w);
                    const double dpow = dL_da * a;
                    o[3] = o[3] + dpow * (-0.5 * dx * dx);
                    o[4] = o[4] + dpow * (-dx * dy);
                    o[5] = o[5] + dpow * (-0.5 * dy * dy);
                    o[6] = o[6] + dpow * (cab.x * dx + cab.y * dy);
                    o[7] = o[7] + dpow * (cab.y * dx + cab.z * dy);
                }
                s0 = s0 + c.x * w;
                s1 = s1 + c.y * w;
                s2 = s2 + c.z * w;
                T_run = T_before;
            }
        }
}

__global__ void k_backward_det_reduce(SplatArrays sp, const uint32_t* __restrict__ vals,
                                      const uint2* __restrict__ ranges, int tiles_x,
                                      const uint32_t* __restrict__ rank, const double* __restrict__ tile_grads,
                                      int n, double* sg) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !sp.valid[i]) return;
    const ushort4 q = sp.rect[i];
    if (sp.tiles[i] == 0) return;
    const uint32_t r = rank[i];
    double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int ty = q.z; ty <= q.w; ++ty)
        for (int tx = q.x; tx <= q.y; ++tx) {
            const uint2 rg = ranges[ty * tiles_x + tx];
            uint32_t lo = rg.x, hi = rg.y;  // first position with rank >= r
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (rank[vals[mid]] < r) lo = mid + 1;
                else hi = mid;
            }
            const double* g = tile_grads + (size_t)lo * 9;
#pragma unroll
            for (int k = 0; k < 9; ++k) acc[k] += g[k];
        }
#pragma unroll
    for (int k = 0; k < 9; ++k) sg[(size_t)i * 9 + k] = acc[k];
}

// project() of one already-sliced Gaussian (rasterizer.cpp:215-276) for the C++
// drop-in's single-Gaussian entry point; SH exactly as the reference (all 16 terms).
__global__ void k_project_one(const double* __restrict__ sl, DevCamera cam, const double* __restrict__ sh,
                              int sh_degree, double opacity_logit, HostSplat* out, int* survived, double* cache) {
    SliceState s;
#pragma unroll
    for (int k = 0; k < 3; ++k) s.mean[k] = sl[k];
#pragma unroll
    for (int k = 0; k < 9; ++k) s.cov[k] = sl[3 + k];
    s.decay = sl[12];
#pragma unroll
    for (int k = 0; k < 3; ++k) s.speed[k] = sl[13 + k];
    ProjState o;
    if (!d_project_geom(s, cam, opacity_logit, o)) {
        *survived = 0;
        return;
    }
    double basis[16];
    d_sh_basis(o.dir, sh_degree, basis);
    HostSplat h;
    bool clamped[3];
    for (int ch = 0; ch < 3; ++ch) {
        double a = sh[ch * 16] * basis[0];
        for (int k = 1; k < 16; ++k) a += sh[ch * 16 + k] * basis[k];
        const double c = a + 0.5;
        clamped[ch] = c < 0;
        h.color[ch] = c < 0 ? 0.0 : c;
    }
    if (cache) {  // ProjectCache (rasterizer.cpp:261-275), layout of rgs_project_sliced_cache
        for (int k = 0; k < 3; ++k) cache[k] = o.p[k];
        for (int k = 0; k < 6; ++k) cache[3 + k] = o.T[k];
        for (int k = 0; k < 4; ++k) cache[9 + k] = o.cov2[k];
        for (int k = 0; k < 3; ++k) cache[13 + k] = o.dir[k];
        cache[16] = o.dist;
        for (int k = 0; k < 16; ++k) cache[17 + k] = basis[k];
        d_sh_basis_grad(o.dir, sh_degree, cache + 33);
        for (int ch = 0; ch < 3; ++ch) cache[81 + ch] = clamped[ch] ? 1.0 : 0.0;
        cache[84] = o.opacity;
    }
    for (int r = 0; r < 2; ++r) {
        double a = o.T[r * 3 + 0] * s.speed[0];
        a += o.T[r * 3 + 1] * s.speed[1];
        a += o.T[r * 3 + 2] * s.speed[2];
        h.flow2[r] = a;
    }
    h.mean2[0] = o.mean2[0];
    h.mean2[1] = o.mean2[1];
    h.conic[0] = o.conic[0];
    h.conic[1] = o.conic[1];
    h.conic[2] = o.conic[2];
    h.depth = o.p[2];
    h.alpha_base = o.alpha_base;
    h.radius = o.radius;
    h.source_index = -1;
    h.pad = 0;
    *out = h;
    *survived = 1;
}

__global__ void k_mark_all_slow(int n, uint32_t* list, int* count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) list[i] = (uint32_t)i;
    if (i == 0) *count = n;
}

// ---------------------------------------------------------------------------
// FP64 backward replay of the listed (slow) pixels, one warp per pixel
// (rasterizer.cpp:437-468).  Lanes evaluate 32 positions (descending) in parallel,
// the T/suffix recursion is replayed by every lane, then each lane scatters its
// splat's nine screen-space gradients with FP64 atomics.
__global__ void __launch_bounds__(256) k_backward_fp64(SplatArrays sp, const uint32_t* __restrict__ vals,
                                                       const uint2* __restrict__ ranges, DevCamera cam,
                                                       double3 bg, const double* __restrict__ final_T,
                                                       const uint32_t* __restrict__ n_contrib,
                                                       const float* __restrict__ dL, const uint32_t* list,
                                                       const int* count, double* sg, unsigned long long* sgx) {
    const int lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int total = *count;
    for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < total; w += nwarps) {
        const uint32_t pix = list[w];
        const int contrib = (int)(n_contrib[pix] & ~kSlowBit);
        if (contrib == 0) continue;
        const int x = pix % cam.width, y = pix / cam.width;
        const int tile = (y / kTile) * cam.tiles_x + (x / kTile);
        const uint2 rg = ranges[tile];
        const double g0 = dL[(size_t)pix * 3 + 0], g1 = dL[(size_t)pix * 3 + 1], g2 = dL[(size_t)pix * 3 + 2];
        const double fT = final_T[pix];
        double T_run = fT;
        double s0 = bg.x * fT, s1 = bg.y * fT, s2 = bg.z * fT;
        // Software pipeline over the 32-entry batches (as k_blend_fp64): ids two batches ahead,
        // records one batch ahead.
        uint32_t idN = 0, id2 = 0;
        if (contrib - 1 - lane >= 0) idN = vals[rg.x + contrib - 1 - lane];
        if (contrib - 33 - lane >= 0) id2 = vals[rg.x + contrib - 33 - lane];
        double2 mN = make_double2(0, 0);
        double4 cabN = make_double4(0, 0, 0, 0), colN = make_double4(0, 0, 0, 0);
        if (contrib - 1 - lane >= 0) {
            mN = sp.mean2[idN];
            cabN = sp.conic_ab[idN];
            colN = sp.color_depth[idN];
        }
        for (int hi = contrib; hi > 0; hi -= 32) {
            const int pos = hi - 1 - lane;
            const uint32_t id = idN;
            const double2 m = mN;
            const double4 cab = cabN, col = colN;
            if (pos - 32 >= 0) {
                idN = id2;
                mN = sp.mean2[id2];
                cabN = sp.conic_ab[id2];
                colN = sp.color_depth[id2];
            }
            if (pos - 64 >= 0) id2 = vals[rg.x + pos - 64];
            bool pass = false;
            double a = 0, raw = 0, dx = 0, dy = 0, c0 = 0, c1 = 0, c2 = 0;
            if (pos >= 0) {
                dx = (double)x - m.x;
                dy = (double)y - m.y;
                const double power = -0.5 * (cab.x * dx * dx + cab.z * dy * dy) - cab.y * dx * dy;
                if (!(power > 0)) {
                    raw = cab.w * rgs_exp::glibc_exp(power);
                    a = smin(kAlphaClamp, raw);
                    pass = !(a < kMinAlpha);
                }
                if (pass) {
                    c0 = col.x;
                    c1 = col.y;
                    c2 = col.z;
                }
            }
            // The back-to-front recursion T_before = T_run / (1 - a), suffix += c a T_before over
            // lanes 0..31 (= descending positions) as warp scans: an inclusive product of (1 - a)
            // and an exclusive sum of the colour contributions.  No decision depends on T here
            // (the forward fixed contrib), so the ~1-ulp reassociation only reaches the values.
            double f = pass ? 1 - a : 1.0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double y = __shfl_up_sync(0xffffffffu, f, o);
                if (lane >= o) f *= y;
            }
            const double my_Tb = T_run / f;
            const double wl = pass ? a * my_Tb : 0.0;
            double e0 = c0 * wl, e1 = c1 * wl, e2 = c2 * wl;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double y0 = __shfl_up_sync(0xffffffffu, e0, o);
                const double y1 = __shfl_up_sync(0xffffffffu, e1, o);
                const double y2 = __shfl_up_sync(0xffffffffu, e2, o);
                if (lane >= o) {
                    e0 += y0;
                    e1 += y1;
                    e2 += y2;
                }
            }
            // exclusive prefix = inclusive - own contribution
            const double my_s0 = s0 + (e0 - c0 * wl), my_s1 = s1 + (e1 - c1 * wl), my_s2 = s2 + (e2 - c2 * wl);
            T_run = T_run / __shfl_sync(0xffffffffu, f, 31);
            s0 = s0 + __shfl_sync(0xffffffffu, e0, 31);
            s1 = s1 + __shfl_sync(0xffffffffu, e1, 31);
            s2 = s2 + __shfl_sync(0xffffffffu, e2, 31);
            if (pass) {
                const double T_before = my_Tb;
                const double wgt = a * T_before;
                double* o = sg + (size_t)id * 9;
                unsigned long long* ox = sgx ? sgx + (size_t)id * 18 : nullptr;
                auto add = [&](int q, double val) {
                    if (ox) fixed_add(ox + 2 * q, val);
                    else atomicAdd(o + q, val);
                };
                add(0, wgt * g0);
                add(1, wgt * g1);
                add(2, wgt * g2);
                const double v0 = c0 * T_before - my_s0 / (1 - a);
                const double v1 = c1 * T_before - my_s1 / (1 - a);
                const double v2 = c2 * T_before - my_s2 / (1 - a);
                double dL_da = g0 * v0;
                dL_da += g1 * v1;
                dL_da += g2 * v2;
                if (raw <= kAlphaClamp) {
                    add(8, dL_da * (a / cab.w));
                    const double dpow = dL_da * a;
                    add(3, dpow * (-0.5 * dx * dx));
                    add(4, dpow * (-dx * dy));
                    add(5, dpow * (-0.5 * dy * dy));
                    add(6, dpow * (cab.x * dx + cab.y * dy));
                    add(7, dpow * (cab.y * dx + cab.z * dy));
                }
            }
        }
    }
}

// K7a's SH loop, one row k per step (compile-time k): loads the row's three coefficients
// (j = 3k + ch) and accumulates acol[ch] += v basis[k], tg[ch][ax] += g_k[ax] v.
template <bool F64, int Kr>
__device__ __forceinline__ void sh_rows(const ParamView& P, int i, int K, const double* dir,
                                        int sh_degree, const double* basis, double* acol, double (*tg)[3]) {
    if constexpr (Kr < 16) {
        if (Kr >= K) return;
        double g3[3];
        d_sh_basis_grad_row<Kr>(dir[0], dir[1], dir[2], sh_degree, g3);
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            const int j = 3 * Kr + ch;
            const double v = ld_coef<F64>(P, i, j);
            if (Kr == 0) {
                acol[ch] = v * basis[0];
#pragma unroll
                for (int ax = 0; ax < 3; ++ax) tg[ch][ax] = g3[ax] * v;
            } else {
                acol[ch] += v * basis[Kr];
#pragma unroll
                for (int ax = 0; ax < 3; ++ax) tg[ch][ax] += g3[ax] * v;
            }
        }
        sh_rows<F64, Kr + 1>(P, i, K, dir, sh_degree, basis, acol, tg);
    }
}

// K7a: colour path of the per-Gaussian backward (rasterizer.cpp:137-147): SH gradients and
// the view-direction term of d mean3, from the forward's direction (K1 stores it; the chain
// is recomputed bit-identically either way).  Split from K7b so neither kernel carries the
// SH basis gradients and the slice state at once (K7 was 255 registers with spills).
template <bool F64>
__global__ void __launch_bounds__(128, 6) k_color_backward(ParamView P, int sh_degree, const uint8_t* __restrict__ valid,
                                                        const double4* __restrict__ dir_dist,
                                                        const double* __restrict__ sgrad, int accumulate,
                                                        float* grads, double* cdm3) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.n || !valid[i]) return;
    const int n = P.n;
    const double4 dd = dir_dist[i];
    struct {
        double dir[3];
        double dist;
    } o = {{dd.x, dd.y, dd.z}, dd.w};
    const double* g9 = sgrad + (size_t)i * 9;
    const double dcol[3] = {g9[0], g9[1], g9[2]};
    // ---- colour path: SH coefficients and view direction (rasterizer.cpp:137-147).
    // The SH blocks are streamed once: the colour (for the clamp flags) and, per channel,
    // t[ch][ax] = sum_k bgrad[k][ax] sh[k][ch] accumulate in the reference's k order.
    const int deg = sh_degree < 0 ? 0 : (sh_degree > 3 ? 3 : sh_degree);
    const int K = (deg + 1) * (deg + 1);
    double basis[16];
    d_sh_basis(o.dir, sh_degree, basis);
    double acol[3] = {0, 0, 0}, tg[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    // one SH row k at a time: its three coefficients (one per channel) and its basis-gradient
    // row (computed on the spot, not a 48-entry array); per channel the k order is the
    // reference's, as in the 48-entry form
    sh_rows<F64, 0>(P, i, K, o.dir, sh_degree, basis, acol, tg);
    bool live[3];
    double dL_ddir[3] = {0, 0, 0};
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        const bool clamped = (acol[ch] + 0.5) < 0;
        live[ch] = !(clamped || dcol[ch] == 0);
        if (!live[ch]) continue;
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) dL_ddir[ax] += dcol[ch] * tg[ch][ax];
    }
    {
        // SH gradients (rasterizer.cpp:139): d_sh(ch, k) = dcol[ch] basis[k] unless clamped
#pragma unroll
        for (int b = 0; b < 12; ++b) {
            float f4[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int j = 4 * b + e, k = j / 3, ch = j - 3 * k;
                f4[e] = live[ch] ? (float)(0.0 + dcol[ch] * basis[k]) : 0.f;
            }
            float4* pb = reinterpret_cast<float4*>(grads + (16 + 4 * (size_t)b) * n) + i;
            if (accumulate) {
                const float4 t = *pb;
                *pb = make_float4(t.x + f4[0], t.y + f4[1], t.z + f4[2], t.w + f4[3]);
            } else {
                *pb = make_float4(f4[0], f4[1], f4[2], f4[3]);
            }
        }
    }
    double dmean3[3] = {0, 0, 0};
    if (dL_ddir[0] != 0 || dL_ddir[1] != 0 || dL_ddir[2] != 0) {
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            double a = 0;
#pragma unroll
            for (int c = 0; c < 3; ++c) a += ((r == c ? 1.0 : 0.0) - o.dir[r] * o.dir[c]) / o.dist * dL_ddir[c];
            dmean3[r] += a;
        }
    }
    cdm3[(size_t)i * 3 + 0] = dmean3[0];
    cdm3[(size_t)i * 3 + 1] = dmean3[1];
    cdm3[(size_t)i * 3 + 2] = dmean3[2];
}

// ---------------------------------------------------------------------------
// K7b: per-Gaussian backward (rasterizer.cpp:134-181, gaussian.cpp:57-101,
// rotor.cpp:138-194).  Recomputes the forward chain from the parameters.
template <bool F64>
__global__ void __launch_bounds__(128, 3) k_gaussian_backward(ParamView P, int sh_degree, DevCamera cam,
                                                           const uint8_t* __restrict__ valid,
                                                           const double* __restrict__ sgrad,
                                                           const double* __restrict__ cdm3, int accumulate,
                                                           float* grads, float* vnorm, int32_t* visible) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.n) return;
    const int n = P.n;
    float4* gm = reinterpret_cast<float4*>(grads);
    float4* gl = reinterpret_cast<float4*>(grads + 4 * (size_t)n);
    float4* gr0 = reinterpret_cast<float4*>(grads + 8 * (size_t)n);
    float4* gr1 = reinterpret_cast<float4*>(grads + 12 * (size_t)n);
    float* gop = grads + 64 * (size_t)n;
    if (!valid[i]) {
        if (!accumulate) {
            const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
            gm[i] = z;
            gl[i] = z;
            gr0[i] = z;
            gr1[i] = z;
#pragma unroll
            for (int b = 0; b < 12; ++b) reinterpret_cast<float4*>(grads + (16 + 4 * (size_t)b) * n)[i] = z;
            gop[i] = 0.f;
            vnorm[i] = 0.f;
            visible[i] = 0;
        }
        return;
    }
    double mean4[4], ls[4], rot[8];
    ld_block<F64>(P, 0, i, mean4);
    ld_block<F64>(P, 1, i, ls);
    ld_block<F64>(P, 2, i, rot);
    ld_block<F64>(P, 3, i, rot + 4);
    const double op = ld_opacity<F64>(P, i);
    SliceState s;
    d_slice(mean4, ls, rot, cam.time, s);
    ProjState o;
    d_project_geom(s, cam, op, o);

    const double* g9 = sgrad + (size_t)i * 9;
    const double dcol[3] = {g9[0], g9[1], g9[2]};
    const double dcon[3] = {g9[3], g9[4], g9[5]};
    const double dm2[2] = {g9[6], g9[7]};
    const double dab = g9[8];

    // out[0..16]: mean4, ls4, rotor8, opacity; the 48 SH gradients are written directly.
    double out[17];
#pragma unroll
    for (int k = 0; k < 17; ++k) out[k] = 0;

    // ---- colour path: K7a (k_color_backward) left its d mean3 term in cdm3
    double dmean3[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) dmean3[r] = 0.0 + cdm3[(size_t)i * 3 + r];
    // ---- alpha_base = opacity * decay
    const double dL_ddecay = dab * o.opacity;
    out[16] += dab * s.decay * o.opacity * (1 - o.opacity);

    // ---- conic = cov2^-1 -> cov2 -> cov3, T
    const double invdet = 1.0 / o.det;
    const double con[4] = {o.cov2[3] * invdet, -o.cov2[1] * invdet, -o.cov2[2] * invdet, o.cov2[0] * invdet};
    const double gh[4] = {dcon[0], dcon[1] / 2, dcon[1] / 2, dcon[2]};
    double P1[4], H[4];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < 2; ++c) P1[r * 2 + c] = (-con[r * 2]) * gh[c] + (-con[r * 2 + 1]) * gh[2 + c];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < 2; ++c) H[r * 2 + c] = P1[r * 2] * con[c] + P1[r * 2 + 1] * con[2 + c];
    double dcov3[9];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        const double q0 = o.T[r] * H[0] + o.T[3 + r] * H[2];
        const double q1 = o.T[r] * H[1] + o.T[3 + r] * H[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) dcov3[r * 3 + c] = q0 * o.T[c] + q1 * o.T[3 + c];
    }
    double dT[6];
    {
        const double HH[4] = {H[0] + H[0], H[1] + H[2], H[2] + H[1], H[3] + H[3]};
        double HT[6];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) HT[r * 3 + c] = HH[r * 2] * o.T[c] + HH[r * 2 + 1] * o.T[3 + c];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                double a = HT[r * 3 + 0] * s.cov[0 * 3 + c];
                a += HT[r * 3 + 1] * s.cov[1 * 3 + c];
                a += HT[r * 3 + 2] * s.cov[2 * 3 + c];
                dT[r * 3 + c] = a;
            }
    }
    // ---- mean2 = pinhole(p_cam); T = J R (J depends on p_cam)
    const double z = o.p[2], z2 = z * z, z3 = z2 * z;
    const double J[6] = {cam.fx / z, 0, -cam.fx * o.p[0] / z2, 0, cam.fy / z, -cam.fy * o.p[1] / z2};
    double dpc[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) dpc[r] = J[r] * dm2[0] + J[3 + r] * dm2[1];
    double dJ[6];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            double a = dT[r * 3 + 0] * cam.R[c * 3 + 0];
            a += dT[r * 3 + 1] * cam.R[c * 3 + 1];
            a += dT[r * 3 + 2] * cam.R[c * 3 + 2];
            dJ[r * 3 + c] = a;
        }
    dpc[0] += dJ[2] * (-cam.fx / z2);
    dpc[1] += dJ[5] * (-cam.fy / z2);
    dpc[2] += dJ[0] * (-cam.fx / z2) + dJ[2] * (2 * cam.fx * o.p[0] / z3) + dJ[4] * (-cam.fy / z2) +
              dJ[5] * (2 * cam.fy * o.p[1] / z3);
#pragma unroll
    for (int r = 0; r < 3; ++r) dmean3[r] += cam.R[r] * dpc[0] + cam.R[3 + r] * dpc[1] + cam.R[6 + r] * dpc[2];

    // ---- slice_backward (gaussian.cpp:57-101), dL_dspeed = 0
    {
        const double W = s.W, lambda = 1 / W, dt = s.dt;
        const double dL_dlambda = dL_ddecay * (-0.5 * dt * dt) * s.decay;
        out[3] += dL_ddecay * lambda * dt * s.decay;
        out[0] += dmean3[0];
        out[1] += dmean3[1];
        out[2] += dmean3[2];
        out[3] += -(s.speed[0] * dmean3[0] + s.speed[1] * dmean3[1] + s.speed[2] * dmean3[2]);
        double dV[3];
#pragma unroll
        for (int r = 0; r < 3; ++r) dV[r] = (dt / W) * dmean3[r];
        const double vdm = s.V[0] * dmean3[0] + s.V[1] * dmean3[1] + s.V[2] * dmean3[2];
        double dW = -(dt * vdm) / (W * W);
        double GV[3], SV[3];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            GV[r] = dcov3[r * 3] * s.V[0] + dcov3[r * 3 + 1] * s.V[1] + dcov3[r * 3 + 2] * s.V[2];
            SV[r] = (dcov3[r * 3] + dcov3[r]) * s.V[0] + (dcov3[r * 3 + 1] + dcov3[3 + r]) * s.V[1] +
                    (dcov3[r * 3 + 2] + dcov3[6 + r]) * s.V[2];
        }
#pragma unroll
        for (int r = 0; r < 3; ++r) dV[r] += (-SV[r]) / W;
        dW += (s.V[0] * GV[0] + s.V[1] * GV[1] + s.V[2] * GV[2]) / (W * W);
        dW += -dL_dlambda / (W * W);
        double G4[16];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) G4[r * 4 + c] = 0;
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) G4[r * 4 + c] = dcov3[r * 3 + c];
#pragma unroll
        for (int r = 0; r < 3; ++r) G4[r * 4 + 3] = dV[r];
        G4[15] = dW;
        d_g4_backward(s, rot, G4, out);
    }
    // ---- write (scene SoA layout)
    float f[17];
#pragma unroll
    for (int k = 0; k < 17; ++k) f[k] = (float)out[k];
    float4 om = make_float4(f[0], f[1], f[2], f[3]);
    float4 ol = make_float4(f[4], f[5], f[6], f[7]);
    float4 o0 = make_float4(f[8], f[9], f[10], f[11]);
    float4 o1 = make_float4(f[12], f[13], f[14], f[15]);
    const float vn = (float)sqrt(dm2[0] * dm2[0] + dm2[1] * dm2[1]);
    if (accumulate) {
        float4 t;
        t = gm[i]; gm[i] = make_float4(t.x + om.x, t.y + om.y, t.z + om.z, t.w + om.w);
        t = gl[i]; gl[i] = make_float4(t.x + ol.x, t.y + ol.y, t.z + ol.z, t.w + ol.w);
        t = gr0[i]; gr0[i] = make_float4(t.x + o0.x, t.y + o0.y, t.z + o0.z, t.w + o0.w);
        t = gr1[i]; gr1[i] = make_float4(t.x + o1.x, t.y + o1.y, t.z + o1.z, t.w + o1.w);
        gop[i] += f[16];
        vnorm[i] += vn;
        visible[i] += 1;
    } else {
        gm[i] = om;
        gl[i] = ol;
        gr0[i] = o0;
        gr1[i] = o1;
        gop[i] = f[16];
        vnorm[i] = vn;
        visible[i] = 1;
    }
}

}  // namespace rgs_dev

// ---------------------------------------------------------------------------
namespace rgs_launch {
using namespace rgs_dev;

static inline int blocks(long long n, int t) { return (int)((n + t - 1) / t); }

void preprocess(const float* params, const double* params64, int n, int sh_degree, const DevCamera& cam,
                const SplatArrays& out, BinState* st, cudaStream_t s, const SliceCacheView* cache) {
    if (n <= 0) return;
    ParamView P{params, n, params64};
    const SliceCacheView C = cache ? *cache : SliceCacheView{nullptr, nullptr};
    if (params64) {
        if (cache) k_preprocess<true, true><<<blocks(n, 128), 128, 0, s>>>(P, sh_degree, cam, out, st, C);
        else k_preprocess<true, false><<<blocks(n, 128), 128, 0, s>>>(P, sh_degree, cam, out, st, C);
    } else {
        if (cache) k_preprocess<false, true><<<blocks(n, 128), 128, 0, s>>>(P, sh_degree, cam, out, st, C);
        else k_preprocess<false, false><<<blocks(n, 128), 128, 0, s>>>(P, sh_degree, cam, out, st, C);
    }
}

size_t slice_cache_bytes(int n) { return (size_t)std::max(n, 1) * (kSliceCacheBlocks * sizeof(double2) + 1) + 64; }

void slice_cache(const float* params, const double* params64, int n, void* buf, SliceCacheView* view, cudaStream_t s) {
    view->blk = static_cast<double2*>(buf);
    view->status = reinterpret_cast<int8_t*>(view->blk + kSliceCacheBlocks * (size_t)std::max(n, 1));
    if (n <= 0) return;
    ParamView P{params, n, params64};
    if (params64) k_slice_cache<true><<<blocks(n, 128), 128, 0, s>>>(P, *view);
    else k_slice_cache<false><<<blocks(n, 128), 128, 0, s>>>(P, *view);
}

void splats_from_host(const void* splats, int n, const DevCamera& cam, const SplatArrays& out, BinState* st,
                      cudaStream_t s) {
    if (n <= 0) return;
    k_splats_from_host<<<blocks(n, 128), 128, 0, s>>>(reinterpret_cast<const HostSplat*>(splats), n, cam, out, st);
}

void mark_all_slow(int n_pixels, uint32_t* slow_list, int* slow_count, cudaStream_t s) {
    k_mark_all_slow<<<blocks(n_pixels, 256), 256, 0, s>>>(n_pixels, slow_list, slow_count);
}

static int persistent_blocks(int max_items) {
    // Persistent grid: 148 SMs x 8 CTAs x 8 warps, capped by the item count.
    const int warps = 148 * 8 * 8;
    const int need = max_items < warps ? max_items : warps;
    return (need + 7) / 8 > 0 ? (need + 7) / 8 : 1;
}

void blend_fp64_pixels(const SplatArrays& sp, const uint32_t* pair_vals, const uint2* ranges, const DevCamera& cam,
                       double3 bg, int flow_mode, float* image, double* image64, double* final_T, uint32_t* n_contrib,
                       const uint32_t* slow_list, const int* slow_count, int max_pixels, cudaStream_t s) {
    if (max_pixels <= 0) return;
    k_blend_fp64<<<persistent_blocks(max_pixels), 256, 0, s>>>(sp, pair_vals, ranges, cam, bg, flow_mode, image,
                                                               image64, final_T, n_contrib, slow_list, slow_count);
}

void backward_deterministic(const SplatArrays& sp, const uint32_t* pair_vals, const uint2* ranges,
                            const DevCamera& cam, double3 bg, const double* final_T, const uint32_t* n_contrib,
                            const float* dL_dimage, const uint32_t* sorted_ids, const int* n_valid_dev, int n,
                            uint32_t* rank, double* tile_grads, double* screen_grads, cudaStream_t s) {
    const int ntiles = cam.tiles_x * cam.tiles_y;
    if (n <= 0 || ntiles <= 0) return;
    k_inverse_rank<<<blocks(n, 256), 256, 0, s>>>(sorted_ids, n_valid_dev, rank);
    k_backward_det_tiles<<<blocks(ntiles, 64), 64, 0, s>>>(sp, pair_vals, ranges, cam, bg, final_T, n_contrib,
                                                           dL_dimage, tile_grads);
    k_backward_det_reduce<<<blocks(n, 128), 128, 0, s>>>(sp, pair_vals, ranges, cam.tiles_x, rank, tile_grads, n,
                                                         screen_grads);
}

int project_one(const double* sliced16_dev, const DevCamera& cam, const double* sh48_dev, int sh_degree,
                double opacity_logit, void* out_dev, int* survived_dev, cudaStream_t s, double* cache_dev) {
    k_project_one<<<1, 1, 0, s>>>(sliced16_dev, cam, sh48_dev, sh_degree, opacity_logit,
                                  reinterpret_cast<HostSplat*>(out_dev), survived_dev, cache_dev);
    return 0;
}

void backward_fp64_pixels(const SplatArrays& sp, const uint32_t* pair_vals, const uint2* ranges,
                          const DevCamera& cam, double3 bg, const double* final_T, const uint32_t* n_contrib,
                          const float* dL_dimage, const uint32_t* slow_list, const int* slow_count, int max_pixels,
                          double* screen_grads, cudaStream_t s, unsigned long long* screen_grads_fixed) {
    if (max_pixels <= 0) return;
    k_backward_fp64<<<persistent_blocks(max_pixels), 256, 0, s>>>(sp, pair_vals, ranges, cam, bg, final_T, n_contrib,
                                                                  dL_dimage, slow_list, slow_count, screen_grads,
                                                                  screen_grads_fixed);
}

}  // namespace rgs_launch
namespace rgs_dev {
__global__ void k_fixed_to_double(const unsigned long long* __restrict__ fixed, size_t n, double* __restrict__ out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        out[i] = fixed_value(fixed + 2 * i);
}
}  // namespace rgs_dev
namespace rgs_launch {
void fixed_to_double(const unsigned long long* fixed, size_t n_values, double* out, cudaStream_t s) {
    if (n_values == 0) return;
    k_fixed_to_double<<<(int)std::min<size_t>((n_values + 255) / 256, 148 * 8), 256, 0, s>>>(fixed, n_values, out);
}

// K7a (part & 1): the colour / SH path; K7b (part & 2): the geometry chain (reads K7a's d mean3).
void gaussian_backward(const float* params, const double* params64, int n, int sh_degree, const DevCamera& cam,
                       const double4* dir_dist, double* color_dmean3, const uint8_t* valid, const double* screen_grads,
                       int accumulate, float* grads, float* vnorm, int32_t* visible, cudaStream_t s, int part) {
    if (n <= 0) return;
    ParamView P{params, n, params64};
    if (params64) {
        if (part & 1)
            k_color_backward<true><<<blocks(n, 128), 128, 0, s>>>(P, sh_degree, valid, dir_dist, screen_grads,
                                                                   accumulate, grads, color_dmean3);
        if (part & 2)
            k_gaussian_backward<true><<<blocks(n, 128), 128, 0, s>>>(P, sh_degree, cam, valid, screen_grads,
                                                                     color_dmean3, accumulate, grads, vnorm, visible);
    } else {
        if (part & 1)
            k_color_backward<false><<<blocks(n, 128), 128, 0, s>>>(P, sh_degree, valid, dir_dist, screen_grads,
                                                                    accumulate, grads, color_dmean3);
        if (part & 2)
            k_gaussian_backward<false><<<blocks(n, 128), 128, 0, s>>>(P, sh_degree, cam, valid, screen_grads,
                                                                      color_dmean3, accumulate, grads, vnorm, visible);
    }
}

}  // namespace rgs_launch
