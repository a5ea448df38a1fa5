// FP32 tile kernels: K5 forward blend and K6 backward replay
// (rasterizer.cpp:97-122 and 437-468).
//
// Every (pixel, splat) evaluation is done in FP32 together with a bound on its error
// against the FP64 reference.  A gate decision (power > 0, alpha < 1/255,
// T(1-alpha) < 1e-4, and the backward's unclamped alpha <= 0.99) whose FP32 value
// lies inside the bound marks the pixel "slow": the thread stops and k_blend_fp64
// (k_fp64.cu) recomputes the whole pixel in FP64.  Every decision the FP32 path keeps
// is therefore the FP64 decision, and K6 replays exactly those.
//
// Layout: one CTA per 16x16 tile, one thread per pixel, each warp owns an 8x4
// sub-tile.  Splats are staged 256 at a time in shared memory; each warp first culls
// the staged splats against its sub-tile with the bounding box of the alpha >= 1/255
// ellipse (a ballot per 32 splats) and then walks only the surviving ones, in depth
// order.  The exponent is kept in log2 units so alpha costs one MUFU.EX2.
#include <cstdlib>

#include "rgs_internal.cuh"

namespace rgs_dev {

// One staged splat of a tile batch (64 B).
struct StagedSplat {
    float4 a;  // (mx, my, ca2, cb2)   mean relative to the tile origin
    float4 b;  // (cc2, D, pa2, cs2n)  D: error floor incl. the mean's FP32 rounding
    float4 c;  // (r, g, b, alpha_base)   flow: (fx, fy, 0, alpha_base)
    float4 d;  // (ex, ey, pc2, R)     culling extents, clamp-gate power, R >= 1 / (1 - alpha_max)
};

// Staged values of one splat, relative to the tile origin (px0, py0); `lmax`: the radial cull's
// eigenvalue bound.  Shared by K5 (structure-of-arrays staging) and K6 (StagedSplat).
template <bool FLOW>
__device__ __forceinline__ void stage_values(const SplatArrays& sp, uint32_t id, double px0, double py0, float4& A,
                                             float4& Bv, float4& C, float4& Dv, float& lmax) {
    const double2 m = sp.mean2[id];
    const float mx = (float)(m.x - px0), my = (float)(m.y - py0);
    const float4 cf = sp.conic_f[id];
    const float4 col = sp.color_f[id];
    const float4 g = sp.guard_f[id];
    const float4 e = sp.ext_f[id];
    const float D = 1.5e-6f + 1.2e-7f * (fabsf(mx) * e.z + fabsf(my) * e.w);
    A = make_float4(mx, my, cf.x, cf.y);
    Bv = make_float4(cf.z, D, col.w, g.x);
    if (FLOW) {
        const double4 f = sp.flow_radius[id];
        C = make_float4((float)f.x, (float)f.y, 0.f, cf.w);
    } else {
        C = make_float4(col.x, col.y, col.z, cf.w);
    }
    // The T-gate's per-blend error growth alpha ln2 M / (1 - alpha) (M bounds the error of the
    // log2 power, so ln2 M bounds the relative error of alpha), with 1 / (1 - alpha) <=
    // 1 / (1 - min(0.99, ab)): R = ln2 / (1 - min(0.99, ab)), rounded up -- and the largest
    // eigenvalue of the (negative definite) log2-power form [[ca2, cb2/2], [cb2/2, cc2]] plus a
    // slack far above its FP32 rounding: p2 <= lmax d^2 at Euclidean distance d from the mean
    // (near-degenerate conics get lmax >= 0: no culling from it).  Both precomputed per splat by K1
    // (d_blend_record, k_fp64.cu).
    Dv = make_float4(e.x, e.y, g.y, g.z);
    lmax = g.w;
}

template <bool FLOW>
__device__ __forceinline__ void stage(const SplatArrays& sp, uint32_t id, double px0, double py0, StagedSplat* dst,
                                      float* lmax) {
    float4 A, Bv, C, Dv;
    float l;
    stage_values<FLOW>(sp, id, px0, py0, A, Bv, C, Dv, l);
    dst->a = A;
    dst->b = Bv;
    dst->c = C;
    dst->d = Dv;
    *lmax = l;
}

// Per-warp culling of a staged splat against the warp's 8 x (H+1) sub-tile with the bounding box
// of its alpha >= 1/255 ellipse (an exact ellipse-rectangle test removed 19% of the evaluations
// but cost more in the ballot phase than it saved: measured, round 1), and a radial bound:
// p2 <= lmax d^2 with d the distance from the mean to the sub-tile's pixel rectangle (shrunk by
// 1e-3 px).  With the error floor D and a 1e-3 margin below the alpha threshold, every pixel of
// the sub-tile certainly skips the splat in FP64, so K5 and K6 (which cull identically) drop it
// without changing any gate decision.
template <int H = 3>
__device__ __forceinline__ bool overlaps_v(const float4& a, const float4& b, const float4& d, float lmax, float sx0,
                                           float sy0) {
    if (!((a.x + d.x >= sx0) && (a.x - d.x <= sx0 + 7.f) && (a.y + d.y >= sy0) && (a.y - d.y <= sy0 + (float)H)))
        return false;
    const float ddx = fmaxf(fmaxf(sx0 - a.x, a.x - (sx0 + 7.f)) - 1e-3f, 0.f);
    const float ddy = fmaxf(fmaxf(sy0 - a.y, a.y - (sy0 + (float)H)) - 1e-3f, 0.f);
    return lmax * fmaf(ddx, ddx, ddy * ddy) >= b.z - b.y - 1e-3f;
}
template <int H = 3>
__device__ __forceinline__ bool overlaps_radial(const StagedSplat& s, float lmax, float sx0, float sy0) {
    return overlaps_v<H>(s.a, s.b, s.d, lmax, sx0, sy0);
}

enum { kSkip = 0, kAccept = 1, kAmbiguous = 2 };

// Gate values shared by K5 and K6: explicit-rounding intrinsics, so both kernels compute
// bit-identical p2 / M and take identical decisions.
__device__ __forceinline__ void gate_values(const float4& a, const float4& b, float fpx, float fpy, float& p, float& M,
                                            float& dx, float& dy) {
    dx = __fsub_rn(fpx, a.x);
    dy = __fsub_rn(fpy, a.y);
    const float t = __fmul_rn(a.z, dx), u = __fmul_rn(b.x, dy), v = __fmul_rn(a.w, dx);
    const float q = __fmaf_rn(t, dx, __fmul_rn(u, dy));  // ca2 dx^2 + cc2 dy^2  (<= 0)
    p = __fmaf_rn(v, dy, q);                             // log2(e) * power
    M = __fmaf_rn(b.w, q, b.y);                          // error bound of p
}
// alpha < 1/255 for certain, or power > 0 for certain
__device__ __forceinline__ bool gate_skip(float p, float M, float pa2) { return (__fadd_rn(p, M) < pa2) | (p > M); }
// (not skipped and) power > 0 or alpha < 1/255 within the bound
__device__ __forceinline__ bool gate_ambiguous(float p, float M, float pa2) {
    return (p > -M) | (__fsub_rn(p, M) <= pa2);
}

// gate_values with paired FP32 instructions (FADD2 / FMUL2, sm_100): the same IEEE operations
// on the same operands, so p2 and M are bit-identical to gate_values (K6 replays K5's decisions).
__device__ __forceinline__ void gate_values_x2(const float4& a, const float4& b, float2 fp, float& p, float& M) {
    const float2 dxy = __fadd2_rn(fp, make_float2(-a.x, -a.y));           // (dx, dy)
    const float2 tv = __fmul2_rn(make_float2(a.z, a.w), make_float2(dxy.x, dxy.x));  // (ca2 dx, cb2 dx)
    const float u = __fmul_rn(b.x, dxy.y);
    const float q = __fmaf_rn(tv.x, dxy.x, __fmul_rn(u, dxy.y));
    p = __fmaf_rn(tv.y, dxy.y, q);
    M = __fmaf_rn(b.w, q, b.y);
}

__device__ __forceinline__ int classify(const float4& a, const float4& b, float fpx, float fpy, float& p, float& M,
                                        float& dx, float& dy) {
    gate_values(a, b, fpx, fpy, p, M, dx, dy);
    if (gate_skip(p, M, b.z)) return kSkip;
    return gate_ambiguous(p, M, b.z) ? kAmbiguous : kAccept;
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// alpha = min(0.99, ab 2^p2), identical in K5 and K6.
__device__ __forceinline__ float blend_alpha(float ab, float p) { return fminf(0.99f, __fmul_rn(ab, ex2_approx(p))); }

constexpr unsigned kFull = 0xffffffffu;

// Shared-memory loads from a 32-bit shared-window address.  The "memory" clobber keeps them
// ordered with the stores and __syncwarp() that publish the survivor list (without it the
// compiler may hoist a load above the barrier).
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
    float4 v;
    asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ float2 lds_f2(uint32_t a) {
    float2 v;
    asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a) : "memory");
    return v;
}

// Transmittance-gate thresholds of K5's common-case test (rasterizer.cpp:111): with a relative
// error bound errN on the FP32 test_T, test_T (1 - errN) > kStopHi certainly continues and
// test_T (1 + errN) < kStopLo certainly stops; the 2e-7 margins cover the rounding of the
// fused products and of the float constant 1e-4f against the double 1e-4.
constexpr float kStopHi = 1.0000002e-4f, kStopLo = 0.9999998e-4f;

// K5: forward blend.  CTA per 16x16 tile, warp per 8x4 sub-tile, one pixel per lane.
// Per batch of 256 splats the CTA stages the blend records in shared memory as structure of
// arrays; per window of 32 staged splats each warp culls them against its sub-tile (a ballot)
// and copies the survivors, in order, into its own compacted list; then every lane walks that
// list with a plain induction pointer.  The gate decisions are the shared gate_values /
// gate_skip / gate_ambiguous of K6; the transmittance gate is one fused test in the common
// case (certainly continue), with stop / ambiguity resolved on the rare path.  A lane that
// stops or turns slow leaves the walk (no per-visit done test).
template <bool FLOW, bool COUNT>
__global__ void __launch_bounds__(256, 5) k_blend_fp32(SplatArrays sp, const uint32_t* __restrict__ vals,
                                                    const uint2* __restrict__ ranges, DevCamera cam, float3 bg,
                                                    float* __restrict__ image, double* __restrict__ final_T,
                                                    uint32_t* __restrict__ n_contrib, uint32_t* slow_list,
                                                    int* slow_count, unsigned long long* counters) {
    constexpr int kWarps = kTilePixels / 32;
    __shared__ float4 s_a[kTilePixels], s_b[kTilePixels], s_c[kTilePixels], s_d[kTilePixels];
    __shared__ float s_l[kTilePixels];
    __shared__ StagedSplat w_list[kWarps][32];  // (a, b, c, (pc2, R, -, -)) of the window's survivors
    __shared__ uint8_t w_k[kWarps][32];
    const int tile = blockIdx.x;
    const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sx0 = (warp & 1) * 8, sy0 = (warp >> 1) * 4;
    const int lx = sx0 + (lane & 7), ly = sy0 + (lane >> 3);
    const int px = tx * kTile + lx, py = ty * kTile + ly;
    const bool inside = px < cam.width && py < cam.height;
    const uint2 rg = ranges[tile];
    const double px0 = tx * kTile, py0 = ty * kTile;
    const float fpx = (float)lx, fpy = (float)ly, fsx0 = (float)sx0, fsy0 = (float)sy0;
    const unsigned lt_mask = (1u << lane) - 1u;

    const float2 fp2 = make_float2(fpx, fpy);
    float T = 1.f, errT3 = 3e-7f, acc2 = 0.f;  // errT3 = errT + 3e-7
    float2 acc01 = make_float2(0.f, 0.f);
    int contrib = 0;
    bool done = !inside, slow = false, stopped = false;
    uint32_t n_eval = 0, n_blend = 0, n_ref = 0;  // COUNT only
    bool warp_done = __all_sync(kFull, done);

    // (loading the next batch's splat ids one batch ahead, with or without an L1 prefetch of
    // their records once the warp has walked its windows: equal time, 0.329-0.332 ms)
    for (uint32_t start = rg.x; start < rg.y; start += kTilePixels) {
        if (__syncthreads_count(done) == kTilePixels) break;
        const uint32_t j = start + threadIdx.x;
        if (j < rg.y) {
            float4 A, Bv, C, Dv;
            float l;
            stage_values<FLOW>(sp, vals[j], px0, py0, A, Bv, C, Dv, l);
            // K5's merged ambiguity test (below) takes the clamp gate as p + M >= pcq with
            // pcq = pc2 for pc2 <= 0 and the smallest positive float otherwise
            Dv.z = Dv.z > 0.f ? __int_as_float(1) : Dv.z;
            s_a[threadIdx.x] = A;
            s_b[threadIdx.x] = Bv;
            s_c[threadIdx.x] = C;
            s_d[threadIdx.x] = Dv;
            s_l[threadIdx.x] = l;
        }
        __syncthreads();
        const int n = (int)min((uint32_t)kTilePixels, rg.y - start);
        if (warp_done) continue;
        for (int c = 0; c < n; c += 32) {
            const int k0 = c + lane;
            bool surv = false;
            float4 a, b, d;
            if (k0 < n) {
                a = s_a[k0];
                b = s_b[k0];
                d = s_d[k0];
                surv = overlaps_v(a, b, d, s_l[k0], fsx0, fsy0);
            }
            const unsigned m = __ballot_sync(kFull, surv);
            if (surv) {
                const int q = __popc(m & lt_mask);
                StagedSplat* e = &w_list[warp][q];
                e->a = a;
                e->b = b;
                e->c = s_c[k0];
                e->d = d;
                w_k[warp][q] = (uint8_t)lane;
            }
            __syncwarp();
            unsigned bmask = 0;  // COUNT only: the window entries this lane blended
            if (!done) {
                // the survivor list walked on one 32-bit shared-memory address (a single
                // induction variable: it is also the `last` record)
                const uint32_t first = (uint32_t)__cvta_generic_to_shared(w_list[warp]);
                const uint32_t end = first + (uint32_t)__popc(m) * (uint32_t)sizeof(StagedSplat);
                // the last blended entry's address (0: none in this window)
                uint32_t last = 0;
                for (uint32_t e = first; e != end; e += (uint32_t)sizeof(StagedSplat)) {
                    // (loading the colour / guard entries before the skip branch as well, with
                    // volatile loads so ptxas keeps them there, measured 0.353 vs 0.328 ms)
                    const float4 a2 = lds_f4(e), b2 = lds_f4(e + 16);
                    float p, M;
                    gate_values_x2(a2, b2, fp2, p, M);
                    if (COUNT) ++n_eval;
                    if (gate_skip(p, M, b2.z)) continue;
                    const float4 cc = lds_f4(e + 32);
                    const float2 pr = lds_f2(e + 56);  // (pcq, R)
                    const float al = blend_alpha(cc.w, p);
                    const float test_T = __fmul_rn(T, __fsub_rn(1.f, al));
                    const float errN = fmaf(al * M, pr.y, errT3);
                    // ambiguous alpha / power gate, or the backward's clamp gate (unclamped
                    // alpha <= 0.99, rasterizer.cpp:356), within their error bounds, as one
                    // superset test: p > -M (exactly: RN(p + M) > 0, i.e. >= the smallest
                    // positive float) or RN(p - M) <= pa2 or [RN(p + M) >= pc2 and
                    // RN(p - M) <= pc2] all imply RN(p + M) >= pcq or RN(p - M) <= pa2 (pcq:
                    // staging).  The extra pixels it sends to the FP64 fix-up are those within
                    // |p| < 0.0145 of the centre of a splat with alpha_base > 0.99.
                    const bool amb_gc = (__fadd_rn(p, M) >= pr.x) | (__fsub_rn(p, M) <= b2.z);
                    if (!amb_gc & (fmaf(-test_T, errN, test_T) > kStopHi)) {  // one branch: both tests evaluated
                        const float w = al * T;
                        acc01 = __ffma2_rn(make_float2(cc.x, cc.y), make_float2(w, w), acc01);
                        acc2 = fmaf(cc.z, w, acc2);
                        T = test_T;
                        errT3 = errN + 3e-7f;
                        last = e;
                        if (COUNT) {
                            ++n_blend;
                            bmask |= 1u << (int)((e - first) / sizeof(StagedSplat));
                        }
                        continue;
                    }
                    // rare: certainly stop (rasterizer.cpp:111, the splat is not blended), or a
                    // decision inside its error bound -> the pixel goes to the FP64 fix-up
                    if (!amb_gc && fmaf(test_T, errN, test_T) < kStopLo) {
                        done = stopped = true;
                        if (COUNT) n_ref = start - rg.x + c + w_k[warp][(e - first) / sizeof(StagedSplat)] + 1;
                        break;
                    }
                    if (COUNT) {
                        // slow-pixel reasons: power > 0 / alpha gate, clamp gate, transmittance gate
                        const bool amb_g = gate_ambiguous(p, M, b2.z);
                        const int r = amb_g ? ((p > -M) ? 3 : 4) : (amb_gc ? 5 : 6);
                        atomicAdd(counters + r, 1ull);
                    }
                    slow = done = true;
                    break;
                }
                if (last) {
                    const int lastq = (int)((last - first) / sizeof(StagedSplat));
                    contrib = (int)(start - rg.x) + c + w_k[warp][lastq] + 1;
                }
            }
            __syncwarp();  // the list is rewritten by the next window
            if (COUNT) {
                // warp visits of the window (entries walked) and those where some lane blended
                const unsigned anyb = __reduce_or_sync(kFull, bmask);
                if (lane == 0 && __popc(m)) {
                    atomicAdd(counters + 7, (unsigned long long)__popc(m));
                    atomicAdd(counters + 8, (unsigned long long)__popc(anyb));
                }
            }
            if (__all_sync(kFull, done)) {
                warp_done = true;
                break;
            }
        }
    }
    if (COUNT) {
        // E of the roofline = evaluations of the reference algorithm (every list entry up
        // to the termination point); n_eval = the ones this kernel actually evaluated.
        unsigned long long e = inside ? (stopped ? n_ref : rg.y - rg.x) : 0, b = n_blend, ke = n_eval;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            e += __shfl_xor_sync(kFull, e, o);
            b += __shfl_xor_sync(kFull, b, o);
            ke += __shfl_xor_sync(kFull, ke, o);
        }
        if (lane == 0) {
            atomicAdd(counters + 0, e);
            atomicAdd(counters + 1, b);
            atomicAdd(counters + 2, ke);
        }
    }
    if (!inside) return;
    const uint32_t pix = (uint32_t)py * cam.width + px;
    if (slow) {
        slow_list[atomicAdd(slow_count, 1)] = pix;
        return;
    }
    if (FLOW) {
        image[(size_t)pix * 2 + 0] = acc01.x;
        image[(size_t)pix * 2 + 1] = acc01.y;
    } else {
        image[(size_t)pix * 3 + 0] = fmaf(T, bg.x, acc01.x);
        image[(size_t)pix * 3 + 1] = fmaf(T, bg.y, acc01.y);
        image[(size_t)pix * 3 + 2] = fmaf(T, bg.z, acc2);
        final_T[pix] = (double)T;
        n_contrib[pix] = (uint32_t)contrib;
    }
}

// K5 (two pixels per lane; the default -- RGS_K5=2 selects one pixel per lane): CTA of 128 threads per 16x16 tile, warp per 8x8 sub-tile,
// lane pixels (x, y) and (x, y + 4) -- the sub-tiles and pixel pairs of K6.  The two pixels share
// dx and every per-splat operand, so the gate, alpha, transmittance and colour arithmetic are
// paired FP32 instructions (bit-identical to the scalar forms); predicated selects keep a pixel
// that skipped unchanged.  A finished pixel (stopped, slow or outside the image) gets the y
// coordinate kGone, so every later splat certainly skips it without a per-visit flag test.
// Decisions per (pixel, splat) are those of k_blend_fp32, including its merged ambiguity test.
constexpr int kX2Threads = 128;
constexpr int kX2Warps = kX2Threads / 32;
// staged splats per batch, one per thread: 0.261 ms per C2 frame vs 0.265 at 256 (two per thread;
// the warps of a block wait less for each other at the batch barrier) and 0.320 at 512 (5 CTAs/SM)
constexpr int kX2Stage = 128;
// CTAs per SM: 7 (71 registers, no spills) -- C2 frame 0.283 ms, 2490 FPS in the pipelined sweep;
// 8 (64 registers, spills in the staging): 0.310 ms, 2213 FPS; 6: 0.287 ms, 2453 FPS.  Loading the
// next entry's gate operands one visit ahead (a rotating register pair) measured 0.322 ms at 6-8.
constexpr int kX2Blocks = 7;
// |dy| = 1e12: q <= cc2 dy^2 is below any alpha threshold for every conic the projection makes,
// the error bound M = cs2n q + D stays far below |q| (|cs2n| << 1), and nothing overflows.
constexpr float kGone = 1e12f;

// Tile order for K5: longest list first (a counting sort on 255 - min(255, length / 4)), so the
// blocks of the last wave are short ones.  One block.
__global__ void __launch_bounds__(1024) k_tile_order(const uint2* __restrict__ ranges, int nt, uint32_t* order) {
    __shared__ uint32_t cnt[256];
    if (threadIdx.x < 256) cnt[threadIdx.x] = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < nt; t += blockDim.x) {
        const uint2 r = ranges[t];
        atomicAdd(&cnt[255 - min(255u, (r.y - r.x) >> 2)], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // exclusive scan of the 256 counts by one warp, 8 per lane
        uint32_t v[8], s = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            v[j] = cnt[threadIdx.x * 8 + j];
            s += v[j];
        }
        uint32_t incl = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, incl, o);
            if ((int)threadIdx.x >= o) incl += y;
        }
        uint32_t run = incl - s;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            cnt[threadIdx.x * 8 + j] = run;
            run += v[j];
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < nt; t += blockDim.x) {
        const uint2 r = ranges[t];
        order[atomicAdd(&cnt[255 - min(255u, (r.y - r.x) >> 2)], 1u)] = (uint32_t)t;
    }
}

template <bool FLOW, bool COUNT, int NB = kX2Blocks, int STAGE = kX2Stage>
__global__ void __launch_bounds__(kX2Threads, NB) k_blend_fp32_x2(SplatArrays sp, const uint32_t* __restrict__ vals,
                                                              const uint2* __restrict__ ranges, DevCamera cam,
                                                              float3 bg, float* __restrict__ image,
                                                              double* __restrict__ final_T,
                                                              uint32_t* __restrict__ n_contrib, uint32_t* slow_list,
                                                              int* slow_count, unsigned long long* counters,
                                                              const uint32_t* __restrict__ tile_order) {
    __shared__ float4 s_a[STAGE], s_b[STAGE], s_c[STAGE], s_d[STAGE];
    __shared__ float s_l[STAGE];
    __shared__ StagedSplat w_list[kX2Warps][32];
    __shared__ uint8_t w_k[kX2Warps][32];
    const int tile = tile_order ? (int)tile_order[blockIdx.x] : (int)blockIdx.x;
    const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sx0 = (warp & 1) * 8, sy0 = (warp >> 1) * 8;
    const int lx = sx0 + (lane & 7), ly = sy0 + (lane >> 3);
    const int px = tx * kTile + lx, py0 = ty * kTile + ly, py1 = py0 + 4;
    const bool in0 = px < cam.width && py0 < cam.height, in1 = px < cam.width && py1 < cam.height;
    const uint2 rg = ranges[tile];
    const double px0 = tx * kTile, py0t = ty * kTile;
    const float fpx = (float)lx, fsx0 = (float)sx0, fsy0 = (float)sy0;
    float2 fpy = make_float2(in0 ? (float)ly : kGone, in1 ? (float)(ly + 4) : kGone);
    const unsigned lt_mask = (1u << lane) - 1u;

    float2 T = make_float2(1.f, 1.f), errT3 = make_float2(3e-7f, 3e-7f);  // errT3 = errT + 3e-7
    float2 acc0 = make_float2(0.f, 0.f), acc1 = acc0, acc2 = acc0;        // channel c of pixels (0, 1)
    int contrib0 = 0, contrib1 = 0;
    bool slow0 = false, slow1 = false, stopped0 = false, stopped1 = false;
    uint32_t n_eval = 0, n_blend = 0, n_ref0 = 0, n_ref1 = 0;  // COUNT only
    bool gone = (fpy.x == kGone) & (fpy.y == kGone);
    bool warp_done = __all_sync(kFull, gone);

    for (uint32_t start = rg.x; start < rg.y; start += STAGE) {
        if (__syncthreads_count(gone) == kX2Threads) break;
#pragma unroll
        for (int h = 0; h < STAGE / kX2Threads; ++h) {
            const int t = threadIdx.x + h * kX2Threads;
            const uint32_t j = start + t;
            if (j < rg.y) {
                float4 A, Bv, C, Dv;
                float l;
                stage_values<FLOW>(sp, vals[j], px0, py0t, A, Bv, C, Dv, l);
                Dv.z = Dv.z > 0.f ? __int_as_float(1) : Dv.z;  // pcq, as in k_blend_fp32
                s_a[t] = A;
                s_b[t] = Bv;
                s_c[t] = C;
                s_d[t] = Dv;
                s_l[t] = l;
            }
        }
        __syncthreads();
        const int n = (int)min((uint32_t)STAGE, rg.y - start);
        if (warp_done) continue;
        for (int c = 0; c < n; c += 32) {
            const int k0 = c + lane;
            bool surv = false;
            float4 a, b, d;
            if (k0 < n) {
                a = s_a[k0];
                b = s_b[k0];
                d = s_d[k0];
                surv = overlaps_v<7>(a, b, d, s_l[k0], fsx0, fsy0);
            }
            const unsigned m = __ballot_sync(kFull, surv);
            if (surv) {
                const int q = __popc(m & lt_mask);
                StagedSplat* e = &w_list[warp][q];
                e->a = a;
                e->b = b;
                e->c = s_c[k0];
                e->d = d;
                w_k[warp][q] = (uint8_t)lane;
            }
            __syncwarp();
            unsigned bmask = 0;  // COUNT only: the window entries this lane blended
            if (!gone) {
                const uint32_t first = (uint32_t)__cvta_generic_to_shared(w_list[warp]);
                const uint32_t end = first + (uint32_t)__popc(m) * (uint32_t)sizeof(StagedSplat);
                uint32_t last0 = 0, last1 = 0;  // the last blended entries' addresses (0: none)
                for (uint32_t e = first; e != end; e += (uint32_t)sizeof(StagedSplat)) {
                    const float4 a2 = lds_f4(e), b2 = lds_f4(e + 16);
                    // gate_values for both pixels (shared dx, paired dy)
                    const float dx = __fsub_rn(fpx, a2.x);
                    const float2 dy = __fadd2_rn(fpy, make_float2(-a2.y, -a2.y));
                    const float2 tv = __fmul2_rn(make_float2(a2.z, a2.w), make_float2(dx, dx));
                    const float2 u = __fmul2_rn(make_float2(b2.x, b2.x), dy);
                    const float2 q2 = __ffma2_rn(make_float2(tv.x, tv.x), make_float2(dx, dx), __fmul2_rn(u, dy));
                    const float2 p = __ffma2_rn(make_float2(tv.y, tv.y), dy, q2);
                    const float2 M = __ffma2_rn(make_float2(b2.w, b2.w), q2, make_float2(b2.y, b2.y));
                    const float2 pM = __fadd2_rn(p, M);
                    if (COUNT) n_eval += (fpy.x != kGone ? 1u : 0u) + (fpy.y != kGone ? 1u : 0u);
                    // act: not certainly below the alpha threshold.  gate_skip's other half, power
                    // > 0 for certain (p > M), is left to the rare path below: such a pixel fails
                    // the merged test (p + M < pcq <= the smallest positive float), so it never
                    // blends, and the rare path skips it without a state change.
                    const bool act0 = !(pM.x < b2.z), act1 = !(pM.y < b2.z);
                    if (!(act0 | act1)) continue;
                    const float4 cc = lds_f4(e + 32);
                    const float2 pr = lds_f2(e + 56);  // (pcq, R)
                    // alpha without blend_alpha's clamp at 0.99: wherever it is used -- a pixel that
                    // blends, or stops, passed the merged test p + M < pcq -- it is already below
                    // 0.99: for ab < 0.99, p < 0 gives ab 2^p < ab; for ab >= 0.99, p < pc2 - M with
                    // M >= 1.5e-6 keeps ab 2^p below 0.99 (1 - 1e-6), far outside the EX2 / rounding
                    // error.  So it equals K6's clamped alpha for every pixel K6 replays.
                    const float2 al = __fmul2_rn(make_float2(cc.w, cc.w), make_float2(ex2_approx(p.x), ex2_approx(p.y)));
                    const float2 test_T = __fmul2_rn(T, __fadd2_rn(make_float2(1.f, 1.f), make_float2(-al.x, -al.y)));
                    const float2 errN = __ffma2_rn(__fmul2_rn(al, M), make_float2(pr.y, pr.y), errT3);
                    const float2 lo = __ffma2_rn(make_float2(-test_T.x, -test_T.y), errN, test_T);
                    const float2 pm = __fadd2_rn(p, make_float2(-M.x, -M.y));
                    // certain decisions (the merged ambiguity test of k_blend_fp32) and certainly
                    // continuing transmittance
                    // (cl implies act: p - M > pa2 gives p + M > pa2)
                    const bool cl0 = (pM.x < pr.x) & (pm.x > b2.z), cl1 = (pM.y < pr.x) & (pm.y > b2.z);
                    const bool ok0 = cl0 & (lo.x > kStopHi), ok1 = cl1 & (lo.y > kStopHi);
                    const float2 w = __fmul2_rn(al, T);
                    const float2 wm = make_float2(ok0 ? w.x : 0.f, ok1 ? w.y : 0.f);
                    acc0 = __ffma2_rn(make_float2(cc.x, cc.x), wm, acc0);
                    acc1 = __ffma2_rn(make_float2(cc.y, cc.y), wm, acc1);
                    if (!FLOW) acc2 = __ffma2_rn(make_float2(cc.z, cc.z), wm, acc2);
                    const float2 eT3 = __fadd2_rn(errN, make_float2(3e-7f, 3e-7f));
                    T = make_float2(ok0 ? test_T.x : T.x, ok1 ? test_T.y : T.y);
                    errT3 = make_float2(ok0 ? eT3.x : errT3.x, ok1 ? eT3.y : errT3.y);
                    last0 = ok0 ? e : last0;
                    last1 = ok1 ? e : last1;
                    if (COUNT) {
                        n_blend += (ok0 ? 1u : 0u) + (ok1 ? 1u : 0u);
                        if (ok0 | ok1) bmask |= 1u << (int)((e - first) / sizeof(StagedSplat));
                    }
                    if ((act0 & !ok0) | (act1 & !ok1)) {
                        // rare: certainly stop (rasterizer.cpp:111, the splat is not blended), or
                        // a decision inside its error bound -> the pixel goes to the FP64 fix-up
                        const float2 hi = __ffma2_rn(test_T, errN, test_T);
                        const int qi = (int)((e - first) / sizeof(StagedSplat));
                        // (a finished pixel only gets here through an overflowing bound -- a
                        // degenerate conic's M at y = kGone -- and stays as it is)
                        if (act0 & !ok0 & !(p.x > M.x) & (fpy.x != kGone)) {
                            if (cl0 && hi.x < kStopLo) {
                                stopped0 = true;
                                if (COUNT) n_ref0 = start - rg.x + c + w_k[warp][qi] + 1;
                            } else {
                                slow0 = true;
                                if (COUNT) {
                                    const bool g = gate_ambiguous(p.x, M.x, b2.z);
                                    atomicAdd(counters + (g ? ((p.x > -M.x) ? 3 : 4) : (!cl0 ? 5 : 6)), 1ull);
                                }
                            }
                            fpy.x = kGone;
                        }
                        if (act1 & !ok1 & !(p.y > M.y) & (fpy.y != kGone)) {
                            if (cl1 && hi.y < kStopLo) {
                                stopped1 = true;
                                if (COUNT) n_ref1 = start - rg.x + c + w_k[warp][qi] + 1;
                            } else {
                                slow1 = true;
                                if (COUNT) {
                                    const bool g = gate_ambiguous(p.y, M.y, b2.z);
                                    atomicAdd(counters + (g ? ((p.y > -M.y) ? 3 : 4) : (!cl1 ? 5 : 6)), 1ull);
                                }
                            }
                            fpy.y = kGone;
                        }
                        gone = (fpy.x == kGone) & (fpy.y == kGone);
                        if (gone) break;
                    }
                }
                if (last0) contrib0 = (int)(start - rg.x) + c + w_k[warp][(last0 - first) / sizeof(StagedSplat)] + 1;
                if (last1) contrib1 = (int)(start - rg.x) + c + w_k[warp][(last1 - first) / sizeof(StagedSplat)] + 1;
            }
            __syncwarp();  // the list is rewritten by the next window
            if (COUNT) {
                // warp visits of the window and those where some lane blended
                const unsigned anyb = __reduce_or_sync(kFull, bmask);
                if (lane == 0 && __popc(m)) {
                    atomicAdd(counters + 7, (unsigned long long)__popc(m));
                    atomicAdd(counters + 8, (unsigned long long)__popc(anyb));
                }
            }
            if (__all_sync(kFull, gone)) {
                warp_done = true;
                break;
            }
        }
    }
    if (COUNT) {
        unsigned long long e = (in0 ? (stopped0 ? n_ref0 : rg.y - rg.x) : 0) +
                               (in1 ? (stopped1 ? n_ref1 : rg.y - rg.x) : 0),
                           b = n_blend, ke = n_eval;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            e += __shfl_xor_sync(kFull, e, o);
            b += __shfl_xor_sync(kFull, b, o);
            ke += __shfl_xor_sync(kFull, ke, o);
        }
        if (lane == 0) {
            atomicAdd(counters + 0, e);
            atomicAdd(counters + 1, b);
            atomicAdd(counters + 2, ke);
        }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        if (!(h ? in1 : in0)) continue;
        const uint32_t pix = (uint32_t)(h ? py1 : py0) * cam.width + px;
        if (h ? slow1 : slow0) {
            slow_list[atomicAdd(slow_count, 1)] = pix;
            continue;
        }
        const float Th = h ? T.y : T.x;
        const float r = h ? acc0.y : acc0.x, g = h ? acc1.y : acc1.x, bb = h ? acc2.y : acc2.x;
        if (FLOW) {
            image[(size_t)pix * 2 + 0] = r;
            image[(size_t)pix * 2 + 1] = g;
        } else {
            image[(size_t)pix * 3 + 0] = fmaf(Th, bg.x, r);
            image[(size_t)pix * 3 + 1] = fmaf(Th, bg.y, g);
            image[(size_t)pix * 3 + 2] = fmaf(Th, bg.z, bb);
            final_T[pix] = (double)Th;
            n_contrib[pix] = (uint32_t)(h ? contrib1 : contrib0);
        }
    }
}

// Reduce-scatter of 9 per-lane partials across the warp (butterfly, 12 shuffles instead of
// 9 x 5): at each level the lanes split their remaining slots in two halves, keep one half
// and receive the partner's contribution to it.  Afterwards lane pairs (l, l^1) hold the
// warp sum of value `idx` (valid when ok) -- 9 lanes then issue their shared-memory
// atomics in one instruction.
template <int K, int OFF>
__device__ __forceinline__ void rs_level(const float* in, float* out, int lane, int& base, int& end) {
    constexpr int LO = (K + 1) / 2;
    const bool hi = (lane & OFF) != 0;
#pragma unroll
    for (int i = 0; i < LO; ++i) {
        const float mine = hi ? (LO + i < K ? in[LO + i] : 0.f) : in[i];
        const float give = hi ? in[i] : (LO + i < K ? in[LO + i] : 0.f);
        out[i] = mine + __shfl_xor_sync(kFull, give, OFF);
    }
    // the lane's slots cover value indices [base, end); keep the low or the high half
    if (hi) base += LO;
    else end = min(end, base + LO);
}

__device__ __forceinline__ float reduce_scatter9(const float* v, int lane, int& idx, bool& ok) {
    float a[5], b[3], c[2], d[1];
    int base = 0, end = 9;
    rs_level<9, 16>(v, a, lane, base, end);  // 9 -> 5 slots
    rs_level<5, 8>(a, b, lane, base, end);   // 5 -> 3
    rs_level<3, 4>(b, c, lane, base, end);   // 3 -> 2
    rs_level<2, 2>(c, d, lane, base, end);   // 2 -> 1
    const float r = d[0] + __shfl_xor_sync(kFull, d[0], 1);
    idx = base;
    ok = base < end;  // padding slots hold zeros and own no value
    return r;
}

// K6: back-to-front replay of the FP32 pixels (rasterizer.cpp:320-397).  128 threads per tile,
// each lane replays kBwdPx = 2 pixels (rows y and y + 4 of its warp's 8x8 sub-tile), so the
// per-splat loop overhead and the warp reduction are shared by 64 pixels (measured: 2 pixels
// 1.10 ms / C3 step, 1 pixel 1.36 ms, 4 pixels 1.28 ms; 48-register cap 1.25 ms).  Warps are
// independent: each stages its own 32-splat windows (no block barriers -- a block-shared
// staging with per-warp shared-memory slots summed per batch measured the same), sums its
// lanes' two partials, reduce-scatters them across the warp and the 9 owner lanes issue one
// FP64 atomic each.  Slow pixels are replayed in FP64 by k_backward_fp64.  The 8x8 cull is
// the union of K5's two 8x4 culls, so every pair K5 evaluated is evaluated here with the same
// FP32 numbers and the same decision.
//
// Per pixel the colour terms fold into scalars: with G = sum_c dL/dc_c * colour_c (per pair)
// and S = sum_c dL/dc_c * s_c (per pixel, s = colour accumulated behind the splat),
// dL/dalpha = T_before G - S / (1 - alpha) and S += w G.
constexpr int kBwdPx = 2;  // pixels per lane, rows y + 4 i
constexpr int kBwdThreads = kTilePixels / kBwdPx;
constexpr int kBwdWarps = kBwdThreads / 32;

template <bool FIXED>
__global__ void __launch_bounds__(kBwdThreads) k_backward_fp32(SplatArrays sp, const uint32_t* __restrict__ vals,
                                                                const uint2* __restrict__ ranges, DevCamera cam,
                                                                float3 bg, const double* __restrict__ final_T,
                                                                const uint32_t* __restrict__ n_contrib,
                                                                const float* __restrict__ dL, double* sg,
                                                                unsigned long long* sgx,
                                                                const uint32_t* __restrict__ tile_order) {
    __shared__ StagedSplat smw[kBwdWarps][32];
    __shared__ float slmw[kBwdWarps][32];
    const int tile = tile_order ? (int)tile_order[blockIdx.x] : (int)blockIdx.x;
    const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sx0 = (warp & 1) * 8, sy0 = (warp >> 1) * 4 * kBwdPx;
    const int lx = sx0 + (lane & 7), ly = sy0 + (lane >> 3);
    const double px0 = tx * kTile, py0 = ty * kTile;
    const uint2 rg = ranges[tile];
    const float fpx = (float)lx, fsx0 = (float)sx0, fsy0 = (float)sy0;
    constexpr float kLn2 = 0.69314718055994531f;
    StagedSplat* sm = smw[warp];
    float* slm = slmw[warp];

    static_assert(kBwdPx == 2, "the replay pairs the lane's two pixels");
    int contrib[kBwdPx];
    float T_run[kBwdPx], g0[kBwdPx], g1[kBwdPx], g2[kBwdPx], S[kBwdPx];
    int cmax = 0;
#pragma unroll
    for (int h = 0; h < kBwdPx; ++h) {
        const int px = tx * kTile + lx, py = ty * kTile + ly + 4 * h;
        contrib[h] = 0;
        T_run[h] = 1.f;
        g0[h] = g1[h] = g2[h] = S[h] = 0.f;
        if (px < cam.width && py < cam.height) {
            const uint32_t pix = (uint32_t)py * cam.width + px;
            const uint32_t c = n_contrib[pix];
            if (!(c & kSlowBit)) {
                contrib[h] = (int)c;
                const float fT = (float)final_T[pix];
                T_run[h] = fT;
                g0[h] = dL[(size_t)pix * 3 + 0];
                g1[h] = dL[(size_t)pix * 3 + 1];
                g2[h] = dL[(size_t)pix * 3 + 2];
                S[h] = fmaf(g0[h], bg.x * fT, fmaf(g1[h], bg.y * fT, g2[h] * (bg.z * fT)));
            }
        }
        cmax = max(cmax, contrib[h]);
    }
    const float2 fpy2 = make_float2((float)ly, (float)(ly + 4));
    float2 T_run2 = make_float2(T_run[0], T_run[1]), S2 = make_float2(S[0], S[1]);
    const float2 g0_2 = make_float2(g0[0], g0[1]), g1_2 = make_float2(g1[0], g1[1]), g2_2 = make_float2(g2[0], g2[1]);
    const int wmax = __reduce_max_sync(kFull, cmax);

    for (int end = wmax; end > 0; end -= 32) {
        const int beg = end > 32 ? end - 32 : 0;
        const int cnt = end - beg;
        uint32_t myid = 0;
        __syncwarp();
        if (lane < cnt) {
            myid = vals[rg.x + beg + lane];
            stage<false>(sp, myid, px0, py0, &sm[lane], &slm[lane]);
            const float pc2 = sm[lane].d.z;
            sm[lane].d.z = pc2 > 0.f ? __int_as_float(1) : pc2;  // pcq, as K5
        }
        __syncwarp();
        unsigned mask = __ballot_sync(kFull, lane < cnt && overlaps_radial<4 * kBwdPx - 1>(sm[lane], slm[lane], fsx0, fsy0));
        while (mask) {
            const int k = 31 - __clz(mask);
            mask &= ~(1u << k);
            // The lane's two pixels (rows y and y + 4) share dx and every per-splat operand: their
            // gate values and replay arithmetic are paired FP32 instructions (FADD2 / FMUL2 /
            // FFMA2); gate_values' operations, so K5's decisions are replayed exactly.  A pixel that
            // does not accept this splat contributes zero through masked weights.
            const float4 a = sm[k].a, b = sm[k].b;
            const float dx = __fsub_rn(fpx, a.x);
            const float2 dy = __fadd2_rn(fpy2, make_float2(-a.y, -a.y));
            const float2 tv = __fmul2_rn(make_float2(a.z, a.w), make_float2(dx, dx));
            const float2 u = __fmul2_rn(make_float2(b.x, b.x), dy);
            const float2 q2 = __ffma2_rn(make_float2(tv.x, tv.x), make_float2(dx, dx), __fmul2_rn(u, dy));
            const float2 p = __ffma2_rn(make_float2(tv.y, tv.y), dy, q2);
            const float2 M = __ffma2_rn(make_float2(b.w, b.w), q2, make_float2(b.y, b.y));
            // K5's blend decision.  A pixel K6 replays is not slow, so every splat before its
            // n_contrib was either blended -- K5's merged test held: p - M > pa2 and p + M < pcq --
            // or certainly skipped (p + M < pa2, or p > M): the merged test alone tells them apart.
            // It also puts every blended splat certainly below the clamp (p < pc2), so the unclamped
            // alpha is the clamped one and the clamp gate's gradient mask is all ones
            // (rasterizer.cpp:356).
            const float2 pM = __fadd2_rn(p, M), pm = __fadd2_rn(p, make_float2(-M.x, -M.y));
            const float pcq = sm[k].d.z;
            const bool acc0 = (beg + k < contrib[0]) & (pm.x > b.z) & (pM.x < pcq);
            const bool acc1 = (beg + k < contrib[1]) & (pm.y > b.z) & (pM.y < pcq);
            const bool act = acc0 | acc1;
            float v[9];
            if (act) {
                const float4 cc = sm[k].c;
                const float2 e = make_float2(ex2_approx(p.x), ex2_approx(p.y));
                const float2 al = __fmul2_rn(make_float2(cc.w, cc.w), e);  // below 0.99 (above)
                const float2 om = __fadd2_rn(make_float2(1.f, 1.f), make_float2(-al.x, -al.y));
                const float2 inv_om = make_float2(rcp_approx(om.x), rcp_approx(om.y));
                const float2 Tb = __fmul2_rn(T_run2, inv_om);
                const float2 w = __fmul2_rn(al, Tb);
                const float2 wm = make_float2(acc0 ? w.x : 0.f, acc1 ? w.y : 0.f);
                const float2 V0 = __fmul2_rn(wm, g0_2), V1 = __fmul2_rn(wm, g1_2), V2 = __fmul2_rn(wm, g2_2);
                const float2 G = __ffma2_rn(g0_2, make_float2(cc.x, cc.x),
                                            __ffma2_rn(g1_2, make_float2(cc.y, cc.y),
                                                       __fmul2_rn(g2_2, make_float2(cc.z, cc.z))));
                const float2 dL_da = __ffma2_rn(Tb, G, __fmul2_rn(make_float2(-S2.x, -S2.y), inv_om));
                // the conic / mean / alpha_base terms (unclamped alpha, al = ab * e)
                const float2 dam = make_float2(acc0 ? dL_da.x : 0.f, acc1 ? dL_da.y : 0.f);
                const float A = -2.f * kLn2 * a.z, B = -kLn2 * a.w, C = -2.f * kLn2 * b.x;
                const float2 dp = __fmul2_rn(dam, al);
                const float2 V8 = __fmul2_rn(dam, e);
                const float2 V3 = __fmul2_rn(dp, make_float2(-0.5f * dx * dx, -0.5f * dx * dx));
                const float2 V4 = __fmul2_rn(dp, __fmul2_rn(make_float2(-dx, -dx), dy));
                const float2 V5 = __fmul2_rn(dp, __fmul2_rn(__fmul2_rn(make_float2(-0.5f, -0.5f), dy), dy));
                const float2 V6 = __fmul2_rn(dp, __ffma2_rn(make_float2(A, A), make_float2(dx, dx),
                                                             __fmul2_rn(make_float2(B, B), dy)));
                const float2 V7 = __fmul2_rn(dp, __ffma2_rn(make_float2(B, B), make_float2(dx, dx),
                                                             __fmul2_rn(make_float2(C, C), dy)));
                v[0] = V0.x + V0.y;
                v[1] = V1.x + V1.y;
                v[2] = V2.x + V2.y;
                v[3] = V3.x + V3.y;
                v[4] = V4.x + V4.y;
                v[5] = V5.x + V5.y;
                v[6] = V6.x + V6.y;
                v[7] = V7.x + V7.y;
                v[8] = V8.x + V8.y;
                S2 = __ffma2_rn(wm, G, S2);
                if (acc0) T_run2.x = Tb.x;
                if (acc1) T_run2.y = Tb.y;
            } else {
#pragma unroll
                for (int q = 0; q < 9; ++q) v[q] = 0.f;
            }
            const unsigned am = __ballot_sync(kFull, act);
            if (am == 0) continue;
            const size_t sid = (size_t)__shfl_sync(kFull, myid, k);
            double* o = sg + sid * 9;
            if (__popc(am) == 1) {
                if (act) {
#pragma unroll
                    for (int q = 0; q < 9; ++q)
                        if (v[q] != 0.f) {
                            if (FIXED) fixed_add(sgx + 18 * sid + 2 * q, (double)v[q]);
                            else atomicAdd(o + q, (double)v[q]);
                        }
                }
            } else {
                int idx;
                bool ok;
                const float r = reduce_scatter9(v, lane, idx, ok);
                if (ok && !(lane & 1) && r != 0.f) {
                    if (FIXED) fixed_add(sgx + 18 * sid + 2 * idx, (double)r);
                    else atomicAdd(o + idx, (double)r);
                }
            }
        }
    }
}

}  // namespace rgs_dev

namespace rgs_launch {
using namespace rgs_dev;

// RGS_K5 (A/B runs): "2" one pixel per lane, "x<N>" two pixels per lane at N (6-8) CTAs per SM;
// default: two pixels per lane at kX2Blocks.  (The round-1 kernel, with separate ambiguity tests,
// is gone: K6 replays the merged test's decisions.)
static int g_k5_variant = 3;
static int g_x2_nb = kX2Blocks;

static bool g_tile_order = true;

template <int NB, int STAGE = kX2Stage>
static void launch_x2(const SplatArrays& sp, const uint32_t* pair_vals, const uint2* ranges, const DevCamera& cam,
                      float3 bg, int flow_mode, float* image, double* final_T, uint32_t* n_contrib,
                      uint32_t* slow_list, int* slow_count, unsigned long long* counters, cudaStream_t s,
                      uint32_t* order) {
    const int tiles = cam.tiles_x * cam.tiles_y;
    if (!g_tile_order) order = nullptr;
    if (order) k_tile_order<<<1, 1024, 0, s>>>(ranges, tiles, order);
    if (flow_mode)
        k_blend_fp32_x2<true, false, NB><<<tiles, kX2Threads, 0, s>>>(sp, pair_vals, ranges, cam, bg, image, final_T,
                                                                      n_contrib, slow_list, slow_count, counters,
                                                                      order);
    else if (counters)
        k_blend_fp32_x2<false, true, NB><<<tiles, kX2Threads, 0, s>>>(sp, pair_vals, ranges, cam, bg, image, final_T,
                                                                      n_contrib, slow_list, slow_count, counters,
                                                                      order);
    else
        k_blend_fp32_x2<false, false, NB, STAGE><<<tiles, kX2Threads, 0, s>>>(sp, pair_vals, ranges, cam, bg, image,
                                                                       final_T, n_contrib, slow_list, slow_count,
                                                                       counters, order);
}

void blend_fp32(const SplatArrays& sp, const uint32_t* pair_vals, const uint2* ranges, const DevCamera& cam,
                float3 bg, int flow_mode, float* image, double* final_T, uint32_t* n_contrib, uint32_t* slow_list,
                int* slow_count, unsigned long long* counters, cudaStream_t s, uint32_t* tile_order) {
    const int tiles = cam.tiles_x * cam.tiles_y;
#define RGS_K5_LAUNCH(K)                                                                                           \
    if (flow_mode)                                                                                                 \
        K<true, false><<<tiles, kTilePixels, 0, s>>>(sp, pair_vals, ranges, cam, bg, image, final_T, n_contrib,    \
                                                     slow_list, slow_count, counters);                            \
    else if (counters)                                                                                             \
        K<false, true><<<tiles, kTilePixels, 0, s>>>(sp, pair_vals, ranges, cam, bg, image, final_T, n_contrib,    \
                                                     slow_list, slow_count, counters);                            \
    else                                                                                                           \
        K<false, false><<<tiles, kTilePixels, 0, s>>>(sp, pair_vals, ranges, cam, bg, image, final_T, n_contrib,   \
                                                      slow_list, slow_count, counters);
    if (g_k5_variant == 2) {
        RGS_K5_LAUNCH(k_blend_fp32)
    } else if (g_x2_nb == 6) {
        launch_x2<6>(sp, pair_vals, ranges, cam, bg, flow_mode, image, final_T, n_contrib, slow_list, slow_count,
                     counters, s, tile_order);
    } else if (g_x2_nb == 8) {
        launch_x2<8>(sp, pair_vals, ranges, cam, bg, flow_mode, image, final_T, n_contrib, slow_list, slow_count,
                     counters, s, tile_order);
    } else {
        launch_x2<kX2Blocks>(sp, pair_vals, ranges, cam, bg, flow_mode, image, final_T, n_contrib, slow_list,
                             slow_count, counters, s, tile_order);
    }
#undef RGS_K5_LAUNCH
}

// Per-device kernel attributes (called from rgs_ctx_create on the context's device).
bool raster_init() {
    const char* v = std::getenv("RGS_K5");
    g_k5_variant = 3;
    g_x2_nb = kX2Blocks;
    if (v && v[0] == '2') g_k5_variant = 2;
    const char* o = std::getenv("RGS_K5_ORDER");
    g_tile_order = !(o && o[0] == '0');
    if (v && v[0] == 'x' && v[1] >= '6' && v[1] <= '8') g_x2_nb = v[1] - '0';
    return true;
}

void backward_fp32(const SplatArrays& sp, const uint32_t* pair_vals, const uint2* ranges, const DevCamera& cam,
                   float3 bg, const double* final_T, const uint32_t* n_contrib, const float* dL_dimage,
                   double* screen_grads, cudaStream_t s, unsigned long long* screen_grads_fixed,
                   uint32_t* tile_order) {
    const int tiles = cam.tiles_x * cam.tiles_y;
    if (!g_tile_order) tile_order = nullptr;
    if (tile_order) k_tile_order<<<1, 1024, 0, s>>>(ranges, tiles, tile_order);
    if (screen_grads_fixed)
        k_backward_fp32<true><<<tiles, kBwdThreads, 0, s>>>(sp, pair_vals, ranges, cam, bg, final_T, n_contrib,
                                                            dL_dimage, screen_grads, screen_grads_fixed, tile_order);
    else
        k_backward_fp32<false><<<tiles, kBwdThreads, 0, s>>>(sp, pair_vals, ranges, cam, bg, final_T, n_contrib,
                                                             dL_dimage, screen_grads, nullptr, tile_order);
}

}  // namespace rgs_launch
