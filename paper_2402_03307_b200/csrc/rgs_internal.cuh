// Internal declarations shared by the device translation units and the C-ABI host code.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace rgs_dev {

// rasterizer.hpp:13-18, gaussian.hpp:57-59
constexpr int kTile = 16;
constexpr int kTilePixels = kTile * kTile;
constexpr double kNearPlane = 0.2;
constexpr double kAlphaClamp = 0.99;
constexpr double kMinAlpha = 1.0 / 255.0;
constexpr double kStopT = 1e-4;
constexpr double kCovDilation = 0.3;
constexpr double kCov3Eps = 1e-9;
constexpr double kTemporalFloor = 1e-12;
constexpr double kVisibility = 16;
constexpr double kEpsBranch = 1e-12;

// Camera in the form the kernels use (camera.hpp:11-27); center = -R^T t is
// computed on the host with the reference's expression order.
struct DevCamera {
    int width, height, tiles_x, tiles_y;
    double fx, fy, cx, cy, time;
    double R[9];  // row-major rotation block
    double t[3];
    double center[3];
};

// Offsets (in elements) of the SoA parameter blocks, see rgs_scene_params().  A scene
// stores its parameters either as float (base) or, for RGS_SCENE_F64, as double
// (base64) with the same element layout.
struct ParamView {
    const float* base;
    int n;
    const double* base64 = nullptr;
    __host__ __device__ const float4* mean() const { return reinterpret_cast<const float4*>(base); }
    __host__ __device__ const float4* ls() const { return reinterpret_cast<const float4*>(base + 4 * (size_t)n); }
    __host__ __device__ const float4* rot0() const { return reinterpret_cast<const float4*>(base + 8 * (size_t)n); }
    __host__ __device__ const float4* rot1() const { return reinterpret_cast<const float4*>(base + 12 * (size_t)n); }
    __host__ __device__ const float4* sh(int m) const {
        return reinterpret_cast<const float4*>(base + (16 + 4 * (size_t)m) * (size_t)n);
    }
    __host__ __device__ const float* opacity() const { return base + 64 * (size_t)n; }
};

// Load one 4-wide parameter block (block b = elements [4bN, 4(b+1)N)) for Gaussian i.
template <bool F64, typename T>
__device__ __forceinline__ void ld_block(const ParamView& P, int blk, int i, T* v) {
    if constexpr (F64) {
        const double2* p = reinterpret_cast<const double2*>(P.base64 + 4 * (size_t)blk * P.n) + 2 * (size_t)i;
        const double2 a = p[0], b = p[1];
        v[0] = (T)a.x; v[1] = (T)a.y; v[2] = (T)b.x; v[3] = (T)b.y;
    } else {
        const float4 f = reinterpret_cast<const float4*>(P.base + 4 * (size_t)blk * P.n)[i];
        v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
    }
}
// SH coefficient j (= 3k + ch) of Gaussian i: element j % 4 of block 4 + j / 4.
template <bool F64>
__device__ __forceinline__ double ld_coef(const ParamView& P, int i, int j) {
    const size_t off = 4 * (size_t)(4 + (j >> 2)) * P.n + 4 * (size_t)i + (j & 3);
    if constexpr (F64) return P.base64[off];
    else return P.base[off];
}
template <bool F64>
__device__ __forceinline__ double ld_opacity(const ParamView& P, int i) {
    if constexpr (F64) return P.base64[64 * (size_t)P.n + i];
    else return P.base[64 * (size_t)P.n + i];
}

// Per-Gaussian splat records written by the preprocess kernel (dense, indexed by
// Gaussian / input-splat index; `valid` marks the ones that produced a splat).
struct SplatArrays {
    uint8_t* valid;
    uint32_t* tiles;         // number of tiles in the rectangle (0 if empty)
    double2* mean2;          // FP64 screen mean
    double4* conic_ab;       // (ca, cb, cc, alpha_base) FP64
    double4* color_depth;    // (r, g, b, depth) FP64
    double4* flow_radius;    // (flow_x, flow_y, radius, 0)
    ushort4* rect;           // tile rectangle (x0, x1, y0, y1), inclusive
    float4* conic_f;         // (ca2, cb2, cc2, alpha_base): -log2(e) * (A/2, B, C/2)
    float4* color_f;         // (r, g, b, pa2): pa2 = log2(1/(255 ab))
    float4* guard_f;         // (cs2n, pc2, R, lmax): error-bound slope, clamp-gate power log2(0.99/ab),
                             // T-gate error growth bound, radial-cull eigenvalue bound
    float4* ext_f;           // (ex, ey, gx2, gy2): alpha-ellipse bbox, max |grad p2| inside it
    int32_t* source_index;   // only for rasterize_forward (else NULL -> index)
    unsigned long long* depth_key;  // order-preserving bits of the FP64 depth (valid splats)
    double4* dir_dist;              // (view direction, distance) of valid splats (scene renders)
};

// Slice cache of a view batch (k_fp64.cu k_slice_cache): 7 double2 blocks of N + N status bytes.
struct SliceCacheView {
    double2* blk;
    int8_t* status;
};

// Error word: (index << 8) | code, minimum wins (lowest failing index).
constexpr unsigned long long kNoError = ~0ull;

// Per-view device counters shared by the preprocess and binning kernels; the host
// reads it back once per view (after the tile-count scan).
struct BinState {
    unsigned long long err;      // rotor error word (kNoError if none)
    unsigned long long key_min;  // min / max depth key over valid splats
    unsigned long long key_max;
    int n_valid;                 // splats produced (RenderRecords::splats.size())
    int slow_count;              // pixels handed to the FP64 fix-up
    int shift;                   // depth-bucket shift
    uint32_t n_big;              // buckets too large for the per-thread sort
    uint32_t n_pairs;            // total (tile, splat) pairs
    uint32_t pair_cap;           // capacity of the pair buffers (set by the host)
    uint32_t n_pairs_eff;        // n_pairs, or 0 when it exceeds pair_cap (overflow)
    uint32_t overflow;           // 1: the view must be re-rendered with larger buffers
    uint32_t tile_blocks_done;   // tile-major scatter: completion counter of k_tile_offsets
    uint32_t pad3;               // (explicit: the whole 64 B are written, so copies read no padding)
};
static_assert(sizeof(BinState) == 64, "BinState is copied as 64 initialised bytes");

// Guard-band constants for the FP32 blend (DESIGN.md §"FP32 blend with FP64 re-decision").
constexpr float kGuardFloor = 1e-6f;

// Packed per-pixel state written by the forward: bit 31 = slow (FP64) pixel.
constexpr uint32_t kSlowBit = 0x80000000u;

// Reproducible accumulation of the screen-space gradients (RGS_FLAG_REPRODUCIBLE): each double
// contribution v is added to a pair of 64-bit integer counters as fixed point -- v 2^20 =
// hi + f (hi = floor, f in [0, 1)), hi into the first (two's complement), f 2^40 (truncated) into
// the second.  Integer addition is associative, so the sums are bitwise independent of the
// order the atomics land in: |sum| < 2^43, resolution 2^-60, up to 2^23 contributions per value.
__device__ __forceinline__ void fixed_add(unsigned long long* hl, double v) {
    const double s = v * 1048576.0;  // 2^20
    const double h = floor(s);
    atomicAdd(hl, (unsigned long long)(long long)h);
    atomicAdd(hl + 1, (unsigned long long)((s - h) * 1099511627776.0));  // 2^40
}
__device__ __forceinline__ double fixed_value(const unsigned long long* hl) {
    return ((double)(long long)hl[0] + (double)hl[1] * 9.094947017729282e-13) * 9.5367431640625e-07;  // 2^-40, 2^-20
}

}  // namespace rgs_dev

// ---------------------------------------------------------------------------
// Kernel launchers (defined in k_fp64.cu / k_fp32.cu).
namespace rgs_launch {
using namespace rgs_dev;

void preprocess(const float* params, const double* params64, int n, int sh_degree, const DevCamera& cam, const SplatArrays& out,
                BinState* st, cudaStream_t s, const SliceCacheView* cache = nullptr);
size_t slice_cache_bytes(int n);
void slice_cache(const float* params, const double* params64, int n, void* buf, SliceCacheView* view, cudaStream_t s);
void splats_from_host(const void* splats, int n, const DevCamera& cam, const SplatArrays& out, BinState* st,
                      cudaStream_t s);
// k_binning.cu
int num_depth_buckets();     // allocation (the largest bucket count)
int depth_bucket_bits(int n);  // the bucket count used for n splats: 1 << depth_bucket_bits(n)
bool binning_init();
bool raster_init();  // k_raster.cu
bool train_init();   // k_train.cu
void exclusive_scan(const uint32_t* in, int n, uint32_t* out, uint32_t* scratch, uint32_t* total, cudaStream_t s,
                    const int* n_dev = nullptr);
size_t scan1_scratch_words(int n);
void exclusive_scan_1p(const uint32_t* in, int n, uint32_t* out, uint32_t* scratch, uint32_t* total, cudaStream_t s,
                       const int* n_dev = nullptr);
void bucket_hist(const uint8_t* valid, const unsigned long long* key, int n, BinState* st, uint32_t* bucket_count,
                 cudaStream_t s);
void depth_ranks(const uint8_t* valid, const unsigned long long* key, const uint32_t* tiles, int n,
                 const int32_t* src, BinState* st, const uint32_t* bucket_count, const uint32_t* bucket_off,
                 uint32_t* bucket_cur, unsigned long long* ent_key, uint32_t* ent_id, uint32_t* sorted_ids,
                 uint32_t* sorted_tiles, uint32_t* big_list, void* big_scratch, cudaStream_t s);
int tile_key_shift(int tiles_x, int tiles_y);
void duplicate(const uint32_t* sorted_ids, const uint32_t* pair_off, const uint32_t* sorted_tiles,
               const ushort4* rect, const BinState* st, int n, int tiles_x, int tiles_y, uint32_t* keys,
               uint32_t* vals, int* aux, cudaStream_t s);
void check_capacity(BinState* st, cudaStream_t s);
void fold_status(const BinState* st, unsigned long long* word, unsigned long long overflow_word, cudaStream_t s);
void frame_init(BinState* st, uint32_t pair_cap, uint32_t* bucket_count, uint32_t* bucket_cur, int n,
                cudaStream_t s);
// Tile-major scatter (images up to 256 x 256 tiles and 8192 tiles; k_binning.cu): per-chunk tile
// counts -> per-chunk prefixes, tile starts, tile ranges and the pair count (into `st`), then the
// pairs' splat ids straight to their sorted positions.
// mode: RGS_BINNING_AUTO (the scatter for single views, the radix passes for the views of a
// batch), RGS_BINNING_RADIX, RGS_BINNING_SCATTER (where it applies); the process default comes
// from the environment variable RGS_BINNING=auto|radix|scatter.
int default_binning_mode();
bool tile_scatter_usable(int tiles_x, int tiles_y, int n, long long pair_cap, bool batch, int mode);
size_t tile_count_words(int n, int n_tiles);
void tile_counts(const uint32_t* sorted_ids, const uint32_t* sorted_tiles, const ushort4* rect, BinState* st, int n,
                 int tiles_x, int tiles_y, uint32_t* counts, uint32_t* starts, uint2* ranges, cudaStream_t s);
void tile_scatter(const uint32_t* sorted_ids, const uint32_t* sorted_tiles, const ushort4* rect, BinState* st,
                  int n, int tiles_x, int tiles_y, const uint32_t* counts, const uint32_t* starts, uint2* ranges,
                  uint32_t* vals, cudaStream_t s);
int radix_blocks(long long n_pairs);
size_t radix_count_entries(long long n_pairs);
// Returns 1 when the sorted pairs end in (keys_b, vals_b) (three passes), 0 for (keys_a, vals_a).
int tile_radix_sort(uint32_t* keys_a, uint32_t* vals_a, uint32_t* keys_b, uint32_t* vals_b, const BinState* st,
                    long long n_pairs, int tiles_x, int tiles_y, uint32_t* status_a, uint32_t* status_b, int* aux,
                    uint2* ranges, cudaStream_t s);
// tile_order (optional, n_tiles u32): K5's blocks take the tiles longest list first (one
// counting-sort kernel before it), so the last wave is made of short tiles.
void blend_fp32(const SplatArrays& sp, const uint32_t* pair_vals, const uint2* ranges, const DevCamera& cam,
                float3 bg, int flow_mode, float* image, double* final_T, uint32_t* n_contrib,
                uint32_t* slow_list, int* slow_count, unsigned long long* counters, cudaStream_t s,
                uint32_t* tile_order = nullptr);
void mark_all_slow(int n_pixels, uint32_t* slow_list, int* slow_count, cudaStream_t s);
void blend_fp64_pixels(const SplatArrays& sp, const uint32_t* pair_vals, const uint2* ranges,
                       const DevCamera& cam, double3 bg, int flow_mode, float* image, double* image64,
                       double* final_T, uint32_t* n_contrib, const uint32_t* slow_list, const int* slow_count,
                       int max_pixels, cudaStream_t s);
void backward_deterministic(const SplatArrays& sp, const uint32_t* pair_vals, const uint2* ranges,
                            const DevCamera& cam, double3 bg, const double* final_T, const uint32_t* n_contrib,
                            const float* dL_dimage, const uint32_t* sorted_ids, const int* n_valid_dev, int n,
                            uint32_t* rank, double* tile_grads, double* screen_grads, cudaStream_t s);
int project_one(const double* sliced16_dev, const DevCamera& cam, const double* sh48_dev, int sh_degree,
                double opacity_logit, void* out_dev, int* survived_dev, cudaStream_t s, double* cache_dev = nullptr);
// screen_grads_fixed (NULL: FP64 atomics into screen_grads): RGS_FLAG_REPRODUCIBLE's fixed-point
// counters (18 u64 per splat, fixed_add), turned into screen_grads by fixed_to_double.
void backward_fp32(const SplatArrays& sp, const uint32_t* pair_vals, const uint2* ranges,
                   const DevCamera& cam, float3 bg, const double* final_T, const uint32_t* n_contrib,
                   const float* dL_dimage, double* screen_grads, cudaStream_t s,
                   unsigned long long* screen_grads_fixed = nullptr,
                   uint32_t* tile_order = nullptr);
void backward_fp64_pixels(const SplatArrays& sp, const uint32_t* pair_vals, const uint2* ranges,
                          const DevCamera& cam, double3 bg, const double* final_T, const uint32_t* n_contrib,
                          const float* dL_dimage, const uint32_t* slow_list, const int* slow_count,
                          int max_pixels, double* screen_grads, cudaStream_t s,
                          unsigned long long* screen_grads_fixed = nullptr);
void fixed_to_double(const unsigned long long* fixed, size_t n_values, double* out, cudaStream_t s);
void gaussian_backward(const float* params, const double* params64, int n, int sh_degree, const DevCamera& cam,
                       const double4* dir_dist, double* color_dmean3, const uint8_t* valid,
                       const double* screen_grads, int accumulate, float* grads, float* vnorm,
                       int32_t* visible, cudaStream_t s, int part = 3);
void export_splats(const SplatArrays& sp, const uint32_t* compact_ids, int n_valid, void* out,
                   cudaStream_t s);
void compact_index(const uint8_t* valid, const uint32_t* scan, int n, uint32_t* compact_ids, cudaStream_t s);
void map_ids(const uint32_t* pair_vals, long long n_pairs, const uint32_t* scan, int32_t* out, cudaStream_t s);
void scene_pack(const float* mean, const float* ls, const float* rot, const float* op, const float* sh,
                int n, float* params, cudaStream_t s);
void scene_pack64(const double* mean, const double* ls, const double* rot, const double* op, const double* sh,
                  int n, double* params, cudaStream_t s);
void scene_unpack(const float* params, const double* params64, int n, double* mean, double* ls, double* rot,
                  double* op, double* sh, cudaStream_t s);
void records_to_soa(const float* rec, int n, float* params, double* params64, cudaStream_t s);
void soa_to_records(const float* params, const double* params64, int n, float* rec, cudaStream_t s);
// (n, 65) double rows (mean4, log_scales4, rotor8, opacity_logit, sh48 channel-major) <-> the SoA
void rows_to_soa(const double* rows, int n, float* params, double* params64, cudaStream_t s);
void soa_to_rows(const float* params, const double* params64, int n, double* rows, cudaStream_t s);
void valid_to_u32(const uint8_t* valid, int n, uint32_t* out, cudaStream_t s);
double ffma_peak(float* out, int blocks, int iters, cudaStream_t s);
double dfma_peak(double* out, int blocks, int iters, cudaStream_t s);
}  // namespace rgs_launch
