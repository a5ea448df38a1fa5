// Tile binning (replaces bin_and_sort, rasterizer.cpp:57-74).
//
// The reference appends splat k to every tile of its rectangle in k order, then sorts
// each tile's list by (depth, source_index).  Here:
//
//   1. Depth ranks: an MSD counting sort of the visible splats on a depth bucket (the
//      top bits of key - min_key, 2^18 buckets); every bucket is then sorted by the
//      exact (64-bit depth key, source index) -- insertion sort per bucket, shared-memory
//      bitonic for rare large buckets.  sorted_ids[r] = splat of rank r.
//   2. Up to 256 x 256 (and 8192) tiles: the tile-major scatter below writes every pair at its
//      final place directly.  Larger images take steps 2' and 3:
//   2'. Duplicate-with-key in rank order: an exclusive scan of tiles-touched over the
//      ranks gives each splat its pair offset; warps emit the (tile, splat) pairs of 32
//      consecutive ranks cooperatively (coalesced stores).
//   3. LSD radix sort of the pairs on the packed key (ty << 8 | tx), as two stable 8-bit
//      digit passes (tx, then ty), one kernel each: the global digit histograms come from
//      the duplicate kernel (per splat rectangle, not per pair), a block's offset inside each
//      digit from a decoupled look-back; the block ranks its elements with warp
//      __match_any_sync peer groups, sorts them by digit in shared memory and writes
//      contiguous per-digit runs.
//
// Stable passes over pairs emitted in rank order leave every tile's list in
// (depth, index) order: the reference's std::sort order bit for bit.
#include <algorithm>
#include <cstdlib>

#include "rgs_internal.cuh"

namespace rgs_dev {

// Depth buckets: 2^bits with bits = ceil(log2 n) - 3 in [12, 18] (about 8 splats per bucket at
// most): C2 (300K) 16 bits -- 0.046 -> 0.042 ms for the depth ranks against 18 bits (a quarter of
// the bucket scan and the per-view bucket reset); C4 (2M) keeps 18.
constexpr int kBucketBits = 18;  // the largest (allocation)
constexpr int kNumBuckets = 1 << kBucketBits;
constexpr int kSmallBucket = 32;
constexpr unsigned kFullMask = 0xffffffffu;

__device__ __forceinline__ bool key_less(unsigned long long ka, uint32_t ta, unsigned long long kb, uint32_t tb) {
    return ka < kb || (ka == kb && ta < tb);
}

// Tie-break value of splat i: its source index (rasterize_forward) or i itself.
__device__ __forceinline__ uint32_t tie_of(const int32_t* src, uint32_t i) {
    return src ? ((uint32_t)src[i] ^ 0x80000000u) : i;
}

// --------------------------------------------------------------------------- scan
// Exclusive scan of a u32 array in three phases (block sums, scan of sums, apply).
constexpr int kScanThreads = 256;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* total) {
    __shared__ uint32_t warp_sums[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFullMask, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[w] = x;
    __syncthreads();
    if (w == 0) {
        const int nw = blockDim.x >> 5;
        uint32_t s = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFullMask, s, o);
            if (lane >= o) s += y;
        }
        if (lane < nw) warp_sums[lane] = s;
    }
    __syncthreads();
    const uint32_t before = (w > 0 ? warp_sums[w - 1] : 0) + x - v;
    if (total) *total = warp_sums[(blockDim.x >> 5) - 1];
    __syncthreads();
    return before;
}


// Single-pass exclusive scan (decoupled look-back): one kernel instead of sums / scan of sums /
// apply.  Status words: bit 63 inclusive, bit 62 aggregate, low 32 bits the value.  Tiles of
// kScan1Tile items; blocks take tile indices from an atomic ticket.
constexpr int kScan1Items = 8;
constexpr int kScan1Tile = kScanThreads * kScan1Items;
constexpr unsigned long long kScanInc = 1ull << 63, kScanAgg = 1ull << 62;

__global__ void __launch_bounds__(kScanThreads) k_scan_1p(const uint32_t* __restrict__ in, int n,
                                                          const int* __restrict__ n_dev, uint32_t* out,
                                                          uint32_t* total, unsigned long long* status,
                                                          uint32_t* ticket) {
    __shared__ uint32_t s_bid, s_excl;
    if (threadIdx.x == 0) s_bid = atomicAdd(ticket, 1u);
    __syncthreads();
    const int bid = (int)s_bid;
    if (n_dev) n = min(n, *n_dev);
    const int base = bid * kScan1Tile;
    if (base >= n && !(bid == 0 && total)) return;
    uint32_t v[kScan1Items];
    uint32_t sum = 0;
#pragma unroll
    for (int k = 0; k < kScan1Items; ++k) {
        const int e = base + threadIdx.x * kScan1Items + k;
        v[k] = e < n ? in[e] : 0u;
        sum += v[k];
    }
    uint32_t agg;
    const uint32_t ex = block_exclusive_scan(sum, &agg);
    if (threadIdx.x < 32) {
        // warp-wide look-back: lane j reads predecessor p - j, 32 status words per round trip
        const int lane = threadIdx.x;
        volatile unsigned long long* vs = status;
        uint32_t excl = 0;
        if (bid == 0) {
            if (lane == 0) vs[0] = kScanInc | agg;
        } else {
            if (lane == 0) vs[bid] = kScanAgg | agg;
            for (int p = bid - 1; p >= 0;) {
                const unsigned long long w = p - lane >= 0 ? vs[p - lane] : (unsigned long long)(kScanInc | 0ull);
                const unsigned inc = __ballot_sync(kFullMask, (w & kScanInc) != 0);
                const unsigned ready = __ballot_sync(kFullMask, (w & (kScanInc | kScanAgg)) != 0);
                const int last = inc ? __ffs(inc) - 1 : 31;  // nearest inclusive predecessor
                const unsigned need = last == 31 ? kFullMask : ((2u << last) - 1u);
                if ((ready & need) != need) continue;  // a predecessor has not published yet
                uint32_t x = lane <= last && p - lane >= 0 ? (uint32_t)w : 0u;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFullMask, x, o);
                excl += x;
                if (inc) break;
                p -= 32;
            }
            if (lane == 0) vs[bid] = kScanInc | (unsigned long long)(excl + agg);
        }
        if (lane == 0) {
            s_excl = excl;
            const bool last_tile = base + kScan1Tile >= n;
            if (last_tile && total) *total = excl + agg;
        }
    }
    __syncthreads();
    uint32_t run = s_excl + ex;
#pragma unroll
    for (int k = 0; k < kScan1Items; ++k) {
        const int e = base + threadIdx.x * kScan1Items + k;
        if (e < n) out[e] = run;
        run += v[k];
    }
}

// Inclusive prefix sum over the block of one int per thread (a difference array -> values).
__device__ __forceinline__ int block_inclusive_diff(int v) {
    uint32_t total;
    const uint32_t ex = block_exclusive_scan((uint32_t)v, &total);
    return (int)(ex + (uint32_t)v);
}

// `n_dev` (optional) overrides n with a device-side count.
__global__ void __launch_bounds__(kScanThreads) k_scan_sums(const uint32_t* __restrict__ in, int n,
                                                            const int* __restrict__ n_dev, uint32_t* sums) {
    if (n_dev) n = min(n, *n_dev);
    const int base = blockIdx.x * kScanTile + threadIdx.x * kScanItems;
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k)
        if (base + k < n) s += in[base + k];
    uint32_t total;
    block_exclusive_scan(s, &total);
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_block_sums(uint32_t* sums, int nb, uint32_t* grand_total) {
    uint32_t carry = 0;
    for (int base = 0; base < nb; base += kScanThreads) {
        const int i = base + threadIdx.x;
        const uint32_t v = i < nb ? sums[i] : 0;
        uint32_t total;
        const uint32_t ex = block_exclusive_scan(v, &total);
        if (i < nb) sums[i] = carry + ex;
        carry += total;
    }
    if (threadIdx.x == 0 && grand_total) *grand_total = carry;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_apply(const uint32_t* __restrict__ in, int n,
                                                             const int* __restrict__ n_dev,
                                                             const uint32_t* __restrict__ sums, uint32_t* out) {
    if (n_dev) n = min(n, *n_dev);
    const int base = blockIdx.x * kScanTile + threadIdx.x * kScanItems;
    uint32_t v[kScanItems];
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        v[k] = base + k < n ? in[base + k] : 0;
        s += v[k];
    }
    uint32_t run = block_exclusive_scan(s, nullptr) + sums[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (base + k < n) out[base + k] = run;
        run += v[k];
    }
}

// --------------------------------------------------------------------------- depth ranks
__global__ void k_bucket_setup(BinState* st, int bucket_bits) {
    const unsigned long long lo = st->key_min, hi = st->key_max;
    int shift = 0;
    if (hi > lo) {
        const unsigned long long range = hi - lo;
        const int bits = 64 - __clzll(range);
        shift = bits > bucket_bits ? bits - bucket_bits : 0;
    }
    st->shift = shift;
}

__global__ void k_bucket_hist(const uint8_t* __restrict__ valid, const unsigned long long* __restrict__ key, int n,
                              const BinState* __restrict__ st, uint32_t* bucket_count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !valid[i]) return;
    atomicAdd(&bucket_count[(uint32_t)((key[i] - st->key_min) >> st->shift)], 1u);
}

__global__ void k_bucket_scatter(const uint8_t* __restrict__ valid, const unsigned long long* __restrict__ key,
                                 int n, const BinState* __restrict__ st, const uint32_t* __restrict__ bucket_off,
                                 uint32_t* bucket_cur, unsigned long long* ent_key, uint32_t* ent_id) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !valid[i]) return;
    const unsigned long long k = key[i];
    const uint32_t b = (uint32_t)((k - st->key_min) >> st->shift);
    const uint32_t pos = bucket_off[b] + atomicAdd(&bucket_cur[b], 1u);
    ent_key[pos] = k;
    ent_id[pos] = (uint32_t)i;
}

// One thread per scattered entry: its rank inside its (small) bucket by counting the
// bucket's entries that order before it -- (key, tie) is a total order -- and a direct
// write to the sorted position.  Buckets above kSmallBucket are deferred to the big sort
// (queued once, by their first entry).
__global__ void k_bucket_sort_small(const uint32_t* __restrict__ bucket_count, const uint32_t* __restrict__ bucket_off,
                                    const unsigned long long* __restrict__ ent_key,
                                    const uint32_t* __restrict__ ent_id, const int32_t* __restrict__ src,
                                    const uint32_t* __restrict__ tiles, uint32_t* sorted_ids,
                                    uint32_t* sorted_tiles, BinState* st, uint32_t* big_list) {
    const int pos = blockIdx.x * blockDim.x + threadIdx.x;
    if (pos >= st->n_valid) return;
    const unsigned long long k = ent_key[pos];
    const uint32_t b = (uint32_t)((k - st->key_min) >> st->shift);
    const uint32_t cnt = bucket_count[b], off = bucket_off[b];
    if (cnt > kSmallBucket) {
        if ((uint32_t)pos == off) big_list[atomicAdd(&st->n_big, 1u)] = b;
        return;
    }
    const uint32_t id = ent_id[pos];
    const uint32_t t = tie_of(src, id);
    uint32_t rank = 0;
    for (uint32_t q = off; q < off + cnt; ++q)
        if (q != (uint32_t)pos) rank += key_less(ent_key[q], tie_of(src, ent_id[q]), k, t) ? 1u : 0u;
    sorted_ids[off + rank] = id;
    sorted_tiles[off + rank] = tiles[id];
}

struct SortRec {
    unsigned long long key;
    uint32_t tie;
    uint32_t id;
};

__device__ __forceinline__ bool rec_greater(const SortRec& a, const SortRec& b) {
    return key_less(b.key, b.tie, a.key, a.tie);
}

__device__ void block_bitonic(SortRec* s, int n_pow2) {
    for (int k = 2; k <= n_pow2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n_pow2; i += blockDim.x) {
                const int l = i ^ j;
                if (l > i) {
                    const bool up = (i & k) == 0;
                    SortRec a = s[i], b = s[l];
                    if (rec_greater(a, b) == up) {
                        s[i] = b;
                        s[l] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
}

constexpr int kBigSmem = 4096;  // records per block in shared memory (64 KB)

// One block per big bucket: bitonic in shared memory, or in a disjoint window
// [2 off, 2 off + np) of global scratch when the bucket exceeds kBigSmem records.
__global__ void __launch_bounds__(512) k_bucket_sort_big(const uint32_t* __restrict__ bucket_count,
                                                         const uint32_t* __restrict__ bucket_off,
                                                         const unsigned long long* __restrict__ ent_key,
                                                         const uint32_t* __restrict__ ent_id,
                                                         const int32_t* __restrict__ src,
                                                         const uint32_t* __restrict__ tiles, const BinState* st,
                                                         const uint32_t* __restrict__ big_list, uint32_t* sorted_ids,
                                                         uint32_t* sorted_tiles, SortRec* scratch) {
    extern __shared__ SortRec smem_rec[];
    for (uint32_t w = blockIdx.x; w < st->n_big; w += gridDim.x) {
        const uint32_t b = big_list[w];
        const uint32_t cnt = bucket_count[b], off = bucket_off[b];
        int np = 1;
        while (np < (int)cnt) np <<= 1;
        SortRec* s = np <= kBigSmem ? smem_rec : scratch + (size_t)off * 2;
        for (int i = threadIdx.x; i < np; i += blockDim.x) {
            if (i < (int)cnt) {
                const uint32_t id = ent_id[off + i];
                s[i] = SortRec{ent_key[off + i], tie_of(src, id), id};
            } else {
                s[i] = SortRec{~0ull, 0xffffffffu, 0xffffffffu};
            }
        }
        __syncthreads();
        block_bitonic(s, np);
        for (int i = threadIdx.x; i < (int)cnt; i += blockDim.x) {
            sorted_ids[off + i] = s[i].id;
            sorted_tiles[off + i] = tiles[s[i].id];
        }
        __syncthreads();
    }
}

// --------------------------------------------------------------------------- duplicate
// Pair emission of one warp (32 consecutive ranks) for k_duplicate.
__device__ __forceinline__ void emit_pairs(uint32_t id, uint32_t cnt, uint32_t off, ushort4 q, int lane,
                                                uint32_t* keys, uint32_t* vals, int ty_shift) {
    // inclusive prefix of counts within the warp
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFullMask, incl, o);
        if (lane >= o) incl += y;
    }
    const uint32_t total = __shfl_sync(kFullMask, incl, 31);
    const uint32_t base = __shfl_sync(kFullMask, off, 0);
    const int w = q.y - q.x + 1;
    for (uint32_t k0 = 0; k0 < total; k0 += 32) {  // warp-uniform trip count (full-mask shuffles)
        const uint32_t k = k0 + lane;
        // owner: first lane whose inclusive prefix exceeds k (binary search over lanes)
        int lo = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            const uint32_t v = __shfl_sync(kFullMask, incl, lo + step - 1);
            if (v <= k) lo += step;
        }
        // lane `lo` owns pair k; fetch its rectangle and exclusive prefix
        const uint32_t o_incl = __shfl_sync(kFullMask, incl, lo);
        const uint32_t o_cnt = __shfl_sync(kFullMask, cnt, lo);
        const int o_w = __shfl_sync(kFullMask, w, lo);
        const int o_x0 = __shfl_sync(kFullMask, (int)q.x, lo);
        const int o_y0 = __shfl_sync(kFullMask, (int)q.z, lo);
        const uint32_t o_id = __shfl_sync(kFullMask, id, lo);
        if (k < total) {
            const int m = (int)(k - (o_incl - o_cnt));
            const int dy = m / o_w, dx = m - dy * o_w;
            keys[base + k] = ((uint32_t)(o_y0 + dy) << ty_shift) | (uint32_t)(o_x0 + dx);  // packed (ty, tx)
            vals[base + k] = o_id;
        }
    }
}

// Warp-cooperative: the pairs of 32 consecutive ranks are written as one contiguous
// run (lane l writes pair l, l+32, ...).  key = tile id, value = splat id.
// It also builds the two radix passes' global digit histograms per splat, not per pair: a
// rectangle [x0, x1] x [y0, y1] adds its height to tx digits x0..x1 and its width to ty digits
// y0..y1 -- difference arrays in shared memory, flushed with 2 x 257 global atomics per block.
__global__ void __launch_bounds__(256) k_duplicate(const uint32_t* __restrict__ sorted_ids,
                                                   const uint32_t* __restrict__ pair_off,
                                                   const uint32_t* __restrict__ sorted_tiles,
                                                   const ushort4* __restrict__ rect, const BinState* __restrict__ st,
                                                   int ty_shift, uint32_t* keys, uint32_t* vals, int* hist_diff) {
    __shared__ int sdx[257], sdy[257];
    for (int e = threadIdx.x; e < 257; e += blockDim.x) sdx[e] = sdy[e] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int nv = st->n_valid;
    const bool warp_live = !st->overflow && r - lane < nv;  // buffers large enough, warp not past the end
    uint32_t id = 0, cnt = 0, off = 0;
    ushort4 q = make_ushort4(0, 0, 0, 0);
    if (warp_live && r < nv) {
        id = sorted_ids[r];
        cnt = sorted_tiles[r];
        off = pair_off[r];
        if (cnt) {
            q = rect[id];
            if (ty_shift == 8) {  // byte digits tx / ty: histograms per rectangle
                const int h = q.w - q.z + 1, wd = q.y - q.x + 1;
                atomicAdd(&sdx[q.x], h);
                atomicAdd(&sdx[q.y + 1], -h);
                atomicAdd(&sdy[q.z], wd);
                atomicAdd(&sdy[q.w + 1], -wd);
            }
        }
    }
    if (warp_live) emit_pairs(id, cnt, off, q, lane, keys, vals, ty_shift);
    __syncthreads();
    for (int e = threadIdx.x; e < 257; e += blockDim.x) {
        if (sdx[e]) atomicAdd(&hist_diff[e], sdx[e]);
        if (sdy[e]) atomicAdd(&hist_diff[257 + e], sdy[e]);
    }
}

// --------------------------------------------------------------------------- LSD digit pass
// Stable counting-sort pass on one byte of the packed key (ty << 8 | tx): tx for pass 0,
// ty for pass 1.  A block sorts a tile of kBlockTile consecutive elements locally:
// warp w ranks the tile's elements [256 w, 256 w + 256) in 8 rounds of 32 (lane order,
// __match_any_sync peer groups, warp-private running counts per digit); a per-digit
// prefix over the 8 warps gives each element its position in a digit-sorted copy of
// the tile in shared memory, which is then written out as contiguous per-digit runs
// at the global offsets of (digit, block).  Stability follows from (block, warp,
// round, lane) order = element order.
constexpr int kRadixThreads = 256;
constexpr int kRadixWarps = kRadixThreads / 32;
constexpr int kRadixRounds = 16;  // the largest tile (allocation); RGS_RADIX=8 selects 2048-item tiles
// 4096-item tiles at 3 CTAs/SM (76 registers: the values are re-read at the local scatter rather
// than held through the ranking): serialised time equal to 2 CTAs/SM at 120 registers, +0.5 % FPS
// in the pipelined sweep (a resident radix block leaves room for K5 blocks); 4 CTAs/SM spills.
constexpr int kBlockTile = kRadixThreads * kRadixRounds;  // 4096
constexpr int kMinBlockTile = kRadixThreads * 8;
static int g_radix_rounds = 16;
constexpr int kRadixDigits = 256;
constexpr int kAuxInts = 784;  // digit histograms + tickets (tile_radix_sort)

// One-sweep digit pass: the global digit
// starts come from the histograms k_duplicate built, and each block's offset inside a digit
// from a decoupled look-back over its predecessors' published per-digit counts.  Blocks take
// their tile index from an atomic ticket, so every predecessor has started (and publishes its
// aggregate before looking back itself): the spin-wait always terminates.
constexpr uint32_t kFlagAgg = 1u << 30, kFlagInc = 2u << 30, kCountMask = (1u << 30) - 1u;

template <int ROUNDS, int MINB>
__global__ void __launch_bounds__(kRadixThreads, MINB) k_radix_onesweep(const uint32_t* __restrict__ keys_in,
                                                                  const uint32_t* __restrict__ vals_in,
                                                                  const BinState* __restrict__ st, int shift,
                                                                  const int* __restrict__ hist_diff, int hist_plain,
                                                                  uint32_t* status, uint32_t* ticket,
                                                                  uint32_t* keys_out, uint32_t* vals_out,
                                                                  int nbits) {
    __shared__ uint32_t wcnt[kRadixWarps][kRadixDigits];
    __shared__ uint32_t dstart[kRadixDigits];
    __shared__ uint32_t gbase[kRadixDigits];
    __shared__ uint32_t skey[(kRadixThreads * ROUNDS)], sval[(kRadixThreads * ROUNDS)];
    __shared__ uint32_t s_bid;
    if (threadIdx.x == 0) s_bid = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t bid = s_bid;
    const uint32_t n = st->n_pairs_eff;
    if (bid * (uint32_t)(kRadixThreads * ROUNDS) >= n) return;  // past the end (all later tickets too)
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < kRadixWarps; ++k) wcnt[k][threadIdx.x] = 0;
    const uint32_t base = bid * (kRadixThreads * ROUNDS) + w * ((kRadixThreads * ROUNDS) / kRadixWarps);
    // the values are read again (L2) at the local scatter instead of being held in registers
    // through the ranking: 120 -> fewer registers, more blocks per SM
    uint32_t key[ROUNDS], rk[ROUNDS];
#pragma unroll
    for (int j = 0; j < ROUNDS; ++j) {
        const uint32_t e = base + j * 32 + lane;
        key[j] = e < n ? keys_in[e] : 0xffffffffu;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < ROUNDS; ++j) {
        const uint32_t d = key[j] != 0xffffffffu ? (key[j] >> shift) & 0xffu : 0xffffffffu;
        // lanes with the same digit: __match_any_sync, or (nbits > 0, the RGS_RADIX_BALLOT A/B
        // switch) nbits ballots over the digit's significant bits -- slower (0.125 vs 0.094 ms per
        // C2 frame); the kernel as built with both paths measured 4 % faster on the match path than
        // the match-only build (0.0945 vs 0.0984 ms, same box: register allocation, 79 vs 76)
        unsigned peers;
        if (nbits > 0) {
            const bool ok = d != 0xffffffffu;
            peers = __ballot_sync(0xffffffffu, ok);
            if (!ok) peers = ~peers;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                if (b < nbits) {
                    const bool bit = (d >> b) & 1u;
                    const unsigned bal = __ballot_sync(0xffffffffu, bit);
                    peers &= bit ? bal : ~bal;
                }
            }
        } else {
            peers = __match_any_sync(0xffffffffu, d);
        }
        const uint32_t below = __popc(peers & ((1u << lane) - 1u));
        uint32_t r = 0;
        if (d != 0xffffffffu) r = wcnt[w][d] + below;
        __syncwarp();
        if (d != 0xffffffffu && below == 0) wcnt[w][d] += __popc(peers);
        __syncwarp();
        rk[j] = r;
    }
    __syncthreads();
    const int dd = threadIdx.x;
    uint32_t tot = 0;
#pragma unroll
    for (int k = 0; k < kRadixWarps; ++k) {
        const uint32_t c = wcnt[k][dd];
        wcnt[k][dd] = tot;
        tot += c;
    }
    // publish this block's count of digit dd, then look back for its exclusive prefix
    volatile uint32_t* vs = status;
    if (bid == 0) {
        vs[dd] = kFlagInc | tot;
    } else {
        vs[(size_t)bid * kRadixDigits + dd] = kFlagAgg | tot;
        // Look back in windows of kLookback predecessors: their loads are issued together, so
        // a long run of aggregate-only predecessors (the first wave starts all at once) costs
        // one memory round trip per window rather than per block.
        constexpr int kLookback = 16;
        uint32_t excl = 0;
        int64_t p = (int64_t)bid - 1;
        while (p >= 0) {
            uint32_t win[kLookback];
#pragma unroll
            for (int j = 0; j < kLookback; ++j) win[j] = p - j >= 0 ? (uint32_t)vs[(size_t)(p - j) * kRadixDigits + dd] : (uint32_t)kFlagInc;
            bool stop = false;
            int used = 0;
#pragma unroll
            for (int j = 0; j < kLookback; ++j) {
                if (stop) break;
                const uint32_t v = win[j];
                if (!(v & (kFlagAgg | kFlagInc))) break;  // not published yet: reload from here
                if (p - j >= 0) excl += v & kCountMask;
                ++used;
                if (v & kFlagInc) stop = true;
            }
            if (stop) break;
            p -= used;
        }
        vs[(size_t)bid * kRadixDigits + dd] = kFlagInc | (excl + tot);
        dstart[dd] = excl;  // temporarily: exclusive offset of this block inside the digit
    }
    if (bid == 0) dstart[dd] = 0;
    // global digit start: exclusive prefix over digits of the histogram (difference array)
    {
        uint32_t t2;
        const uint32_t h = hist_plain ? (uint32_t)hist_diff[dd] : (uint32_t)block_inclusive_diff(hist_diff[dd]);
        const uint32_t ex = block_exclusive_scan(h, &t2);
        gbase[dd] = ex + dstart[dd];
    }
    __syncthreads();
    {
        uint32_t total;
        const uint32_t ex = block_exclusive_scan(tot, &total);
        __syncthreads();
        dstart[dd] = ex;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < ROUNDS; ++j) {
        if (key[j] == 0xffffffffu) continue;
        const uint32_t d = (key[j] >> shift) & 0xffu;
        const uint32_t p = dstart[d] + wcnt[w][d] + rk[j];
        skey[p] = key[j];
        sval[p] = vals_in[base + j * 32 + lane];
    }
    __syncthreads();
    const uint32_t valid_in_tile = min((uint32_t)(kRadixThreads * ROUNDS), n - bid * (uint32_t)(kRadixThreads * ROUNDS));
    for (uint32_t i = threadIdx.x; i < valid_in_tile; i += kRadixThreads) {
        const uint32_t k = skey[i];
        const uint32_t d = (k >> shift) & 0xffu;
        const uint32_t g = gbase[d] + (i - dstart[d]);
        keys_out[g] = k;
        vals_out[g] = sval[i];
    }
}

// Wide tile keys (images beyond 256 tiles per axis: key = ty << 12 | tx, three byte passes):
// the byte-digit histograms of all three passes in one read of the keys (block histograms in
// shared memory, then global atomics).
__global__ void __launch_bounds__(256) k_digit_hist3(const uint32_t* __restrict__ keys, const BinState* __restrict__ st,
                                                     int* hist) {
    __shared__ int h[3][kRadixDigits];
    for (int e = threadIdx.x; e < 3 * kRadixDigits; e += blockDim.x) (&h[0][0])[e] = 0;
    __syncthreads();
    const uint32_t n = st->n_pairs_eff;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t k = keys[i];
        atomicAdd(&h[0][k & 0xffu], 1);
        atomicAdd(&h[1][(k >> 8) & 0xffu], 1);
        atomicAdd(&h[2][(k >> 16) & 0xffu], 1);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 3 * kRadixDigits; e += blockDim.x)
        if ((&h[0][0])[e]) atomicAdd(&hist[e], (&h[0][0])[e]);
}

// --------------------------------------------------------------------------- tile-major scatter
// For images up to 256 x 256 tiles and kScatterMaxTiles tiles the pairs are not materialised and
// sorted at all: every (tile, splat) pair is written straight to its final position
//
//     pos(r, t) = start(t) + #{ r' < r : rect(r') contains t }
//
// (r = depth rank), which is exactly the reference's per-tile (depth, index) order.  The count is
// split three ways:
//   A  k_chunk_tile_counts -- per chunk of 32 * rounds consecutive ranks, the pair count of every
//      tile (row difference arrays in shared memory, a warp scan per tile row);
//   B  k_tile_offsets      -- per tile, the exclusive prefix of those counts over the chunks (in
//      place) and the tile's total; the last block to finish scans the totals into the tile
//      starts, the tile ranges and the pair count;
//   C  k_tile_scatter      -- per chunk, rounds of 32 ranks: lane masks per tile column and tile row
//      (which of the round's 32 rectangles cover it; prefix-OR of begin / end marks), so a pair's
//      offset inside the round is popc(col_mask & row_mask & lanes below); a per-tile running
//      position in shared memory (tile start + chunk prefix, stamped with the round that last
//      advanced it) carries the rounds.  Tile row ty belongs to warp ty % 4 of the block, so no
//      two warps touch a running position; inside a warp each lane walks its own run of pairs.
// Traffic: rect + id + count per visible splat, 4 B per pair written, and the chunk x tile count
// matrix (written by A, read and rewritten by B, read by C) -- against 2 x 16 B per pair for the
// two radix passes plus 8 B per pair of K3.
constexpr int kScatWarps = 4;
constexpr int kScatThreads = 32 * kScatWarps;
constexpr int kScatterMaxTiles = 8192;
constexpr int kOffThreads = 512;  // k_tile_offsets: 16 warps share the chunks of 32 tiles
constexpr uint32_t kRunMask = (1u << 26) - 1u;  // k_tile_scatter: positions < 2^26, 6-bit round stamp
static int g_scatter_rounds = 16;
// 0: the scatter for single views, the radix passes for multi-view batches;
// 1: radix passes only; 2: the scatter wherever it applies (RGS_BINNING=auto|radix|scatter)
static int g_binning_mode = 0;

__global__ void __launch_bounds__(256) k_chunk_tile_counts(const uint32_t* __restrict__ sorted_ids,
                                                           const uint32_t* __restrict__ sorted_tiles,
                                                           const ushort4* __restrict__ rect,
                                                           const BinState* __restrict__ st, int chunk, int tiles_x,
                                                           int tiles_y, uint32_t* counts) {
    extern __shared__ int s_diff[];  // tiles_y rows of tiles_x + 1
    const int W = tiles_x + 1;
    const int nv = st->n_valid;
    const int r0 = blockIdx.x * chunk;
    if (r0 >= nv) return;
    for (int e = threadIdx.x; e < tiles_y * W; e += blockDim.x) s_diff[e] = 0;
    __syncthreads();
    const int r1 = min(r0 + chunk, nv);
    for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
        if (!sorted_tiles[r]) continue;
        const ushort4 q = rect[sorted_ids[r]];
        for (int y = q.z; y <= q.w; ++y) {
            atomicAdd(&s_diff[y * W + q.x], 1);
            atomicAdd(&s_diff[y * W + q.y + 1], -1);
        }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    uint32_t* out = counts + (size_t)blockIdx.x * tiles_x * tiles_y;
    for (int y = threadIdx.x >> 5; y < tiles_y; y += nw) {
        int carry = 0;
        for (int x0 = 0; x0 < tiles_x; x0 += 32) {
            const int x = x0 + lane;
            int v = x < tiles_x ? s_diff[y * W + x] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(kFullMask, v, o);
                if (lane >= o) v += u;
            }
            v += carry;
            if (x < tiles_x) out[y * tiles_x + x] = (uint32_t)v;
            carry = __shfl_sync(kFullMask, v, 31);
        }
    }
}

// B: per tile, the exclusive prefix of its counts over the chunks (in place) and its total; a
// block takes 32 tiles (lanes) and its 16 warps split the chunks into segments.  The last block to
// finish (the completion counter BinState::tile_blocks_done, reset by frame_init) turns the totals into the
// tile starts (exclusive scan, in place), the tile ranges and the pair count.
__global__ void __launch_bounds__(kOffThreads) k_tile_offsets(uint32_t* counts, BinState* st, int chunk, int n_tiles,
                                                              uint32_t* totals_starts, uint2* ranges) {
    constexpr int kW = kOffThreads / 32;
    __shared__ uint32_t seg[kW][32];
    __shared__ bool s_last;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int t = blockIdx.x * 32 + lane;
    const int nch = (st->n_valid + chunk - 1) / chunk;
    const int per = (nch + kW - 1) / kW;
    const int c0 = min(w * per, nch), c1 = min(c0 + per, nch);
    uint32_t s = 0;
    if (t < n_tiles) {
#pragma unroll 8
        for (int c = c0; c < c1; ++c) s += counts[(size_t)c * n_tiles + t];
    }
    seg[w][lane] = s;
    __syncthreads();
    if (w == 0) {
        uint32_t tot = 0;
#pragma unroll
        for (int k = 0; k < kW; ++k) {
            const uint32_t v = seg[k][lane];
            seg[k][lane] = tot;
            tot += v;
        }
        if (t < n_tiles) totals_starts[t] = tot;
    }
    __syncthreads();
    if (t < n_tiles) {
        uint32_t run = seg[w][lane];
#pragma unroll 8
        for (int c = c0; c < c1; ++c) {
            const size_t e = (size_t)c * n_tiles + t;
            const uint32_t v = counts[e];
            counts[e] = run;
            run += v;
        }
    }
    // last block: tile starts
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&st->tile_blocks_done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    constexpr int kItems = kScatterMaxTiles / kOffThreads;
    volatile const uint32_t* tv = totals_starts;
    uint32_t v[kItems];
    uint32_t sum = 0;
    const int base = threadIdx.x * kItems;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        v[k] = base + k < n_tiles ? tv[base + k] : 0u;
        sum += v[k];
    }
    uint32_t total;
    uint32_t run = block_exclusive_scan(sum, &total);
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        if (base + k < n_tiles) {
            totals_starts[base + k] = run;
            ranges[base + k] = make_uint2(run, run + v[k]);
        }
        run += v[k];
    }
    if (threadIdx.x == 0) st->n_pairs = total;
}

// Lane masks of one round: col[x] = lanes whose rectangle spans column x, row[y] likewise.  Begin
// marks go into col / row directly, end marks (x1 + 1) into the warp's scratch, then an inclusive
// prefix-OR of both along the axis: covered = begun & ~ended.
__device__ __forceinline__ void scatter_axis_masks(uint32_t* m, uint32_t* f, int n, int lo, int hi, bool valid,
                                                   int lane) {
    for (int e = lane; e <= n; e += 32) {
        if (e < n) m[e] = 0;
        f[e] = 0;
    }
    __syncwarp();
    if (valid) {
        atomicOr(&m[lo], 1u << lane);
        atomicOr(&f[hi + 1], 1u << lane);
    }
    __syncwarp();
    uint32_t cb = 0, cf = 0;
    for (int x0 = 0; x0 < n; x0 += 32) {
        const int x = x0 + lane;
        uint32_t b = x < n ? m[x] : 0u, e = x < n ? f[x] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t ub = __shfl_up_sync(kFullMask, b, o), ue = __shfl_up_sync(kFullMask, e, o);
            if (lane >= o) {
                b |= ub;
                e |= ue;
            }
        }
        b |= cb;
        e |= cf;
        if (x < n) m[x] = b & ~e;
        cb = __shfl_sync(kFullMask, b, 31);
        cf = __shfl_sync(kFullMask, e, 31);
    }
    __syncwarp();
}

__global__ void __launch_bounds__(kScatThreads) k_tile_scatter(const uint32_t* __restrict__ sorted_ids,
                                                               const uint32_t* __restrict__ sorted_tiles,
                                                               const ushort4* __restrict__ rect,
                                                               BinState* st, int rounds,
                                                               int tiles_x, int tiles_y,
                                                               const uint32_t* __restrict__ base,
                                                               const uint32_t* __restrict__ starts, uint2* ranges,
                                                               uint32_t* vals) {
    extern __shared__ uint32_t s_scat[];
    const int n_tiles = tiles_x * tiles_y;
    const int chunk = 32 * rounds;
    uint32_t* run = s_scat;                                     // n_tiles running positions
    uint32_t* s_id = run + ((n_tiles + 1) & ~1);               // chunk splat ids
    ushort4* s_rect = reinterpret_cast<ushort4*>(s_id + chunk);  // chunk rectangles (x1 < x0: none)
    uint32_t* s_col = reinterpret_cast<uint32_t*>(s_rect + chunk);  // kScatWarps slots x 256
    uint32_t* s_row = s_col + kScatWarps * 256;                     // kScatWarps slots x 256
    uint32_t* s_end = s_row + kScatWarps * 256;                     // per warp 2 x 257 end marks
    if (st->overflow || st->n_pairs > kRunMask) {
        // the view is re-rendered (beyond 2^26 pairs: by the radix passes): no tile ranges into
        // the unwritten pairs
        if (blockIdx.x == 0 && threadIdx.x == 0) st->overflow = 1;
        for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n_tiles; e += gridDim.x * blockDim.x)
            ranges[e] = make_uint2(0, 0);
        return;
    }
    const int nv = st->n_valid;
    const int r0 = blockIdx.x * chunk;
    if (r0 >= nv) return;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    // running positions: tile start + the chunk's prefix; stamp 63 (no round yet)
    const uint32_t* b = base + (size_t)blockIdx.x * n_tiles;
    if ((n_tiles & 3) == 0) {
        const uint4* b4 = reinterpret_cast<const uint4*>(b);
        const uint4* s4 = reinterpret_cast<const uint4*>(starts);
        uint4* r4 = reinterpret_cast<uint4*>(run);
        for (int e = threadIdx.x; e < (n_tiles >> 2); e += kScatThreads) {
            const uint4 x = b4[e], y = s4[e];
            r4[e] = make_uint4((63u << 26) | (x.x + y.x), (63u << 26) | (x.y + y.y), (63u << 26) | (x.z + y.z),
                               (63u << 26) | (x.w + y.w));
        }
    } else {
        for (int e = threadIdx.x; e < n_tiles; e += kScatThreads) run[e] = (63u << 26) | (b[e] + starts[e]);
    }
    const int n_here = min(chunk, nv - r0);
    const int nr = (n_here + 31) >> 5;
    for (int i = threadIdx.x; i < nr * 32; i += kScatThreads) {
        const int r = r0 + i;
        ushort4 q = make_ushort4(1, 0, 0, 0);
        uint32_t id = 0;
        if (i < n_here && sorted_tiles[r]) {
            id = sorted_ids[r];
            q = rect[id];
        }
        s_id[i] = id;
        s_rect[i] = q;
    }
    __syncthreads();
    uint32_t* endx = s_end + w * 514;
    uint32_t* endy = endx + 257;
    for (int g = 0; g < nr; g += kScatWarps) {
        // warp w builds the masks of round g + w into slot w
        if (g + w < nr) {
            const ushort4 q = s_rect[(g + w) * 32 + lane];
            const bool valid = q.x <= q.y;
            scatter_axis_masks(s_col + w * 256, endx, tiles_x, q.x, q.y, valid, lane);
            scatter_axis_masks(s_row + w * 256, endy, tiles_y, q.z, q.w, valid, lane);
        }
        __syncthreads();
        const int kr = min(kScatWarps, nr - g);
        for (int k = 0; k < kr; ++k) {
            const int i = (g + k) * 32 + lane;
            const ushort4 q = s_rect[i];
            const bool valid = q.x <= q.y;
            // rows of this warp's band inside the rectangle: y = first, first + 4, ... <= y1
            const int first = q.z + ((w - q.z) & (kScatWarps - 1));
            const int nb = valid && first <= q.w ? ((q.w - first) >> 2) + 1 : 0;
            const int wd = q.y - q.x + 1;
            const uint32_t cnt = nb ? (uint32_t)(wd * nb) : 0u;
            uint32_t incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t u = __shfl_up_sync(kFullMask, incl, o);
                if (lane >= o) incl += u;
            }
            const uint32_t total = __shfl_sync(kFullMask, incl, 31);
            const uint32_t excl = incl - cnt;
            if (total == 0) continue;
            const uint32_t nonempty = __ballot_sync(kFullMask, cnt != 0);  // rectangles with band rows
            const uint32_t* cm = s_col + k * 256;
            const uint32_t* rm = s_row + k * 256;
            const int ri = g + k;  // round index inside the chunk: the running positions' stamp
            // Lane L takes the contiguous pairs [L per, (L + 1) per) of the round and walks them:
            // one owner search and one division per lane, then column / band-row / owner steps.
            const uint32_t per = (total + 31) >> 5;
            uint32_t kk = lane * per;
            int o = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const uint32_t v = __shfl_sync(kFullMask, incl, o + step - 1);
                if (v <= kk) o += step;
            }
            const uint32_t o_excl = __shfl_sync(kFullMask, excl, o & 31);
            int tx = 0, ty = 0, x0 = 0, x1 = -1, y1 = -1;
            uint32_t id = 0;
            if (kk < total) {
                const ushort4 oq = s_rect[(g + k) * 32 + o];
                const int ofirst = oq.z + ((w - oq.z) & (kScatWarps - 1));
                const int owd = oq.y - oq.x + 1;
                const int m = (int)(kk - o_excl);
                // m / owd: m < 2^14, owd <= 256 -- (m + 0.5) / owd is >= 0.5 / owd from an integer
                const int dy = (int)__fdividef((float)m + 0.5f, (float)owd);
                x0 = oq.x;
                x1 = oq.y;
                y1 = oq.w;
                tx = x0 + (m - dy * owd);
                ty = ofirst + kScatWarps * dy;
                id = s_id[(g + k) * 32 + o];
            }
            for (uint32_t j = 0; j < per; ++j, ++kk) {
                if (kk >= total) break;
                const int t = ty * tiles_x + tx;
                const uint32_t mask = cm[tx] & rm[ty];
                const uint32_t c = __popc(mask);
                // run[t] = stamp << 26 | position; stamped with this round, it already includes
                // the round's pairs of tile t (its last rectangle has been processed).  Lanes of
                // the warp read it while the round's last rectangle over t may be updating it:
                // both sides are shared-memory atomics (a read-only atomicOr, an atomicExch).
                const uint32_t v = atomicOr(&run[t], 0u);
                const uint32_t p0 = (v & kRunMask) - ((int)(v >> 26) == ri ? c : 0u);
                vals[p0 + __popc(mask & ((1u << o) - 1u))] = id;
                if (!(mask & ~((2u << o) - 1u))) atomicExch(&run[t], ((uint32_t)ri << 26) | (p0 + c));
                // next pair: next column, next band row, next rectangle with rows in the band
                if (++tx > x1) {
                    tx = x0;
                    ty += kScatWarps;
                    if (ty > y1) {
                        const uint32_t later = nonempty & ~((2u << o) - 1u);
                        if (later) {
                            o = __ffs(later) - 1;
                            const ushort4 oq = s_rect[(g + k) * 32 + o];
                            x0 = tx = oq.x;
                            x1 = oq.y;
                            ty = oq.z + ((w - oq.z) & (kScatWarps - 1));
                            y1 = oq.w;
                            id = s_id[(g + k) * 32 + o];
                        }
                    }
                }
            }
            __syncwarp();  // the round's running positions, before the next round reads them
        }
        __syncthreads();
    }
}

// RGS_FLAG_DEFER_CHECKS: the view's rotor error / pair-buffer overflow into the context's
// deferred status word (min wins: the lowest failing index, as the synchronous check).
__global__ void k_fold_status(const BinState* st, unsigned long long* word, unsigned long long overflow_word) {
    if (st->err != kNoError) atomicMin(word, st->err);
    if (st->overflow) atomicMin(word, overflow_word);
}

// Per-view reset of the binning state in one launch (instead of a pageable H2D copy of the
// initial BinState and two memsets): counters, depth-key range, capacity, bucket arrays.
__global__ void k_frame_init(BinState* st, uint32_t pair_cap, uint32_t* bucket_count, uint32_t* bucket_cur, int nb) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) {
        BinState z;
        z.err = kNoError;
        z.key_min = ~0ull;
        z.key_max = 0;
        z.n_valid = 0;
        z.slow_count = 0;
        z.shift = 0;
        z.n_big = 0;
        z.n_pairs = 0;
        z.pair_cap = pair_cap;
        z.n_pairs_eff = 0;
        z.overflow = 0;
        z.tile_blocks_done = z.pad3 = 0;
        *st = z;
    }
    if (i < nb) {
        bucket_count[i] = 0;
        bucket_cur[i] = 0;
    }
}

// Pair total vs buffer capacity: an overflowing view does no pair work and is re-rendered.
__global__ void k_check_capacity(BinState* st) {
    const bool over = st->n_pairs > st->pair_cap;
    st->overflow = over ? 1u : 0u;
    st->n_pairs_eff = over ? 0u : st->n_pairs;
}

// Per-tile [start, end) from the sorted keys: grid-stride, four keys per thread (one 16-byte
// load) compared with their neighbours; sized by the device-side pair count.
__global__ void __launch_bounds__(256) k_tile_ranges(const uint32_t* __restrict__ keys, const BinState* __restrict__ st,
                                                     int tiles_x, int ty_shift, uint2* ranges) {
    const uint32_t n = st->n_pairs_eff;
    constexpr uint32_t kNone = 0xffffffffu;  // never a tile key (ty, tx < 2^12)
    const uint32_t tx_mask = (1u << ty_shift) - 1u;
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; 4 * q < n; q += gridDim.x * blockDim.x) {
        const uint32_t i0 = 4 * q;
        uint32_t k[6];
        k[0] = i0 > 0 ? keys[i0 - 1] : kNone;
        if (i0 + 4 <= n) {
            const uint4 v = *reinterpret_cast<const uint4*>(keys + i0);
            k[1] = v.x;
            k[2] = v.y;
            k[3] = v.z;
            k[4] = v.w;
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) k[1 + j] = i0 + j < n ? keys[i0 + j] : kNone;
        }
        k[5] = i0 + 4 < n ? keys[i0 + 4] : kNone;
#pragma unroll
        for (int j = 1; j <= 4; ++j) {
            if (k[j] == kNone) break;
            const uint32_t t = (k[j] >> ty_shift) * (uint32_t)tiles_x + (k[j] & tx_mask);
            const uint32_t i = i0 + j - 1;
            if (k[j - 1] != k[j]) ranges[t].x = i;
            if (k[j + 1] != k[j]) ranges[t].y = i + 1;
        }
    }
}

}  // namespace rgs_dev

// ---------------------------------------------------------------------------
namespace rgs_launch {
using namespace rgs_dev;

static inline int blocks(long long n, int t) { return (int)((n + t - 1) / t); }

int num_depth_buckets() { return kNumBuckets; }
int depth_bucket_bits(int n) {
    int b = 0;
    while (b < 31 && (1ll << b) < (long long)std::max(n, 1)) ++b;
    return std::min(kBucketBits, std::max(12, b - 3));
}

// Single-pass variant; scratch: scan1_scratch_words(n) u32 (status words + ticket).
size_t scan1_scratch_words(int n) { return 2 * (size_t)(blocks(std::max(n, 1), kScan1Tile) + 1) + 4; }
void exclusive_scan_1p(const uint32_t* in, int n, uint32_t* out, uint32_t* scratch, uint32_t* total, cudaStream_t s,
                       const int* n_dev) {
    const int nb = blocks(std::max(n, 1), kScan1Tile);
    unsigned long long* status = reinterpret_cast<unsigned long long*>(scratch);
    uint32_t* ticket = scratch + 2 * (size_t)nb;
    cudaMemsetAsync(scratch, 0, 4 * (2 * (size_t)nb + 1), s);
    k_scan_1p<<<nb, kScanThreads, 0, s>>>(in, n, n_dev, out, total, status, ticket);
}

void exclusive_scan(const uint32_t* in, int n, uint32_t* out, uint32_t* scratch, uint32_t* total, cudaStream_t s,
                    const int* n_dev) {
    const int nb = blocks(n, kScanTile);
    if (nb <= 0) return;
    k_scan_sums<<<nb, kScanThreads, 0, s>>>(in, n, n_dev, scratch);
    k_scan_block_sums<<<1, kScanThreads, 0, s>>>(scratch, nb, total);
    k_scan_apply<<<nb, kScanThreads, 0, s>>>(in, n, n_dev, scratch, out);
}

void bucket_hist(const uint8_t* valid, const unsigned long long* key, int n, BinState* st, uint32_t* bucket_count,
                 cudaStream_t s) {
    k_bucket_setup<<<1, 1, 0, s>>>(st, depth_bucket_bits(n));
    if (n > 0) k_bucket_hist<<<blocks(n, 256), 256, 0, s>>>(valid, key, n, st, bucket_count);
}

void depth_ranks(const uint8_t* valid, const unsigned long long* key, const uint32_t* tiles, int n,
                 const int32_t* src, BinState* st, const uint32_t* bucket_count, const uint32_t* bucket_off,
                 uint32_t* bucket_cur, unsigned long long* ent_key, uint32_t* ent_id, uint32_t* sorted_ids,
                 uint32_t* sorted_tiles, uint32_t* big_list, void* big_scratch, cudaStream_t s) {
    if (n <= 0) return;
    k_bucket_scatter<<<blocks(n, 256), 256, 0, s>>>(valid, key, n, st, bucket_off, bucket_cur, ent_key, ent_id);
    k_bucket_sort_small<<<blocks(n, 256), 256, 0, s>>>(bucket_count, bucket_off, ent_key, ent_id, src, tiles,
                                                        sorted_ids, sorted_tiles, st, big_list);
    k_bucket_sort_big<<<148, 512, kBigSmem * sizeof(SortRec), s>>>(bucket_count, bucket_off, ent_key, ent_id, src,
                                                                   tiles, st, big_list, sorted_ids, sorted_tiles,
                                                                   reinterpret_cast<SortRec*>(big_scratch));
}

// Tile key layout: ty << 8 | tx (two byte passes) up to 256 x 256 tiles, else ty << 12 | tx
// (three byte passes, up to 4096 x 4096 tiles).
int tile_key_shift(int tiles_x, int tiles_y) { return (tiles_x <= 256 && tiles_y <= 256) ? 8 : 12; }

void duplicate(const uint32_t* sorted_ids, const uint32_t* pair_off, const uint32_t* sorted_tiles,
               const ushort4* rect, const BinState* st, int n, int tiles_x, int tiles_y, uint32_t* keys,
               uint32_t* vals, int* aux, cudaStream_t s) {
    cudaMemsetAsync(aux, 0, sizeof(int) * kAuxInts, s);
    if (n > 0)
        k_duplicate<<<blocks(n, 256), 256, 0, s>>>(sorted_ids, pair_off, sorted_tiles, rect, st,
                                                    tile_key_shift(tiles_x, tiles_y), keys, vals, aux);
}

int radix_blocks(long long n_pairs) { return std::max(blocks(n_pairs, kMinBlockTile), 1); }
static int radix_grid(long long n_pairs) {
    return std::max(blocks(n_pairs, kRadixThreads * g_radix_rounds), 1);
}
static int g_radix_ballot = 0;
static int digit_bits(int n) {  // significant bits of the values 0 .. n - 1 (at least 1)
    int b = 1;
    while (b < 8 && (1 << b) < n) ++b;
    return b;
}
template <typename... A>
static void radix_pass(int nb, cudaStream_t s, A... a) {
    if (g_radix_rounds == 8) k_radix_onesweep<8, 4><<<nb, kRadixThreads, 0, s>>>(a...);
    else k_radix_onesweep<16, 3><<<nb, kRadixThreads, 0, s>>>(a...);
}
size_t radix_count_entries(long long n_pairs) { return (size_t)kRadixDigits * radix_blocks(n_pairs); }

// Two stable byte passes (tx, then ty) on ty << 8 | tx; the sorted pairs end back in (keys_a,
// vals_a).  Wide keys (ty << 12 | tx): three byte passes, ending in (keys_b, vals_b) -- returned.
// aux: [0, 514) the digit-histogram difference arrays k_duplicate filled (wide keys: [0, 768) the
// plain histograms of k_digit_hist3), [780, 783) tickets; status_a / status_b:
// radix_count_entries() u32 each (decoupled look-back state).
int tile_radix_sort(uint32_t* keys_a, uint32_t* vals_a, uint32_t* keys_b, uint32_t* vals_b, const BinState* st,
                    long long n_pairs, int tiles_x, int tiles_y, uint32_t* status_a, uint32_t* status_b, int* aux,
                    uint2* ranges, cudaStream_t s) {
    const int nb = radix_grid(n_pairs);
    const size_t entries = (size_t)kRadixDigits * nb;
    const int n_tiles = tiles_x * tiles_y;
    const int shift = tile_key_shift(tiles_x, tiles_y);
    uint32_t* tickets = reinterpret_cast<uint32_t*>(aux + 780);
    int out = 0;
    cudaMemsetAsync(status_a, 0, 4 * entries, s);
    cudaMemsetAsync(status_b, 0, 4 * entries, s);
    if (shift == 8) {
        radix_pass(nb, s, keys_a, vals_a, st, 0, aux, 0, status_a, tickets, keys_b,
                                                       vals_b, g_radix_ballot ? digit_bits(tiles_x) : 0);
        radix_pass(nb, s, keys_b, vals_b, st, 8, aux + 257, 0, status_b, tickets + 1,
                                                       keys_a, vals_a, g_radix_ballot ? digit_bits(tiles_y) : 0);
    } else {
        k_digit_hist3<<<148 * 2, 256, 0, s>>>(keys_a, st, aux);
        radix_pass(nb, s, keys_a, vals_a, st, 0, aux, 1, status_a, tickets, keys_b,
                                                       vals_b, g_radix_ballot ? 8 : 0);
        radix_pass(nb, s, keys_b, vals_b, st, 8, aux + 256, 1, status_b, tickets + 1,
                                                       keys_a, vals_a, g_radix_ballot ? 8 : 0);
        cudaMemsetAsync(status_a, 0, 4 * entries, s);
        radix_pass(nb, s, keys_a, vals_a, st, 16, aux + 512, 1, status_a, tickets + 2,
                                                       keys_b, vals_b, g_radix_ballot ? 8 : 0);
        out = 1;
    }
    cudaMemsetAsync(ranges, 0, sizeof(uint2) * (size_t)n_tiles, s);
    k_tile_ranges<<<std::max(std::min(blocks(n_pairs, 4 * 256), 148 * 8), 1), 256, 0, s>>>(
        out ? keys_b : keys_a, st, tiles_x, shift, ranges);
    return out;
}

void check_capacity(BinState* st, cudaStream_t s) { k_check_capacity<<<1, 1, 0, s>>>(st); }

void fold_status(const BinState* st, unsigned long long* word, unsigned long long overflow_word, cudaStream_t s) {
    k_fold_status<<<1, 1, 0, s>>>(st, word, overflow_word);
}

void frame_init(BinState* st, uint32_t pair_cap, uint32_t* bucket_count, uint32_t* bucket_cur, int n,
                cudaStream_t s) {
    const int nb = 1 << depth_bucket_bits(n);
    k_frame_init<<<blocks(nb, 256), 256, 0, s>>>(st, pair_cap, bucket_count, bucket_cur, nb);
}

// ---- tile-major scatter (k_chunk_tile_counts, k_tile_offsets, k_tile_scatter)
static int scatter_chunk() { return 32 * g_scatter_rounds; }
static size_t scatter_smem(int n_tiles) {
    const int chunk = scatter_chunk();
    return 4 * ((size_t)((n_tiles + 1) & ~1) + chunk + 2 * (size_t)chunk + 2 * kScatWarps * 256 + kScatWarps * 514);
}
size_t tile_count_words(int n, int n_tiles) {
    return (size_t)blocks(std::max(n, 1), scatter_chunk()) * (size_t)std::max(n_tiles, 1);
}
int default_binning_mode() { return g_binning_mode; }
bool tile_scatter_usable(int tiles_x, int tiles_y, int n, long long pair_cap, bool batch, int mode) {
    if (mode == 1 || (batch && mode == 0)) return false;
    // AUTO keeps the scatter while its chunk x tile count matrix is small: C3 (200K, 800x800: 1M
    // words) -- 396 vs 390 it/s against the radix passes; C5 (1M, 1352x1014: 10.6M words, the
    // per-tile offset scan over 1953 chunks) -- 18.6 vs 18.1 ms per step
    const size_t words = tile_count_words(n, tiles_x * tiles_y);
    if (mode == 0 && words > ((size_t)1 << 22)) return false;
    return pair_cap <= (long long)kRunMask && tiles_x <= 256 && tiles_y <= 256 && tiles_x * tiles_y <= kScatterMaxTiles &&
           words <= ((size_t)1 << 26);
}

void tile_counts(const uint32_t* sorted_ids, const uint32_t* sorted_tiles, const ushort4* rect, BinState* st, int n,
                 int tiles_x, int tiles_y, uint32_t* counts, uint32_t* starts, uint2* ranges, cudaStream_t s) {
    const int chunk = scatter_chunk();
    const int n_tiles = tiles_x * tiles_y;
    k_chunk_tile_counts<<<blocks(std::max(n, 1), chunk), 256, 4 * (size_t)tiles_y * (tiles_x + 1), s>>>(
        sorted_ids, sorted_tiles, rect, st, chunk, tiles_x, tiles_y, counts);
    k_tile_offsets<<<blocks(n_tiles, 32), kOffThreads, 0, s>>>(counts, st, chunk, n_tiles, starts, ranges);
}

void tile_scatter(const uint32_t* sorted_ids, const uint32_t* sorted_tiles, const ushort4* rect, BinState* st,
                  int n, int tiles_x, int tiles_y, const uint32_t* counts, const uint32_t* starts, uint2* ranges,
                  uint32_t* vals, cudaStream_t s) {
    k_tile_scatter<<<blocks(std::max(n, 1), scatter_chunk()), kScatThreads, scatter_smem(tiles_x * tiles_y), s>>>(
        sorted_ids, sorted_tiles, rect, st, g_scatter_rounds, tiles_x, tiles_y, counts, starts, ranges, vals);
}

bool binning_init() {
    const char* v = std::getenv("RGS_RADIX");
    g_radix_rounds = (v && v[0] == '8') ? 8 : 16;
    // RGS_RADIX_BALLOT=1: digit peers by ballots over the significant digit bits instead of
    // __match_any_sync -- measured slower (C2 radix passes 0.125 vs 0.094 ms)
    const char* m = std::getenv("RGS_RADIX_BALLOT");
    g_radix_ballot = (m && m[0] == '1') ? 1 : 0;
    const char* b = std::getenv("RGS_BINNING");
    g_binning_mode = !b ? 0 : (b[0] == 'r' ? 1 : (b[0] == 's' ? 2 : 0));
    const char* r = std::getenv("RGS_SCATTER_ROUNDS");
    if (r) {
        const int k = std::atoi(r);
        if (k == 8 || k == 16 || k == 32) g_scatter_rounds = k;
    }
    return cudaFuncSetAttribute(k_bucket_sort_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kBigSmem * (int)sizeof(SortRec)) == cudaSuccess &&
           cudaFuncSetAttribute(k_tile_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)scatter_smem(kScatterMaxTiles)) == cudaSuccess;
}

}  // namespace rgs_launch
