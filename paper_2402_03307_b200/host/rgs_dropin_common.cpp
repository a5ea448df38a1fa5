// Shared state and helpers of the C++ drop-ins (rgs_dropin_common.hpp).
#include "rgs_dropin_common.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <malloc.h>
#include <mutex>
#include <stdexcept>
#include <thread>
#include <vector>

namespace rgs {
namespace dropin {

rgs_ctx* context() {
    static rgs_ctx* c = [] {
        // The reference API hands ~100 MB per-Gaussian structs (StoreGrads, RenderRecords) across
        // every call; above glibc's mmap threshold each one is a fresh mmap whose pages fault and
        // zero on first touch.  Serve them from the heap instead, so freed blocks are reused
        // (RGS_DROPIN_NO_MALLOPT=1 leaves the process's malloc settings alone).
        if (!std::getenv("RGS_DROPIN_NO_MALLOPT")) {
            mallopt(M_MMAP_THRESHOLD, 1 << 30);
            mallopt(M_TRIM_THRESHOLD, 1 << 30);
        }
        rgs_ctx* h = nullptr;
        const char* dev = std::getenv("RGS_DEVICE");
        if (rgs_ctx_create(dev ? std::atoi(dev) : 0, &h) != RGS_OK)
            throw std::runtime_error("rgs_b200: no CUDA device (the B200 path has no CPU fallback)");
        return h;
    }();
    return c;
}

namespace {

uint64_t hash_chunk(const unsigned char* b, size_t bytes, uint64_t h) {
    const size_t nw = bytes / 8;
    uint64_t l[4] = {h ^ 0x9e3779b97f4a7c15ull, h + 0xc2b2ae3d27d4eb4full, h * 31 + 1, ~h};
    size_t i = 0;
    for (; i + 4 <= nw; i += 4) {
        for (int k = 0; k < 4; ++k) {
            uint64_t w;
            std::memcpy(&w, b + 8 * (i + k), 8);
            l[k] = (l[k] ^ w) * 0x100000001b3ull;
            l[k] = (l[k] << 29) | (l[k] >> 35);
        }
    }
    for (; i < nw; ++i) {
        uint64_t w;
        std::memcpy(&w, b + 8 * i, 8);
        l[0] = (l[0] ^ w) * 0x100000001b3ull;
        l[0] = (l[0] << 29) | (l[0] >> 35);
    }
    for (size_t j = 8 * nw; j < bytes; ++j) l[1] = (l[1] ^ b[j]) * 0x100000001b3ull;
    return (l[0] * 3 + l[1]) * 0x9e3779b97f4a7c15ull ^ (l[2] * 5 + l[3]);
}

}  // namespace

uint64_t hash_bytes(const void* p, size_t bytes, uint64_t seed) {
    // fixed 4 MiB chunks (the value does not depend on the thread count), hashed in parallel
    constexpr size_t kChunk = size_t(4) << 20;
    const unsigned char* b = static_cast<const unsigned char*>(p);
    const size_t nc = (bytes + kChunk - 1) / kChunk;
    if (nc <= 1) return hash_chunk(b, bytes, seed);
    std::vector<uint64_t> hs(nc);
    const unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), (unsigned)nc));
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < nt; ++t)
        pool.emplace_back([&, t] {
            for (size_t c = t; c < nc; c += nt)
                hs[c] = hash_chunk(b + c * kChunk, std::min(kChunk, bytes - c * kChunk), seed + c);
        });
    for (auto& th : pool) th.join();
    return hash_chunk(reinterpret_cast<const unsigned char*>(hs.data()), 8 * nc, seed ^ bytes);
}

uint64_t params_hash(const GaussianStore& st) {
    uint64_t h = 0x5bd1e995u ^ (uint64_t)st.size() ^ ((uint64_t)st.active_sh_degree << 40);
    h = hash_vec(st.mean, h);
    h = hash_vec(st.log_scales, h);
    h = hash_vec(st.rotor, h);
    h = hash_vec(st.opacity_logit, h);
    return hash_vec(st.sh, h);
}

uint64_t moments_hash(const GaussianStore& st) {
    uint64_t h = 0x27d4eb2f ^ (uint64_t)st.size();
    for (const auto* v : {&st.m_mean, &st.v_mean, &st.m_ls, &st.v_ls}) h = hash_vec(*v, h);
    h = hash_vec(st.m_rot, h);
    h = hash_vec(st.v_rot, h);
    h = hash_vec(st.m_op, h);
    h = hash_vec(st.v_op, h);
    h = hash_vec(st.m_sh, h);
    return hash_vec(st.v_sh, h);
}

uint64_t stats_hash(const GaussianStore& st) {
    return hash_vec(st.grad_count, hash_vec(st.grad_accum, 0x165667b1 ^ (uint64_t)st.size()));
}

namespace {
struct Pool {
    std::mutex m;
    std::vector<std::pair<size_t, void*>> free;
    std::vector<std::pair<void*, size_t>> sizes;
};
Pool& pool() {
    static Pool p;
    return p;
}
}  // namespace

void* pool_get(size_t bytes) {
    bytes = std::max<size_t>(bytes, 256);
    Pool& p = pool();
    {
        std::lock_guard<std::mutex> g(p.m);
        size_t best = (size_t)-1;
        for (size_t i = 0; i < p.free.size(); ++i)
            if (p.free[i].first >= bytes && (best == (size_t)-1 || p.free[i].first < p.free[best].first)) best = i;
        if (best != (size_t)-1) {
            void* q = p.free[best].second;
            p.free.erase(p.free.begin() + best);
            return q;
        }
    }
    void* q = rgs_malloc(context(), bytes);
    if (!q) throw std::runtime_error("rgs_b200: out of device memory");
    std::lock_guard<std::mutex> g(p.m);
    p.sizes.push_back({q, bytes});
    return q;
}

void pool_put(void* q) {
    if (!q) return;
    Pool& p = pool();
    std::lock_guard<std::mutex> g(p.m);
    for (const auto& e : p.sizes)
        if (e.first == q) {
            p.free.push_back({e.second, q});
            return;
        }
}

namespace {
struct Published {
    uint64_t hash = 0;
    int n = -1, sh = -1;
    const double* params = nullptr;
};
Published& published() {
    static Published p;
    return p;
}
}  // namespace

void publish_params(uint64_t h, int n, int sh_degree, const double* dev_params64) {
    published() = Published{h, n, sh_degree, dev_params64};
}

const double* published_params(uint64_t h, int n, int sh_degree) {
    const Published& p = published();
    return (p.params && p.hash == h && p.n == n && p.sh == sh_degree) ? p.params : nullptr;
}

}  // namespace dropin
}  // namespace rgs
