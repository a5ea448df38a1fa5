// Shared by the two C++ drop-ins (rgs_adapter.cpp: rasterizer.hpp; rgs_train_adapter.cpp: image /
// ssim / loss / knn / optim): one CUDA context, content hashes of host stores, pooled device
// buffers, and the device copy of the store the training side last wrote (so the next render
// copies it device to device instead of uploading the host store again).
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <thread>
#include <vector>

#include "rgs/gaussian.hpp"
#include "rgs_cuda.h"

namespace rgs {
namespace dropin {

// The drop-ins' context (RGS_DEVICE selects the device, default 0); throws without a device.
rgs_ctx* context();

// 64-bit hash of a byte range, computed in parallel chunks (deterministic for any thread count).
uint64_t hash_bytes(const void* p, size_t bytes, uint64_t seed);

template <typename V>
uint64_t hash_vec(const V& v, uint64_t seed) {
    return hash_bytes(v.data(), v.size() * sizeof(typename V::value_type), seed);
}

// f(begin, end) over [0, n) split into contiguous ranges on up to hardware_concurrency threads
// (the host-side layout conversions between the reference's per-Gaussian structs and the
// device SoA; every index is written by exactly one range, so the result is thread-count free).
template <typename F>
void parallel_for(size_t n, F&& f) {
    const size_t kMinPerThread = 4096;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t nt = std::min<size_t>({(size_t)hw, (n + kMinPerThread - 1) / kMinPerThread, 32});
    if (nt <= 1) {
        f(size_t(0), n);
        return;
    }
    std::vector<std::thread> pool;
    pool.reserve(nt - 1);
    const size_t per = (n + nt - 1) / nt;
    for (size_t t = 1; t < nt; ++t) {
        const size_t b = t * per, e = std::min(n, b + per);
        if (b < e) pool.emplace_back([&f, b, e] { f(b, e); });
    }
    f(size_t(0), std::min(n, per));
    for (auto& th : pool) th.join();
}

// Grow-only host scratch vectors, reused across calls (per element type and slot): their pages
// stay mapped, so the 50-100 MB layout conversions of a large store pay no page faults or zero
// fills per call.  Returns a vector of at least n elements (contents unspecified).
template <typename T>
std::vector<T>& scratch(int slot, size_t n) {
    static thread_local std::vector<T> bufs[8];
    std::vector<T>& v = bufs[slot];
    if (v.size() < n) v.resize(n);
    return v;
}

// The parameters a render reads (gaussian.hpp:79-85) and the SH degree.
uint64_t params_hash(const GaussianStore& s);
// Adam moments and densification statistics (gaussian.hpp:87-95).
uint64_t moments_hash(const GaussianStore& s);
uint64_t stats_hash(const GaussianStore& s);

// Grow-only device buffers recycled between calls (no cudaMalloc / cudaFree per call).
void* pool_get(size_t bytes);
void pool_put(void* p);

// The FP64 device parameters the training side last wrote (rgs_scene_params_f64 of its
// scene), published under params_hash of the host store it downloaded them into.
void publish_params(uint64_t params_hash, int n, int sh_degree, const double* dev_params64);
const double* published_params(uint64_t params_hash, int n, int sh_degree);

}  // namespace dropin
}  // namespace rgs
