// Shared by the two C++ drop-ins (rgs_adapter.cpp: rasterizer.hpp; rgs_train_adapter.cpp: image /
// ssim / loss / knn / optim): one CUDA context, content hashes of host stores, pooled device
// buffers, and the device copy of the store the training side last wrote (so the next render
// copies it device to device instead of uploading the host store again).
#pragma once

#include <cstddef>
#include <cstdint>

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
