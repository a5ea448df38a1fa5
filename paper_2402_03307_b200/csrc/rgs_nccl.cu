// Multi-GPU batch reduction over NCCL (trainer.cpp:33-53 + StoreGrads::add,
// gaussian.cpp:199-209, across ranks): the C-ABI entry points of include/rgs_cuda.h
// "multi-GPU".  NCCL is resolved at run time from the process (the caller's libnccl, e.g. the
// one torch loaded, so a communicator made by the caller can be passed in) or else from
// libnccl.so.2; the library has no link dependency on it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "../../include/rgs_cuda.h"

namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
};

template <typename F>
bool resolve(void* h, const char* name, F& f) {
    f = reinterpret_cast<F>(dlsym(h, name));
    return f != nullptr;
}

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* handles[2] = {RTLD_DEFAULT, nullptr};
        for (int k = 0; k < 2 && !api.ok; ++k) {
            void* h = handles[k];
            if (k == 1) {
                h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
                if (!h) {
                    api.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
                    break;
                }
            }
            api.ok = resolve(h, "ncclGetUniqueId", api.get_unique_id) &&
                     resolve(h, "ncclCommInitRank", api.comm_init_rank) &&
                     resolve(h, "ncclCommDestroy", api.comm_destroy) && resolve(h, "ncclAllReduce", api.all_reduce) &&
                     resolve(h, "ncclGroupStart", api.group_start) && resolve(h, "ncclGroupEnd", api.group_end) &&
                     resolve(h, "ncclGetErrorString", api.error_string);
        }
        if (!api.ok && api.why.empty()) api.why = "NCCL symbols not found";
    });
    return api;
}

}  // namespace

// The context's current stream (rgs_capi.cu).
extern "C" void* rgs_ctx_stream(rgs_ctx* c);
extern "C" const char* rgs_ctx_last_error(const rgs_ctx* c);
namespace rgs_host {
int set_ctx_error(rgs_ctx* c, int code, const char* msg);
}

extern "C" {

int rgs_nccl_available(void) { return nccl().ok ? 1 : 0; }

int rgs_nccl_unique_id(unsigned char* id128) {
    if (!id128) return RGS_E_INVALID;
    const NcclApi& a = nccl();
    if (!a.ok) return RGS_E_NO_DEVICE;
    ncclUniqueId id;
    if (a.get_unique_id(&id) != ncclSuccess) return RGS_E_CUDA;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id128, &id, sizeof id);
    return RGS_OK;
}

int rgs_nccl_comm_create(rgs_ctx* ctx, int nranks, int rank, const unsigned char* id128, void** comm) {
    if (!ctx || !id128 || !comm || nranks < 1 || rank < 0 || rank >= nranks) return RGS_E_INVALID;
    const NcclApi& a = nccl();
    if (!a.ok) return rgs_host::set_ctx_error(ctx, RGS_E_NO_DEVICE, a.why.c_str());
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    ncclComm_t c = nullptr;
    const ncclResult_t r = a.comm_init_rank(&c, nranks, id, rank);
    if (r != ncclSuccess) return rgs_host::set_ctx_error(ctx, RGS_E_CUDA, a.error_string(r));
    *comm = c;
    return RGS_OK;
}

void rgs_nccl_comm_destroy(void* comm) {
    if (comm && nccl().ok) nccl().comm_destroy(static_cast<ncclComm_t>(comm));
}

int rgs_allreduce_grads(rgs_ctx* ctx, void* comm, float* grads_vnorm, size_t n_floats, int32_t* visible,
                        size_t n_visible, double* losses, int n_losses) {
    if (!ctx || !comm || (n_floats && !grads_vnorm) || (n_visible && !visible) || (n_losses > 0 && !losses))
        return RGS_E_INVALID;
    const NcclApi& a = nccl();
    if (!a.ok) return rgs_host::set_ctx_error(ctx, RGS_E_NO_DEVICE, a.why.c_str());
    cudaStream_t s = static_cast<cudaStream_t>(rgs_ctx_stream(ctx));
    ncclComm_t c = static_cast<ncclComm_t>(comm);
    // One NCCL group: the three reductions go out as a single fused launch.
    ncclResult_t r = a.group_start();
    if (r == ncclSuccess && n_floats) r = a.all_reduce(grads_vnorm, grads_vnorm, n_floats, ncclFloat32, ncclSum, c, s);
    if (r == ncclSuccess && n_visible) r = a.all_reduce(visible, visible, n_visible, ncclInt32, ncclSum, c, s);
    if (r == ncclSuccess && n_losses > 0) r = a.all_reduce(losses, losses, (size_t)n_losses, ncclFloat64, ncclSum, c, s);
    const ncclResult_t e = a.group_end();
    if (r == ncclSuccess) r = e;
    if (r != ncclSuccess) return rgs_host::set_ctx_error(ctx, RGS_E_CUDA, a.error_string(r));
    return RGS_OK;
}

}  // extern "C"
