// NCCL, loaded at run time (dlopen) for the multi-GPU contexts of the library
// (SURVEY.md §8(b) {rank, world, ncclUniqueId}; §8(e) the one exchange step).
//
// The library does not link against NCCL: a single-GPU user needs no NCCL at all, and in
// a PyTorch process dlopen("libnccl.so.2") returns the NCCL torch already loaded (same
// soname), so the library and torch.distributed share one NCCL.  PA_NCCL_LIB overrides
// the library name.  Types and enum values come from nccl.h (stable C ABI).
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <mutex>

namespace pa {

struct NcclApi {
    bool ok = false;
    const char *why = "not loaded";
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*Reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                           cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GetVersion)(int *) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

inline NcclApi &nccl_api() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char *name = getenv("PA_NCCL_LIB");
        void *h = dlopen(name && *name ? name : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = "dlopen(libnccl.so.2) failed (set PA_NCCL_LIB)";
            return;
        }
        bool all = true;
        auto sym = [&](auto &fn, const char *s) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, s));
            if (!fn) all = false;
        };
        sym(api.GetUniqueId, "ncclGetUniqueId");
        sym(api.CommInitRank, "ncclCommInitRank");
        sym(api.CommDestroy, "ncclCommDestroy");
        sym(api.CommAbort, "ncclCommAbort");
        sym(api.Reduce, "ncclReduce");
        sym(api.AllGather, "ncclAllGather");
        sym(api.GetVersion, "ncclGetVersion");
        sym(api.GetErrorString, "ncclGetErrorString");
        if (!all) {
            api.why = "libnccl.so.2 lacks an expected symbol";
            return;
        }
        api.ok = true;
        api.why = "";
    });
    return api;
}

}  // namespace pa
