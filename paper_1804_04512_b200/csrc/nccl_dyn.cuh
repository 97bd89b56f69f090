// nccl_dyn.cuh -- NCCL loaded on first use (dlopen "libnccl.so.2"), so the library has no
// link-time NCCL dependency and, inside a process that already imported torch, binds to the
// NCCL torch loaded (same soname). Only the calls the data-parallel step needs.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

#include "runtime.cuh"

namespace b2n {

struct NcclApi {
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*commGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*commAbort)(ncclComm_t) = nullptr;
    const char* (*errStr)(ncclResult_t) = nullptr;
};

inline NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) throw Error(B2N_ENCCL, std::string("cannot load libnccl.so.2: ") + dlerror());
        a.getUniqueId = reinterpret_cast<decltype(a.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        a.commInitRank = reinterpret_cast<decltype(a.commInitRank)>(dlsym(h, "ncclCommInitRank"));
        a.allReduce = reinterpret_cast<decltype(a.allReduce)>(dlsym(h, "ncclAllReduce"));
        a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(h, "ncclCommDestroy"));
        a.errStr = reinterpret_cast<decltype(a.errStr)>(dlsym(h, "ncclGetErrorString"));
        a.commGetAsyncError = reinterpret_cast<decltype(a.commGetAsyncError)>(dlsym(h, "ncclCommGetAsyncError"));
        a.commAbort = reinterpret_cast<decltype(a.commAbort)>(dlsym(h, "ncclCommAbort"));
        if (!a.getUniqueId || !a.commInitRank || !a.allReduce || !a.commDestroy)
            throw Error(B2N_ENCCL, "libnccl.so.2 lacks a required symbol");
        return a;
    }();
    return api;
}

inline void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw Error(B2N_ENCCL, std::string(what) + ": " + (nccl().errStr ? nccl().errStr(r) : "nccl error"));
}

// one communicator per replica (one process per GPU, rank = process rank). While the host waits on
// a step (spin_sync) the communicator is polled: ncclCommGetAsyncError reporting an error, or a wait
// longer than B2N_NCCL_TIMEOUT seconds (default 600), aborts it (ncclCommAbort releases the kernels
// blocked in the collective) and throws B2N_ENCCL -- a dead peer fails the step instead of hanging it.
struct DpComm : WaitWatch {
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1;
    double timeout_s = 600.0;
    bool aborted = false;
    void init(const char id[128], int r, int w) {
        ncclUniqueId uid;
        static_assert(sizeof(uid.internal) == 128, "ncclUniqueId size");
        std::memcpy(uid.internal, id, 128);
        nccl_check(nccl().commInitRank(&comm, w, uid, r), "ncclCommInitRank");
        rank = r;
        world = w;
        if (const char* e = std::getenv("B2N_NCCL_TIMEOUT")) timeout_s = std::atof(e);
        wait_watches().push_back(this);
    }
    void poll(double waited_s) override {
        if (!comm || aborted) return;
        ncclResult_t st = ncclSuccess;
        if (nccl().commGetAsyncError && nccl().commGetAsyncError(comm, &st) != ncclSuccess) st = ncclSystemError;
        const bool err = st != ncclSuccess && st != ncclInProgress;
        if (!err && !(timeout_s > 0 && waited_s > timeout_s)) return;
        if (nccl().commAbort) nccl().commAbort(comm);
        aborted = true;
        comm = nullptr;
        throw Error(B2N_ENCCL, err ? std::string("NCCL asynchronous error: ") + (nccl().errStr ? nccl().errStr(st) : "?")
                                   : "NCCL collective exceeded B2N_NCCL_TIMEOUT; communicator aborted");
    }
    ~DpComm() {
        auto& w = wait_watches();
        w.erase(std::remove(w.begin(), w.end(), static_cast<WaitWatch*>(this)), w.end());
        if (comm) nccl().commDestroy(comm);
    }
    void allreduce_f32(float* buf, size_t n, cudaStream_t st) const {
        nccl_check(nccl().allReduce(buf, buf, n, ncclFloat32, ncclSum, comm, st), "ncclAllReduce");
    }
    void allreduce_f64(double* buf, size_t n, cudaStream_t st) const {
        nccl_check(nccl().allReduce(buf, buf, n, ncclFloat64, ncclSum, comm, st), "ncclAllReduce");
    }
};

}  // namespace b2n
