// comm.cu -- row-sharded multi-GPU support: NCCL loaded at run time.
//
// With a communicator attached, each rank holds a contiguous row block A_g of
// A (and the matching rows of Q); B', W, G and every b x b / l x b Gram are
// replicated.  The engine all-reduces (sum) exactly the products that
// contract over the rows of A:
//     ||A||_F^2,  W = A'Y,  [Q|Y]'Y,  Y'Y,  Q'Y
// (SURVEY.md section 8(e)).  NCCL's all-reduce hands every rank the same bits,
// so all ranks take the same convergence / redraw decisions.
//
// libnccl.so.2 is dlopen()ed on first use (torch's bundled copy when it is
// already loaded, else the system one): single-GPU users need no NCCL.
//
// The host backend (fqb_comm_attach_host) runs the same reduction points through a
// caller's all-reduce on pinned host copies (D2H, callback, H2D on the handle's
// stream).  It is what a host application with its own transport (MPI, gloo) binds,
// and it lets several ranks share one GPU in a test without any kernel waiting on
// another rank's kernel: every exchange is a host round trip.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "engine.hpp"

namespace farqb {
namespace {

struct NcclApi {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    bool ok = false;
    std::string why;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
        api.get_unique_id = reinterpret_cast<decltype(&ncclGetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        api.comm_init_rank = reinterpret_cast<decltype(&ncclCommInitRank)>(dlsym(h, "ncclCommInitRank"));
        api.comm_destroy = reinterpret_cast<decltype(&ncclCommDestroy)>(dlsym(h, "ncclCommDestroy"));
        api.all_reduce = reinterpret_cast<decltype(&ncclAllReduce)>(dlsym(h, "ncclAllReduce"));
        api.error_string = reinterpret_cast<decltype(&ncclGetErrorString)>(dlsym(h, "ncclGetErrorString"));
        api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_reduce && api.error_string;
        if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
    });
    if (!api.ok) throw Error(kStatusNccl, api.why);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw Error(kStatusNccl, std::string(what) + ": " + nccl().error_string(r));
}

}  // namespace

void comm_unique_id(void* out128) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(out128, &id, sizeof id);
}

void comm_attach(Handle& h, const void* id128, int nranks, int rank) {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw Error(kStatusInvalid, "bad rank / nranks");
    comm_detach(h);
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    ncclComm_t c = nullptr;
    nccl_check(nccl().comm_init_rank(&c, nranks, id, rank), "ncclCommInitRank");
    h.comm = c;
    h.nranks = nranks;
    h.rank = rank;
}

void comm_detach(Handle& h) {
    if (h.comm) {
        cudaStreamSynchronize(h.stream);
        nccl().comm_destroy(static_cast<ncclComm_t>(h.comm));
    }
    if (h.host_ar_buf) {
        cudaStreamSynchronize(h.stream);
        cudaFreeHost(h.host_ar_buf);
    }
    h.comm = nullptr;
    h.host_ar = nullptr;
    h.host_ar_user = nullptr;
    h.host_ar_buf = nullptr;
    h.host_ar_cap = 0;
    h.nranks = 1;
    h.rank = 0;
}

void comm_attach_host(Handle& h, fqb_host_allreduce_fn fn, void* user, int nranks, int rank) {
    if (!fn) throw Error(kStatusInvalid, "null all-reduce callback");
    if (nranks < 1 || rank < 0 || rank >= nranks) throw Error(kStatusInvalid, "bad rank / nranks");
    comm_detach(h);
    h.host_ar = fn;
    h.host_ar_user = user;
    h.nranks = nranks;
    h.rank = rank;
}

void comm_allreduce_sum(Handle& h, double* buf, size_t count, cudaStream_t s) {
    if (count == 0) return;
    if (h.host_ar) {
        if (count > h.host_ar_cap) {
            if (h.host_ar_buf) {
                FQB_CUDA(cudaStreamSynchronize(s));
                FQB_CUDA(cudaFreeHost(h.host_ar_buf));
                h.host_ar_buf = nullptr;
            }
            FQB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h.host_ar_buf), count * sizeof(double)));
            h.host_ar_cap = count;
        }
        FQB_CUDA(cudaMemcpyAsync(h.host_ar_buf, buf, count * sizeof(double), cudaMemcpyDeviceToHost, s));
        FQB_CUDA(cudaStreamSynchronize(s));
        if (h.host_ar(h.host_ar_user, h.host_ar_buf, int64_t(count)) != 0)
            throw Error(kStatusNccl, "host all-reduce callback failed");
        FQB_CUDA(cudaMemcpyAsync(buf, h.host_ar_buf, count * sizeof(double), cudaMemcpyHostToDevice, s));
        ++h.collectives;
        return;
    }
    if (!h.comm) return;
    nccl_check(nccl().all_reduce(buf, buf, count, ncclFloat64, ncclSum, static_cast<ncclComm_t>(h.comm), s),
               "ncclAllReduce");
    ++h.collectives;
}

}  // namespace farqb
