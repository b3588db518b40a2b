// NCCL for the shard-by-k apply: the library's own communicator, resolved at run
// time with dlopen so libpcop_b200.so loads (and its single-GPU paths run) on hosts without NCCL.
//
// The reference has no parallel path at all: its k-loop (pc_operator.cpp:49-54) is serial.  Here
// each rank applies its block of terms and the partial outputs are combined by ONE fp64 sum
// reduction of the real cropped outputs (N*8 bytes per vector):
// ncclAllReduce (every rank gets the full apply) or ncclReduce (rank 0 gets it).
//
// dlopen("libnccl.so.2") returns the copy already mapped into the process when there is one
// (e.g. torch's bundled NCCL under torch.distributed), else the system library.  Types come from
// the system <nccl.h>; only the handful of entry points below are bound.
#include "comm.h"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

namespace pcb {
namespace {

struct NcclApi {
    void* so = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*comm_count)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                           cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    ncclResult_t (*get_version)(int*) = nullptr;
    std::string err;
};

NcclApi& api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* n : names) {
            a.so = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
            if (a.so) break;
        }
        if (!a.so) {
            a.err = std::string("NCCL not found (dlopen libnccl.so.2): ") + (dlerror() ? dlerror() : "");
            return;
        }
#define PCB_BIND(field, sym) a.field = reinterpret_cast<decltype(a.field)>(dlsym(a.so, sym))
        PCB_BIND(get_unique_id, "ncclGetUniqueId");
        PCB_BIND(comm_init_rank, "ncclCommInitRank");
        PCB_BIND(comm_destroy, "ncclCommDestroy");
        PCB_BIND(comm_count, "ncclCommCount");
        PCB_BIND(all_reduce, "ncclAllReduce");
        PCB_BIND(reduce, "ncclReduce");
        PCB_BIND(group_start, "ncclGroupStart");
        PCB_BIND(group_end, "ncclGroupEnd");
        PCB_BIND(error_string, "ncclGetErrorString");
        PCB_BIND(get_version, "ncclGetVersion");
#undef PCB_BIND
        if (!a.get_unique_id || !a.comm_init_rank || !a.comm_destroy || !a.all_reduce || !a.reduce)
            a.err = "NCCL library lacks the required entry points";
    });
    return a;
}

std::string nccl_msg(const char* what, ncclResult_t r) {
    NcclApi& a = api();
    return std::string(what) + ": " + (a.error_string ? a.error_string(r) : "NCCL error") + " (" +
           std::to_string((int)r) + ")";
}

}  // namespace

bool comm_available(std::string* why) {
    NcclApi& a = api();
    if (!a.err.empty() && why) *why = a.err;
    return a.err.empty();
}

int comm_version() {
    NcclApi& a = api();
    int v = 0;
    if (a.err.empty() && a.get_version) a.get_version(&v);
    return v;
}

std::string comm_unique_id(void* out128) {
    NcclApi& a = api();
    if (!a.err.empty()) return a.err;
    ncclUniqueId id;
    const ncclResult_t r = a.get_unique_id(&id);
    if (r != ncclSuccess) return nccl_msg("ncclGetUniqueId", r);
    static_assert(sizeof(ncclUniqueId) == PCB_COMM_ID_BYTES, "ncclUniqueId size");
    std::memcpy(out128, &id, sizeof(id));
    return "";
}

std::string comm_init(const void* id128, int nranks, int rank, void** out) {
    NcclApi& a = api();
    *out = nullptr;
    if (!a.err.empty()) return a.err;
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclComm_t c = nullptr;
    const ncclResult_t r = a.comm_init_rank(&c, nranks, id, rank);
    if (r != ncclSuccess) return nccl_msg("ncclCommInitRank", r);
    *out = c;
    return "";
}

void comm_destroy(void* c) {
    if (c && api().comm_destroy) api().comm_destroy(static_cast<ncclComm_t>(c));
}

// in-place fp64 sum: root < 0 -> all-reduce, else reduce to `root`
std::string comm_sum(void* c, double* buf, size_t count, int root, cudaStream_t st) {
    NcclApi& a = api();
    const ncclComm_t comm = static_cast<ncclComm_t>(c);
    const ncclResult_t r = root < 0 ? a.all_reduce(buf, buf, count, ncclFloat64, ncclSum, comm, st)
                                    : a.reduce(buf, buf, count, ncclFloat64, ncclSum, root, comm, st);
    if (r != ncclSuccess) return nccl_msg(root < 0 ? "ncclAllReduce" : "ncclReduce", r);
    return "";
}

}  // namespace pcb
