// Native NCCL data plane for the distributed SaP handle: neighbour exchanges of spike tips,
// interface rows and operator halos as grouped ncclSend / ncclRecv on the handle's stream (no host
// synchronisation), Krylov reductions as ncclAllReduce on device scalars.
//
// libnccl is resolved at run time (dlopen): the copy torch already loaded into the process when there is
// one (RTLD_NOLOAD, so both share one NCCL), else the system's libnccl.so.2. nccl.h supplies the types.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <string>

#include "comm_nccl.h"

namespace sapgpu {

namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string error;
    bool ok = false;
};

NcclApi& api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) {
            a.error = std::string("libnccl.so.2 not found: ") + dlerror();
            return;
        }
        auto sym = [&](const char* name) {
            void* p = dlsym(lib, name);
            if (!p && a.error.empty()) a.error = std::string("libnccl.so.2 lacks ") + name;
            return p;
        };
        a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
        a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
        a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
        a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
        a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
        a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
        a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
        a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
        a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
        a.ok = a.error.empty();
    });
    return a;
}

void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        NcclApi& a = api();
        throw CommFailure(std::string("sap: ") + what + " failed: " + (a.GetErrorString ? a.GetErrorString(r) : "?"));
    }
}

NcclApi& need() {
    NcclApi& a = api();
    if (!a.ok) throw CommFailure("sap: NCCL unavailable (" + a.error + ")");
    return a;
}

}  // namespace

struct NcclComm {
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1;
};

void nccl_unique_id(unsigned char* out) {
    static_assert(sizeof(ncclUniqueId) == kNcclIdBytes, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    check(need().GetUniqueId(&id), "ncclGetUniqueId");
    memcpy(out, &id, sizeof(id));
}

NcclComm* nccl_create(const unsigned char* id_bytes, int rank, int world) {
    NcclApi& a = need();
    ncclUniqueId id;
    memcpy(&id, id_bytes, sizeof(id));
    auto* c = new NcclComm;
    c->rank = rank;
    c->world = world;
    const ncclResult_t r = a.CommInitRank(&c->comm, world, id, rank);
    if (r != ncclSuccess) {
        delete c;
        check(r, "ncclCommInitRank");
    }
    return c;
}

void nccl_destroy(NcclComm* c) {
    if (!c) return;
    if (c->comm && api().ok) api().CommDestroy(c->comm);
    delete c;
}

// One group: receives from / sends to the left (rank - 1) and right (rank + 1) neighbours, stream-ordered.
void nccl_exchange(NcclComm* c, const double* sl, int n_sl, const double* sr, int n_sr, double* rl, int n_rl,
                   double* rr, int n_rr, cudaStream_t s) {
    if (!(n_sl || n_sr || n_rl || n_rr)) return;
    NcclApi& a = need();
    check(a.GroupStart(), "ncclGroupStart");
    if (n_rl) check(a.Recv(rl, (size_t)n_rl, ncclFloat64, c->rank - 1, c->comm, s), "ncclRecv");
    if (n_rr) check(a.Recv(rr, (size_t)n_rr, ncclFloat64, c->rank + 1, c->comm, s), "ncclRecv");
    if (n_sl) check(a.Send(sl, (size_t)n_sl, ncclFloat64, c->rank - 1, c->comm, s), "ncclSend");
    if (n_sr) check(a.Send(sr, (size_t)n_sr, ncclFloat64, c->rank + 1, c->comm, s), "ncclSend");
    check(a.GroupEnd(), "ncclGroupEnd");
}

void nccl_allreduce(NcclComm* c, double* d, int count, cudaStream_t s) {
    if (count <= 0) return;
    check(need().AllReduce(d, d, (size_t)count, ncclFloat64, ncclSum, c->comm, s), "ncclAllReduce");
}

bool nccl_available(std::string* why) {
    NcclApi& a = api();
    if (!a.ok && why) *why = a.error;
    return a.ok;
}

}  // namespace sapgpu
