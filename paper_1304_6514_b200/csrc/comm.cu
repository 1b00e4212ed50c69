// Multi-GPU transport for the sharded runs (north_star subsystem 4): one context
// per GPU (one process or thread each), slices split into contiguous blocks, and the only data
// exchange is the paper's final compose step — the block maps gathered to rank 0 (TREE) or the
// running state handed rank to rank (CHAIN, the λ chain of PAPER.md:218-222). Replaces the
// reference's simulated wire (inject_latency + message counters, nievergelt.cpp:73-79, 95-101).
//
// Two transports behind one interface:
//  * NCCL (ncclSend / ncclRecv on the context's stream, over NVLink/NVSwitch on the box);
//  * host callbacks (the caller moves host buffers: MPI, torch.distributed gloo, ...). The device
//    buffer is staged through pinned memory; used by the CPU-side tests of the sharded logic and by
//    callers without NCCL. No kernel ever waits on another rank's kernel with this transport.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <type_traits>
#include <vector>

#include "pint_internal.cuh"

struct pint_comm {
    int rank = 0, world = 1;
    ncclComm_t nccl = nullptr;
    pint_send_fn send = nullptr;
    pint_recv_fn recv = nullptr;
    void* user = nullptr;
    void* staging = nullptr;  // pinned host staging (callback transport)
    size_t staging_bytes = 0;
    int64_t messages = 0, bytes = 0;  // exchanged by this rank since the last reset
};

namespace {

// NCCL is resolved at run time (dlopen of libnccl.so.2 when the first NCCL communicator is made),
// not linked: a link-time dependency would load the system NCCL with libpint_cuda.so, and a process
// that loads this library before torch could then not load torch (libtorch_cuda needs its own,
// newer NCCL under the same soname). In a torch process the already-loaded NCCL is the one found.
struct Nccl {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        auto sym = [&](auto& f, const char* name) { f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name)); };
        sym(n.GetUniqueId, "ncclGetUniqueId");
        sym(n.CommInitRank, "ncclCommInitRank");
        sym(n.CommInitAll, "ncclCommInitAll");
        sym(n.CommDestroy, "ncclCommDestroy");
        sym(n.Send, "ncclSend");
        sym(n.Recv, "ncclRecv");
        sym(n.GroupStart, "ncclGroupStart");
        sym(n.GroupEnd, "ncclGroupEnd");
        sym(n.GetErrorString, "ncclGetErrorString");
        n.ok = n.GetUniqueId && n.CommInitRank && n.CommInitAll && n.CommDestroy && n.Send && n.Recv && n.GroupStart &&
               n.GroupEnd && n.GetErrorString;
    });
    return n;
}

int nccl_err(pint_ctx* ctx, ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return PINT_OK;
    return pint_set_error(ctx, PINT_E_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

void* staging(pint_comm* c, size_t bytes) {
    if (c->staging_bytes < bytes) {
        if (c->staging) cudaFreeHost(c->staging);
        c->staging = nullptr;
        c->staging_bytes = 0;
        if (cudaHostAlloc(&c->staging, bytes, cudaHostAllocDefault) != cudaSuccess) return nullptr;
        c->staging_bytes = bytes;
    }
    return c->staging;
}

}  // namespace

int comm_send(pint_ctx* ctx, const void* dev_buf, size_t bytes, int peer) {
    pint_comm* c = ctx->comm;
    ++c->messages;
    c->bytes += static_cast<int64_t>(bytes);
    if (c->nccl) return nccl_err(ctx, nccl().Send(dev_buf, bytes, ncclChar, peer, c->nccl, ctx->stream), "ncclSend");
    void* h = staging(c, bytes);
    if (!h) return pint_set_error(ctx, PINT_E_CUDA, "comm: pinned staging allocation failed");
    if (cudaMemcpyAsync(h, dev_buf, bytes, cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess)
        return pint_set_error(ctx, PINT_E_CUDA, "comm: D2H staging failed");
    if (c->send(c->user, peer, h, bytes) != 0) return pint_set_error(ctx, PINT_E_NCCL, "comm: send callback failed");
    return PINT_OK;
}

int comm_recv(pint_ctx* ctx, void* dev_buf, size_t bytes, int peer) {
    pint_comm* c = ctx->comm;
    if (c->nccl) return nccl_err(ctx, nccl().Recv(dev_buf, bytes, ncclChar, peer, c->nccl, ctx->stream), "ncclRecv");
    void* h = staging(c, bytes);
    if (!h) return pint_set_error(ctx, PINT_E_CUDA, "comm: pinned staging allocation failed");
    if (c->recv(c->user, peer, h, bytes) != 0) return pint_set_error(ctx, PINT_E_NCCL, "comm: recv callback failed");
    if (cudaMemcpyAsync(dev_buf, h, bytes, cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess)  // (the staging is reused by the next call)
        return pint_set_error(ctx, PINT_E_CUDA, "comm: H2D staging failed");
    return PINT_OK;
}

// Gather `bytes` from every rank to root: slot r of `gathered` (root) holds rank r's `mine`. NCCL:
// one grouped send/recv set (the W - 1 transfers run together over NVSwitch).
int comm_gather(pint_ctx* ctx, const void* mine, void* gathered, size_t bytes, int root) {
    pint_comm* c = ctx->comm;
    if (c->rank == root && cudaMemcpyAsync(static_cast<char*>(gathered) + bytes * root, mine, bytes,
                                           cudaMemcpyDeviceToDevice, ctx->stream) != cudaSuccess)
        return pint_set_error(ctx, PINT_E_CUDA, "comm_gather: local copy failed");
    if (c->world == 1) return PINT_OK;
    if (c->nccl) {
        if (const int rc = nccl_err(ctx, nccl().GroupStart(), "ncclGroupStart")) return rc;
        int rc = PINT_OK;
        if (c->rank == root) {
            for (int r = 0; r < c->world && !rc; ++r)
                if (r != root) rc = comm_recv(ctx, static_cast<char*>(gathered) + bytes * r, bytes, r);
        } else {
            rc = comm_send(ctx, mine, bytes, root);
        }
        const int rg = nccl_err(ctx, nccl().GroupEnd(), "ncclGroupEnd");
        return rc ? rc : rg;
    }
    if (c->rank != root) return comm_send(ctx, mine, bytes, root);
    for (int r = 0; r < c->world; ++r)
        if (r != root)
            if (const int rc = comm_recv(ctx, static_cast<char*>(gathered) + bytes * r, bytes, r)) return rc;
    return PINT_OK;
}

void comm_counters(pint_ctx* ctx, int64_t* messages, int64_t* bytes, bool reset) {
    pint_comm* c = ctx->comm;
    if (messages) *messages = c ? c->messages : 0;
    if (bytes) *bytes = c ? c->bytes : 0;
    if (c && reset) c->messages = c->bytes = 0;
}

void comm_free(pint_ctx* ctx) {
    if (!ctx->comm) return;
    if (ctx->comm->nccl) nccl().CommDestroy(ctx->comm->nccl);
    if (ctx->comm->staging) cudaFreeHost(ctx->comm->staging);
    delete ctx->comm;
    ctx->comm = nullptr;
}

extern "C" {

int pint_comm_unique_id(void* id_out) {
    if (!id_out) return PINT_E_INVALID;
    if (!nccl().ok) return PINT_E_NCCL;
    ncclUniqueId id;
    if (nccl().GetUniqueId(&id) != ncclSuccess) return PINT_E_NCCL;
    std::memcpy(id_out, &id, sizeof id);
    return PINT_OK;
}

int pint_comm_init(pint_ctx* ctx, const void* id, int rank, int world) {
    if (!ctx || !id || world < 1 || rank < 0 || rank >= world) return PINT_E_INVALID;
    if (!nccl().ok) return pint_set_error(ctx, PINT_E_NCCL, "pint_comm_init: libnccl.so.2 not found");
    comm_free(ctx);
    cudaSetDevice(ctx->device);
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    auto* c = new pint_comm();
    c->rank = rank;
    c->world = world;
    if (const int rc = nccl_err(ctx, nccl().CommInitRank(&c->nccl, world, uid, rank), "ncclCommInitRank")) {
        delete c;
        return rc;
    }
    ctx->comm = c;
    return PINT_OK;
}

int pint_comm_init_all(pint_ctx** ctxs, int world) {
    if (!ctxs || world < 1) return PINT_E_INVALID;
    if (!nccl().ok) return ctxs[0] ? pint_set_error(ctxs[0], PINT_E_NCCL, "pint_comm_init_all: libnccl.so.2 not found")
                                   : PINT_E_NCCL;
    std::vector<ncclComm_t> comms(static_cast<size_t>(world));
    std::vector<int> devs(static_cast<size_t>(world));
    for (int r = 0; r < world; ++r) {
        if (!ctxs[r]) return PINT_E_INVALID;
        comm_free(ctxs[r]);
        devs[r] = ctxs[r]->device;
    }
    if (const int rc = nccl_err(ctxs[0], nccl().CommInitAll(comms.data(), world, devs.data()), "ncclCommInitAll")) return rc;
    for (int r = 0; r < world; ++r) {
        auto* c = new pint_comm();
        c->rank = r;
        c->world = world;
        c->nccl = comms[r];
        ctxs[r]->comm = c;
    }
    return PINT_OK;
}

int pint_comm_init_callbacks(pint_ctx* ctx, int rank, int world, pint_send_fn send, pint_recv_fn recv, void* user) {
    if (!ctx || world < 1 || rank < 0 || rank >= world || (world > 1 && (!send || !recv))) return PINT_E_INVALID;
    comm_free(ctx);
    auto* c = new pint_comm();
    c->rank = rank;
    c->world = world;
    c->send = send;
    c->recv = recv;
    c->user = user;
    ctx->comm = c;
    return PINT_OK;
}

int pint_comm_rank(const pint_ctx* ctx, int* rank, int* world) {
    if (!ctx || !ctx->comm) return PINT_E_INVALID;
    if (rank) *rank = ctx->comm->rank;
    if (world) *world = ctx->comm->world;
    return PINT_OK;
}

int pint_comm_destroy(pint_ctx* ctx) {
    if (!ctx) return PINT_E_INVALID;
    comm_free(ctx);
    return PINT_OK;
}

}  // extern "C"
