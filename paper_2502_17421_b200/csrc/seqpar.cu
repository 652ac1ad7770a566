// seqpar.cu -- sequence-parallel Hybrid Tree Attention (one process per GPU, or P virtual ranks
// of one process on one GPU: the loopback communicator).
//
// The prefix KV is sharded contiguously along the sequence; rank r computes the prefix pass on
// its slice (split-KV on its own SMs), combines its splits into ONE partial per query row laid
// out destination-major [P][B][T][H/P][d] (+ LSE), exchanges the head slices all-to-all (the only
// cross-rank step), and merges the P received prefix partials with the tree partial of its own
// H/P heads.  Exactness: Appendix C applied P+1 ways.  The paper runs on one
// GPU; this exchange is new here.
//
// Every rank runs the same three per-rank phases (local parts -> exchange -> final merge, then
// the optional all-gather + reassembly); only the transport of the exchange differs:
//  * NCCL: a grouped ncclSend/ncclRecv all-to-all over NVLink (ncclAllGather for the output).
//    NCCL is resolved with dlopen("libnccl.so.2") at hta_comm_create, so libhta has no link-time
//    NCCL dependency; inside a PyTorch process this finds the NCCL torch already loaded.
//  * loopback: all P ranks live in this process on the current device; the exchange is the
//    same destination-major block copies done with cudaMemcpyAsync.  This runs the P > 1 code
//    (destination-major send layout, rank > 0 head offsets, P-way final merge, reassembly) on
//    one GPU, which is how the tests check it against the oracle.
#include <dlfcn.h>

#include <cstring>
#include <new>
#include <vector>

#include "hta_internal.h"

using namespace hta;

namespace {

typedef struct ncclCommOpaque *nccl_comm_t;
typedef struct {
    char internal[128];
} nccl_uid_t;
typedef int nccl_result_t;
enum { kNcclFloat32 = 7, kNcclUint8 = 1 };

struct NcclApi {
    bool ok = false;
    nccl_result_t (*GetUniqueId)(nccl_uid_t *) = nullptr;
    nccl_result_t (*CommInitRank)(nccl_comm_t *, int, nccl_uid_t, int) = nullptr;
    nccl_result_t (*CommDestroy)(nccl_comm_t) = nullptr;
    nccl_result_t (*CommGetAsyncError)(nccl_comm_t, nccl_result_t *) = nullptr;
    nccl_result_t (*GroupStart)() = nullptr;
    nccl_result_t (*GroupEnd)() = nullptr;
    nccl_result_t (*Send)(const void *, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
    nccl_result_t (*Recv)(void *, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
    nccl_result_t (*AllGather)(const void *, void *, size_t, int, nccl_comm_t, cudaStream_t) = nullptr;
};

NcclApi &nccl() {
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
        if (h == nullptr) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (h == nullptr) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (h != nullptr) {
#define HTA_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name))
            HTA_SYM(GetUniqueId, "ncclGetUniqueId");
            HTA_SYM(CommInitRank, "ncclCommInitRank");
            HTA_SYM(CommDestroy, "ncclCommDestroy");
            HTA_SYM(CommGetAsyncError, "ncclCommGetAsyncError");
            HTA_SYM(GroupStart, "ncclGroupStart");
            HTA_SYM(GroupEnd, "ncclGroupEnd");
            HTA_SYM(Send, "ncclSend");
            HTA_SYM(Recv, "ncclRecv");
            HTA_SYM(AllGather, "ncclAllGather");
#undef HTA_SYM
            api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.CommGetAsyncError &&
                     api.GroupStart && api.GroupEnd && api.Send && api.Recv && api.AllGather;
        }
    }
    return api;
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
size_t round16(size_t x) { return (x + 15) & ~size_t(15); }

// Per-rank exchange block: O [B][T][Hp][d] followed by LSE [B][Hp][T] (floats, 16-byte rounded).
size_t block_floats(const hta_shape_t &s, int P) { return seqpar_block_floats(s.B, s.T, s.H / P, s.d); }

// One rank's workspace, carved in this order (all 16-byte aligned):
//   prefix split partials | send blocks [P][blk] | receive blocks [P][blk] |
//   own output slice (O [B,T,Hp,d] dtype, LSE [B,Hp,T]) | gathered slices [P] (O) then [P] (LSE)
struct RankWs {
    float *parts;
    size_t parts_bytes;
    float *sendb, *recvb;
    uint8_t *own_o;
    float *own_l;
    uint8_t *gat_o, *gat_l;
};

struct Geometry {
    hta_shape_t s;
    int P, Hp;
    size_t es;        // bytes per output element
    size_t blk;       // floats per exchange block
    size_t o_slice;   // bytes of one rank's O head slice
    size_t l_slice;   // bytes of one rank's LSE head slice
    size_t ws_bytes;  // workspace per rank
    int sms;
};

hta_status_t geometry(const hta_shape_t *shape, int P, int sms, Geometry *g) {
    if (shape == nullptr || P < 1 || shape->H % P != 0) return HTA_ERR_INVALID_ARGUMENT;
    const size_t base = hta_workspace_size(shape, sms);
    if (base == size_t(-1)) return HTA_ERR_INVALID_ARGUMENT;
    g->s = *shape;
    g->P = P;
    g->Hp = shape->H / P;
    g->es = shape->dtype == HTA_BF16 ? 2 : 4;
    g->blk = block_floats(*shape, P);
    g->o_slice = size_t(shape->B) * shape->T * g->Hp * shape->d * g->es;
    g->l_slice = size_t(shape->B) * g->Hp * shape->T * 4;
    g->sms = sms;
    g->ws_bytes = round16(base) + 2 * round16(P * g->blk * sizeof(float)) + round16(g->o_slice) +
                  round16(g->l_slice) + round16(P * g->o_slice) + round16(P * g->l_slice);
    return HTA_OK;
}

RankWs carve(const Geometry &g, void *ws) {
    uint8_t *w = static_cast<uint8_t *>(ws);
    RankWs r;
    r.parts = reinterpret_cast<float *>(w);
    r.parts_bytes = hta_workspace_size(&g.s, g.sms);
    w += round16(r.parts_bytes);
    r.sendb = reinterpret_cast<float *>(w);
    w += round16(g.P * g.blk * sizeof(float));
    r.recvb = reinterpret_cast<float *>(w);
    w += round16(g.P * g.blk * sizeof(float));
    r.own_o = w;
    w += round16(g.o_slice);
    r.own_l = reinterpret_cast<float *>(w);
    w += round16(g.l_slice);
    r.gat_o = w;
    w += round16(g.P * g.o_slice);
    r.gat_l = w;
    return r;
}

// Phase 1 of rank r: prefix pass over its slice, splits combined into the destination-major
// send blocks.
hta_status_t phase_local(const Geometry &g, const RankWs &w, const void *q, const void *k, const void *v,
                         const int32_t *seqlens, cudaStream_t st) {
    return seqpar_local_parts(&g.s, q, k, v, seqlens, w.parts, w.parts_bytes, w.sendb, g.P, st);
}

// Phase 3 of rank r: the P received prefix partials + the tree pass of heads [r*Hp, (r+1)*Hp).
// recvb: the P received blocks (rank r's own block included).
hta_status_t phase_merge(const Geometry &g, const RankWs &w, int r, const void *q, const void *kt, const void *vt,
                         const uint8_t *mask, int64_t mbs, const int32_t *parents, int64_t pbs, const float *recvb,
                         void *o, float *lse, int gather, cudaStream_t st) {
    void *o_local = gather ? static_cast<void *>(w.own_o) : o;
    float *l_local = gather ? w.own_l : lse;
    return seqpar_final_merge(&g.s, g.P, r, q, kt, vt, mask, mbs, parents, pbs, recvb, g.blk, o_local, l_local, st);
}

// Phase 4 (gather_output): the P gathered head slices [P][B,T,Hp,d] -> o [B,T,H,d] (and LSE).
hta_status_t phase_reassemble(const Geometry &g, const RankWs &w, void *o, float *lse, cudaStream_t st) {
    const hta_shape_t &s = g.s;
    const size_t row = size_t(g.Hp) * s.d * g.es;
    for (int p = 0; p < g.P; ++p) {
        if (cudaMemcpy2DAsync(static_cast<uint8_t *>(o) + p * row, size_t(s.H) * s.d * g.es, w.gat_o + p * g.o_slice,
                              row, row, size_t(s.B) * s.T, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
            return HTA_ERR_CUDA;
        if (lse != nullptr) {
            const size_t lrow = size_t(g.Hp) * s.T * 4;
            if (cudaMemcpy2DAsync(reinterpret_cast<uint8_t *>(lse) + p * lrow, size_t(s.H) * s.T * 4,
                                  w.gat_l + p * g.l_slice, lrow, lrow, size_t(s.B), cudaMemcpyDeviceToDevice,
                                  st) != cudaSuccess)
                return HTA_ERR_CUDA;
        }
    }
    return HTA_OK;
}

}  // namespace

// Peer-memory exchange state of one rank (or of every virtual rank of a loopback communicator):
// a double-buffered receive buffer recv [2][P][cap] floats (block q = source rank q: O then LSE)
// and P flags + 1 epoch counter (uint32), and the peers' views of theirs (IPC-mapped over NVLink).
struct P2pRank {
    float *recv = nullptr;
    uint32_t *flags = nullptr;  // [P] flags, [P] step counter, [P+1] block counter, [P+2] error word
    float *peer_recv[kMaxP2pRanks] = {};
    uint32_t *peer_flags[kMaxP2pRanks] = {};
    bool owned = true;          // allocated here (else IPC-opened or a loopback alias)
};

struct hta_comm_s {
    nccl_comm_t comm;  // nullptr for a loopback communicator
    int nranks;
    int rank;          // -1 for a loopback communicator (it holds every rank)
    // peer-memory exchange (hta_comm_p2p_*): per rank (one for NCCL, nranks for loopback)
    bool p2p = false;
    size_t p2p_cap = 0;  // floats per block
    std::vector<P2pRank> p2p_ranks;
};

namespace {
// rank r's phases 1-3 of the sequence-parallel step over the peer-memory exchange
hta_status_t p2p_combine(const Geometry &g, const RankWs &w, const hta_comm_s &c, int r, const void *q,
                         const void *k, const void *v, const int32_t *seqlens, cudaStream_t st) {
    P2pOut out{};
    const P2pRank &me = c.p2p_ranks[c.rank >= 0 ? 0 : r];
    for (int p = 0; p < g.P; ++p) {
        out.dst[p] = me.peer_recv[p] + size_t(r) * c.p2p_cap;
        out.peer_flags[p] = me.peer_flags[p];
    }
    out.epoch = me.flags + g.P;
    out.counter = me.flags + g.P + 1;
    out.rank = r;
    out.parity = int64_t(g.P) * int64_t(c.p2p_cap);
    return seqpar_local_parts(&g.s, q, k, v, seqlens, w.parts, w.parts_bytes, w.sendb, g.P, st, &out);
}
hta_status_t p2p_merge(const Geometry &g, const hta_comm_s &c, int r, const void *q, const void *kt, const void *vt,
                       const uint8_t *mask, int64_t mbs, const int32_t *parents, int64_t pbs, void *o, float *lse,
                       cudaStream_t st) {
    const P2pRank &me = c.p2p_ranks[c.rank >= 0 ? 0 : r];
    P2pIn in{me.flags + g.P, me.flags, int64_t(g.P) * int64_t(c.p2p_cap)};
    return seqpar_final_merge(&g.s, g.P, r, q, kt, vt, mask, mbs, parents, pbs, me.recv, c.p2p_cap, o, lse, st,
                              &in);
}
void p2p_release(hta_comm_s &c) {
    for (size_t i = 0; i < c.p2p_ranks.size(); ++i) {
        P2pRank &pr = c.p2p_ranks[i];
        if (c.rank >= 0)  // NCCL communicator: close the peers' IPC mappings
            for (int q = 0; q < c.nranks; ++q)
                if (q != c.rank && pr.peer_recv[q] != nullptr) {
                    cudaIpcCloseMemHandle(pr.peer_recv[q]);
                    cudaIpcCloseMemHandle(pr.peer_flags[q]);
                }
        if (pr.owned) {
            cudaFree(pr.recv);
            cudaFree(pr.flags);
        }
    }
    c.p2p_ranks.clear();
    c.p2p = false;
}
hta_status_t p2p_alloc_rank(P2pRank &pr, int P, size_t cap) {
    if (cudaMalloc(&pr.recv, 2 * size_t(P) * cap * sizeof(float)) != cudaSuccess) return HTA_ERR_CUDA;
    if (cudaMalloc(&pr.flags, (P + 3) * sizeof(uint32_t)) != cudaSuccess) return HTA_ERR_CUDA;
    if (cudaMemset(pr.flags, 0, (P + 3) * sizeof(uint32_t)) != cudaSuccess) return HTA_ERR_CUDA;
    return cudaDeviceSynchronize() == cudaSuccess ? HTA_OK : HTA_ERR_CUDA;
}
}  // namespace

extern "C" {

hta_status_t hta_comm_unique_id(void *unique_id_128) {
    if (unique_id_128 == nullptr) return HTA_ERR_INVALID_ARGUMENT;
    NcclApi &api = nccl();
    if (!api.ok) return HTA_ERR_NCCL;
    nccl_uid_t id;
    if (api.GetUniqueId(&id) != 0) return HTA_ERR_NCCL;
    std::memcpy(unique_id_128, &id, sizeof(id));
    return HTA_OK;
}

hta_status_t hta_comm_create(const void *unique_id_128, int32_t nranks, int32_t rank, hta_comm_t *comm) {
    if (unique_id_128 == nullptr || comm == nullptr || nranks < 1 || rank < 0 || rank >= nranks)
        return HTA_ERR_INVALID_ARGUMENT;
    NcclApi &api = nccl();
    if (!api.ok) return HTA_ERR_NCCL;
    nccl_uid_t id;
    std::memcpy(&id, unique_id_128, sizeof(id));
    nccl_comm_t c = nullptr;
    if (api.CommInitRank(&c, nranks, id, rank) != 0) return HTA_ERR_NCCL;
    hta_comm_s *h = new (std::nothrow) hta_comm_s{c, nranks, rank};
    if (h == nullptr) {
        api.CommDestroy(c);
        return HTA_ERR_INVALID_ARGUMENT;
    }
    *comm = h;
    return HTA_OK;
}

hta_status_t hta_comm_create_loopback(int32_t nranks, hta_comm_t *comm) {
    if (comm == nullptr || nranks < 1 || nranks > 64) return HTA_ERR_INVALID_ARGUMENT;
    hta_comm_s *h = new (std::nothrow) hta_comm_s{nullptr, nranks, -1};
    if (h == nullptr) return HTA_ERR_INVALID_ARGUMENT;
    *comm = h;
    return HTA_OK;
}

hta_status_t hta_comm_destroy(hta_comm_t comm) {
    if (comm == nullptr) return HTA_ERR_INVALID_ARGUMENT;
    hta_status_t r = HTA_OK;
    p2p_release(*comm);
    if (comm->comm != nullptr) {
        NcclApi &api = nccl();
        if (api.ok && api.CommDestroy(comm->comm) != 0) r = HTA_ERR_NCCL;
    }
    delete comm;
    return r;
}

hta_status_t hta_comm_p2p_alloc(hta_comm_t comm, size_t block_capacity_floats, void *ipc_handles_128) {
    if (comm == nullptr || ipc_handles_128 == nullptr || block_capacity_floats == 0) return HTA_ERR_INVALID_ARGUMENT;
    if (comm->nranks > kMaxP2pRanks) return HTA_ERR_UNSUPPORTED;
    p2p_release(*comm);
    const int n = comm->rank >= 0 ? 1 : comm->nranks;
    comm->p2p_ranks.assign(n, P2pRank{});
    comm->p2p_cap = (block_capacity_floats + 3) & ~size_t(3);  // (16-byte aligned blocks)
    for (int i = 0; i < n; ++i) {
        hta_status_t r = p2p_alloc_rank(comm->p2p_ranks[i], comm->nranks, comm->p2p_cap);
        if (r != HTA_OK) {
            p2p_release(*comm);
            return r;
        }
    }
    if (comm->rank < 0) {  // loopback: every virtual rank's peers are the other virtual ranks' buffers
        for (int i = 0; i < n; ++i)
            for (int q = 0; q < n; ++q) {
                comm->p2p_ranks[i].peer_recv[q] = comm->p2p_ranks[q].recv;
                comm->p2p_ranks[i].peer_flags[q] = comm->p2p_ranks[q].flags;
            }
        std::memset(ipc_handles_128, 0, 128);
        comm->p2p = true;
        return HTA_OK;
    }
    cudaIpcMemHandle_t h[2];
    if (cudaIpcGetMemHandle(&h[0], comm->p2p_ranks[0].recv) != cudaSuccess ||
        cudaIpcGetMemHandle(&h[1], comm->p2p_ranks[0].flags) != cudaSuccess) {
        p2p_release(*comm);
        return HTA_ERR_CUDA;
    }
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    std::memcpy(ipc_handles_128, h, 128);
    return HTA_OK;
}

hta_status_t hta_comm_p2p_set(hta_comm_t comm, int32_t enabled) {
    if (comm == nullptr) return HTA_ERR_INVALID_ARGUMENT;
    if (enabled && comm->p2p_ranks.empty()) return HTA_ERR_INVALID_ARGUMENT;
    comm->p2p = enabled != 0 && (comm->rank < 0 || comm->p2p_ranks[0].peer_recv[comm->rank] != nullptr);
    return enabled && !comm->p2p ? HTA_ERR_INVALID_ARGUMENT : HTA_OK;
}

hta_status_t hta_comm_p2p_error(hta_comm_t comm) {
    if (comm == nullptr) return HTA_ERR_INVALID_ARGUMENT;
    for (const P2pRank &pr : comm->p2p_ranks) {
        uint32_t err = 0;
        if (cudaMemcpy(&err, pr.flags + comm->nranks + 2, sizeof(err), cudaMemcpyDeviceToHost) != cudaSuccess)
            return HTA_ERR_CUDA;
        if (err != 0) return HTA_ERR_CUDA;
    }
    return HTA_OK;
}

hta_status_t hta_comm_p2p_open(hta_comm_t comm, const void *ipc_handles_all) {
    if (comm == nullptr || ipc_handles_all == nullptr || comm->p2p_ranks.empty()) return HTA_ERR_INVALID_ARGUMENT;
    if (comm->rank < 0) return HTA_OK;  // loopback: wired by hta_comm_p2p_alloc
    P2pRank &me = comm->p2p_ranks[0];
    const uint8_t *all = static_cast<const uint8_t *>(ipc_handles_all);
    for (int q = 0; q < comm->nranks; ++q) {
        if (q == comm->rank) {
            me.peer_recv[q] = me.recv;
            me.peer_flags[q] = me.flags;
            continue;
        }
        cudaIpcMemHandle_t h[2];
        std::memcpy(h, all + size_t(q) * 128, 128);
        void *pr = nullptr, *pf = nullptr;
        if (cudaIpcOpenMemHandle(&pr, h[0], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
            cudaIpcOpenMemHandle(&pf, h[1], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            cudaGetLastError();
            p2p_release(*comm);
            return HTA_ERR_CUDA;
        }
        me.peer_recv[q] = static_cast<float *>(pr);
        me.peer_flags[q] = static_cast<uint32_t *>(pf);
    }
    comm->p2p = true;
    return HTA_OK;
}

hta_status_t hta_comm_async_error(hta_comm_t comm) {
    if (comm == nullptr) return HTA_ERR_INVALID_ARGUMENT;
    if (comm->comm == nullptr) return HTA_OK;  // loopback: no asynchronous transport
    NcclApi &api = nccl();
    if (!api.ok) return HTA_ERR_NCCL;
    nccl_result_t async = 0;
    if (api.CommGetAsyncError(comm->comm, &async) != 0 || async != 0) return HTA_ERR_NCCL;
    return HTA_OK;
}

size_t hta_workspace_size_seqpar(const hta_shape_t *shape_local, int32_t num_sms, int32_t nranks) {
    Geometry g;
    if (geometry(shape_local, nranks, num_sms > 0 ? num_sms : 148, &g) != HTA_OK) return size_t(-1);
    return g.ws_bytes;
}

}  // extern "C"

// hta_forward_seqpar / hta_forward_seqpar_tree: the tree's visibility from the mask or (mask ==
// nullptr) the parent array.
static hta_status_t seqpar_forward(hta_comm_t comm, const hta_shape_t *shape_local, const void *q,
                                   const void *k_cache_local, const void *v_cache_local,
                                   const int32_t *cache_seqlens_local, const void *k_tree, const void *v_tree,
                                   const uint8_t *mask, int64_t mask_batch_stride, const int32_t *parents,
                                   int64_t parents_bs, void *o, float *lse_out, int32_t gather_output, void *ws,
                                   size_t ws_bytes, hta_stream_t stream) {
    if (comm == nullptr || shape_local == nullptr) return HTA_ERR_INVALID_ARGUMENT;
    if (comm->comm == nullptr) return HTA_ERR_INVALID_ARGUMENT;  // loopback: hta_forward_seqpar_loopback
    if (!q || !k_cache_local || !v_cache_local || !k_tree || !v_tree || (!mask && !parents) || !o)
        return HTA_ERR_INVALID_ARGUMENT;
    if (!aligned16(q) || !aligned16(k_cache_local) || !aligned16(v_cache_local) || !aligned16(k_tree) ||
        !aligned16(v_tree) || !aligned16(o) || !aligned16(ws))
        return HTA_ERR_INVALID_ARGUMENT;
    const int P = comm->nranks, r = comm->rank;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    Geometry g;
    hta_status_t rc = geometry(shape_local, P, sms, &g);
    if (rc != HTA_OK) return rc;
    if (ws == nullptr || ws_bytes < g.ws_bytes) return HTA_ERR_WORKSPACE;
    NcclApi &api = nccl();
    if (!api.ok) return HTA_ERR_NCCL;
    if ((rc = hta_comm_async_error(comm)) != HTA_OK) return rc;  // an earlier step's NCCL failure
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const RankWs w = carve(g, ws);

    if (comm->p2p && !gather_output && g.blk <= comm->p2p_cap) {
        // peer-memory exchange: the split combine writes each head block straight into its rank's
        // receive buffer over NVLink, one signal kernel flags them, the final merge waits for the flags
        if ((rc = p2p_combine(g, w, *comm, r, q, k_cache_local, v_cache_local, cache_seqlens_local, st)) != HTA_OK)
            return rc;
        return p2p_merge(g, *comm, r, q, k_tree, v_tree, mask, mask_batch_stride, parents, parents_bs, o, lse_out, st);
    }
    // 1) local prefix pass -> one destination-major partial per row
    if ((rc = phase_local(g, w, q, k_cache_local, v_cache_local, cache_seqlens_local, st)) != HTA_OK) return rc;
    // 2) all-to-all of head slices: block p of sendb goes to rank p, block p of recvb comes from p
    // (one rank: its single block is merged straight from the send buffer)
    if (P > 1 && cudaMemcpyAsync(w.recvb + size_t(r) * g.blk, w.sendb + size_t(r) * g.blk, g.blk * sizeof(float),
                                 cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return HTA_ERR_CUDA;
    if (P > 1) {
        if (api.GroupStart() != 0) return HTA_ERR_NCCL;
        for (int peer = 0; peer < P; ++peer) {
            if (peer == r) continue;
            if (api.Send(w.sendb + size_t(peer) * g.blk, g.blk, kNcclFloat32, peer, comm->comm, st) != 0 ||
                api.Recv(w.recvb + size_t(peer) * g.blk, g.blk, kNcclFloat32, peer, comm->comm, st) != 0) {
                api.GroupEnd();
                return HTA_ERR_NCCL;
            }
        }
        if (api.GroupEnd() != 0) return HTA_ERR_NCCL;
    }
    // 3) merge the P prefix partials with the tree partial of heads [r*Hp, (r+1)*Hp)
    if ((rc = phase_merge(g, w, r, q, k_tree, v_tree, mask, mask_batch_stride, parents, parents_bs,
                          P > 1 ? w.recvb : w.sendb, o, lse_out, gather_output, st)) != HTA_OK)
        return rc;
    if (!gather_output) return HTA_OK;
    // 4) all-gather of the head slices, then [P][B,T,Hp,d] -> [B,T,H,d]
    if (api.GroupStart() != 0) return HTA_ERR_NCCL;
    if (api.AllGather(w.own_o, w.gat_o, g.o_slice, kNcclUint8, comm->comm, st) != 0 ||
        (lse_out != nullptr && api.AllGather(w.own_l, w.gat_l, g.l_slice, kNcclUint8, comm->comm, st) != 0)) {
        api.GroupEnd();
        return HTA_ERR_NCCL;
    }
    if (api.GroupEnd() != 0) return HTA_ERR_NCCL;
    return phase_reassemble(g, w, o, lse_out, st);
}

extern "C" {

hta_status_t hta_forward_seqpar(hta_comm_t comm, const hta_shape_t *shape_local, const void *q,
                                const void *k_cache_local, const void *v_cache_local,
                                const int32_t *cache_seqlens_local, const void *k_tree, const void *v_tree,
                                const uint8_t *mask, int64_t mask_batch_stride, void *o, float *lse_out,
                                int32_t gather_output, void *ws, size_t ws_bytes, hta_stream_t stream) {
    if (mask == nullptr) return HTA_ERR_INVALID_ARGUMENT;
    return seqpar_forward(comm, shape_local, q, k_cache_local, v_cache_local, cache_seqlens_local, k_tree, v_tree,
                          mask, mask_batch_stride, nullptr, 0, o, lse_out, gather_output, ws, ws_bytes, stream);
}

hta_status_t hta_forward_seqpar_tree(hta_comm_t comm, const hta_shape_t *shape_local, const void *q,
                                     const void *k_cache_local, const void *v_cache_local,
                                     const int32_t *cache_seqlens_local, const void *k_tree, const void *v_tree,
                                     const int32_t *parents, int64_t parents_batch_stride, void *o, float *lse_out,
                                     int32_t gather_output, void *ws, size_t ws_bytes, hta_stream_t stream) {
    if (parents == nullptr) return HTA_ERR_INVALID_ARGUMENT;
    return seqpar_forward(comm, shape_local, q, k_cache_local, v_cache_local, cache_seqlens_local, k_tree, v_tree,
                          nullptr, 0, parents, parents_batch_stride, o, lse_out, gather_output, ws, ws_bytes, stream);
}

hta_status_t hta_forward_seqpar_loopback(hta_comm_t comm, const hta_shape_t *shape_local, const void *q,
                                         const void *const *k_cache_local, const void *const *v_cache_local,
                                         const int32_t *const *cache_seqlens_local, const void *k_tree,
                                         const void *v_tree, const uint8_t *mask, int64_t mask_batch_stride,
                                         void *const *o, float *const *lse_out, int32_t gather_output, void *ws,
                                         size_t ws_bytes, hta_stream_t stream) {
    if (comm == nullptr || comm->comm != nullptr || shape_local == nullptr) return HTA_ERR_INVALID_ARGUMENT;
    if (!k_cache_local || !v_cache_local || !o || !q || !k_tree || !v_tree || !mask) return HTA_ERR_INVALID_ARGUMENT;
    const int P = comm->nranks;
    for (int r = 0; r < P; ++r) {
        if (!k_cache_local[r] || !v_cache_local[r] || !o[r]) return HTA_ERR_INVALID_ARGUMENT;
        if (!aligned16(k_cache_local[r]) || !aligned16(v_cache_local[r]) || !aligned16(o[r]))
            return HTA_ERR_INVALID_ARGUMENT;
    }
    if (!aligned16(q) || !aligned16(k_tree) || !aligned16(v_tree) || !aligned16(ws)) return HTA_ERR_INVALID_ARGUMENT;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    Geometry g;
    hta_status_t rc = geometry(shape_local, P, sms, &g);
    if (rc != HTA_OK) return rc;
    const size_t per = round16(g.ws_bytes);
    if (ws == nullptr || ws_bytes < per * P) return HTA_ERR_WORKSPACE;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    std::vector<RankWs> w(P);
    for (int r = 0; r < P; ++r) w[r] = carve(g, static_cast<uint8_t *>(ws) + per * r);
    auto sl = [&](int r) { return cache_seqlens_local ? cache_seqlens_local[r] : nullptr; };
    auto lse = [&](int r) { return lse_out ? lse_out[r] : nullptr; };
    if (comm->p2p && !gather_output && g.blk <= comm->p2p_cap) {  // the peer-memory exchange, all ranks
        for (int r = 0; r < P; ++r)
            if ((rc = p2p_combine(g, w[r], *comm, r, q, k_cache_local[r], v_cache_local[r], sl(r), st)) != HTA_OK)
                return rc;
        for (int r = 0; r < P; ++r)
            if ((rc = p2p_merge(g, *comm, r, q, k_tree, v_tree, mask, mask_batch_stride, nullptr, 0, o[r], lse(r),
                                st)) != HTA_OK)
                return rc;
        return HTA_OK;
    }
    for (int r = 0; r < P; ++r)
        if ((rc = phase_local(g, w[r], q, k_cache_local[r], v_cache_local[r], sl(r), st)) != HTA_OK) return rc;
    // the all-to-all: block dst of rank src's send buffer -> block src of rank dst's receive buffer
    for (int dst = 0; dst < P; ++dst)
        for (int src = 0; src < P; ++src)
            if (cudaMemcpyAsync(w[dst].recvb + size_t(src) * g.blk, w[src].sendb + size_t(dst) * g.blk,
                                g.blk * sizeof(float), cudaMemcpyDeviceToDevice, st) != cudaSuccess)
                return HTA_ERR_CUDA;
    for (int r = 0; r < P; ++r)
        if ((rc = phase_merge(g, w[r], r, q, k_tree, v_tree, mask, mask_batch_stride, nullptr, 0, w[r].recvb, o[r],
                              lse(r), gather_output, st)) != HTA_OK)
            return rc;
    if (!gather_output) return HTA_OK;
    // the all-gather: rank src's own slice -> slot src of every rank's gather buffer
    for (int dst = 0; dst < P; ++dst)
        for (int src = 0; src < P; ++src) {
            if (cudaMemcpyAsync(w[dst].gat_o + src * g.o_slice, w[src].own_o, g.o_slice, cudaMemcpyDeviceToDevice,
                                st) != cudaSuccess)
                return HTA_ERR_CUDA;
            if (lse_out != nullptr &&
                cudaMemcpyAsync(w[dst].gat_l + src * g.l_slice, w[src].own_l, g.l_slice, cudaMemcpyDeviceToDevice,
                                st) != cudaSuccess)
                return HTA_ERR_CUDA;
        }
    for (int r = 0; r < P; ++r)
        if ((rc = phase_reassemble(g, w[r], o[r], lse(r), st)) != HTA_OK) return rc;
    return HTA_OK;
}

}  // extern "C"
