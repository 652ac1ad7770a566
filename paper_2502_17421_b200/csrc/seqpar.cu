// seqpar.cu -- sequence-parallel Hybrid Tree Attention over NCCL (one process per GPU).
//
// The prefix KV is sharded contiguously along the sequence; rank r computes the prefix pass on
// its slice (split-KV on its own SMs), combines its splits into ONE partial per query row laid
// out destination-major [P][B][T][H/P][d] (+ LSE), exchanges the head slices with a grouped
// ncclSend/ncclRecv all-to-all (the only cross-device step), and merges the P received prefix
// partials with the tree partial of its own H/P heads.  Exactness: Appendix C applied P+1 ways
// (PAPER.md:662-671).  The paper runs on one GPU; this exchange is new here.
//
// NCCL is resolved at hta_comm_create time with dlopen("libnccl.so.2") so libhta has no
// link-time NCCL dependency; inside a PyTorch process this finds the NCCL torch already loaded.
#include <dlfcn.h>

#include <cstring>
#include <new>

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
            HTA_SYM(GroupStart, "ncclGroupStart");
            HTA_SYM(GroupEnd, "ncclGroupEnd");
            HTA_SYM(Send, "ncclSend");
            HTA_SYM(Recv, "ncclRecv");
            HTA_SYM(AllGather, "ncclAllGather");
#undef HTA_SYM
            api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.GroupStart && api.GroupEnd &&
                     api.Send && api.Recv && api.AllGather;
        }
    }
    return api;
}

// Per-rank exchange block: O [B][T][Hp][d] followed by LSE [B][Hp][T] (floats).
size_t block_floats(const hta_shape_t &s, int P) {
    const size_t Hp = size_t(s.H / P);
    return size_t(s.B) * s.T * Hp * s.d + size_t(s.B) * Hp * s.T;
}

size_t round16(size_t x) { return (x + 15) & ~size_t(15); }

}  // namespace

struct hta_comm_s {
    nccl_comm_t comm;
    int nranks;
    int rank;
};

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

hta_status_t hta_comm_destroy(hta_comm_t comm) {
    if (comm == nullptr) return HTA_ERR_INVALID_ARGUMENT;
    NcclApi &api = nccl();
    hta_status_t r = HTA_OK;
    if (api.ok && api.CommDestroy(comm->comm) != 0) r = HTA_ERR_NCCL;
    delete comm;
    return r;
}

size_t hta_workspace_size_seqpar(const hta_shape_t *shape_local, int32_t num_sms, int32_t nranks) {
    if (shape_local == nullptr || nranks < 1 || shape_local->H % nranks != 0) return size_t(-1);
    const size_t base = hta_workspace_size(shape_local, num_sms);
    if (base == size_t(-1)) return base;
    const hta_shape_t &s = *shape_local;
    const size_t blk = block_floats(s, nranks) * sizeof(float);
    const size_t es = s.dtype == HTA_BF16 ? 2 : 4;
    const size_t gat = round16(size_t(s.B) * s.T * s.H * s.d * es) + round16(size_t(s.B) * s.H * s.T * 4);
    return round16(base) + 2 * round16(size_t(nranks) * blk) + 2 * gat;
}

hta_status_t hta_forward_seqpar(hta_comm_t comm, const hta_shape_t *shape_local, const void *q,
                                const void *k_cache_local, const void *v_cache_local,
                                const int32_t *cache_seqlens_local, const void *k_tree, const void *v_tree,
                                const uint8_t *mask, int64_t mask_batch_stride, void *o, float *lse_out,
                                int32_t gather_output, void *ws, size_t ws_bytes, hta_stream_t stream) {
    if (comm == nullptr || shape_local == nullptr) return HTA_ERR_INVALID_ARGUMENT;
    const int P = comm->nranks, r = comm->rank;
    if (shape_local->H % P != 0) return HTA_ERR_INVALID_ARGUMENT;
    const size_t need = hta_workspace_size_seqpar(shape_local, 0, P);
    if (need == size_t(-1)) return HTA_ERR_INVALID_ARGUMENT;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t need_dev = hta_workspace_size_seqpar(shape_local, sms, P);
    if (ws == nullptr || ws_bytes < need_dev) return HTA_ERR_WORKSPACE;
    if (!q || !k_cache_local || !v_cache_local || !k_tree || !v_tree || !mask || !o) return HTA_ERR_INVALID_ARGUMENT;
    NcclApi &api = nccl();
    if (!api.ok) return HTA_ERR_NCCL;

    hta_shape_t s = *shape_local;
    const int Hp = s.H / P;
    const int d = s.d;
    const size_t es = s.dtype == HTA_BF16 ? 2 : 4;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);

    // carve the workspace
    uint8_t *w = static_cast<uint8_t *>(ws);
    const size_t base = round16(hta_workspace_size(&s, sms));
    float *prefix_parts = reinterpret_cast<float *>(w);
    const size_t blk = block_floats(s, P);
    float *sendb = reinterpret_cast<float *>(w + base);
    float *recvb = reinterpret_cast<float *>(w + base + round16(P * blk * sizeof(float)));
    uint8_t *gsend = w + base + 2 * round16(P * blk * sizeof(float));
    const size_t gat_o = round16(size_t(s.B) * s.T * s.H * d * es);
    const size_t gat_l = round16(size_t(s.B) * s.H * s.T * 4);

    // 1) local prefix pass -> split partials -> one destination-major partial per row
    hta_status_t rc = seqpar_local_parts(&s, q, k_cache_local, v_cache_local, cache_seqlens_local, prefix_parts,
                                         hta_workspace_size(&s, sms), sendb, P, st);
    if (rc != HTA_OK) return rc;
    // 2) all-to-all of head slices
    const size_t own = size_t(r) * blk;
    if (cudaMemcpyAsync(recvb + own, sendb + own, blk * sizeof(float), cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return HTA_ERR_CUDA;
    if (P > 1) {
        if (api.GroupStart() != 0) return HTA_ERR_NCCL;
        for (int peer = 0; peer < P; ++peer) {
            if (peer == r) continue;
            if (api.Send(sendb + size_t(peer) * blk, blk, kNcclFloat32, peer, comm->comm, st) != 0 ||
                api.Recv(recvb + size_t(peer) * blk, blk, kNcclFloat32, peer, comm->comm, st) != 0) {
                api.GroupEnd();
                return HTA_ERR_NCCL;
            }
        }
        if (api.GroupEnd() != 0) return HTA_ERR_NCCL;
    }
    // 3) merge the P prefix partials with the tree partial of heads [r*Hp, (r+1)*Hp)
    void *o_local = gather_output ? static_cast<void *>(gsend) : o;
    float *lse_local = gather_output ? reinterpret_cast<float *>(gsend + gat_o) : lse_out;
    rc = seqpar_final_merge(&s, P, r, q, k_tree, v_tree, mask, mask_batch_stride, recvb, blk, o_local, lse_local,
                                st);
    if (rc != HTA_OK || !gather_output) return rc;
    // 4) optional all-gather of the head slices, then [P][B,T,Hp,d] -> [B,T,H,d]
    const size_t o_slice = size_t(s.B) * s.T * Hp * d * es;
    const size_t l_slice = size_t(s.B) * Hp * s.T * 4;
    uint8_t *gro = gsend + gat_o + gat_l;
    uint8_t *grl = gro + round16(P * o_slice);
    // LSE slice is packed right after the O slice inside gsend (o_local then lse_local).
    if (api.GroupStart() != 0) return HTA_ERR_NCCL;
    if (api.AllGather(gsend, gro, o_slice, kNcclUint8, comm->comm, st) != 0 ||
        (lse_out != nullptr && api.AllGather(gsend + gat_o, grl, l_slice, kNcclUint8, comm->comm, st) != 0)) {
        api.GroupEnd();
        return HTA_ERR_NCCL;
    }
    if (api.GroupEnd() != 0) return HTA_ERR_NCCL;
    for (int peer = 0; peer < P; ++peer) {
        if (cudaMemcpy2DAsync(static_cast<uint8_t *>(o) + size_t(peer) * Hp * d * es, size_t(s.H) * d * es,
                              gro + peer * o_slice, size_t(Hp) * d * es, size_t(Hp) * d * es, size_t(s.B) * s.T,
                              cudaMemcpyDeviceToDevice, st) != cudaSuccess)
            return HTA_ERR_CUDA;
        if (lse_out != nullptr &&
            cudaMemcpy2DAsync(reinterpret_cast<uint8_t *>(lse_out) + size_t(peer) * Hp * s.T * 4,
                              size_t(s.H) * s.T * 4, grl + peer * l_slice, size_t(Hp) * s.T * 4,
                              size_t(Hp) * s.T * 4, size_t(s.B), cudaMemcpyDeviceToDevice, st) != cudaSuccess)
            return HTA_ERR_CUDA;
    }
    return HTA_OK;
}

}  // extern "C"
