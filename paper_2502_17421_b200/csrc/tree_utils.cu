// tree_utils.cu -- tree mask construction and the greedy accepted path (bit-exact integer work).
//
// Mask (reading Z4): mask[i][j] = 1 iff j == i or j is an ancestor of i.
//   Host: bit-parallel rows, row(i) = row(parent(i)) | bit(i) in index order (parents[i] < i).
//   Device: one thread per node walks its parent chain (depth <= T <= 256).
// Accepted path (reading Z12).  Host: forward pass marks accepted nodes
//   (acc[v] = acc[parent] && draft[v] == target_argmax[parent]), a reverse pass computes the
//   longest accepted continuation below every node, and the walk from the root takes, at
//   each level, the smallest-index child that still reaches the maximal length -- the
//   lexicographically smallest among the longest accepted paths.  Device: the same result
//   computed by a block of T threads (see accept_kernel).
#include <cstring>

#include "hta_internal.h"
#include "ptx_sm100.cuh"

namespace hta {

// ----------------------------------------------------------------------------- mask

int host_build_mask(const int32_t *parents, int T, uint8_t *mask) {
    constexpr int W = 4;  // 4 x 64 bits = 256 nodes
    uint64_t rows[256][W];
    for (int i = 0; i < T; ++i)
        if (parents[i] < -1 || parents[i] >= i) return -1;
    for (int i = 0; i < T; ++i) {
        const int pa = parents[i];
        for (int w = 0; w < W; ++w) rows[i][w] = pa >= 0 ? rows[pa][w] : 0ull;
        rows[i][i >> 6] |= 1ull << (i & 63);
        for (int j = 0; j < T; ++j) mask[static_cast<int64_t>(i) * T + j] = (rows[i][j >> 6] >> (j & 63)) & 1ull;
    }
    return 0;
}

__global__ void __launch_bounds__(256) build_mask_kernel(const int32_t *__restrict__ parents, int T,
                                                         uint8_t *__restrict__ mask) {
    __shared__ int32_t par[256];
    const int i = threadIdx.x;
    // the next kernel (hta_forward's prefix pass, which needs no mask) may start its prologue now;
    // whoever reads the mask does so after griddepcontrol.wait
    pdl_launch_dependents();
    if (i < T) par[i] = parents[i];  // one coalesced load; the chain walks below hit smem
    __syncthreads();
    if (i >= T) return;
    uint32_t bits[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    bool ok = true;
    int a = i;
    while (a >= 0) {  // parent indices strictly decrease, so this terminates
        bits[a >> 5] |= 1u << (a & 31);
        const int pa = par[a];
        if (pa < -1 || pa >= a) {
            ok = false;
            break;
        }
        a = pa;
    }
    uint8_t *row = mask + static_cast<int64_t>(i) * T;
    if (!ok)
        for (int w = 0; w < 8; ++w) bits[w] = 0u;
    if ((T & 3) == 0) {  // rows are 4-byte aligned: store 4 mask bytes at a time
        for (int j = 0; j < T; j += 4) {
            const uint32_t nib = (bits[j >> 5] >> (j & 31)) & 0xFu;
            const uint32_t word = (nib & 1u) | ((nib & 2u) << 7) | ((nib & 4u) << 14) | ((nib & 8u) << 21);
            *reinterpret_cast<uint32_t *>(row + j) = word;
        }
    } else {
        for (int j = 0; j < T; ++j) row[j] = static_cast<uint8_t>((bits[j >> 5] >> (j & 31)) & 1u);
    }
}

cudaError_t launch_build_mask(const int32_t *parents, int T, uint8_t *mask, cudaStream_t s) {
    if (T <= 0 || T > 256) return cudaErrorInvalidValue;
    build_mask_kernel<<<1, 256, 0, s>>>(parents, T, mask);
    return cudaGetLastError();
}

// ----------------------------------------------------------------------------- accept

// Shared by host and device: returns -1 on invalid input.
__host__ __device__ static int accept_impl(const int32_t *parents, const int32_t *draft, const int32_t *tgt, int T,
                                           int root, int ctx, int32_t *path, int32_t *path_len, int32_t *bonus,
                                           uint8_t *acc, int16_t *height) {
    if (T < 1 || T > 256 || root < -1 || root >= T) return -1;
    for (int i = 0; i < T; ++i)
        if (parents[i] < -1 || parents[i] >= i) return -1;
    for (int v = 0; v < T; ++v) {
        const int pa = parents[v];
        if (root >= 0)
            acc[v] = (v == root) || (v > root && pa >= 0 && acc[pa] && draft[v] == tgt[pa]);
        else
            acc[v] = pa < 0 ? (draft[v] == ctx) : (acc[pa] && draft[v] == tgt[pa]);
        height[v] = 0;
    }
    for (int v = T - 1; v >= 0; --v) {
        const int pa = parents[v];
        if (acc[v] && pa >= 0 && acc[pa] && (root < 0 || v != root) && height[v] + 1 > height[pa])
            height[pa] = static_cast<int16_t>(height[v] + 1);
    }
    int len = 0, cur = -1;
    if (root >= 0) {
        cur = root;
    } else {
        int best = -1;
        for (int v = 0; v < T; ++v)
            if (parents[v] < 0 && acc[v] && height[v] > best) best = height[v];
        for (int v = 0; v < T && best >= 0; ++v)
            if (parents[v] < 0 && acc[v] && height[v] == best) {
                cur = v;
                break;
            }
    }
    if (cur < 0) {
        *path_len = 0;
        *bonus = ctx;
        return 0;
    }
    path[len++] = cur;
    while (height[cur] > 0) {
        int nxt = -1;
        for (int c = cur + 1; c < T; ++c)
            if (parents[c] == cur && acc[c] && height[c] == height[cur] - 1) {
                nxt = c;
                break;
            }
        if (nxt < 0) break;  // unreachable for consistent heights
        cur = nxt;
        path[len++] = cur;
    }
    *path_len = len;
    *bonus = tgt[cur];
    return 0;
}

int host_accept(const int32_t *parents, const int32_t *draft, const int32_t *tgt, int T, int root, int ctx,
                int32_t *path, int32_t *path_len, int32_t *bonus) {
    uint8_t acc[256];
    int16_t height[256];
    return accept_impl(parents, draft, tgt, T, root, ctx, path, path_len, bonus, acc, height);
}

// Device version: one block, thread v = node v.  Pointer jumping over the parent chains gives,
// for every node, whether its whole root path matches (AND of the per-node match bits) and its
// depth, in ceil(log2 T) rounds; the maximal accepted depth is a block max; the nodes on some
// maximal accepted path are marked by walking up from the maximal endpoints; the walk from
// the root then takes the smallest marked child at each level (lexicographically smallest).
__global__ void __launch_bounds__(256) accept_kernel(const int32_t *parents, const int32_t *draft,
                                                     const int32_t *tgt, int T, int root, int ctx, int32_t *path,
                                                     int32_t *path_len, int32_t *bonus) {
    __shared__ int32_t par[256], tg[256], anc[256], dep[256];
    __shared__ uint8_t ok[256], good[256];
    __shared__ int s_err, s_L, s_next;
    const int v = threadIdx.x;
    const bool in = v < T;
    if (v == 0) {
        s_err = 0;
        s_L = 0;
    }
    int pa = -1, dr = 0;
    if (in) {
        pa = parents[v];
        dr = draft[v];
        tg[v] = tgt[v];
        par[v] = pa;
    }
    __syncthreads();
    if (in && (pa < -1 || pa >= v)) atomicOr(&s_err, 1);
    if (v == 0 && (root < -1 || root >= T)) atomicOr(&s_err, 1);
    // match bit and first jump target of every node
    int my_anc = -1, my_dep = 0;
    uint8_t my_ok = 0;
    if (in) {
        my_dep = 1;
        pa = (pa >= -1 && pa < v) ? pa : -1;  // invalid input is reported below; never index with it
        if (root >= 0) {
            my_ok = (v == root) ? 1 : (pa >= 0 && dr == tg[pa]);
            my_anc = (v == root) ? -1 : pa;
        } else {
            my_ok = pa < 0 ? (dr == ctx) : (dr == tg[pa]);
            my_anc = pa;
        }
        anc[v] = my_anc;
        dep[v] = my_dep;
        ok[v] = my_ok;
    }
    __syncthreads();
    if (s_err) {
        if (v == 0) {
            *path_len = -1;
            *bonus = -1;
        }
        return;
    }
    for (int round = 0; round < 8; ++round) {  // 2^8 = 256 >= any depth
        int a2 = my_anc, d2 = my_dep;
        uint8_t o2 = my_ok;
        if (in && my_anc >= 0) {
            o2 = my_ok & ok[my_anc];
            d2 = my_dep + dep[my_anc];
            a2 = anc[my_anc];
        }
        __syncthreads();
        if (in) {
            my_anc = a2;
            my_dep = d2;
            my_ok = o2;
            anc[v] = a2;
            dep[v] = d2;
            ok[v] = o2;
        }
        __syncthreads();
    }
    // in root mode only root's subtree counts: every other chain ends at a top node with ok = 0
    if (in && my_ok) atomicMax(&s_L, my_dep);
    if (in) good[v] = 0;
    __syncthreads();
    const int L = s_L;
    if (L == 0) {  // forest mode with no accepted depth-1 node
        if (v == 0) {
            *path_len = 0;
            *bonus = ctx;
        }
        return;
    }
    if (in && my_ok && my_dep == L) {  // mark the nodes of every maximal accepted path
        int a = v;
        while (a >= 0 && (root < 0 || a != root)) {
            good[a] = 1;
            a = par[a];
        }
        if (root >= 0) good[root] = 1;
    }
    __syncthreads();
    int cur;
    if (root >= 0) {
        cur = root;
    } else {
        if (v == 0) s_next = 0x7fffffff;
        __syncthreads();
        if (in && par[v] < 0 && good[v]) atomicMin(&s_next, v);
        __syncthreads();
        cur = s_next;
    }
    if (v == 0) path[0] = cur;
    for (int len = 1; len < L; ++len) {
        __syncthreads();
        if (v == 0) s_next = 0x7fffffff;
        __syncthreads();
        if (in && par[v] == cur && good[v]) atomicMin(&s_next, v);
        __syncthreads();
        cur = s_next;
        if (v == 0) path[len] = cur;
    }
    if (v == 0) {
        *path_len = L;
        *bonus = tg[cur];
    }
}

cudaError_t launch_accept(const int32_t *parents, const int32_t *draft, const int32_t *tgt, int T, int root, int ctx,
                          int32_t *path, int32_t *path_len, int32_t *bonus, cudaStream_t s) {
    if (T < 1 || T > 256) return cudaErrorInvalidValue;
    accept_kernel<<<1, 256, 0, s>>>(parents, draft, tgt, T, root, ctx, path, path_len, bonus);
    return cudaGetLastError();
}

// ----------------------------------------------------------------------------- commit

// One CTA per batch entry b: path_len[b] rows of H_kv * d elements each (K and V) copied as
// 16-byte chunks by all threads, then the committed length updated by thread 0 after a barrier
// (so seqlens_out may alias cache_seqlens).
__global__ void __launch_bounds__(256) commit_kv_kernel(const int32_t *__restrict__ path, int64_t path_stride,
                                                        const int32_t *__restrict__ path_len, const uint8_t *kt,
                                                        const uint8_t *vt, uint8_t *kc, uint8_t *vc,
                                                        const int32_t *seqlens, int32_t *seqlens_out, CommitGeom gm) {
    const int b = blockIdx.x;
    __shared__ int s_rows;
    __shared__ int s_node[256];
    __shared__ int64_t s_n;
    // every load at once (one round trip): the path entries, the committed length, the path length
    if (threadIdx.x < gm.T) s_node[threadIdx.x] = path[b * path_stride + threadIdx.x];
    if (threadIdx.x == 0) {
        s_n = seqlens[b];
        s_rows = path_len[b];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int L = s_rows > 0 ? s_rows : 0;
        if (L > gm.T) L = gm.T;
        int rows = 0;
        while (rows < L && s_n + rows < gm.N_max && s_node[rows] >= 0 && s_node[rows] < gm.T)
            ++rows;  // stop at N_max or at the first invalid node
        s_rows = rows;
    }
    __syncthreads();
    const int rows = s_rows;
    const int64_t n = s_n;
    const int chunks = gm.row_bytes / 16;  // per head: d * esize / 16
    for (int idx = threadIdx.x; idx < rows * gm.H_kv * chunks; idx += blockDim.x) {
        const int c = idx % chunks;
        const int hh = (idx / chunks) % gm.H_kv;
        const int i = idx / (chunks * gm.H_kv);
        const int node = s_node[i];
        const int64_t src = (b * gm.ts0 + node * gm.ts1 + hh * gm.ts2) * gm.esize + c * 16;
        const int64_t dst = (b * gm.ks0 + (n + i) * gm.ks1 + hh * gm.ks2) * gm.esize + c * 16;
        *reinterpret_cast<uint4 *>(kc + dst) = *reinterpret_cast<const uint4 *>(kt + src);
        *reinterpret_cast<uint4 *>(vc + dst) = *reinterpret_cast<const uint4 *>(vt + src);
    }
    __syncthreads();
    if (threadIdx.x == 0) seqlens_out[b] = static_cast<int32_t>(n + rows);
}

cudaError_t launch_commit_kv(const int32_t *path, int64_t path_stride, const int32_t *path_len, const void *kt,
                             const void *vt, void *kc, void *vc, const int32_t *seqlens, int32_t *seqlens_out,
                             const CommitGeom &gm, int B, cudaStream_t s) {
    commit_kv_kernel<<<B, 256, 0, s>>>(path, path_stride, path_len, static_cast<const uint8_t *>(kt),
                                       static_cast<const uint8_t *>(vt), static_cast<uint8_t *>(kc),
                                       static_cast<uint8_t *>(vc), seqlens, seqlens_out, gm);
    return cudaGetLastError();
}

}  // namespace hta
