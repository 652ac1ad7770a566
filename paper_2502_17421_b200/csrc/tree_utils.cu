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

cudaError_t launch_build_mask(const int32_t *parents, int T, uint8_t *mask, cudaStream_t s) {
    return launch_tree_step(parents, T, mask, nullptr, nullptr, 0, 0, nullptr, nullptr, nullptr, s);
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

// Device version of both utilities: one block, thread v = node v (T <= 256), no loop over the
// tree depth other than the ancestor walk.
//  * Mask: thread v walks its parent chain in shared memory and collects its ancestor set (itself
//    included) as a 256-bit mask anc(v) = row v of the tree mask (Z4).
//  * Accept (Z12), bit-parallel: with match(u) = draft[u] == target[parent(u)] (context_argmax for
//    a node without parent; the root always matches in root mode) as a 256-bit set M, the path of
//    node v is P(v) = anc(v) (minus the ancestors of the root in root mode, where v must lie in
//    the root's subtree) and v is accepted iff P(v) is inside M.  Its length is popcount P(v).
//    Among the longest accepted paths the lexicographically smallest node sequence is the one
//    whose lowest differing node is its own, i.e. the largest mask when bit 0 of word 0 is the
//    most significant bit: a block-wide max over the bit-reversed masks.  The path is then the
//    winner's set bits in ascending order (one thread per node writes its position).
// The kernel lets the next kernel on the stream launch at once (programmatic dependent launch:
// hta_forward's prefix pass, which reads neither the mask nor the path, overlaps its prologue);
// a kernel that reads these outputs does so after its griddepcontrol.wait.
__global__ void __launch_bounds__(256) tree_step_kernel(const int32_t *__restrict__ parents, int T,
                                                        uint8_t *__restrict__ mask, const int32_t *__restrict__ draft,
                                                        const int32_t *__restrict__ tgt, int root, int ctx,
                                                        int32_t *path, int32_t *path_len, int32_t *bonus) {
    __shared__ int32_t par[256], tg[256];
    __shared__ uint32_t match_w[8], err_w[8], root_anc[8];
    __shared__ uint32_t best_key[8][9];  // per warp: its best (depth, 8 words of bit-reversed mask)
    __shared__ int best_node[8];
    const int v = threadIdx.x;
    const int lane = v & 31, warp = v >> 5;
    pdl_launch_dependents();
    const bool in = v < T;
    const bool do_acc = draft != nullptr;
    // every input load at once (one round trip)
    int pa = -1, dr = 0;
    if (in) {
        pa = parents[v];
        if (do_acc) {
            dr = draft[v];
            tg[v] = tgt[v];
        }
        par[v] = pa;
    }
    const bool bad = in && (pa < -1 || pa >= v);
    __syncthreads();
    // match bit of every node (its draft token vs the target's argmax at its parent)
    const int tgt_par = (do_acc && in && !bad) ? (pa >= 0 ? tg[pa] : ctx) : 0;
    const bool mt = do_acc && in && !bad && (root >= 0 ? (v == root || (pa >= 0 && dr == tgt_par)) : dr == tgt_par);
    const uint32_t mw = __ballot_sync(0xffffffffu, mt);
    const uint32_t ew = __ballot_sync(0xffffffffu, bad);
    if (lane == 0) {
        match_w[warp] = mw;
        err_w[warp] = ew;
    }
    if (do_acc) __syncthreads();
    uint32_t bits[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    bool ok = in && !bad;
    if (ok) {
        int a = v;
        while (a >= 0) {  // parent indices strictly decrease, so this terminates
            bits[a >> 5] |= 1u << (a & 31);
            const int pp = par[a];
            if (pp < -1 || pp >= a) {
                ok = false;
                break;
            }
            a = pp;
        }
        if (!ok)
#pragma unroll
            for (int w = 0; w < 8; ++w) bits[w] = 0u;
    }
    if (mask != nullptr && in) {
        uint8_t *row = mask + static_cast<int64_t>(v) * T;
        if ((T & 3) == 0) {  // rows are 4-byte aligned: store 4 mask bytes at a time
            for (int j = 0; j < T; j += 4) {
                const uint32_t nib = (bits[j >> 5] >> (j & 31)) & 0xFu;
                *reinterpret_cast<uint32_t *>(row + j) =
                    (nib & 1u) | ((nib & 2u) << 7) | ((nib & 4u) << 14) | ((nib & 8u) << 21);
            }
        } else {
            for (int j = 0; j < T; ++j) row[j] = static_cast<uint8_t>((bits[j >> 5] >> (j & 31)) & 1u);
        }
    }
    if (!do_acc) return;
    bool any_err = root < -1 || root >= T;
#pragma unroll
    for (int w = 0; w < 8; ++w) any_err |= err_w[w] != 0u;
    if (any_err) {
        if (v == 0) {
            *path_len = -1;
            *bonus = -1;
        }
        return;
    }
    if (root >= 0 && v == root) {
#pragma unroll
        for (int w = 0; w < 8; ++w) root_anc[w] = bits[w] & ~(w == (root >> 5) ? 1u << (root & 31) : 0u);
    }
    __syncthreads();
    // this node's path and whether it is accepted
    bool accepted = in;
    int depth = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        if (root >= 0) bits[w] &= ~root_anc[w];
        accepted &= (bits[w] & ~match_w[w]) == 0u;
        depth += __popc(bits[w]);
    }
    if (root >= 0) accepted &= ((bits[root >> 5] >> (root & 31)) & 1u) != 0u;
    // key: depth, then the bit-reversed mask words (lexicographically smallest path = largest key)
    uint32_t key[9];
    key[0] = accepted ? static_cast<uint32_t>(depth) : 0u;
#pragma unroll
    for (int w = 0; w < 8; ++w) key[w + 1] = accepted ? __brev(bits[w]) : 0u;
    int node = accepted ? v : -1;
    auto greater = [](const uint32_t (&a)[9], const uint32_t (&b)[9]) {
#pragma unroll
        for (int w = 0; w < 9; ++w)
            if (a[w] != b[w]) return a[w] > b[w];
        return false;
    };
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        uint32_t other[9];
#pragma unroll
        for (int w = 0; w < 9; ++w) other[w] = __shfl_xor_sync(0xffffffffu, key[w], off);
        const int on = __shfl_xor_sync(0xffffffffu, node, off);
        if (greater(other, key)) {
#pragma unroll
            for (int w = 0; w < 9; ++w) key[w] = other[w];
            node = on;
        }
    }
    if (lane == 0) {
#pragma unroll
        for (int w = 0; w < 9; ++w) best_key[warp][w] = key[w];
        best_node[warp] = node;
    }
    __syncthreads();
    // every thread reduces the (at most 8) warp winners the same way
    uint32_t bk[9];
    int bn = -1;
#pragma unroll
    for (int w = 0; w < 9; ++w) bk[w] = 0u;
    for (int i = 0; i < (T + 31) / 32; ++i) {
        uint32_t c[9];
#pragma unroll
        for (int w = 0; w < 9; ++w) c[w] = best_key[i][w];
        if (greater(c, bk)) {
#pragma unroll
            for (int w = 0; w < 9; ++w) bk[w] = c[w];
            bn = best_node[i];
        }
    }
    const int L = static_cast<int>(bk[0]);
    if (L == 0 || bn < 0) {  // forest mode with no accepted depth-1 node
        if (v == 0) {
            *path_len = 0;
            *bonus = ctx;
        }
        return;
    }
    // the winner's path: its mask (bit-reversed back), one thread per member node
    if (in && ((__brev(bk[1 + (v >> 5)]) >> (v & 31)) & 1u)) {
        int pos = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            const uint32_t m = __brev(bk[1 + w]);
            if (w < (v >> 5)) pos += __popc(m);
            else if (w == (v >> 5)) pos += __popc(m & ((1u << (v & 31)) - 1u));
        }
        path[pos] = v;
    }
    if (v == 0) {
        *path_len = L;
        *bonus = tg[bn];
    }
}

cudaError_t launch_tree_step(const int32_t *parents, int T, uint8_t *mask, const int32_t *draft, const int32_t *tgt,
                             int root, int ctx, int32_t *path, int32_t *path_len, int32_t *bonus, cudaStream_t s) {
    if (T <= 0 || T > 256) return cudaErrorInvalidValue;
    tree_step_kernel<<<1, 256, 0, s>>>(parents, T, mask, draft, tgt, root, ctx, path, path_len, bonus);
    return cudaGetLastError();
}

cudaError_t launch_accept(const int32_t *parents, const int32_t *draft, const int32_t *tgt, int T, int root, int ctx,
                          int32_t *path, int32_t *path_len, int32_t *bonus, cudaStream_t s) {
    return launch_tree_step(parents, T, nullptr, draft, tgt, root, ctx, path, path_len, bonus, s);
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
        const int32_t n0 = seqlens[b];
        s_n = n0 < 0 ? 0 : n0;  // a negative committed length counts as empty
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
