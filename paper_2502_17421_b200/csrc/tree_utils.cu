// tree_utils.cu -- tree mask construction and the greedy accepted path (bit-exact integer work).
//
// Mask (reading Z4): mask[i][j] = 1 iff j == i or j is an ancestor of i.
//   Host: bit-parallel rows, row(i) = row(parent(i)) | bit(i) in index order (parents[i] < i).
//   Device: one thread per node walks its parent chain (depth <= T <= 256).
// Accepted path (reading Z12): forward pass marks accepted nodes
//   (acc[v] = acc[parent] && draft[v] == target_argmax[parent]), a reverse pass computes the
//   longest accepted continuation below every node, and the walk from the root takes, at
//   each level, the smallest-index child that still reaches the maximal length.  That is the
//   lexicographically smallest among the longest accepted paths.
#include <cstring>

#include "hta_internal.h"

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

__global__ void build_mask_kernel(const int32_t *__restrict__ parents, int T, uint8_t *__restrict__ mask) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= T) return;
    uint8_t *row = mask + static_cast<int64_t>(i) * T;
    for (int j = 0; j < T; ++j) row[j] = 0;
    bool ok = true;
    int a = i;
    while (a >= 0) {  // parent indices strictly decrease, so this terminates
        row[a] = 1;
        const int pa = parents[a];
        if (pa < -1 || pa >= a) {
            ok = false;
            break;
        }
        a = pa;
    }
    if (!ok)
        for (int j = 0; j < T; ++j) row[j] = 0;
}

cudaError_t launch_build_mask(const int32_t *parents, int T, uint8_t *mask, cudaStream_t s) {
    if (T <= 0) return cudaSuccess;
    build_mask_kernel<<<(T + 127) / 128, 128, 0, s>>>(parents, T, mask);
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

__global__ void accept_kernel(const int32_t *parents, const int32_t *draft, const int32_t *tgt, int T, int root,
                              int ctx, int32_t *path, int32_t *path_len, int32_t *bonus) {
    __shared__ uint8_t acc[256];
    __shared__ int16_t height[256];
    if (threadIdx.x != 0) return;
    if (accept_impl(parents, draft, tgt, T, root, ctx, path, path_len, bonus, acc, height) != 0) {
        *path_len = -1;
        *bonus = -1;
    }
}

cudaError_t launch_accept(const int32_t *parents, const int32_t *draft, const int32_t *tgt, int T, int root, int ctx,
                          int32_t *path, int32_t *path_len, int32_t *bonus, cudaStream_t s) {
    accept_kernel<<<1, 32, 0, s>>>(parents, draft, tgt, T, root, ctx, path, path_len, bonus);
    return cudaGetLastError();
}

}  // namespace hta
