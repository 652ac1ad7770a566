// prefix_simt.cu -- fp32 prefix pass on the FP32 (FFMA) pipe.
//
// Same contract as the tcgen05 kernel (unmasked attention of the tree queries over a KV split,
// PAPER.md:195-201, normalised partial + natural-log LSE) for dtype fp32,
// where TF32 tensor cores (10-bit mantissa) could not meet the 1e-5 relative bound
// (BASELINE.json north_star).  One warp per (query row, split); each lane holds d/32
// elements of q; 8 keys per step give 8 independent shuffle reductions; the running max is
// updated once per step with accurate expf.  Dot products and the running max are kept in
// fp64 (B200 runs FP64 at half the FP32 rate): fp32 rounding of a 128-term dot product is
// ~1e-5 of a logit near 100, which would spend the whole 1e-5 budget on extreme inputs.
#include "hta_internal.h"
#include "ptx_sm100.cuh"

namespace hta {

template <int D>
__global__ void __launch_bounds__(128) prefix_simt_kernel(const PrefixParams p) {
    constexpr int E = D / 32;
    constexpr int U = 16;  // keys in flight per round trip (= kSimtBlock: one round trip per split block)
    const int row = blockIdx.x * 4 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    pdl_launch_dependents();  // the dependent tree/merge grid may start its tree pass now
    if (row >= p.B * p.T * p.H) return;
    const int h = row % p.H;
    const int t = (row / p.H) % p.T;
    const int b = row / (p.H * p.T);
    const int g = h / p.G;
    const int split = blockIdx.y;

    int64_t n_b = p.N_max;
    if (p.seqlens != nullptr) {
        n_b = p.seqlens[b];
        n_b = n_b < 0 ? 0 : (n_b > p.N_max ? p.N_max : n_b);
    }
    const int64_t lo = static_cast<int64_t>(split) * p.tiles_per_split * kSimtBlock;
    int64_t hi = lo + static_cast<int64_t>(p.tiles_per_split) * kSimtBlock;
    if (hi > n_b || split == p.splits - 1) hi = n_b;  // the last split runs to the length

    const float *q = static_cast<const float *>(p.q) + b * p.qs0 + t * p.qs1 + h * p.qs2 + lane * E;
    const float *K = static_cast<const float *>(p.k) + b * p.ks0 + g * p.ks2 + lane * E;
    const float *V = static_cast<const float *>(p.v) + b * p.ks0 + g * p.ks2 + lane * E;
    float qv[E], o[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        qv[e] = q[e];
        o[e] = 0.f;
    }
    double m = -INFINITY;
    float l = 0.f;
    for (int64_t j = lo; j < hi; j += U) {
        // the K and V rows of U keys in flight at once: one round trip per U keys
        float kk[U][E], vv[U][E];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t jj = j + u < hi ? j + u : j;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                kk[u][e] = K[jj * p.ks1 + e];
                vv[u][e] = V[jj * p.ks1 + e];
            }
        }
        double z[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            double acc = 0.0;
#pragma unroll
            for (int e = 0; e < E; ++e) acc = fma(static_cast<double>(qv[e]), static_cast<double>(kk[u][e]), acc);
            z[u] = acc;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1)
#pragma unroll
            for (int u = 0; u < U; ++u) z[u] += __shfl_xor_sync(0xffffffffu, z[u], off);
        double mx = m;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            z[u] = (j + u < hi) ? z[u] * static_cast<double>(p.scale) : -INFINITY;
            mx = z[u] > mx ? z[u] : mx;
        }
        const float corr = expf(static_cast<float>(m - mx));  // m = -inf on the first step -> 0
        l *= corr;
#pragma unroll
        for (int e = 0; e < E; ++e) o[e] *= corr;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const float w = (j + u < hi) ? expf(static_cast<float>(z[u] - mx)) : 0.f;
            l += w;
#pragma unroll
            for (int e = 0; e < E; ++e) o[e] = fmaf(w, vv[u][e], o[e]);
        }
        m = mx;
    }
    float *dst = p.o_out + static_cast<int64_t>(split) * p.o_split_stride +
                 ((static_cast<int64_t>(b) * p.T + t) * p.H + h) * D + lane * E;
    const float inv = l > 0.f ? 1.0f / l : 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) dst[e] = o[e] * inv;
    if (lane == 0)
        p.lse_out[static_cast<int64_t>(split) * p.lse_split_stride + (static_cast<int64_t>(b) * p.H + h) * p.T + t] =
            l > 0.f ? static_cast<float>(m + static_cast<double>(logf(l))) : -INFINITY;
}

cudaError_t launch_prefix_simt(const PrefixParams &p, cudaStream_t s) {
    const int rows = p.B * p.T * p.H;
    dim3 grid((rows + 3) / 4, p.splits);
    if (p.d == 128)
        prefix_simt_kernel<128><<<grid, 128, 0, s>>>(p);
    else if (p.d == 64)
        prefix_simt_kernel<64><<<grid, 128, 0, s>>>(p);
    else
        return cudaErrorInvalidValue;
    return cudaGetLastError();
}

}  // namespace hta
