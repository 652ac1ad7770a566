// tree_merge.cu -- the tree pass and the LSE merge, one warp per output row (b, t, h).
//
// Tree pass: query (b,t,h) attends to the speculative keys s with
// mask[b][t][s] != 0 only.  The visible keys of a row are found with one ballot per 32 mask
// bytes; each key row (d contiguous elements) is read by the whole warp with one vectorised
// load per lane, dot products are reduced with xor shuffles (four keys in flight), and an
// online softmax in fp32 (natural exp) gives the normalised tree partial and its LSE.
// The tree is tiny (<= depth+1 visible keys per row for beam trees), so this pass is
// latency-bound; it needs no tensor cores and no shared memory.
//
// Merge (Appendix C): the n prefix partials (split-KV and/or
// sequence-parallel ranks) and the tree partial are combined in one max-shifted pass
// (reading Z11): M = max LSE_i, W = sum exp(LSE_i - M), O = sum exp(LSE_i - M) O_i / W,
// LSE = M + log W.  All-sentinel rows give O = 0, LSE = -inf without NaN.
//
// Precision: bf16 inputs accumulate dot products in fp32 (bf16 x bf16 products are exact in
// fp32); fp32 inputs accumulate them in fp64 so the 1e-5 relative bound holds even for logits
// near 100 (value distribution V2), where fp32 rounding of a 128-term dot product alone is
// ~1e-5 of a logit.
#include <cuda_bf16.h>

#include <type_traits>

#include "hta_internal.h"
#include "ptx_sm100.cuh"

namespace hta {

template <typename T, int E>
struct VecIO;
template <>
struct VecIO<float, 4> {
    static __device__ __forceinline__ void load(const float *p, float (&v)[4]) {
        const float4 x = *reinterpret_cast<const float4 *>(p);
        v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    }
    static __device__ __forceinline__ void store(float *p, const float (&v)[4]) {
        *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
    }
};
template <>
struct VecIO<float, 2> {
    static __device__ __forceinline__ void load(const float *p, float (&v)[2]) {
        const float2 x = *reinterpret_cast<const float2 *>(p);
        v[0] = x.x; v[1] = x.y;
    }
    static __device__ __forceinline__ void store(float *p, const float (&v)[2]) {
        *reinterpret_cast<float2 *>(p) = make_float2(v[0], v[1]);
    }
};
template <>
struct VecIO<__nv_bfloat16, 4> {
    static __device__ __forceinline__ void load(const __nv_bfloat16 *p, float (&v)[4]) {
        const uint2 x = *reinterpret_cast<const uint2 *>(p);
        const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162 *>(&x.x);
        const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162 *>(&x.y);
        v[0] = __low2float(a); v[1] = __high2float(a); v[2] = __low2float(b); v[3] = __high2float(b);
    }
    static __device__ __forceinline__ void store(__nv_bfloat16 *p, const float (&v)[4]) {
        uint2 x;
        x.x = pack_bf16x2(v[0], v[1]);
        x.y = pack_bf16x2(v[2], v[3]);
        *reinterpret_cast<uint2 *>(p) = x;
    }
};
template <>
struct VecIO<__nv_bfloat16, 2> {
    static __device__ __forceinline__ void load(const __nv_bfloat16 *p, float (&v)[2]) {
        const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162 *>(p);
        v[0] = __low2float(a); v[1] = __high2float(a);
    }
    static __device__ __forceinline__ void store(__nv_bfloat16 *p, const float (&v)[2]) {
        *reinterpret_cast<uint32_t *>(p) = pack_bf16x2(v[0], v[1]);
    }
};

// Tree pass of one output row: normalised tree partial in ot[] and its natural-log LSE.
template <typename Tin, int D>
__device__ __forceinline__ float tree_row(const TreeMergeParams &p, int b, int t, int h, int lane,
                                          float (&ot)[D / 32]) {
    constexpr int E = D / 32;
    const int g = h / p.G;
#pragma unroll
    for (int e = 0; e < E; ++e) ot[e] = 0.f;
    float qv[E];
    VecIO<Tin, E>::load(static_cast<const Tin *>(p.q) + b * p.qs0 + t * p.qs1 + h * p.qs2 + lane * E, qv);
    const Tin *Kt = static_cast<const Tin *>(p.kt) + b * p.ts0 + g * p.ts2 + lane * E;
    const Tin *Vt = static_cast<const Tin *>(p.vt) + b * p.ts0 + g * p.ts2 + lane * E;
    const uint8_t *mrow = p.mask + b * p.mask_bs + static_cast<int64_t>(t) * p.T;
    using Acc = typename std::conditional<std::is_same<Tin, float>::value, double, float>::type;
    float l = 0.f;
    Acc m_acc = static_cast<Acc>(-INFINITY);  // running max kept at accumulation precision
    for (int c0 = 0; c0 < p.T; c0 += 32) {
        const int s = c0 + lane;
        uint32_t bits = __ballot_sync(0xffffffffu, s < p.T && mrow[s] != 0);
        while (bits) {
            int idx[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (bits) {
                    idx[u] = c0 + __ffs(bits) - 1;
                    bits &= bits - 1;
                } else {
                    idx[u] = -1;
                }
            }
            Acc z[4];
            float vv[4][E];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                float kk[E];
                const int sidx = idx[u] < 0 ? idx[0] : idx[u];
                VecIO<Tin, E>::load(Kt + sidx * p.ts1, kk);
                VecIO<Tin, E>::load(Vt + sidx * p.ts1, vv[u]);
                Acc a = 0;
#pragma unroll
                for (int e = 0; e < E; ++e) a = fma(static_cast<Acc>(qv[e]), static_cast<Acc>(kk[e]), a);
                z[u] = a;
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1)
#pragma unroll
                for (int u = 0; u < 4; ++u) z[u] += __shfl_xor_sync(0xffffffffu, z[u], off);
            Acc mx = m_acc;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                z[u] = idx[u] >= 0 ? z[u] * static_cast<Acc>(p.scale) : static_cast<Acc>(-INFINITY);
                mx = z[u] > mx ? z[u] : mx;
            }
            const float corr = expf(static_cast<float>(m_acc - mx));
            l *= corr;
#pragma unroll
            for (int e = 0; e < E; ++e) ot[e] *= corr;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float w = expf(static_cast<float>(z[u] - mx));  // 0 for unused slots
                l += w;
#pragma unroll
                for (int e = 0; e < E; ++e) ot[e] = fmaf(w, vv[u][e], ot[e]);
            }
            m_acc = mx;
        }
    }
    if (!(l > 0.f)) return -INFINITY;
    const float inv = 1.0f / l;
#pragma unroll
    for (int e = 0; e < E; ++e) ot[e] *= inv;
    return static_cast<float>(m_acc + static_cast<Acc>(logf(l)));
}

// One warp per output row, R rows per warp (rows warp, warp + W, ...; W = total warps).  The
// tree passes of all R rows run first -- with programmatic dependent launch they overlap the
// prefix kernel, which lets this grid start early -- and the merges with the prefix partials
// run after griddepcontrol.wait.
template <typename Tin, typename Tout, int D, int R>
__global__ void __launch_bounds__(128) tree_merge_kernel(const TreeMergeParams p) {
    constexpr int E = D / 32;
    const int nrows = p.B * p.T * p.Hr;
    const int warp_id = blockIdx.x * 4 + (threadIdx.x >> 5);
    const int nwarps = gridDim.x * 4;
    const int lane = threadIdx.x & 31;

    // ------------------------------------------------------------- tree pass
    float ot[R][E], lse_t[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
        const int row = warp_id + k * nwarps;
        lse_t[k] = -INFINITY;
#pragma unroll
        for (int e = 0; e < E; ++e) ot[k][e] = 0.f;
        if (row < nrows && p.do_tree) {
            const int hl = row % p.Hr, t = (row / p.Hr) % p.T, b = row / (p.Hr * p.T);
            lse_t[k] = tree_row<Tin, D>(p, b, t, p.h0 + hl, lane, ot[k]);
        }
    }
    if (p.n_parts > 0) pdl_wait_primary();  // the partials come from the preceding prefix kernel

    // ------------------------------------------------------------- merge with prefix parts
#pragma unroll
    for (int k = 0; k < R; ++k) {
        const int row = warp_id + k * nwarps;
        if (row >= nrows) break;
        const int hl = row % p.Hr, t = (row / p.Hr) % p.T, b = row / (p.Hr * p.T);
        float out[E];
        float lse_out = lse_t[k];
#pragma unroll
        for (int e = 0; e < E; ++e) out[e] = ot[k][e];
        if (p.n_parts > 0) {
            const int64_t lrow = (static_cast<int64_t>(b) * p.Hr + hl) * p.T + t;
            const int64_t orow = ((static_cast<int64_t>(b) * p.T + t) * p.Hr + hl) * D + lane * E;
            float mx = lse_t[k];
            for (int s = lane; s < p.n_parts; s += 32) mx = fmaxf(mx, p.lse_parts[s * p.lse_part_stride + lrow]);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
            if (mx == -INFINITY) {
#pragma unroll
                for (int e = 0; e < E; ++e) out[e] = 0.f;
                lse_out = -INFINITY;
            } else {
                float W = 0.f, acc[E];
                const float wt = expf(lse_t[k] - mx);  // 0 when the tree part is a sentinel
                W += wt;
#pragma unroll
                for (int e = 0; e < E; ++e) acc[e] = wt * ot[k][e];
                for (int s0 = 0; s0 < p.n_parts; s0 += 32) {
                    const int s = s0 + lane;
                    const float ws = s < p.n_parts ? expf(p.lse_parts[s * p.lse_part_stride + lrow] - mx) : 0.f;
                    const int cnt = min(32, p.n_parts - s0);
                    // eight partial rows in flight per lane (the partials are L2-resident)
                    for (int u = 0; u < cnt; u += 8) {
                        float w8[8], v8[8][E];
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            w8[j] = __shfl_sync(0xffffffffu, ws, (u + j) & 31);
                            if (u + j < cnt) {
                                VecIO<float, E>::load(p.o_parts + (s0 + u + j) * p.o_part_stride + orow, v8[j]);
                            } else {
                                w8[j] = 0.f;
#pragma unroll
                                for (int e = 0; e < E; ++e) v8[j][e] = 0.f;
                            }
                        }
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            W += w8[j];
#pragma unroll
                            for (int e = 0; e < E; ++e) acc[e] = fmaf(w8[j], v8[j][e], acc[e]);
                        }
                    }
                }
                const float inv = 1.0f / W;
#pragma unroll
                for (int e = 0; e < E; ++e) out[e] = acc[e] * inv;
                lse_out = mx + logf(W);
            }
        }
        const int blk = hl / p.out_hb, hh = hl % p.out_hb;
        Tout *dst = static_cast<Tout *>(p.o) + blk * p.o_block_stride + b * p.os0 + t * p.os1 + hh * p.os2 + lane * E;
        VecIO<Tout, E>::store(dst, out);
        if (p.lse != nullptr && lane == 0)
            p.lse[blk * p.lse_block_stride + (static_cast<int64_t>(b) * p.out_hb + hh) * p.T + t] = lse_out;
    }
}

static int num_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) !=
                                                       cudaSuccess || n <= 0)
            n = 148;
    }
    return n;
}

template <typename Tin, typename Tout, int D>
static cudaError_t launch_tm_d(const TreeMergeParams &p, bool pdl, cudaStream_t s) {
    const int rows = p.B * p.T * p.Hr;
    if (rows == 0) return cudaSuccess;
    // with PDL the grid should fit beside the prefix kernel (one 4-warp block per SM): up to 8
    // rows per warp; without PDL one row per warp spreads the latency-bound work widest
#ifndef HTA_TM_RMAX
#define HTA_TM_RMAX 1
#endif
    int R = 1;
    if (pdl)
        while (R < HTA_TM_RMAX && static_cast<int64_t>(num_sms()) * 4 * R < rows) R *= 2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((rows + 4 * R - 1) / (4 * R));
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaError_t e;
    switch (R) {
        case 1: e = cudaLaunchKernelEx(&cfg, tree_merge_kernel<Tin, Tout, D, 1>, p); break;
        case 2: e = cudaLaunchKernelEx(&cfg, tree_merge_kernel<Tin, Tout, D, 2>, p); break;
        case 4: e = cudaLaunchKernelEx(&cfg, tree_merge_kernel<Tin, Tout, D, 4>, p); break;
        default: e = cudaLaunchKernelEx(&cfg, tree_merge_kernel<Tin, Tout, D, 8>, p); break;
    }
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

template <typename Tin, typename Tout>
static cudaError_t launch_tm(const TreeMergeParams &p, int d, bool pdl, cudaStream_t s) {
    if (d == 128) return launch_tm_d<Tin, Tout, 128>(p, pdl, s);
    if (d == 64) return launch_tm_d<Tin, Tout, 64>(p, pdl, s);
    return cudaErrorInvalidValue;
}

cudaError_t launch_tree_merge(const TreeMergeParams &p, int d, hta_dtype_t in_dtype, hta_dtype_t out_dtype,
                              bool pdl, cudaStream_t s) {
    if (in_dtype == HTA_BF16)
        return out_dtype == HTA_BF16 ? launch_tm<__nv_bfloat16, __nv_bfloat16>(p, d, pdl, s)
                                     : launch_tm<__nv_bfloat16, float>(p, d, pdl, s);
    return out_dtype == HTA_BF16 ? launch_tm<float, __nv_bfloat16>(p, d, pdl, s)
                                 : launch_tm<float, float>(p, d, pdl, s);
}

}  // namespace hta
