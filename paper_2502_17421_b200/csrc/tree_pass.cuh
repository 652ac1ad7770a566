// tree_pass.cuh -- row-level device functions of the tree pass and the LSE merge, shared by
// the tree/merge kernel (tree_merge.cu) and the fused epilogue of the prefix kernel
// (prefix_tc.cu).  One warp per output row (b, t, h); lane l holds elements [l*E, l*E + E) of
// the d-vector, E = d / 32.
//
// Tree pass: query (b,t,h) attends to the speculative keys s with
// mask[b][t][s] != 0 only.  The visible keys of a row are found with one ballot per 32 mask
// bytes; each key row is read by the whole warp with one vectorised load per lane, dot products
// are reduced with xor shuffles (four keys in flight), and an online softmax in fp32 (natural
// exp) gives the normalised tree partial and its LSE.
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
#pragma once
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

// Tree pass of one output row: normalised tree partial in ot[] and its natural-log LSE.  W = 64-bit
// words of the row's visibility (1 for T <= 64, 4 for T <= 256): the set is built and walked with
// 64-bit ballots / find-first-set, so a small tree costs no per-word selects.
template <typename Tin, int D, int W>
__device__ __forceinline__ float tree_row_w(const TreeMergeParams &p, int b, int t, int h, int lane,
                                            float (&ot)[D / 32]) {
    constexpr int E = D / 32;
    constexpr int kKeys = 8;  // visible keys whose K and V rows are in flight at once
    const int g = h / p.G;
#pragma unroll
    for (int e = 0; e < E; ++e) ot[e] = 0.f;
    // one round trip for q and the whole mask row (T <= 64 W: up to 2 W bytes per lane)
    float qv[E];
    VecIO<Tin, E>::load(static_cast<const Tin *>(p.q) + b * p.qs0 + t * p.qs1 + h * p.qs2 + lane * E, qv);
    uint64_t vis[W];
    if (p.mask != nullptr) {
        const uint8_t *mrow = p.mask + b * p.mask_bs + static_cast<int64_t>(t) * p.T;
        uint8_t mb[2 * W];
#pragma unroll
        for (int c = 0; c < 2 * W; ++c) mb[c] = c * 32 + lane < p.T ? mrow[c * 32 + lane] : 0;
#pragma unroll
        for (int c = 0; c < W; ++c)
            vis[c] = static_cast<uint64_t>(__ballot_sync(0xffffffffu, mb[2 * c] != 0)) |
                     (static_cast<uint64_t>(__ballot_sync(0xffffffffu, mb[2 * c + 1] != 0)) << 32);
    } else {
        // hta_forward_tree: the row's visible keys are t and its ancestors (Z4), found by walking
        // the parent links held in registers (lane l: parents[32c + l]); a chain through an
        // invalid link (parents[a] < -1 or >= a) hides the whole row, as hta_build_tree_mask does
        const int32_t *prow = p.parents + b * p.par_bs;
        int par[2 * W];
#pragma unroll
        for (int c = 0; c < 2 * W; ++c) par[c] = c * 32 + lane < p.T ? prow[c * 32 + lane] : -1;
#pragma unroll
        for (int c = 0; c < W; ++c) vis[c] = 0ull;
        int a = t;  // (warp-uniform)
        while (a >= 0) {
            int pa = -1;
#pragma unroll
            for (int c = 0; c < 2 * W; ++c) {
                const int x = __shfl_sync(0xffffffffu, par[c], a & 31);
                if (c == (a >> 5)) pa = x;
            }
#pragma unroll
            for (int c = 0; c < W; ++c)
                if (c == (a >> 6)) vis[c] |= 1ull << (a & 63);
            if (pa < -1 || pa >= a) {
#pragma unroll
                for (int c = 0; c < W; ++c) vis[c] = 0ull;
                break;
            }
            a = pa;
        }
    }
    const Tin *Kt = static_cast<const Tin *>(p.kt) + b * p.ts0 + g * p.ts2 + lane * E;
    const Tin *Vt = static_cast<const Tin *>(p.vt) + b * p.ts0 + g * p.ts2 + lane * E;
    using Acc = typename std::conditional<std::is_same<Tin, float>::value, double, float>::type;
    float l = 0.f;
    Acc m_acc = static_cast<Acc>(-INFINITY);  // running max kept at accumulation precision
    while (true) {
        // next (up to) kKeys visible keys in index order
        int idx[kKeys];
        int n = 0;
#pragma unroll
        for (int u = 0; u < kKeys; ++u) {
            idx[u] = -1;
#pragma unroll
            for (int c = 0; c < W; ++c) {
                if (idx[u] < 0 && vis[c] != 0ull) {
                    idx[u] = c * 64 + __ffsll(static_cast<long long>(vis[c])) - 1;
                    vis[c] &= vis[c] - 1ull;
                }
            }
            n += idx[u] >= 0 ? 1 : 0;
        }
        if (n == 0) break;
        Acc z[kKeys];
        float vv[kKeys][E];
        float kk[kKeys][E];
#pragma unroll
        for (int u = 0; u < kKeys; ++u) {  // all loads first: one round trip per batch
            const int sidx = idx[u] < 0 ? idx[0] : idx[u];
            VecIO<Tin, E>::load(Kt + sidx * p.ts1, kk[u]);
            VecIO<Tin, E>::load(Vt + sidx * p.ts1, vv[u]);
        }
#pragma unroll
        for (int u = 0; u < kKeys; ++u) {
            Acc a = 0;
#pragma unroll
            for (int e = 0; e < E; ++e) a = fma(static_cast<Acc>(qv[e]), static_cast<Acc>(kk[u][e]), a);
            z[u] = a;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1)
#pragma unroll
            for (int u = 0; u < kKeys; ++u) z[u] += __shfl_xor_sync(0xffffffffu, z[u], off);
        Acc mx = m_acc;
#pragma unroll
        for (int u = 0; u < kKeys; ++u) {
            z[u] = idx[u] >= 0 ? z[u] * static_cast<Acc>(p.scale) : static_cast<Acc>(-INFINITY);
            mx = z[u] > mx ? z[u] : mx;
        }
        const float corr = expf(static_cast<float>(m_acc - mx));
        l *= corr;
#pragma unroll
        for (int e = 0; e < E; ++e) ot[e] *= corr;
#pragma unroll
        for (int u = 0; u < kKeys; ++u) {
            const float w = expf(static_cast<float>(z[u] - mx));  // 0 for unused slots
            l += w;
#pragma unroll
            for (int e = 0; e < E; ++e) ot[e] = fmaf(w, vv[u][e], ot[e]);
        }
        m_acc = mx;
        if (n < kKeys) break;
    }
    if (!(l > 0.f)) return -INFINITY;
    const float inv = 1.0f / l;
#pragma unroll
    for (int e = 0; e < E; ++e) ot[e] *= inv;
    return static_cast<float>(m_acc + static_cast<Acc>(logf(l)));
}

template <typename Tin, int D>
__device__ __forceinline__ float tree_row(const TreeMergeParams &p, int b, int t, int h, int lane, float (&ot)[D / 32]) {
    return p.T <= 64 ? tree_row_w<Tin, D, 1>(p, b, t, h, lane, ot) : tree_row_w<Tin, D, 4>(p, b, t, h, lane, ot);
}

// Loads of partials written during the same kernel by other CTAs: L2 only (ld.global.cg).
template <int E>
__device__ __forceinline__ void load_cg(const float *p, float (&v)[E]) {
    if constexpr (E == 4) {
        const float4 x = __ldcg(reinterpret_cast<const float4 *>(p));
        v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    } else {
        const float2 x = __ldcg(reinterpret_cast<const float2 *>(p));
        v[0] = x.x; v[1] = x.y;
    }
}

// Merge of row (b, t, hl) -- hl = h - h0 -- : the tree partial (ot, lse_t; a sentinel when there
// is no tree part) with the p.n_parts prefix partials, written to p.o (Tout) and p.lse.  CG: read
// the partials through L2 only (they were written by other CTAs of the running kernel).
#ifndef HTA_FAST_PARTS
#define HTA_FAST_PARTS 12
#endif
constexpr int kFastParts = HTA_FAST_PARTS;  // partials merged with all loads in flight at once

template <typename Tout, int D, bool CG>
__device__ __forceinline__ void merge_row(const TreeMergeParams &p, int b, int t, int hl, int lane,
                                          const float (&ot)[D / 32], float lse_t) {
    constexpr int E = D / 32;
    float out[E];
    float lse_out = lse_t;
#pragma unroll
    for (int e = 0; e < E; ++e) out[e] = ot[e];
    if (p.n_parts > 0) {
        // (peer-memory exchange, role 2: this step's half of the double-buffered receive blocks)
        const int64_t par_off = p.p2p_role == 2 ? static_cast<int64_t>((*p.p2p_epoch - 1u) & 1u) * p.p2p_parity : 0;
        const int64_t lrow = (static_cast<int64_t>(b) * p.Hr + hl) * p.T + t;
        const int64_t orow = ((static_cast<int64_t>(b) * p.T + t) * p.Hr + hl) * D + lane * E;
        if (p.n_parts <= kFastParts) {
            // every load of the row in flight at once: one round trip (partials are L2-resident)
            float v16[kFastParts][E];
            const float ls = lane < p.n_parts ? (CG ? __ldcg(p.lse_parts + par_off + lane * p.lse_part_stride + lrow)
                                                    : (p.lse_parts + par_off)[lane * p.lse_part_stride + lrow])
                                              : -INFINITY;
#pragma unroll
            for (int j = 0; j < kFastParts; ++j) {
                if (j < p.n_parts) {
                    const float *src = p.o_parts + par_off + j * p.o_part_stride + orow;
                    if (CG)
                        load_cg<E>(src, v16[j]);
                    else
                        VecIO<float, E>::load(src, v16[j]);
                }
            }
            float mx = fmaxf(lse_t, ls);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
            if (mx == -INFINITY) {
#pragma unroll
                for (int e = 0; e < E; ++e) out[e] = 0.f;
                lse_out = -INFINITY;
            } else {
                const float wl = expf(ls - mx);
                const float wt = expf(lse_t - mx);  // 0 when the tree part is a sentinel
                float W = wt, acc[E];
#pragma unroll
                for (int e = 0; e < E; ++e) acc[e] = wt * ot[e];
#pragma unroll
                for (int j = 0; j < kFastParts; ++j) {
                    if (j < p.n_parts) {
                        const float w = __shfl_sync(0xffffffffu, wl, j);
                        W += w;
#pragma unroll
                        for (int e = 0; e < E; ++e) acc[e] = fmaf(w, v16[j][e], acc[e]);
                    }
                }
                const float inv = 1.0f / W;
#pragma unroll
                for (int e = 0; e < E; ++e) out[e] = acc[e] * inv;
                lse_out = mx + logf(W);
            }
        } else {
        float mx = lse_t;
        for (int s = lane; s < p.n_parts; s += 32)
            mx = fmaxf(mx, CG ? __ldcg(p.lse_parts + par_off + s * p.lse_part_stride + lrow)
                              : (p.lse_parts + par_off)[s * p.lse_part_stride + lrow]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        if (mx == -INFINITY) {
#pragma unroll
            for (int e = 0; e < E; ++e) out[e] = 0.f;
            lse_out = -INFINITY;
        } else {
            float W = 0.f, acc[E];
            const float wt = expf(lse_t - mx);  // 0 when the tree part is a sentinel
            W += wt;
#pragma unroll
            for (int e = 0; e < E; ++e) acc[e] = wt * ot[e];
            for (int s0 = 0; s0 < p.n_parts; s0 += 32) {
                const int s = s0 + lane;
                const float ls = s < p.n_parts ? (CG ? __ldcg(p.lse_parts + par_off + s * p.lse_part_stride + lrow)
                                                     : (p.lse_parts + par_off)[s * p.lse_part_stride + lrow])
                                               : -INFINITY;
                const float ws = expf(ls - mx);
                const int cnt = min(32, p.n_parts - s0);
                // eight partial rows in flight per lane (the partials are L2-resident)
                for (int u = 0; u < cnt; u += 8) {
                    float w8[8], v8[8][E];
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        w8[j] = __shfl_sync(0xffffffffu, ws, (u + j) & 31);
                        if (u + j < cnt) {
                            const float *src = p.o_parts + par_off + (s0 + u + j) * p.o_part_stride + orow;
                            if (CG)
                                load_cg<E>(src, v8[j]);
                            else
                                VecIO<float, E>::load(src, v8[j]);
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
    }
    const int blk = hl / p.out_hb, hh = hl % p.out_hb;
    if (p.p2p_role == 1) {  // straight into rank blk's receive buffer (fp32 partials), then fenced
        float *base = p.p2p_dst[blk] + static_cast<int64_t>(*p.p2p_epoch & 1u) * p.p2p_parity;
        VecIO<float, E>::store(base + b * p.os0 + t * p.os1 + hh * p.os2 + lane * E,
                               reinterpret_cast<const float(&)[E]>(out));
        if (lane == 0) base[p.p2p_lse_off + (static_cast<int64_t>(b) * p.out_hb + hh) * p.T + t] = lse_out;
        return;  // (the kernel's last block fences and signals: tree_merge_kernel)
    }
    Tout *dst = static_cast<Tout *>(p.o) + blk * p.o_block_stride + b * p.os0 + t * p.os1 + hh * p.os2 + lane * E;
    VecIO<Tout, E>::store(dst, out);
    if (p.lse != nullptr && lane == 0)
        p.lse[blk * p.lse_block_stride + (static_cast<int64_t>(b) * p.out_hb + hh) * p.T + t] = lse_out;
}

}  // namespace hta
