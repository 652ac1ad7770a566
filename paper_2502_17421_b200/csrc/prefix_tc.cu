// prefix_tc.cu -- the prefix pass of Hybrid Tree Attention on sm_100a tensor cores.
//
// Computes, for every (batch b, KV head g, split s), the UNMASKED attention of the T*G query
// rows that share KV head g over the keys [s*L, (s+1)*L) of the cache (PAPER.md:195, 199-201:
// "the queries and the cached key-value pairs {K_cache, V_cache} do not require additional
// masks"), producing a normalised partial O and its LSE.  The paper calls
// FlashDecoding for this step (PAPER.md:108 footnote); this kernel is the B200-native
// replacement:
//
//  * rows: the T tree tokens x the G query heads of one KV head form the M dimension
//    (row r = t*G + j, head h = g*G + j), 128 rows per tcgen05 tile, NT (1 or 2) tiles per CTA
//    so each KV tile is read from HBM once for up to 256 rows;
//  * warp 0 streams K and V tiles (128 keys x d, bf16) with TMA into a ring of smem slots
//    (128B swizzle, the canonical UMMA layout);
//  * warp 1 (one elected lane) issues tcgen05.mma: S = Q K^T into TMEM (fp32), and, once the
//    softmax warps have written P (bf16) back into TMEM over S, O += P V with A = P read from
//    TMEM (the "TS" form) and B = V from smem (MN-major descriptor); O lives in TMEM;
//  * softmax warpgroups (one thread per row = one TMEM lane) read S with tcgen05.ld, keep the
//    running max / sum in registers, rescale O in TMEM only when the max grows by more than
//    2^8 (exact: the final division uses the same stale max), and write P with tcgen05.st;
//  * the epilogue divides O by the row sum and writes fp32 partials + natural-log LSE.
// A split/row tile with no visible key writes the sentinel (O = 0, LSE = -inf).
#include <cuda_bf16.h>
#include <cstdio>

#include "hta_internal.h"
#include "ptx_sm100.cuh"

namespace hta {

template <int D, int NT>
struct TcCfg {
    static constexpr int kKB = D / 64;                       // 128-byte K-blocks of the head dim
    static constexpr int kRegionBytes = 128 * 128;           // 128 rows x 128 B
    static constexpr int kQTileBytes = kRowsPerTile * D * 2;  // one 128-row Q tile
    static constexpr int kSlotBytes = kBlockN * D * 2;       // one K or V tile
    static constexpr int kSlotsRaw = (224 * 1024 - NT * kQTileBytes) / kSlotBytes;
    static constexpr int kSlots = kSlotsRaw > 8 ? 8 : kSlotsRaw;
    // warp 0: TMA producer, warp 1: MMA issuer + TMEM owner, then the softmax warpgroups
    // (4 consecutive warps cover the four TMEM lane quarters via warp % 4).
    static constexpr int kFirstSoftmaxWarp = 2;
    static constexpr int kThreads = 32 * kFirstSoftmaxWarp + 128 * NT;
    static constexpr int kBarOffset = NT * kQTileBytes + kSlots * kSlotBytes;
    static constexpr int kSmemBytes = 1024 + kBarOffset + 512;
    static_assert(kSlots >= 3, "need at least 3 KV slots");
    static_assert(kSmemBytes <= 232448, "shared memory budget");
};

// TMEM column map: S buffer `buf` at 256*buf, O of tile `tile` at 256*tile + 128.
__device__ __forceinline__ uint32_t s_col(int buf) { return 256u * static_cast<uint32_t>(buf); }
__device__ __forceinline__ uint32_t o_col(int tile) { return 256u * static_cast<uint32_t>(tile) + 128u; }

template <int D, int NT>
__global__ void __launch_bounds__(TcCfg<D, NT>::kThreads, 1)
    prefix_tc_kernel(const __grid_constant__ CUtensorMap tmap_k, const __grid_constant__ CUtensorMap tmap_v,
                     const PrefixParams p) {
    using C = TcCfg<D, NT>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sQ = smem;
    uint8_t *sKV = smem + NT * C::kQTileBytes;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + C::kBarOffset);
    uint64_t *kv_full = bars;                 // [kSlots]
    uint64_t *kv_empty = bars + C::kSlots;    // [kSlots]
    uint64_t *s_full = bars + 2 * C::kSlots;  // [2]
    uint64_t *p_full = s_full + 2;            // [2]
    uint64_t *pv_done = p_full + 2;           // [1]  (NT == 1)
    uint64_t *o_final = pv_done + 1;          // [1]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(o_final + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    // ---- work item: (b, g, split, row group)
    int rest = blockIdx.x;
    const int mg = rest % p.n_mgroups;
    rest /= p.n_mgroups;
    const int split = rest % p.splits;
    rest /= p.splits;
    const int g = rest % p.H_kv;
    const int b = rest / p.H_kv;
    int64_t n_b = p.N_max;
    if (p.seqlens != nullptr) {
        n_b = p.seqlens[b];
        n_b = n_b < 0 ? 0 : (n_b > p.N_max ? p.N_max : n_b);
    }
    const int64_t key_lo = static_cast<int64_t>(split) * p.tiles_per_split * kBlockN;
    int64_t key_hi = key_lo + static_cast<int64_t>(p.tiles_per_split) * kBlockN;
    if (key_hi > n_b) key_hi = n_b;
    const int n_tiles = key_hi > key_lo ? static_cast<int>((key_hi - key_lo + kBlockN - 1) / kBlockN) : 0;
    const int row0 = mg * kRowsPerTile * NT;
    const int tiles_active = (p.M - row0) >= kRowsPerTile ? NT : 1;  // NT==2: is tile 1 needed?

    float *o_base = p.o_out + static_cast<int64_t>(split) * p.o_split_stride;
    float *lse_base = p.lse_out + static_cast<int64_t>(split) * p.lse_split_stride;

    if (n_tiles == 0) {  // empty split: sentinel rows
        for (int r = threadIdx.x; r < kRowsPerTile * NT; r += blockDim.x) {
            const int grow = row0 + r;
            if (grow >= p.M) continue;
            const int t = grow / p.G, h = g * p.G + grow % p.G;
            float4 *dst = reinterpret_cast<float4 *>(o_base + ((static_cast<int64_t>(b) * p.T + t) * p.H + h) * D);
#pragma unroll
            for (int c = 0; c < D / 4; ++c) dst[c] = make_float4(0.f, 0.f, 0.f, 0.f);
            lse_base[(static_cast<int64_t>(b) * p.H + h) * p.T + t] = -INFINITY;
        }
        return;
    }

    // ---- one-time setup
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmap_k);
        tma_prefetch_desc(&tmap_v);
    }
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < C::kSlots; ++s) {
            mbar_init(&kv_full[s], 1);
            mbar_init(&kv_empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 4);
        }
        mbar_init(pv_done, 1);
        mbar_init(o_final, 1);
        fence_mbar_init();
    }
    if (warp == 1) {
        tmem_alloc(tmem_slot, 512);
        tmem_relinquish();
    }
    {   // Q rows -> smem in the canonical K-major SWIZZLE_128B layout
        const __nv_bfloat16 *q = static_cast<const __nv_bfloat16 *>(p.q);
        constexpr int kChunks = D / 8;  // 16-byte chunks per row
        for (int idx = threadIdx.x; idx < NT * kRowsPerTile * kChunks; idx += blockDim.x) {
            const int row = idx / kChunks, ch = idx % kChunks;
            const int tile = row / kRowsPerTile, r = row % kRowsPerTile;
            const int grow = row0 + row;
            uint4 val = make_uint4(0u, 0u, 0u, 0u);
            if (grow < p.M) {
                const int t = grow / p.G, h = g * p.G + grow % p.G;
                val = *reinterpret_cast<const uint4 *>(q + b * p.qs0 + t * p.qs1 + h * p.qs2 + ch * 8);
            }
            uint8_t *dst = sQ + (tile * C::kKB + ch / 8) * C::kRegionBytes + r * 128 + (((ch & 7) ^ (r & 7)) << 4);
            *reinterpret_cast<uint4 *>(dst) = val;
        }
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // production index: K_j -> 2j, V_j -> 2j+1
    auto slot_of = [](int idx) { return idx % C::kSlots; };
    auto phase_of = [](int idx) { return static_cast<uint32_t>((idx / C::kSlots) & 1); };

    if (warp == 0) {
        // ================= TMA producer
        if (lane == 0) {
            int idx = 0;
            for (int j = 0; j < n_tiles; ++j) {
                const int n0 = static_cast<int>(key_lo) + j * kBlockN;
#pragma unroll
                for (int kv = 0; kv < 2; ++kv, ++idx) {
                    const int slot = slot_of(idx);
                    mbar_wait(&kv_empty[slot], phase_of(idx) ^ 1u);
                    mbar_arrive_expect_tx(&kv_full[slot], C::kSlotBytes);
                    uint8_t *dst = sKV + slot * C::kSlotBytes;
#pragma unroll
                    for (int kb = 0; kb < C::kKB; ++kb)
                        tma_load_4d(dst + kb * (kBlockN * 128), kv ? static_cast<const void *>(&tmap_v)
                                                                  : static_cast<const void *>(&tmap_k),
                                    &kv_full[slot], kb * 64, g, n0, b, kPolicyEvictFirst);
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ================= MMA issuer (lane 0 issues; the warp zeroes invalid V rows)
        const uint32_t idesc_qk = idesc_bf16_f32(128, kBlockN, 0);
        const uint32_t idesc_pv = idesc_bf16_f32(128, D, 1);
        const uint32_t sQa = smem_u32(sQ), sKVa = smem_u32(sKV);
        auto issue_S = [&](int tile, int buf, int slot) {
            const uint32_t d_t = tmem + s_col(buf);
#pragma unroll
            for (int k = 0; k < D / 16; ++k) {
                const uint32_t qa = sQa + (tile * C::kKB + k / 4) * C::kRegionBytes + (k % 4) * 32;
                const uint32_t ka = sKVa + slot * C::kSlotBytes + (k / 4) * (kBlockN * 128) + (k % 4) * 32;
                mma_bf16_ss(d_t, sdesc_sw128(qa, 16, 1024), sdesc_sw128(ka, 16, 1024), idesc_qk, k > 0 ? 1u : 0u);
            }
        };
        auto issue_PV = [&](int tile, int buf, int slot, bool acc) {
            const uint32_t d_t = tmem + o_col(tile);
            const uint32_t a_t = tmem + s_col(buf);
#pragma unroll
            for (int k = 0; k < kBlockN / 16; ++k) {
                const uint32_t va = sKVa + slot * C::kSlotBytes + k * 2048;
                mma_bf16_ts(d_t, a_t + k * 8, sdesc_sw128(va, kBlockN * 128, 1024), idesc_pv,
                            (acc || k > 0) ? 1u : 0u);
            }
        };
        // Rows of the last V tile past the valid sequence may hold garbage (even NaN) that
        // P = 0 would not cancel; zero them (reading Z13).
        auto zero_tail = [&](int j, int slot) {
            const int64_t kbase = key_lo + static_cast<int64_t>(j) * kBlockN;
            const int valid = static_cast<int>(key_hi - kbase);
            if (j == n_tiles - 1 && valid < kBlockN && key_hi == n_b && n_b < p.N_max) {
                uint8_t *base = sKV + slot * C::kSlotBytes;
                const int nrows = kBlockN - valid;
                for (int i = lane; i < C::kKB * nrows * 8; i += 32) {
                    const int kb = i / (nrows * 8), rr = (i / 8) % nrows, c = i % 8;
                    *reinterpret_cast<uint4 *>(base + kb * (kBlockN * 128) + (valid + rr) * 128 + c * 16) =
                        make_uint4(0u, 0u, 0u, 0u);
                }
                fence_proxy_async_smem();
            }
            __syncwarp();
        };

        if (NT == 2) {
            const bool two = tiles_active == 2;
            mbar_wait(&kv_full[slot_of(0)], phase_of(0));
            tc_fence_after();
            if (lane == 0) {
                issue_S(0, 0, slot_of(0));
                tc_commit(&s_full[0]);
                if (two) {
                    issue_S(1, 1, slot_of(0));
                    tc_commit(&s_full[1]);
                }
                tc_commit(&kv_empty[slot_of(0)]);
            }
            __syncwarp();
            for (int j = 0; j < n_tiles; ++j) {
                const int vi = 2 * j + 1, ki = 2 * j + 2;
                const uint32_t ph = j & 1;
                mbar_wait(&kv_full[slot_of(vi)], phase_of(vi));
                zero_tail(j, slot_of(vi));
                mbar_wait(&p_full[0], ph);
                tc_fence_after();
                if (lane == 0) issue_PV(0, 0, slot_of(vi), j > 0);
                __syncwarp();
                if (j + 1 < n_tiles) {
                    mbar_wait(&kv_full[slot_of(ki)], phase_of(ki));
                    tc_fence_after();
                    if (lane == 0) {
                        issue_S(0, 0, slot_of(ki));
                        tc_commit(&s_full[0]);
                    }
                    __syncwarp();
                }
                if (two) {
                    mbar_wait(&p_full[1], ph);
                    tc_fence_after();
                    if (lane == 0) issue_PV(1, 1, slot_of(vi), j > 0);
                    __syncwarp();
                }
                if (lane == 0) {
                    tc_commit(&kv_empty[slot_of(vi)]);
                    if (j + 1 < n_tiles) {
                        if (two) {
                            issue_S(1, 1, slot_of(ki));
                            tc_commit(&s_full[1]);
                        }
                        tc_commit(&kv_empty[slot_of(ki)]);
                    }
                }
                __syncwarp();
            }
        } else {
            // NT == 1: one row tile, S double-buffered (buffers 0 and 1), O at o_col(0).
            for (int j0 = 0; j0 < 2 && j0 < n_tiles; ++j0) {
                mbar_wait(&kv_full[slot_of(2 * j0)], phase_of(2 * j0));
                tc_fence_after();
                if (lane == 0) {
                    issue_S(0, j0, slot_of(2 * j0));
                    tc_commit(&s_full[j0]);
                    tc_commit(&kv_empty[slot_of(2 * j0)]);
                }
                __syncwarp();
            }
            for (int j = 0; j < n_tiles; ++j) {
                const int vi = 2 * j + 1, ki = 2 * (j + 2);
                const int buf = j & 1;
                mbar_wait(&kv_full[slot_of(vi)], phase_of(vi));
                zero_tail(j, slot_of(vi));
                mbar_wait(&p_full[buf], static_cast<uint32_t>((j >> 1) & 1));
                tc_fence_after();
                if (lane == 0) {
                    issue_PV(0, buf, slot_of(vi), j > 0);
                    tc_commit(pv_done);
                    tc_commit(&kv_empty[slot_of(vi)]);
                }
                __syncwarp();
                if (j + 2 < n_tiles) {
                    mbar_wait(&kv_full[slot_of(ki)], phase_of(ki));
                    tc_fence_after();
                    if (lane == 0) {
                        issue_S(0, buf, slot_of(ki));
                        tc_commit(&s_full[buf]);
                        tc_commit(&kv_empty[slot_of(ki)]);
                    }
                    __syncwarp();
                }
            }
        }
        if (lane == 0) tc_commit(o_final);
        __syncwarp();
    } else if (warp >= C::kFirstSoftmaxWarp) {
        // ================= softmax warpgroups: one thread per row (TMEM lane)
        const int wg = (warp - C::kFirstSoftmaxWarp) >> 2;
        if (wg < tiles_active) {
            const int quarter = warp & 3;
            const int r = quarter * 32 + lane;
            const int grow = row0 + wg * kRowsPerTile + r;
            const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
            const float c = p.scale_log2;
            float m_run = -INFINITY, l_run = 0.f;
            for (int j = 0; j < n_tiles; ++j) {
                const int buf = NT == 2 ? wg : (j & 1);
                const uint32_t sph = NT == 2 ? static_cast<uint32_t>(j & 1) : static_cast<uint32_t>((j >> 1) & 1);
                mbar_wait(&s_full[buf], sph);
                tc_fence_after();
                float s[kBlockN];
                tmem_ld64(tmem + lane_off + s_col(buf), *reinterpret_cast<float(*)[64]>(&s[0]));
                tmem_ld64(tmem + lane_off + s_col(buf) + 64, *reinterpret_cast<float(*)[64]>(&s[64]));
                const int64_t kbase = key_lo + static_cast<int64_t>(j) * kBlockN;
                const int valid = static_cast<int>(key_hi - kbase < kBlockN ? key_hi - kbase : kBlockN);
                if (valid < kBlockN) {
#pragma unroll
                    for (int cc = 0; cc < kBlockN; ++cc)
                        if (cc >= valid) s[cc] = -INFINITY;
                }
                float mx = s[0];
#pragma unroll
                for (int cc = 1; cc < kBlockN; ++cc) mx = fmaxf(mx, s[cc]);
                const float mt = mx * c;
                const float m_new = (mt > m_run + 8.0f) ? mt : m_run;
                // P = exp2(S*c - m) -> bf16, written over S in TMEM (A operand of O += P V)
                const float neg = -m_new;
                float lsum0 = 0.f, lsum1 = 0.f;
                uint32_t pk[kBlockN / 2];
#pragma unroll
                for (int cc = 0; cc < kBlockN / 2; ++cc) {
                    const float p0 = fast_exp2(fmaf(s[2 * cc], c, neg));
                    const float p1 = fast_exp2(fmaf(s[2 * cc + 1], c, neg));
                    lsum0 += p0;
                    lsum1 += p1;
                    pk[cc] = pack_bf16x2(p0, p1);
                }
                tmem_st32(tmem + lane_off + s_col(buf), *reinterpret_cast<uint32_t(*)[32]>(&pk[0]));
                tmem_st32(tmem + lane_off + s_col(buf) + 32, *reinterpret_cast<uint32_t(*)[32]>(&pk[32]));
                // Rescale O only when the running max moved (rare after the first tiles).  O must
                // hold P_{j-1} V_{j-1}: for NT == 2 that is implied by S_j having completed (MMAs
                // complete in issue order); for NT == 1 wait for it explicitly.  Every PV
                // completion is observed before the next can occur, so parity waits stay exact.
                if (NT == 1 && j > 0) mbar_wait(pv_done, static_cast<uint32_t>((j - 1) & 1));
                const bool need = (j > 0) && (m_new != m_run);
                const float f = need ? fast_exp2(m_run - m_new) : 1.0f;
                l_run = l_run * f + (lsum0 + lsum1);
                if (__any_sync(0xffffffffu, need)) {
                    const int tile = NT == 2 ? wg : 0;
#pragma unroll 1
                    for (int ch = 0; ch < D / 32; ++ch) {
                        float o[32];
                        tmem_ld32(tmem + lane_off + o_col(tile) + ch * 32, o);
#pragma unroll
                        for (int e = 0; e < 32; ++e) o[e] *= f;
                        tmem_st32(tmem + lane_off + o_col(tile) + ch * 32, *reinterpret_cast<uint32_t(*)[32]>(o));
                    }
                }
                m_run = m_new;
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&p_full[buf]);
            }
            // ---- epilogue
            mbar_wait(o_final, 0);
            tc_fence_after();
            pdl_launch_dependents();
            const float inv = 1.0f / l_run;
            const int tile = NT == 2 ? wg : 0;
            const bool row_ok = grow < p.M;
            int t = 0, h = 0;
            if (row_ok) {
                t = grow / p.G;
                h = g * p.G + grow % p.G;
            }
            float4 *dst = reinterpret_cast<float4 *>(o_base + ((static_cast<int64_t>(b) * p.T + t) * p.H + h) * D);
#pragma unroll
            for (int ch = 0; ch < D / 32; ++ch) {
                float o[32];
                tmem_ld32(tmem + lane_off + o_col(tile) + ch * 32, o);
                if (row_ok) {
#pragma unroll
                    for (int e = 0; e < 8; ++e)
                        dst[ch * 8 + e] = make_float4(o[4 * e] * inv, o[4 * e + 1] * inv, o[4 * e + 2] * inv,
                                                      o[4 * e + 3] * inv);
                }
            }
            if (row_ok)
                lse_base[(static_cast<int64_t>(b) * p.H + h) * p.T + t] =
                    (m_run + log2f(l_run)) * 0.69314718055994530942f;
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

template <int D, int NT>
static cudaError_t launch_tc(const PrefixParams &p, const CUtensorMap &tk, const CUtensorMap &tv, cudaStream_t s) {
    using C = TcCfg<D, NT>;
    auto kern = prefix_tc_kernel<D, NT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e != cudaSuccess) return e;
    const int grid = p.n_mgroups * p.splits * p.H_kv * p.B;
    kern<<<grid, C::kThreads, C::kSmemBytes, s>>>(tk, tv, p);
    return cudaGetLastError();
}

int prefix_tc_smem_bytes(int d, int nt) {
    if (d == 128) return nt == 2 ? TcCfg<128, 2>::kSmemBytes : TcCfg<128, 1>::kSmemBytes;
    return nt == 2 ? TcCfg<64, 2>::kSmemBytes : TcCfg<64, 1>::kSmemBytes;
}

cudaError_t launch_prefix_tc(const PrefixParams &p, const CUtensorMap &tk, const CUtensorMap &tv, int, cudaStream_t s) {
    if (p.d == 128) return p.nt == 2 ? launch_tc<128, 2>(p, tk, tv, s) : launch_tc<128, 1>(p, tk, tv, s);
    if (p.d == 64) return p.nt == 2 ? launch_tc<64, 2>(p, tk, tv, s) : launch_tc<64, 1>(p, tk, tv, s);
    return cudaErrorInvalidValue;
}

}  // namespace hta
