// prefix_tc.cu -- the prefix pass of Hybrid Tree Attention on sm_100a tensor cores.
//
// Computes, for every (batch b, KV head g, row group, split s), the UNMASKED attention of the
// query rows that share KV head g over the keys [s*L, (s+1)*L) of the cache (PAPER.md:195,
// 199-201: "the queries and the cached key-value pairs {K_cache, V_cache} do not require
// additional masks"), producing a normalised partial O and its LSE.  The
// paper calls FlashDecoding for this step (PAPER.md:108 footnote); this kernel is the B200-native
// replacement:
//
//  * rows: the T tree tokens x the G query heads of one KV head form the M dimension
//    (row r = t*G + j, head h = g*G + j).  Each CTA owns 128 rows (one TMEM lane per row).
//  * PAIR (M > 128, d = 128): a cluster of two CTAs on one TPC runs tcgen05.mma.cta_group::2
//    with M = 256: each CTA holds its 128 Q rows, HALF of every K tile (64 keys) and HALF of
//    every V tile (64 head-dim columns), so each KV byte is read from HBM once for 256 rows and
//    each SM streams only half of the operand bytes through shared memory.
//  * warp 0 (one lane) streams K and V tiles with TMA into two rings of smem slots (128B
//    swizzle, the canonical UMMA layout) so K tiles can run ahead of V tiles; in a pair both
//    CTAs' bytes are counted on the leader's barriers.
//  * warp 1 of the leader CTA issues the MMAs from a non-blocking, warp-converged loop
//    (elect.sync per instruction, descriptors advanced by constants): S = Q K^T into one of two
//    TMEM buffers (fp32) as soon as a K tile and a buffer are free, and O_h += P_h V_h for each
//    half h of the tile's keys (A = P read from TMEM, the "TS" form; B = V from smem, MN-major)
//    as soon as that half's P and the V tile are ready.
//  * warps 2-9: two independent softmax warpgroups; warpgroup h owns key columns
//    [64h, 64h + 64) of every tile with its own running max / sum and its own accumulator O_h
//    in TMEM, so the two never wait on each other and overlap each other's latency.  Per tile:
//    tcgen05.ld of its 64 S values, row max, exp2 (3/8 of the pairs on the FMA pipe by
//    polynomial, the rest on MUFU), row sum, P -> bf16 -> tcgen05.st over S.  O_h is rescaled in
//    TMEM only when its running max grows by more than 2^8 (exact: the final normalisation
//    uses the same, possibly stale, max).  The epilogue merges the two halves exactly (the
//    log-sum-exp merge of PAPER.md:207-218 applied inside the row).
//  * the epilogue divides O by the row sum and writes fp32 partials + natural-log LSE.
// A split with no visible key writes the sentinel (O = 0, LSE = -inf).
#include <cuda_bf16.h>
#include <cstdio>

#include "hta_internal.h"
#include "ptx_sm100.cuh"

namespace hta {

// Optional pipeline timeline (build with -DHTA_TRACE, tools/trace_prefix.py): lane 0 of each
// traced warp of CTA g_trace_cta appends (event, tag, j, clock) records.
#ifdef HTA_TRACE
__device__ unsigned long long *g_trace = nullptr;
__device__ int g_trace_cta = 0;
#define HTA_TR(ev, tag, jj)                                                                              \
    do {                                                                                                 \
        if (g_trace != nullptr && blockIdx.x == g_trace_cta && lane == 0 && tr_n < 2048)                \
            g_trace[warp * 2048 + tr_n++] = (static_cast<unsigned long long>(ev) << 56) |                \
                                            (static_cast<unsigned long long>(tag) << 52) |               \
                                            (static_cast<unsigned long long>((jj) & 0xFFFFF) << 32) |    \
                                            static_cast<unsigned long long>(static_cast<uint32_t>(clock64())); \
    } while (0)
#else
#define HTA_TR(ev, tag, jj) do { } while (0)
#endif

// Diagnostics only (tools/): HTA_SKIP=1 skips the softmax math, HTA_SKIP=2 also the MMAs,
// leaving the TMA stream and the barrier protocol; HTA_SKIP=3 runs the MMAs with no TMA traffic
// (operands are whatever sits in smem) and no softmax; HTA_SKIP=4 = 3 with the softmax.
// Product builds use 0.
#ifndef HTA_SKIP
#define HTA_SKIP 0
#endif

template <int D, bool PAIR>
struct TcCfg {
    static_assert(!PAIR || D == 128, "CTA pairs split the 128-column V tile in two 64-column halves");
    static constexpr int kKB = D / 64;                          // 128-byte K-blocks of the head dim
    static constexpr int kRegionBytes = 128 * 128;              // 128 rows x 128 B
    static constexpr int kQBytes = kRowsPerTile * D * 2;        // this CTA's 128 Q rows
    static constexpr int kKRows = PAIR ? kBlockN / 2 : kBlockN; // keys of a K tile held by this CTA
    static constexpr int kVCols = PAIR ? D / 2 : D;             // head-dim columns of a V tile held here
    static constexpr int kKBytes = kKRows * D * 2;
    static constexpr int kVBytes = kBlockN * kVCols * 2;
    static constexpr int kRingBytes = 192 * 1024;
    static constexpr int kSlotsK = (kRingBytes / 2) / kKBytes;
    static constexpr int kSlotsV = (kRingBytes / 2) / kVBytes;
    static constexpr int kSBufs = 2;                            // S/P buffers in TMEM
    static constexpr int kSoftmaxWarps = 8;                     // two warpgroups
    static constexpr int kThreads = 64 + 32 * kSoftmaxWarps;    // warp 0 TMA, warp 1 MMA + TMEM
    static constexpr int kVOff = kQBytes + kSlotsK * kKBytes;   // start of the V ring
    static constexpr int kRedOff = kVOff + kSlotsV * kVBytes;   // row-max / row-sum exchange
    static constexpr int kBarOff = kRedOff + 4 * kRowsPerTile * 4;  // (m, l) of both halves
    static constexpr int kSmemBytes = kBarOff + 512;  // base is 1024-aligned (__align__ below)
    static_assert(kSlotsK >= 3 && kSlotsV >= 3, "need at least 3 slots per ring");
    static_assert(kSmemBytes <= 232448, "shared memory budget");
};

// TMEM column map: S/P buffer b at 128*b (b = 0, 1), O_h (accumulator of key half h) at 256 + 128*h.
__device__ __forceinline__ uint32_t s_col(int buf) { return 128u * static_cast<uint32_t>(buf); }
__device__ __forceinline__ uint32_t o_col(int half) { return 256u + 128u * static_cast<uint32_t>(half); }

template <int D, bool PAIR>
__global__ void __launch_bounds__(TcCfg<D, PAIR>::kThreads, 1)
    prefix_tc_kernel(const __grid_constant__ CUtensorMap tmap_k, const __grid_constant__ CUtensorMap tmap_v,
                     const PrefixParams p) {
    using C = TcCfg<D, PAIR>;
    extern __shared__ __align__(1024) uint8_t smem[];  // 128B-swizzled tiles need 1024B alignment
    uint8_t *sQ = smem;
    uint8_t *sK = smem + C::kQBytes;
    uint8_t *sV = smem + C::kVOff;
    float *red = reinterpret_cast<float *>(smem + C::kRedOff);   // epilogue (m, l) exchange [4][128]
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + C::kBarOff);
    uint64_t *k_full = bars;                       // [kSlotsK]  (the leader's copy is the one used)
    uint64_t *k_empty = k_full + C::kSlotsK;       // [kSlotsK]
    uint64_t *v_full = k_empty + C::kSlotsK;       // [kSlotsV]  (the leader's copy is the one used)
    uint64_t *v_empty = v_full + C::kSlotsV;       // [kSlotsV]
    uint64_t *s_full = v_empty + C::kSlotsV;       // [2 bufs]
    uint64_t *p_full = s_full + 2;                 // [2 halves][2 bufs] (the leader's copy is used)
    uint64_t *pv_done = p_full + 4;                // [2 halves][2 bufs]: PV_h(j) -> pv_done[2h + j%2]
    uint64_t *o_final = pv_done + 4;               // [1]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(o_final + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
#ifdef HTA_TRACE
    int tr_n = 0;
#endif
    const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
    const bool leader = rank == 0;

    // ---- work item: (b, g, split, row group); a pair shares one work item
    int rest = PAIR ? (blockIdx.x >> 1) : blockIdx.x;
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
    const int row0 = mg * kRowsPerTile * (PAIR ? 2 : 1) + static_cast<int>(rank) * kRowsPerTile;
    // the last tile of a split that ends at the sequence end may hold garbage rows (Z13)
    const int tail_valid = static_cast<int>(key_hi - (key_lo + static_cast<int64_t>(n_tiles - 1) * kBlockN));
    const bool tail_zero = n_tiles > 0 && tail_valid < kBlockN && key_hi == n_b && n_b < p.N_max;

    float *o_base = p.o_out + static_cast<int64_t>(split) * p.o_split_stride;
    float *lse_base = p.lse_out + static_cast<int64_t>(split) * p.lse_split_stride;

    if (n_tiles == 0) {  // empty split: sentinel rows (both CTAs of a pair take this branch)
        for (int r = threadIdx.x; r < kRowsPerTile; r += blockDim.x) {
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
    if (threadIdx.x == 0 && (smem_u32(smem) & 1023u) != 0u) __trap();  // swizzle atoms need 1 KiB alignment
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmap_k);
        tma_prefetch_desc(&tmap_v);
    }
    if (warp == 1 && lane == 0) {
        for (int i = 0; i < C::kSlotsK; ++i) {
            mbar_init(&k_full[i], 1);
            mbar_init(&k_empty[i], 1);
        }
        for (int i = 0; i < C::kSlotsV; ++i) {
            mbar_init(&v_full[i], 1);
            mbar_init(&v_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) mbar_init(&s_full[i], 1);
        for (int i = 0; i < 4; ++i) {
            mbar_init(&p_full[i], (C::kSoftmaxWarps / 2) * (PAIR ? 2 : 1));
            mbar_init(&pv_done[i], 1);
        }
        mbar_init(o_final, 1);
        fence_mbar_init();
    }
    if (warp == 1) {
        if (PAIR) {
            tmem_alloc2(tmem_slot, 512);
            tmem_relinquish2();
        } else {
            tmem_alloc(tmem_slot, 512);
            tmem_relinquish();
        }
    }
    {   // this CTA's 128 Q rows -> smem in the canonical K-major SWIZZLE_128B layout
        const __nv_bfloat16 *q = static_cast<const __nv_bfloat16 *>(p.q);
        constexpr int kChunks = D / 8;  // 16-byte chunks per row
        for (int idx = threadIdx.x; idx < kRowsPerTile * kChunks; idx += blockDim.x) {
            const int r = idx / kChunks, ch = idx % kChunks;
            const int grow = row0 + r;
            uint4 val = make_uint4(0u, 0u, 0u, 0u);
            if (grow < p.M) {
                const int t = grow / p.G, h = g * p.G + grow % p.G;
                val = *reinterpret_cast<const uint4 *>(q + b * p.qs0 + t * p.qs1 + h * p.qs2 + ch * 8);
            }
            uint8_t *dst = sQ + (ch / 8) * C::kRegionBytes + r * 128 + (((ch & 7) ^ (r & 7)) << 4);
            *reinterpret_cast<uint4 *>(dst) = val;
        }
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync();  // barrier inits and TMEM allocation visible to the peer
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ================= TMA producer: K and V rings filled independently (K runs ahead)
        if (lane == 0 && HTA_SKIP < 3) {
            const uint32_t kfull0 = PAIR ? mapa_shared(smem_u32(&k_full[0]), 0) : 0u;
            const uint32_t vfull0 = PAIR ? mapa_shared(smem_u32(&v_full[0]), 0) : 0u;
            int kj = 0, vj = 0;
            uint32_t idle = 0;
            while (kj < n_tiles || vj < n_tiles) {
                bool did = false;
                if (kj < n_tiles && mbar_test(&k_empty[kj % C::kSlotsK], ((kj / C::kSlotsK) & 1) ^ 1u)) {
                    const int slot = kj % C::kSlotsK;
                    const int n0 = static_cast<int>(key_lo) + kj * kBlockN;
                    uint8_t *dst = sK + slot * C::kKBytes;
                    HTA_TR(30, 0, kj);
                    if (PAIR) {
                        if (leader) mbar_arrive_expect_tx(&k_full[slot], 2u * C::kKBytes);
#pragma unroll
                        for (int kb = 0; kb < C::kKB; ++kb)
                            tma_load_4d_pair(dst + kb * (C::kKRows * 128), &tmap_k, kfull0 + 8u * slot, kb * 64, g,
                                             n0 + static_cast<int>(rank) * C::kKRows, b, kPolicyEvictFirst);
                    } else {
                        mbar_arrive_expect_tx(&k_full[slot], C::kKBytes);
#pragma unroll
                        for (int kb = 0; kb < C::kKB; ++kb)
                            tma_load_4d(dst + kb * (kBlockN * 128), &tmap_k, &k_full[slot], kb * 64, g, n0, b,
                                        kPolicyEvictFirst);
                    }
                    ++kj;
                    did = true;
                }
                if (vj < kj && mbar_test(&v_empty[vj % C::kSlotsV], ((vj / C::kSlotsV) & 1) ^ 1u)) {
                    const int slot = vj % C::kSlotsV;
                    const int n0 = static_cast<int>(key_lo) + vj * kBlockN;
                    uint8_t *dst = sV + slot * C::kVBytes;
                    HTA_TR(31, 0, vj);
                    if (PAIR) {
                        if (leader) mbar_arrive_expect_tx(&v_full[slot], 2u * C::kVBytes);
                        tma_load_4d_pair(dst, &tmap_v, vfull0 + 8u * slot, static_cast<int>(rank) * 64, g, n0, b,
                                         kPolicyEvictFirst);
                    } else {
                        mbar_arrive_expect_tx(&v_full[slot], C::kVBytes);
#pragma unroll
                        for (int kb = 0; kb < C::kKB; ++kb)
                            tma_load_4d(dst + kb * (kBlockN * 128), &tmap_v, &v_full[slot], kb * 64, g, n0, b,
                                        kPolicyEvictFirst);
                    }
                    ++vj;
                    did = true;
                }
                if (!did) {
                    if (++idle > (1u << 26)) {
                        printf("hta: producer stalled (block %d)\n", blockIdx.x);
                        __trap();
                    }
                    __nanosleep(20);
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ================= MMA issuer: the whole warp of the leader CTA runs this loop with
        // warp-uniform values and elect.sync issues each tcgen05 op (one lane, no waterfall);
        // descriptors are built once and advanced by constants, so the tensor pipe is never
        // starved by issue overhead (a single divergent lane issues at half the N=128 MMA rate).
        if (leader) {
            constexpr int kM = PAIR ? 256 : 128;
            const uint32_t idesc_qk = idesc_bf16_f32(kM, kBlockN, 0);
            const uint32_t idesc_pv = idesc_bf16_f32(kM, D, 1);
            const uint64_t qd0 = sdesc_sw128(smem_u32(sQ), 16, 1024);
            const uint64_t kd0 = sdesc_sw128(smem_u32(sK), 16, 1024);
            const uint64_t vd0 = sdesc_sw128(smem_u32(sV), kBlockN * 128, 1024);
            auto commit = [](uint64_t *bar) {
                if (PAIR)
                    tc_commit2_mc_elect(bar);
                else
                    tc_commit_elect(bar);
            };
            auto issue_S = [&](int buf, int slot) {
                if (HTA_SKIP == 1 || HTA_SKIP == 2) return;
                const uint32_t d_t = tmem + s_col(buf);
                const uint64_t kd = kd0 + static_cast<uint32_t>((slot * C::kKBytes) >> 4);
#pragma unroll
                for (int k = 0; k < D / 16; ++k) {
                    // K-major SW128: +32 B per K step inside a 128-B atom, next atom = next region
                    const uint32_t qo = ((k / 4) * C::kRegionBytes + (k % 4) * 32) >> 4;
                    const uint32_t ko = ((k / 4) * (C::kKRows * 128) + (k % 4) * 32) >> 4;
                    if (PAIR)
                        mma2_bf16_ss_elect(d_t, qd0 + qo, kd + ko, idesc_qk, k > 0 ? 1u : 0u);
                    else
                        mma_bf16_ss_elect(d_t, qd0 + qo, kd + ko, idesc_qk, k > 0 ? 1u : 0u);
                }
            };
            // O_h += P_h V_h over the 64 keys [64h, 64h + 64) of the tile (K steps 4h .. 4h+3);
            // P_h sits packed in TMEM columns [64h, 64h + 32) of the S buffer
            auto issue_PV = [&](int half, int buf, int slot, bool acc) {
                if (HTA_SKIP == 1 || HTA_SKIP == 2) return;
                const uint32_t a_t = tmem + s_col(buf) + 64u * half;
                const uint64_t vd = vd0 + static_cast<uint32_t>((slot * C::kVBytes) >> 4);
#pragma unroll
                for (int kk = 0; kk < kBlockN / 32; ++kk) {
                    const int k = half * (kBlockN / 32) + kk;
                    // MN-major SW128: 16 keys = two 8-row groups = +2048 B per K step
                    if (PAIR)
                        mma2_bf16_ts_elect(tmem + o_col(half), a_t + kk * 8, vd + static_cast<uint32_t>(k * 128),
                                           idesc_pv, (acc || kk > 0) ? 1u : 0u);
                    else
                        mma_bf16_ts_elect(tmem + o_col(half), a_t + kk * 8, vd + static_cast<uint32_t>(k * 128),
                                          idesc_pv, (acc || kk > 0) ? 1u : 0u);
                }
            };
            // warp-uniform probe (lane 0's view is broadcast)
            auto ready = [](uint64_t *bar, uint32_t parity) {
                return __shfl_sync(0xffffffffu, mbar_test(bar, parity) ? 1 : 0, 0) != 0;
            };
            constexpr bool kNoMem = HTA_SKIP >= 3;
            int ns = 0, np[2] = {0, 0};  // next S, next PV per key half
            uint32_t idle = 0;
            while (np[0] < n_tiles || np[1] < n_tiles) {
                bool did = false;
                // S_ns into buffer ns % 2 once its K tile landed and both PV halves of tile ns-2
                // (the last readers of that buffer) have been issued.  The tail tile the softmax
                // warps sanitise also needs its V tile in smem before they see S.
                if (ns < n_tiles && ns < min(np[0], np[1]) + 2 &&
                    (kNoMem || ready(&k_full[ns % C::kSlotsK], (ns / C::kSlotsK) & 1)) &&
                    (kNoMem || !(tail_zero && ns == n_tiles - 1) ||
                     ready(&v_full[ns % C::kSlotsV], (ns / C::kSlotsV) & 1))) {
                    tc_fence_after();
                    issue_S(ns & 1, ns % C::kSlotsK);
                    commit(&s_full[ns & 1]);
                    commit(&k_empty[ns % C::kSlotsK]);
                    HTA_TR(21, 0, ns);
                    ++ns;
                    did = true;
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int j = np[h];
                    if (j < ns && (kNoMem || ready(&v_full[j % C::kSlotsV], (j / C::kSlotsV) & 1)) &&
                        ready(&p_full[2 * h + (j & 1)], (j >> 1) & 1)) {
                        HTA_TR(1, h, j);
                        tc_fence_after();
                        issue_PV(h, j & 1, j % C::kSlotsV, j > 0);
                        commit(&pv_done[2 * h + (j & 1)]);
                        if (np[1 - h] > j) commit(&v_empty[j % C::kSlotsV]);  // both halves read V_j
                        ++np[h];
                        did = true;
                    }
                }
                if (did) {
                    idle = 0;
                } else if (++idle > (1u << 26)) {
                    if (lane == 0) printf("hta: MMA issuer stalled (block %d)\n", blockIdx.x);
                    __trap();
                }
            }
            commit(o_final);
        }
        __syncwarp();
    } else {
        // ================= softmax warpgroup `half`: key columns [64*half, 64*half + 64) of every
        // tile, its own running max / sum and its own accumulator O_half
        const int half = (warp - 2) >> 2;
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;
        const int grow = row0 + r;
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        const float c = p.scale_log2;
        const uint32_t pfull0 = PAIR ? mapa_shared(smem_u32(&p_full[0]), 0) : 0u;
        constexpr int kHalfCols = kBlockN / 2;
        float m_run = -INFINITY, l_run = 0.f;
        for (int j = 0; j < n_tiles; ++j) {
            const int buf = j & 1;
            mbar_wait(&s_full[buf], static_cast<uint32_t>((j >> 1) & 1));
            if (quarter == 0) HTA_TR(10, half, j);
            tc_fence_after();
            const bool last = j == n_tiles - 1;
            float mt = 0.f, lsum = 0.f;
            uint32_t pk[kHalfCols / 2];
            if (HTA_SKIP < 1 || HTA_SKIP == 4) {
                float s[kHalfCols];
                tmem_ld64(tmem + lane_off + s_col(buf) + half * kHalfCols, s);
                if (last && tail_valid < kBlockN) {
                    // keys past the split end -> -inf (last tile only; the empty asm keeps this a
                    // real branch instead of per-element selects on every tile)
                    asm volatile("" ::: "memory");
#pragma unroll
                    for (int cc = 0; cc < kHalfCols; ++cc)
                        if (half * kHalfCols + cc >= tail_valid) s[cc] = -INFINITY;
                }
                float mx0 = s[0], mx1 = s[1], mx2 = s[2], mx3 = s[3];
#pragma unroll
                for (int cc = 4; cc < kHalfCols; cc += 8) {
                    mx0 = fmaxf(mx0, fmaxf(s[cc], s[cc + 4]));
                    mx1 = fmaxf(mx1, fmaxf(s[cc + 1], s[cc + 5]));
                    mx2 = fmaxf(mx2, fmaxf(s[cc + 2], s[cc + 6]));
                    mx3 = fmaxf(mx3, fmaxf(s[cc + 3], s[cc + 7]));
                }
                mt = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3)) * c;
                if (quarter == 0) HTA_TR(11, half, j);
                // a half with every key masked (tail) keeps its state: P = 0 below
                const float m_new = (mt > m_run + 8.0f) ? mt : m_run;
                const float m_use = m_new == -INFINITY ? 0.f : m_new;
                // P = exp2(S*c - m) -> bf16 over S in TMEM.  3 of every 8 column pairs use the
                // FMA-pipe polynomial, the rest MUFU ex2 (MUFU alone would co-limit the MMAs).
                const float2 c2 = make_float2(c, c), neg2 = make_float2(-m_use, -m_use);
                float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
                const float2 *s2 = reinterpret_cast<const float2 *>(s);
#pragma unroll
                for (int i = 0; i < kHalfCols / 2; ++i) {
                    const float2 x = __ffma2_rn(s2[i], c2, neg2);
                    float2 pp;
                    if ((i & 7) < 3) {
                        pp = exp2_poly2(x);
                    } else {
                        pp.x = fast_exp2(x.x);
                        pp.y = fast_exp2(x.y);
                    }
                    if (i & 1)
                        acc1 = __fadd2_rn(acc1, pp);
                    else
                        acc0 = __fadd2_rn(acc0, pp);
                    pk[i] = pack_bf16x2(pp.x, pp.y);
                }
                // P_half packed (bf16 x 2 per column) into the first 32 of this half's own 64 S
                // columns: it never overwrites S values the other half may still be reading
                tmem_st32(tmem + lane_off + s_col(buf) + half * kHalfCols, pk);
                lsum = (acc0.x + acc1.x) + (acc0.y + acc1.y);
                mt = m_new;
            } else {
                mt = 0.f;
                lsum = 1.f;
            }
            if (quarter == 0) HTA_TR(12, half, j);
            // Rescale O_half only when this half's running max moved.  O_half must then hold
            // P_{j-1} V_{j-1} first: wait for PV_half(j-1) on pv_done[2*half + (j-1)%2].  That
            // barrier cannot run two phases ahead (PV_half(j+1) needs P_half(j+1), not yet
            // published), so the parity wait is exact although most tiles never wait.
            const bool need = (j > 0) && (mt != m_run) && (m_run != -INFINITY);
            const float f = need ? fast_exp2(m_run - mt) : 1.0f;
            l_run = l_run * f + lsum;
            if (__any_sync(0xffffffffu, need)) {
                mbar_wait(&pv_done[2 * half + ((j - 1) & 1)], static_cast<uint32_t>(((j - 1) >> 1) & 1));
                tc_fence_after();
                if (quarter == 0) HTA_TR(14, half, j);
#pragma unroll 1
                for (int ch = 0; ch < D / 32; ++ch) {
                    float o[32];
                    tmem_ld32(tmem + lane_off + o_col(half) + ch * 32, o);
#pragma unroll
                    for (int e = 0; e < 32; ++e) o[e] *= f;
                    tmem_st32(tmem + lane_off + o_col(half) + ch * 32, *reinterpret_cast<uint32_t(*)[32]>(o));
                }
            }
            m_run = mt;
            if (last && tail_zero) {
                if (r >= tail_valid) {
                    // V rows past the sequence end: zero this half of this CTA's row (may be NaN)
                    uint8_t *vrow = sV + ((n_tiles - 1) % C::kSlotsV) * C::kVBytes + r * 128;
                    constexpr int kChunks16 = C::kVCols * 2 / 16;  // 16-byte chunks in this CTA's row
#pragma unroll
                    for (int cch = half * (kChunks16 / 2); cch < (half + 1) * (kChunks16 / 2); ++cch)
                        *reinterpret_cast<uint4 *>(vrow + (cch / 8) * (kBlockN * 128) + (cch % 8) * 16) =
                            make_uint4(0u, 0u, 0u, 0u);
                }
                fence_proxy_async_smem();
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                const int pi = 2 * half + buf;
                if (!PAIR)
                    mbar_arrive(&p_full[pi]);
                else if (last && tail_zero)
                    mbar_arrive_remote_release_cluster(pfull0 + 8u * pi);  // publishes zeroed V rows
                else
                    mbar_arrive_remote(pfull0 + 8u * pi);
            }
            if (quarter == 0) HTA_TR(13, half, j);
        }
        // ---- epilogue: merge the two halves' (m, O_h, l) exactly; warpgroup h writes output
        // columns [D/2 * h, D/2 * h + D/2)
        red[half * kRowsPerTile + r] = m_run;
        red[(2 + half) * kRowsPerTile + r] = l_run;
        mbar_wait(o_final, 0);
        named_bar_sync(1, 32 * C::kSoftmaxWarps);
        tc_fence_after();
        pdl_launch_dependents();
        const float m0 = red[r], m1 = red[kRowsPerTile + r];
        const float l0 = red[2 * kRowsPerTile + r], l1 = red[3 * kRowsPerTile + r];
        const float mm = fmaxf(m0, m1);
        const float w0 = m0 == -INFINITY ? 0.f : fast_exp2(m0 - mm);
        const float w1 = m1 == -INFINITY ? 0.f : fast_exp2(m1 - mm);
        const float l_tot = l0 * w0 + l1 * w1;
        const float inv = 1.0f / l_tot;
        const float a0 = w0 * inv, a1 = w1 * inv;
        const bool row_ok = grow < p.M;
        int t = 0, h = 0;
        if (row_ok) {
            t = grow / p.G;
            h = g * p.G + grow % p.G;
        }
        float4 *dst = reinterpret_cast<float4 *>(o_base + ((static_cast<int64_t>(b) * p.T + t) * p.H + h) * D);
#pragma unroll
        for (int ch = half * (D / 64); ch < (half + 1) * (D / 64); ++ch) {
            float x0[32], x1[32];
            tmem_ld32(tmem + lane_off + o_col(0) + ch * 32, x0);
            tmem_ld32(tmem + lane_off + o_col(1) + ch * 32, x1);
            if (row_ok) {
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    dst[ch * 8 + e] = make_float4(x0[4 * e] * a0 + x1[4 * e] * a1, x0[4 * e + 1] * a0 + x1[4 * e + 1] * a1,
                                                  x0[4 * e + 2] * a0 + x1[4 * e + 2] * a1,
                                                  x0[4 * e + 3] * a0 + x1[4 * e + 3] * a1);
            }
        }
        if (row_ok && half == 0)
            lse_base[(static_cast<int64_t>(b) * p.H + h) * p.T + t] = (mm + log2f(l_tot)) * 0.69314718055994530942f;
    }

    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync();  // no CTA of the pair leaves while the peer may still signal it
    if (warp == 1) {
        tc_fence_after();
        if (PAIR)
            tmem_dealloc2(tmem, 512);
        else
            tmem_dealloc(tmem, 512);
    }
}

#ifdef HTA_TRACE
extern "C" __attribute__((visibility("default"))) int hta_debug_set_trace(void *buf, int cta) {
    if (cudaMemcpyToSymbol(g_trace, &buf, sizeof(buf)) != cudaSuccess) return -1;
    return cudaMemcpyToSymbol(g_trace_cta, &cta, sizeof(cta)) == cudaSuccess ? 0 : -1;
}
#endif

template <int D, bool PAIR>
static cudaError_t launch_tc(const PrefixParams &p, const CUtensorMap &tk, const CUtensorMap &tv, cudaStream_t s) {
    using C = TcCfg<D, PAIR>;
    auto kern = prefix_tc_kernel<D, PAIR>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.n_mgroups * p.splits * p.H_kv * p.B * (PAIR ? 2 : 1));
    cfg.blockDim = dim3(C::kThreads);
    cfg.dynamicSmemBytes = C::kSmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = PAIR ? 2 : 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, tk, tv, p);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

int prefix_tc_smem_bytes(int d, int nt) {
    if (d == 128) return nt == 2 ? TcCfg<128, true>::kSmemBytes : TcCfg<128, false>::kSmemBytes;
    return TcCfg<64, false>::kSmemBytes;
}

cudaError_t launch_prefix_tc(const PrefixParams &p, const CUtensorMap &tk, const CUtensorMap &tv, int, cudaStream_t s) {
    if (p.d == 128) return p.nt == 2 ? launch_tc<128, true>(p, tk, tv, s) : launch_tc<128, false>(p, tk, tv, s);
    if (p.d == 64 && p.nt == 1) return launch_tc<64, false>(p, tk, tv, s);
    return cudaErrorInvalidValue;
}

}  // namespace hta
