// prefix_tc_3w.cu -- EXPERIMENT (DESIGN.md §11 item 1): the prefix kernel with three softmax warps
// per SM sub-partition (12 in all), one row per thread and a third of the 192 columns per warp;
// the three warps of a row agree on the speculative-max redo per tile through a named barrier.
// Build: tools/lib_variants.sh CMD "3w:@tools/variants_src/prefix_tc_3w.cu" (192-key tiles only).
//
// Based on prefix_tc.cu:
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
//  * KV tiles of kBlockN = 192 keys: TMEM holds two S/P buffers of 192 fp32 columns and the
//    128-column O accumulator (512 columns), and the fixed per-tile costs of the softmax warps
//    (barrier checks, publication, reduction latency) are spread over 192 keys.
//  * PAIR (M > 128, d = 128): a cluster of two CTAs on one TPC runs tcgen05.mma.cta_group::2
//    with M = 256: each CTA holds its 128 Q rows, HALF of every K tile (96 keys) and HALF of
//    every V tile (64 head-dim columns), so each KV byte is read from HBM once for 256 rows and
//    each SM streams only half of the operand bytes through shared memory.
//  * warp 0 (one lane) streams K and V tiles with TMA into two rings of smem slots (128B
//    swizzle, the canonical UMMA layout) so K tiles can run ahead of V tiles; in a pair both
//    CTAs' bytes are counted on the leader's barriers.
//  * warp 1 of the leader CTA issues the MMAs in a fixed order with suspended barrier waits, one
//    elected lane issuing each group (descriptors are warp-uniform and advanced by constants):
//    S = Q K^T into one of two TMEM buffers (fp32) once a K tile and a buffer are free, and
//    O += P V with A = P read from TMEM (the "TS" form) and B = V from smem (MN-major) once P and
//    the V tile are ready.
//  * warps 2-9 (softmax): the two warps that share a TMEM lane quarter own disjoint 16-row halves
//    of it, and each row is shared by a pair of threads (lanes t and t+16) that each hold 96 of
//    its 192 S values (tcgen05.ld .16x32bx2).  Per tile: row max (one shuffle between the pair),
//    exp2 (3/8 of the pairs on the FMA pipe by polynomial, the rest on MUFU), row sum, P -> bf16
//    -> tcgen05.st over S.  No two warps ever exchange data, so they drift freely and overlap
//    each other's latency.  O is rescaled in TMEM only when the running max grows by more than
//    2^8 (exact: the final normalisation uses the same, possibly stale, max).
//  * the epilogue divides O by the row sum and writes fp32 partials + natural-log LSE.
// A split with no visible key writes the sentinel (O = 0, LSE = -inf).
#include <cuda_bf16.h>
#include <cstdio>
#include <type_traits>

#include "hta_internal.h"
#include "ptx_sm100.cuh"

namespace hta {

// Optional pipeline timeline (build with -DHTA_TRACE, tools/trace_prefix.py): lane 0 of each
// traced warp of CTA g_trace_cta appends (event, tag, j, clock) records.
#ifdef HTA_TRACE
__device__ unsigned long long *g_trace = nullptr;
__device__ int g_trace_cta = 0;
__device__ unsigned long long g_cta_times[1024][4];  // per CTA: entry ns, loop start ns/clk, exit ns, exit clk
constexpr int kTraceRecs = 2048;  // per warp, written straight to g_trace (traced CTA only)
#define HTA_TR(ev, tag, jj)                                                                              \
    do {                                                                                                 \
        if (lane == 0 && tr_on && tr_n < kTraceRecs)                                                     \
            tr_buf[warp * kTraceRecs + tr_n++] = (static_cast<unsigned long long>(ev) << 56) |              \
                                                 (static_cast<unsigned long long>(tag) << 52) |           \
                                                 (static_cast<unsigned long long>((jj) & 0xFFFFF) << 32) |\
                                                 static_cast<unsigned long long>(static_cast<uint32_t>(clock64())); \
    } while (0)
__device__ __forceinline__ uint64_t trace_globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// clock and wall time (ns) side by side: the SM clock the kernel actually ran at
#define HTA_TR_CLK(ev)                                                                                   \
    do {                                                                                                 \
        const uint32_t c_ = static_cast<uint32_t>(clock64());                                            \
        const uint32_t t_ = static_cast<uint32_t>(trace_globaltimer());                                  \
        if (lane == 0 && tr_on && tr_n + 1 < kTraceRecs) {                                               \
            tr_buf[warp * kTraceRecs + tr_n++] = (static_cast<unsigned long long>(ev) << 56) | c_;       \
            tr_buf[warp * kTraceRecs + tr_n++] = (static_cast<unsigned long long>(ev + 1) << 56) | t_;   \
        }                                                                                                \
    } while (0)
#else
#define HTA_TR(ev, tag, jj) do { } while (0)
#define HTA_TR_CLK(ev) do { } while (0)
#endif

// Diagnostics only (tools/): HTA_SKIP=1 skips the softmax math, HTA_SKIP=2 also the MMAs,
// leaving the TMA stream and the barrier protocol; HTA_SKIP=3 runs the MMAs with no TMA traffic
// (operands are whatever sits in smem) and no softmax; HTA_SKIP=4 = 3 with the softmax.
// Product builds use 0.
// Publish P_j at the start of tile j+1 (see the softmax loop).
#ifndef HTA_DEFER
#define HTA_DEFER 1
#endif
#ifndef HTA_SKIP
#define HTA_SKIP 0
#endif
// Pairs of every 8 whose exp2 runs on the FMA pipe (polynomial) instead of MUFU.
#ifndef HTA_SPEC_MAX
#define HTA_SPEC_MAX 1
#endif
// Diagnostics: 1 = the contiguous-cache producers loop with the whole warp waiting on each
// mbarrier (+2 us on Llama-8B-64k); 0 = lane 0 alone loops (the other lanes are parked at the
// __syncwarp after the loop).  The paged producers always wait converged: their lanes take part
// in every tile (block-table lookups, shuffles), and a lane-0-only wait with the other 31 lanes
// at a per-tile __syncwarp made the paged pass 2x slower (profiles/r01b/README.md).
#ifndef HTA_CONV
#define HTA_CONV 0
#endif
#ifndef HTA_RING_KB
#define HTA_RING_KB 192
#endif
#ifndef HTA_POLY
#define HTA_POLY 3
#endif

#ifndef HTA_KV_POLICY
#define HTA_KV_POLICY kPolicyEvictFirst
#endif
constexpr uint64_t kKvPolicy = HTA_KV_POLICY;  // L2 policy of the streamed K/V tiles (read once)

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
    static constexpr int kRingBytes = (PAIR || D == 64 ? HTA_RING_KB : 192) * 1024;
#ifdef HTA_KRING_PCT  // diagnostics: share of the ring given to K tiles (percent)
    static constexpr int kSlotsK = (kRingBytes * HTA_KRING_PCT / 100) / kKBytes;
    static constexpr int kSlotsV = (kRingBytes - kSlotsK * kKBytes) / kVBytes;
#else
    static constexpr int kSlotsK = (kRingBytes / 2) / kKBytes;
    static constexpr int kSlotsV = (kRingBytes / 2) / kVBytes;
#endif
    static constexpr int kSBufs = 384 / kBlockN;                // S/P buffers in TMEM (2 x 192 or 3 x 128)
    static constexpr int kSoftmaxWarps = 12;                    // three per SM sub-partition
    static constexpr int kFirstSoftmaxWarp = 3;                 // warp 0 K TMA, 1 MMA + TMEM, 2 V TMA
    static constexpr int kThreads = 32 * (kFirstSoftmaxWarp + kSoftmaxWarps);
    static constexpr int kVOff = kQBytes + kSlotsK * kKBytes;   // start of the V ring
    static constexpr int kBarOff = kVOff + kSlotsV * kVBytes;
    static constexpr int kSmemBytes = kBarOff + 512 + 128 + 4 * 3 * 32 * 4;  // + row exchange
    static_assert(kSlotsK >= 2 && kSlotsV >= 2, "need at least 2 slots per ring");
    static_assert(kSmemBytes <= 232448, "shared memory budget");
};


__device__ __forceinline__ void tmem_ld_32x64_nowait(uint32_t taddr, float *v) {
    uint32_t *r = reinterpret_cast<uint32_t *>(v);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
                 : "r"(taddr)
                 : "memory");
}
__device__ __forceinline__ void tmem_st_32x16_nowait(uint32_t taddr, const uint32_t *r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
                 : "memory");
}

// TMEM column map: S/P buffer b at 128*b (b = 0, 1, 2), O at 384.
__device__ __forceinline__ uint32_t s_col(int buf) { return static_cast<uint32_t>(kBlockN * buf); }
constexpr uint32_t kOCol = 384u;  // O: 128 fp32 columns after the S buffers (384 + 128 = 512)

// this thread's N S values (N = 64 or 96; the other half of the warp at +N columns) and the wait
template <int N>
__device__ __forceinline__ void tmem_ld_S(uint32_t taddr, float *v) {
    if constexpr (N == 96) {
        tmem_ld_x96<96>(taddr, v);
    } else if constexpr (N == 48) {
        tmem_ld_x48<48>(taddr, v);
    } else {
        tmem_ld_x64_nowait<64>(taddr, v);
        tmem_ld_wait_fence<64>(v);
    }
}

// Pool row of logical key k of batch b (paged KV); pages past the table or negative entries read
// page 0 (such keys are past cache_seqlens: masked, and their V rows zeroed).
__device__ __forceinline__ int paged_row(const PrefixParams &p, int b, int k) {
    int page = k / p.page_size;
    page = page < p.max_pages ? page : p.max_pages - 1;
    int e = p.block_table[b * p.bt_stride + page];
    e = e < 0 ? 0 : e;
    return e * p.page_size + k % p.page_size;
}

template <int D, bool PAIR>
__global__ void __launch_bounds__(TcCfg<D, PAIR>::kThreads, 1)
    prefix_tc_kernel(const __grid_constant__ CUtensorMap tmap_q, const __grid_constant__ CUtensorMap tmap_k,
                     const __grid_constant__ CUtensorMap tmap_v, const PrefixParams p) {
    using C = TcCfg<D, PAIR>;
    extern __shared__ __align__(1024) uint8_t smem[];  // 128B-swizzled tiles need 1024B alignment
    uint8_t *sQ = smem;
    uint8_t *sK = smem + C::kQBytes;
    uint8_t *sV = smem + C::kVOff;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + C::kBarOff);
    uint64_t *k_full = bars;                       // [kSlotsK]  (the leader's copy is the one used)
    uint64_t *k_empty = k_full + C::kSlotsK;       // [kSlotsK]
    uint64_t *v_full = k_empty + C::kSlotsK;       // [kSlotsV]  (the leader's copy is the one used)
    uint64_t *v_empty = v_full + C::kSlotsV;       // [kSlotsV]
    uint64_t *s_full = v_empty + C::kSlotsV;       // [kSBufs]
    uint64_t *p_full = s_full + C::kSBufs;         // [kSBufs]   (the leader's copy is the one used)
    uint64_t *pv_done = p_full + C::kSBufs;        // [kSBufs]   PV_j arrives on pv_done[j % kSBufs]
    uint64_t *o_final = pv_done + C::kSBufs;       // [1]
    uint64_t *q_full = o_final + 1;                // [1]       Q staged (the leader's copy is the one used)
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(q_full + 1);

    const int warp = threadIdx.x >> 5;
#ifdef HTA_TRACE
    if (threadIdx.x == 0 && blockIdx.x < 1024) g_cta_times[blockIdx.x][0] = trace_globaltimer();
#endif
    const int lane = threadIdx.x & 31;
#ifdef HTA_TRACE
    int tr_n = 0;
    unsigned long long *tr_buf = g_trace;
    const bool tr_on = g_trace != nullptr && static_cast<int>(blockIdx.x) == g_trace_cta;
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
    // ---- one-time setup (reads no input: it overlaps the previous kernel under programmatic
    // dependent launch)
    if (threadIdx.x == 0 && (smem_u32(smem) & 1023u) != 0u) __trap();  // swizzle atoms need 1 KiB alignment
    if (warp == 0 && lane == 0) {
        if (p.q_tma) tma_prefetch_desc(&tmap_q);
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
        for (int i = 0; i < C::kSBufs; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], C::kSoftmaxWarps * (PAIR ? 2 : 1));
            mbar_init(&pv_done[i], 1);
        }
        mbar_init(o_final, 1);
        mbar_init(q_full, p.q_tma ? 1 : C::kSoftmaxWarps * (PAIR ? 2 : 1));
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
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync();  // barrier inits and TMEM allocation visible to the peer
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // Inputs (q, K/V, seqlens) may come from the kernel before this one on the stream: wait for it
    // (griddepcontrol.wait; a no-op unless it triggered this grid's launch early, as the tree-mask
    // kernel does).  The tree/merge kernel after this one reads the mask after its own wait.
    pdl_wait_primary();

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


    if (warp == 0) HTA_TR_CLK(50);
#ifdef HTA_TRACE
    if (threadIdx.x == 0 && blockIdx.x < 1024) {
        g_cta_times[blockIdx.x][1] = trace_globaltimer();
        g_cta_times[blockIdx.x][2] = clock64();
    }
#endif
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
    } else if (warp == 0) {
        // ================= TMA producer of Q and the K ring (K_j is consumed by S_j).  K and V
        // have producers of their own, so K tiles run ahead of V tiles by as many slots as the
        // K ring has (S_j frees K_j long before PV_j frees V_j).
        if (lane == 0 && p.q_tma) {  // Q first: it gates S_0 and must not queue behind K/V
            const int t0 = row0 / p.G;
            if (PAIR) {
                if (leader) mbar_arrive_expect_tx(q_full, 2u * C::kQBytes);
                const uint32_t qfull0 = mapa_shared(smem_u32(q_full), 0);
#pragma unroll
                for (int kb = 0; kb < C::kKB; ++kb)
                    tma_load_4d_pair(sQ + kb * C::kRegionBytes, &tmap_q, qfull0, kb * 64, g * p.G, t0, b,
                                     kPolicyEvictNormal);  // re-read by every split
            } else {
                mbar_arrive_expect_tx(q_full, C::kQBytes);
#pragma unroll
                for (int kb = 0; kb < C::kKB; ++kb)
                    tma_load_4d(sQ + kb * C::kRegionBytes, &tmap_q, q_full, kb * 64, g * p.G, t0, b,
                                kPolicyEvictNormal);
            }
        }
        if (p.page_size > 0 && HTA_SKIP < 3) {
            // paged KV: the whole warp runs the loop; lane i translates box i (16 keys) of the
            // tile through the block table, lane 0 issues the TMA boxes
            const uint32_t kfull0 = PAIR ? mapa_shared(smem_u32(&k_full[0]), 0) : 0u;
            constexpr int kBoxes = C::kKRows / 16;
            for (int j = 0; j < n_tiles; ++j) {
                const int n0 = static_cast<int>(key_lo) + j * kBlockN + (PAIR ? static_cast<int>(rank) * C::kKRows : 0);
                const int prow = paged_row(p, b, n0 + 16 * (lane < kBoxes ? lane : 0));
                const int slot = j % C::kSlotsK;
                mbar_wait(&k_empty[slot], ((j / C::kSlotsK) & 1) ^ 1u);  // the whole warp waits (converged)
                __syncwarp();
                HTA_TR(30, 0, j);
                uint8_t *dst = sK + slot * C::kKBytes;
                if (lane == 0) {
                    if (PAIR) {
                        if (leader) mbar_arrive_expect_tx(&k_full[slot], 2u * C::kKBytes);
                    } else {
                        mbar_arrive_expect_tx(&k_full[slot], C::kKBytes);
                    }
                }
#pragma unroll
                for (int i = 0; i < kBoxes; ++i) {
                    const int r = __shfl_sync(0xffffffffu, prow, i);
                    if (lane == 0) {
#pragma unroll
                        for (int kb = 0; kb < C::kKB; ++kb) {
                            uint8_t *dd = dst + kb * (C::kKRows * 128) + i * 2048;
                            if (PAIR)
                                tma_load_4d_pair(dd, &tmap_k, kfull0 + 8u * slot, kb * 64, g, r, 0, kKvPolicy);
                            else
                                tma_load_4d(dd, &tmap_k, &k_full[slot], kb * 64, g, r, 0, kKvPolicy);
                        }
                    }
                }
            }
        } else if ((HTA_CONV || lane == 0) && HTA_SKIP < 3) {
            const uint32_t kfull0 = PAIR ? mapa_shared(smem_u32(&k_full[0]), 0) : 0u;
            for (int j = 0; j < n_tiles; ++j) {
                const int n0 = static_cast<int>(key_lo) + j * kBlockN;
                const int slot = j % C::kSlotsK;
                mbar_wait(&k_empty[slot], ((j / C::kSlotsK) & 1) ^ 1u);
                uint8_t *dst = sK + slot * C::kKBytes;
                HTA_TR(30, 0, j);
                if (lane != 0) {
                } else if (PAIR) {
                    if (leader) mbar_arrive_expect_tx(&k_full[slot], 2u * C::kKBytes);
#pragma unroll
                    for (int kb = 0; kb < C::kKB; ++kb)
                        tma_load_4d_pair(dst + kb * (C::kKRows * 128), &tmap_k, kfull0 + 8u * slot, kb * 64, g,
                                         n0 + static_cast<int>(rank) * C::kKRows, b, kKvPolicy);
                } else {
                    mbar_arrive_expect_tx(&k_full[slot], C::kKBytes);
#pragma unroll
                    for (int kb = 0; kb < C::kKB; ++kb)
                        tma_load_4d(dst + kb * (kBlockN * 128), &tmap_k, &k_full[slot], kb * 64, g, n0, b, kKvPolicy);
                }
                if (HTA_CONV) __syncwarp();
            }
        }
        __syncwarp();
    } else if (warp == 2) {
        // ================= TMA producer of the V ring (V_j is consumed by PV_j)
        if (p.page_size > 0 && HTA_SKIP < 3) {
            const uint32_t vfull0 = PAIR ? mapa_shared(smem_u32(&v_full[0]), 0) : 0u;
            constexpr int kBoxes = kBlockN / 16;
            for (int j = 0; j < n_tiles; ++j) {
                const int n0 = static_cast<int>(key_lo) + j * kBlockN;
                const int prow = paged_row(p, b, n0 + 16 * (lane < kBoxes ? lane : 0));
                const int slot = j % C::kSlotsV;
                mbar_wait(&v_empty[slot], ((j / C::kSlotsV) & 1) ^ 1u);
                __syncwarp();
                HTA_TR(31, 0, j);
                uint8_t *dst = sV + slot * C::kVBytes;
                if (lane == 0) {
                    if (PAIR) {
                        if (leader) mbar_arrive_expect_tx(&v_full[slot], 2u * C::kVBytes);
                    } else {
                        mbar_arrive_expect_tx(&v_full[slot], C::kVBytes);
                    }
                }
#pragma unroll
                for (int i = 0; i < kBoxes; ++i) {
                    const int r = __shfl_sync(0xffffffffu, prow, i);
                    if (lane == 0) {
                        if (PAIR) {
                            tma_load_4d_pair(dst + i * 2048, &tmap_v, vfull0 + 8u * slot, static_cast<int>(rank) * 64,
                                             g, r, 0, kKvPolicy);
                        } else {
#pragma unroll
                            for (int kb = 0; kb < C::kKB; ++kb)
                                tma_load_4d(dst + kb * (kBlockN * 128) + i * 2048, &tmap_v, &v_full[slot], kb * 64, g,
                                            r, 0, kKvPolicy);
                        }
                    }
                }
            }
        } else if ((HTA_CONV || lane == 0) && HTA_SKIP < 3) {
            const uint32_t vfull0 = PAIR ? mapa_shared(smem_u32(&v_full[0]), 0) : 0u;
            for (int j = 0; j < n_tiles; ++j) {
                const int n0 = static_cast<int>(key_lo) + j * kBlockN;
                const int slot = j % C::kSlotsV;
                mbar_wait(&v_empty[slot], ((j / C::kSlotsV) & 1) ^ 1u);
                uint8_t *dst = sV + slot * C::kVBytes;
                HTA_TR(31, 0, j);
                if (lane != 0) {
                } else if (PAIR) {
                    if (leader) mbar_arrive_expect_tx(&v_full[slot], 2u * C::kVBytes);
                    tma_load_4d_pair(dst, &tmap_v, vfull0 + 8u * slot, static_cast<int>(rank) * 64, g, n0, b,
                                     kKvPolicy);
                } else {
                    mbar_arrive_expect_tx(&v_full[slot], C::kVBytes);
#pragma unroll
                    for (int kb = 0; kb < C::kKB; ++kb)
                        tma_load_4d(dst + kb * (kBlockN * 128), &tmap_v, &v_full[slot], kb * 64, g, n0, b, kKvPolicy);
                }
                if (HTA_CONV) __syncwarp();
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
            // One elected lane issues each group of MMAs; the descriptors are warp-uniform values
            // computed outside the elected branch, so ptxas keeps them in uniform registers and
            // each tcgen05.mma costs a few instructions (issue must stay well under 64 cycles per
            // N=128 MMA, and this warp shares its sub-partition with two softmax warps).
            auto commit = [](uint64_t *bar) {
                if (PAIR)
                    tc_commit2_mc(bar);
                else
                    tc_commit(bar);
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
                        mma2_bf16_ss(d_t, qd0 + qo, kd + ko, idesc_qk, k > 0 ? 1u : 0u);
                    else
                        mma_bf16_ss(d_t, qd0 + qo, kd + ko, idesc_qk, k > 0 ? 1u : 0u);
                }
            };
            auto issue_PV = [&](int buf, int slot, bool acc) {
                if (HTA_SKIP == 1 || HTA_SKIP == 2) return;
                const uint32_t a_t = tmem + s_col(buf);
                const uint64_t vd = vd0 + static_cast<uint32_t>((slot * C::kVBytes) >> 4);
#pragma unroll
                for (int k = 0; k < kBlockN / 16; ++k) {
                    // MN-major SW128: 16 keys = two 8-row groups = +2048 B per K step
                    if (PAIR)
                        mma2_bf16_ts(tmem + kOCol, a_t + k * 8, vd + static_cast<uint32_t>(k * 128), idesc_pv,
                                     (acc || k > 0) ? 1u : 0u);
                    else
                        mma_bf16_ts(tmem + kOCol, a_t + k * 8, vd + static_cast<uint32_t>(k * 128), idesc_pv,
                                    (acc || k > 0) ? 1u : 0u);
                }
            };
            const bool issuer = elect_one() != 0;
            // Fixed order with hardware-suspended waits (no polling: a spinning issuer would take
            // issue slots from the softmax warps sharing its SM sub-partition):
            //   S_0, S_1, then for every j: PV_j (needs V_j and P_j), S_{j+2} (needs K_{j+2}; its
            //   buffer was last read by PV_j, issued just before).
            constexpr bool kNoMem = HTA_SKIP >= 3;
            auto wait_all = [](uint64_t *bar, uint32_t parity) {
                mbar_wait(bar, parity);
                __syncwarp();
            };
            auto start_S = [&](int jj) {
                if (!kNoMem) {
                    wait_all(&k_full[jj % C::kSlotsK], (jj / C::kSlotsK) & 1);
                    HTA_TR(23, 0, jj);
                    if (tail_zero && jj == n_tiles - 1)  // the softmax warps sanitise V of this tile
                        wait_all(&v_full[jj % C::kSlotsV], (jj / C::kSlotsV) & 1);
                }
                tc_fence_after();
                if (issuer) {
                    issue_S(jj % C::kSBufs, jj % C::kSlotsK);
                    commit(&s_full[jj % C::kSBufs]);
                    commit(&k_empty[jj % C::kSlotsK]);
                }
                __syncwarp();
                HTA_TR(21, 0, jj);
            };
            if (PAIR && !p.q_tma)
                mbar_wait_cluster(q_full, 0);  // staged by both CTAs' threads (generic proxy)
            else
                mbar_wait(q_full, 0);
            __syncwarp();
            HTA_TR(22, 0, 0);
            for (int jj = 0; jj < C::kSBufs && jj < n_tiles; ++jj) start_S(jj);
            for (int j = 0; j < n_tiles; ++j) {
                if (!kNoMem) wait_all(&v_full[j % C::kSlotsV], (j / C::kSlotsV) & 1);
                HTA_TR(24, 0, j);
                wait_all(&p_full[j % C::kSBufs], (j / C::kSBufs) & 1);
                HTA_TR(1, 0, j);
                tc_fence_after();
                if (issuer) {
                    issue_PV(j % C::kSBufs, j % C::kSlotsV, j > 0);
                    commit(&pv_done[j % C::kSBufs]);
                    commit(&v_empty[j % C::kSlotsV]);
                }
                __syncwarp();
                if (j + C::kSBufs < n_tiles) start_S(j + C::kSBufs);
            }
            if (issuer) commit(o_final);
        }
        __syncwarp();
    } else {
        // ================= softmax: warp w owns rows 32*(w%4) + 16*rh .. +15 of the tile (rh =
        // (w-3)/4); lane t holds row (t & 15) of them, keys [96*(t>>4), 96*(t>>4) + 96)
        const int sw = warp - C::kFirstSoftmaxWarp;
        if (!p.q_tma) {  // this CTA's 128 Q rows -> smem in the canonical K-major SWIZZLE_128B
            // layout (G does not divide 128: no TMA box), staged by the softmax warps
            const __nv_bfloat16 *q = static_cast<const __nv_bfloat16 *>(p.q);
            constexpr int kQThreads = 32 * C::kSoftmaxWarps;
            constexpr int kChunks = D / 8;  // 16-byte chunks per row
            constexpr int kPer = (kRowsPerTile * kChunks + kQThreads - 1) / kQThreads;
            const int qt = threadIdx.x - 32 * C::kFirstSoftmaxWarp;
            // all loads of a thread in flight at once (a load/store loop would serialise kPer cold
            // HBM latencies)
            uint4 val[kPer];
#pragma unroll
            for (int i = 0; i < kPer; ++i) {
                const int idx = qt + i * kQThreads;
                const int r = idx / kChunks, ch = idx % kChunks;
                const int grow = row0 + r;
                val[i] = make_uint4(0u, 0u, 0u, 0u);
                if (idx < kRowsPerTile * kChunks && grow < p.M) {
                    const int t = grow / p.G, h = g * p.G + grow % p.G;
                    val[i] = __ldg(reinterpret_cast<const uint4 *>(q + b * p.qs0 + t * p.qs1 + h * p.qs2 + ch * 8));
                }
            }
#pragma unroll
            for (int i = 0; i < kPer; ++i) {
                const int idx = qt + i * kQThreads;
                const int r = idx / kChunks, ch = idx % kChunks;
                if (idx < kRowsPerTile * kChunks)
                    *reinterpret_cast<uint4 *>(sQ + (ch / 8) * C::kRegionBytes + r * 128 + (((ch & 7) ^ (r & 7)) << 4)) =
                        val[i];
            }
            fence_proxy_async_smem();  // generic-proxy stores -> read by the tensor core
            __syncwarp();
            HTA_TR(14, sw, 0);
            if (lane == 0) {
                if (PAIR)
                    mbar_arrive_remote_release_cluster(mapa_shared(smem_u32(q_full), 0));
                else
                    mbar_arrive(q_full);
            }
        }
        // Three softmax warps per lane quarter (one per third of the 192 columns); lane = row.
        const int quarter = warp & 3;
        const int third = sw >> 2;                       // 0, 1, 2: columns [64*third, +64)
        constexpr int kCols = kBlockN / 3;               // 64 S columns per thread
        static_assert(kBlockN % 48 == 0 && kCols % 16 == 0, "thirds of 16-pair chunks");
        const int r = quarter * 32 + lane;
        const int grow = row0 + r;
        const bool pad_warp = row0 + quarter * 32 >= p.M;  // the quarter's 3 warps agree
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        const uint32_t bar_id = 1u + static_cast<uint32_t>(quarter);  // named barrier of the 3 warps
        int *xflag = reinterpret_cast<int *>(smem + C::kBarOff + 512);           // [2][4][3]
        float *xval = reinterpret_cast<float *>(smem + C::kBarOff + 512 + 128);  // [4][3][32]
        float *my_x = xval + (quarter * 3 + third) * 32 + lane;
        const float c = p.scale_log2;
        const uint32_t pfull0 = PAIR ? mapa_shared(smem_u32(&p_full[0]), 0) : 0u;
        float m_run = -INFINITY, l_run = 0.f;  // l_run: this thread's third of the row
        auto publish = [&](int jp) {
            tmem_st_wait();
            if (jp == n_tiles - 1 && tail_zero) {
                for (int kr = r; kr < kBlockN; kr += kRowsPerTile) {
                    if (kr < tail_valid) continue;
                    uint8_t *vrow = sV + ((n_tiles - 1) % C::kSlotsV) * C::kVBytes + kr * 128;
                    constexpr int kChunks16 = C::kVCols * 2 / 16;
                    for (int cch = third; cch < kChunks16; cch += 3)
                        *reinterpret_cast<uint4 *>(vrow + (cch / 8) * (kBlockN * 128) + (cch % 8) * 16) =
                            make_uint4(0u, 0u, 0u, 0u);
                }
                fence_proxy_async_smem();
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                const int pb = jp % C::kSBufs;
                if (!PAIR)
                    mbar_arrive(&p_full[pb]);
                else if (jp == n_tiles - 1 && tail_zero)
                    mbar_arrive_remote_release_cluster(pfull0 + 8u * pb);
                else
                    mbar_arrive_remote(pfull0 + 8u * pb);
            }
            HTA_TR(13, sw, jp);
        };
        // the three warps of a row exchange one float per row (xval), between two named barriers
        auto row_reduce = [&](float v, bool is_max) {
            *my_x = v;
            named_bar_sync(bar_id, 96);
            const float *q0 = xval + quarter * 96 + lane;
            const float a = q0[0], b2 = q0[32], c3 = q0[64];
            named_bar_sync(bar_id, 96);  // the slots are free again
            return is_max ? fmaxf(a, fmaxf(b2, c3)) : (a + b2) + c3;
        };
        for (int j = 0; j < n_tiles; ++j) {
            const int buf = j % C::kSBufs;
            mbar_wait(&s_full[buf], static_cast<uint32_t>((j / C::kSBufs) & 1));
            HTA_TR(10, sw, j);
            tc_fence_after();
            const bool last = j == n_tiles - 1;
            float mt = m_run, lsum = 0.f;
            if (pad_warp) {
                if (j > 0) publish(j - 1);
            } else {
                float s[kCols];
                if (j > 0) publish(j - 1);
                tmem_ld_32x64_nowait(tmem + lane_off + s_col(buf) + kCols * third, s);
                tmem_ld_wait_fence<kCols>(s);
                if (last && tail_valid < kBlockN) {
                    asm volatile("" ::: "memory");
                    const int lim = tail_valid - third * kCols;
#pragma unroll
                    for (int cc = 0; cc < kCols; ++cc)
                        if (cc >= lim) s[cc] = -INFINITY;
                }
                float xmax_poly = -INFINITY;
                auto exp_store = [&](float m_use, auto spec) {
                    constexpr bool kSpec = decltype(spec)::value;
                    const float2 c2 = make_float2(c, c), neg2 = make_float2(-m_use, -m_use);
                    float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
                    const float2 *s2 = reinterpret_cast<const float2 *>(s);
                    uint32_t pk[16];
#pragma unroll
                    for (int i = 0; i < kCols / 2; ++i) {
                        const float2 x = __ffma2_rn(s2[i], c2, neg2);
                        float2 pp;
                        if ((i & 7) < HTA_POLY) {
                            if (kSpec) xmax_poly = max3f(xmax_poly, x.x, x.y);
                            pp = exp2_poly2<!kSpec>(x);
                        } else {
                            pp.x = fast_exp2(x.x);
                            pp.y = fast_exp2(x.y);
                        }
                        if (i & 1)
                            acc1 = __fadd2_rn(acc1, pp);
                        else
                            acc0 = __fadd2_rn(acc0, pp);
                        pk[i & 15] = pack_bf16x2(pp.x, pp.y);
                        if ((i & 15) == 15)
                            tmem_st_32x16_nowait(tmem + lane_off + s_col(buf) + (kCols / 2) * third + (i - 15), pk);
                    }
                    return (acc0.x + acc1.x) + (acc0.y + acc1.y);
                };
                HTA_TR(11, sw, j);
                lsum = exp_store(m_run, std::true_type{});
                // the three warps of the row agree on a redo (flag per warp, double-buffered by tile)
                const int mine = __any_sync(0xffffffffu, !(lsum <= 0x1p60f) || xmax_poly > 60.f) ? 1 : 0;
                int *fl = xflag + (j & 1) * 12 + quarter * 3;
                if (lane == 0) fl[third] = mine;
                named_bar_sync(bar_id, 96);
                if (fl[0] | fl[1] | fl[2]) {
                    tmem_st_wait();
                    float mx0 = s[0], mx1 = s[1], mx2 = s[2], mx3 = s[3];
#pragma unroll
                    for (int cc = 4; cc < kCols; cc += 4) {
                        mx0 = fmaxf(mx0, s[cc]);
                        mx1 = fmaxf(mx1, s[cc + 1]);
                        mx2 = fmaxf(mx2, s[cc + 2]);
                        mx3 = fmaxf(mx3, s[cc + 3]);
                    }
                    const float mx = row_reduce(fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3)), true) * c;
                    mt = mx > m_run ? mx : m_run;
                    lsum = exp_store(mt, std::false_type{});
                }
            }
            HTA_TR(12, sw, j);
            const bool need = (j > 0) && (mt != m_run);
            const float f = need ? fast_exp2(m_run - mt) : 1.0f;
            l_run = l_run * f + lsum;
            if (__any_sync(0xffffffffu, need)) {
                mbar_wait(&pv_done[(j - 1) % C::kSBufs], static_cast<uint32_t>(((j - 1) / C::kSBufs) & 1));
                tc_fence_after();
#pragma unroll 1
                for (int ch = third; ch < D / 32; ch += 3) {  // this warp's 32-column chunks of O
                    float o[32];
                    tmem_ld32(tmem + lane_off + kOCol + 32 * ch, *reinterpret_cast<float(*)[32]>(o));
#pragma unroll
                    for (int e = 0; e < 32; ++e) o[e] *= f;
                    tmem_st32(tmem + lane_off + kOCol + 32 * ch, *reinterpret_cast<uint32_t(*)[32]>(o));
                }
            }
            m_run = mt;
        }
        if (n_tiles > 0) publish(n_tiles - 1);
        mbar_wait(o_final, 0);
        tc_fence_after();
        pdl_launch_dependents();
        const float l_tot = pad_warp ? 1.f : row_reduce(l_run, false);
        const float inv = 1.0f / l_tot;
        const bool row_ok = grow < p.M;
        int t = 0, h = 0;
        if (row_ok) {
            t = grow / p.G;
            h = g * p.G + grow % p.G;
        }
        float *dst = o_base + ((static_cast<int64_t>(b) * p.T + t) * p.H + h) * D;
        for (int ch = third; ch < D / 32; ch += 3) {
            float o[32];
            tmem_ld32(tmem + lane_off + kOCol + 32 * ch, *reinterpret_cast<float(*)[32]>(o));
            if (row_ok) {
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    reinterpret_cast<float4 *>(dst + 32 * ch)[e] =
                        make_float4(o[4 * e] * inv, o[4 * e + 1] * inv, o[4 * e + 2] * inv, o[4 * e + 3] * inv);
            }
        }
        if (row_ok && third == 0)
            lse_base[(static_cast<int64_t>(b) * p.H + h) * p.T + t] = (m_run + log2f(l_tot)) * 0.69314718055994530942f;
    }

#ifdef HTA_TRACE
    if (warp == 3) HTA_TR_CLK(52);
    if (threadIdx.x == 96 && blockIdx.x < 1024) {
        g_cta_times[blockIdx.x][3] = trace_globaltimer();
        g_cta_times[blockIdx.x][2] = clock64() - g_cta_times[blockIdx.x][2];
    }
#endif
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
extern "C" __attribute__((visibility("default"))) int hta_debug_cta_times(void *host_out) {
    return cudaMemcpyFromSymbol(host_out, g_cta_times, sizeof(g_cta_times)) == cudaSuccess ? 0 : -1;
}
#endif

template <int D, bool PAIR>
static cudaError_t launch_tc(const PrefixParams &p, const CUtensorMap &tq, const CUtensorMap &tk, const CUtensorMap &tv,
                             cudaStream_t s) {
    using C = TcCfg<D, PAIR>;
    auto kern = prefix_tc_kernel<D, PAIR>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.n_mgroups * p.splits * p.H_kv * p.B * (PAIR ? 2 : 1));
    cfg.blockDim = dim3(C::kThreads);
    cfg.dynamicSmemBytes = C::kSmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = PAIR ? 2 : 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    // programmatic dependent launch: the prologue (barriers, TMEM, descriptor prefetch) overlaps
    // the previous kernel when it allows it (griddepcontrol.wait guards every input read)
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    e = cudaLaunchKernelEx(&cfg, kern, tq, tk, tv, p);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

int prefix_tc_smem_bytes(int d, int nt) {
    if (d == 128) return nt == 2 ? TcCfg<128, true>::kSmemBytes : TcCfg<128, false>::kSmemBytes;
    return TcCfg<64, false>::kSmemBytes;
}

cudaError_t launch_prefix_tc(const PrefixParams &p, const CUtensorMap &tq, const CUtensorMap &tk, const CUtensorMap &tv,
                             int, cudaStream_t s) {
    if (p.d == 128)
        return p.nt == 2 ? launch_tc<128, true>(p, tq, tk, tv, s) : launch_tc<128, false>(p, tq, tk, tv, s);
    if (p.d == 64 && p.nt == 1) return launch_tc<64, false>(p, tq, tk, tv, s);
    return cudaErrorInvalidValue;
}

}  // namespace hta
