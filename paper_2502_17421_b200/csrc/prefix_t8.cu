// prefix_t8.cu -- the prefix pass (split-KV partials as in prefix_tc.cu)
// over an FP8 (E4M3) KV cache for units of at most 64 query rows (MHA with T <= 64, e.g.
// LongChat-16k; the draft frontier), in TRANSPOSED form:
//
//   S^T_j = K_j Q^T        A = K_j (128 keys x d, f16) in TMEM,   B = Q (64 rows x d) in smem
//   O^T  += V_j^T P_j^T    A = V_j^T (d x 128 keys, f16) in smem, B = P_j^T (128 keys x 64 rows) in smem
//
// so the MMAs have no padding rows (N = 64 query rows; the untransposed f16 kernel, prefix_tc.cu
// KV8, runs M = 128 with 64 padding rows for such units).  The E4M3 K tiles land by TMA (128-byte
// swizzle) in a staging ring and are widened straight into TMEM (tcgen05.st, thread = key), so
// the f16 K never touches shared memory; the E4M3 V tiles land in the upper half of f16 slots and
// are widened in place (rows are independent for 128-byte rows), V^T being the MN-major view of
// the f16 V tile.  Shared-memory traffic per 128-key tile: TMA 32 KB, widening 16 + 16 KB read
// and 32 KB written, Q 16 KB, P^T 16 KB written and read, V 32 KB read = 176 KB (224 KB for the
// untransposed kernel).
//
// Softmax in the transposed layout: S^T has one key per TMEM lane and one query row per column,
// so a thread holds 16 rows of ONE key.  The row max is speculative (the running max m of the
// earlier tiles, in shared memory): a tile is exponentiated against it unless some key exceeds it
// by more than 15 (f16 P's range, 2^15); the four warps that share a row quarter vote on that with
// one bar.red.or.  An overflowing tile (the first tile of a split, a jump of the logits) finds
// the row maxima with an in-warp transposing reduction and a 4-warp exchange, raises m, rescales
// the row sums and O^T, and is then exponentiated.  Row sums are accumulated per (thread = key,
// row) in registers and reduced once, in the epilogue.
//
// Warps (26, one CTA per SM): 0-15 softmax (lane quarter w % 4, rows 16*(w/4)..+15), 16-19 K
// widening (lane quarter w % 4), 20-23 V widening (32 key rows each), 24 TMA, 25 MMA + TMEM.
// TMEM (512 columns allocated): S^T x3 at 0/64/128, K x2 at 192/256, O^T at 320.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "hta_internal.h"
#include "ptx_sm100.cuh"

#if HTA_T8

namespace hta {

// Pipeline timeline (diagnostics: libhta_trace.so, tools/trace_prefix.py with FP8=1): lane 0 of
// every warp of CTA g_trace_t8_cta records (event, tile, clock).
#ifdef HTA_TRACE
__device__ unsigned long long *g_trace_t8 = nullptr;
__device__ int g_trace_t8_cta = 0;
#define T8_TR(ev, jj)                                                                                      \
    do {                                                                                                   \
        if (tr_on && lane == 0 && tr_n < 1024)                                                             \
            tr_buf[warp * 1024 + tr_n++] = (static_cast<unsigned long long>(ev) << 56) |                   \
                                           (static_cast<unsigned long long>((jj) & 0xFFFFFF) << 32) |      \
                                           static_cast<uint32_t>(clock64());                               \
    } while (0)
#define T8_TRS(k) tr_c[k] = static_cast<uint32_t>(clock64())
#define T8_TRFLUSH(jj)                                                                                     \
    do {                                                                                                   \
        for (int k_ = 0; k_ < 4; ++k_)                                                                     \
            if (tr_on && lane == 0 && tr_n < 1024)                                                         \
                tr_buf[warp * 1024 + tr_n++] = (static_cast<unsigned long long>(50 + k_) << 56) |          \
                                               (static_cast<unsigned long long>((jj) & 0xFFFFFF) << 32) | tr_c[k_]; \
    } while (0)
extern "C" __attribute__((visibility("default"))) int hta_debug_set_trace_t8(void *buf, int cta) {
    if (cudaMemcpyToSymbol(g_trace_t8, &buf, sizeof(buf)) != cudaSuccess) return -1;
    return cudaMemcpyToSymbol(g_trace_t8_cta, &cta, sizeof(cta)) == cudaSuccess ? 0 : -1;
}
#else
#define T8_TR(ev, jj) \
    do {              \
    } while (0)
#define T8_TRS(k) \
    do {          \
    } while (0)
#define T8_TRFLUSH(jj) \
    do {               \
    } while (0)
#endif

namespace {

constexpr int kT8Keys = 128;  // keys per tile (M of both MMAs is 128: keys for S^T, d for O^T)
constexpr int kT8Rows = 64;   // query rows per unit (N of both MMAs)
constexpr int kT8Stages = 5;  // E4M3 K staging slots
constexpr int kT8VSlots = 3;  // f16 V slots (E4M3 landed in the upper half, widened in place)
constexpr int kT8SWarps = 16;                    // softmax warps: lane quarter w % 4, row quarter w / 4
constexpr int kT8RW = kT8Rows / (kT8SWarps / 4);  // query rows per softmax warp (16)
constexpr int kT8WarpKW = 16, kT8WarpVW = 20, kT8WarpTma = 24, kT8WarpMma = 25;
constexpr int kT8Threads = 26 * 32;  // 832 threads at 72 registers (7 warps x 32 x 72 <= 16 K per sub-partition)

constexpr uint32_t kT8SCol = 0, kT8KCol = 192, kT8OCol = 320;

constexpr int kT8QBytes = kT8Rows * 128 * 2;      // Q f16, K-major SW128: 2 atoms [64 rows][128 B]
constexpr int kT8PBytes = kT8Keys * kT8Rows * 2;  // P^T f16, MN-major SW128: [128 keys][64 rows]
constexpr int kT8StBytes = kT8Keys * 128;         // one E4M3 K tile [128 keys][128 B], 128-byte swizzle
constexpr int kT8VBytes = kT8Keys * 128 * 2;      // f16 V tile: 2 atoms [128 keys][128 B], SW128
constexpr int kT8OffP = kT8QBytes;
constexpr int kT8OffKs = kT8OffP + 2 * kT8PBytes;
constexpr int kT8OffV = kT8OffKs + kT8Stages * kT8StBytes;
constexpr int kT8OffBar = kT8OffV + kT8VSlots * kT8VBytes;
constexpr int kT8NumBars = 2 * kT8Stages + 3 * kT8VSlots + 2 + 2 + 2 + 3 + 3 + 2 + 2;
constexpr int kT8OffM = (kT8OffBar + 8 * kT8NumBars + 15) / 16 * 16;  // m_run[64], fac[64], red[4][64], tmem slot
constexpr int kT8SmemBytes = kT8OffM + (64 + 64 + 256) * 4 + 16;
static_assert(kT8SmemBytes <= 232448, "shared memory budget");
static_assert(kT8OffKs % 1024 == 0 && kT8StBytes % 1024 == 0, "swizzled tiles need 1 KiB alignment");

constexpr uint64_t kT8KvPolicy = kPolicyEvictFirst;  // streamed once
constexpr float kT8Limit = 15.0f;                    // P <= 2^15 (f16)
#ifndef HTA_T8_L2_AHEAD
#define HTA_T8_L2_AHEAD 6
#endif
constexpr int kT8L2Ahead = HTA_T8_L2_AHEAD;  // tiles staged in L2 beyond the ring

__device__ __forceinline__ void t8_st32(uint32_t taddr, const uint32_t *r) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
__device__ __forceinline__ void t8_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t *r = reinterpret_cast<uint32_t *>(v);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr)
                 : "memory");
    tmem_ld_wait_fence<16>(v);
}
__device__ __forceinline__ void t8_st16(uint32_t taddr, const uint32_t *r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
                     taddr),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
                 "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
                 : "memory");
}
// Named barrier over n threads that returns the OR of v over them.
__device__ __forceinline__ bool bar_red_or(uint32_t id, uint32_t n, bool v) {
    uint32_t r;
    asm volatile(
        "{\n\t.reg .pred p, q;\n\tsetp.ne.u32 q, %1, 0;\n\tbar.red.or.pred p, %2, %3, q;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(r)
        : "r"(static_cast<uint32_t>(v)), "r"(id), "r"(n)
        : "memory");
    return r != 0u;
}
// Transposing reduction: lane L holds v[0..N-1] (one value per row); afterwards v[0] of lane L
// is the reduction over the 32 lanes of row L % N (N - 1 + log2(32 / N) shuffles).
template <bool MAX, int N>
__device__ __forceinline__ float xreduce(float (&v)[N], int lane) {
#pragma unroll
    for (int o = N / 2; o >= 1; o >>= 1) {
        const bool hi = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const float keep = hi ? v[i + o] : v[i];
            const float send = hi ? v[i] : v[i + o];
            const float got = __shfl_xor_sync(0xffffffffu, send, o);
            v[i] = MAX ? fmaxf(keep, got) : keep + got;
        }
    }
#pragma unroll
    for (int o = N; o < 32; o <<= 1) {
        const float got = __shfl_xor_sync(0xffffffffu, v[0], o);
        v[0] = MAX ? fmaxf(v[0], got) : v[0] + got;
    }
    return v[0];
}

__global__ void __launch_bounds__(kT8Threads, 1)
    prefix_t8_kernel(const __grid_constant__ CUtensorMap tmap_k, const __grid_constant__ CUtensorMap tmap_v,
                     const PrefixParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *sQ = smem;
    uint8_t *sP = smem + kT8OffP;
    uint8_t *sKs = smem + kT8OffKs;
    uint8_t *sV = smem + kT8OffV;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + kT8OffBar);
    uint64_t *kst_land = bars;                  // [S] E4M3 K tile landed (TMA bytes)
    uint64_t *kst_free = kst_land + kT8Stages;  // [S] ... read by the 4 K widening warps
    uint64_t *v_land = kst_free + kT8Stages;    // [3] E4M3 V tile landed (TMA bytes)
    uint64_t *v_full = v_land + kT8VSlots;      // [3] ... widened (4 arrivals)
    uint64_t *v_free = v_full + kT8VSlots;      // [3] PV done with the slot (commit)
    uint64_t *k_full = v_free + kT8VSlots;      // [2] K_j in TMEM (4 arrivals)
    uint64_t *k_free = k_full + 2;              // [2] S^T_j done (commit)
    uint64_t *pv_done = k_free + 2;             // [2] PV_j done (commit): frees P^T buffer j % 2
    uint64_t *s_full = pv_done + 2;             // [3] S^T_j in TMEM (commit)
    uint64_t *s_free = s_full + 3;              // [3] S^T_j loaded by the 8 softmax warps
    uint64_t *p_full = s_free + 3;              // [2] P^T_j in smem (8 arrivals)
    uint64_t *o_final = p_full + 2;             // [1]
    uint64_t *q_full = o_final + 1;             // [1] Q staged (8 arrivals)
    float *m_run = reinterpret_cast<float *>(smem + kT8OffM);  // [64] running max (log2 units, x c)
    float *fac = m_run + 64;                                    // [64] rescale factors of an overflow tile
    float *red = fac + 64;                                      // [4][64] cross-warp exchange
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(red + 256);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
#ifdef HTA_TRACE
    unsigned long long *const tr_buf = g_trace_t8;
    const bool tr_on = tr_buf != nullptr && static_cast<int>(blockIdx.x) == g_trace_t8_cta;
    int tr_n = 0;
    uint32_t tr_c[4] = {0, 0, 0, 0};
#endif
    T8_TR(0, 0);
    int rest = blockIdx.x;
    const int split = rest % p.splits;
    rest /= p.splits;
    const int g = rest % p.H_kv;
    const int b = rest / p.H_kv;

    if (threadIdx.x == 0 && (smem_u32(smem) & 1023u) != 0u) __trap();
    if (warp == kT8WarpTma && lane == 0) {
        tma_prefetch_desc(&tmap_k);
        tma_prefetch_desc(&tmap_v);
    }
    if (warp == kT8WarpMma && lane == 0) {
        for (int i = 0; i < kT8Stages; ++i) {
            mbar_init(&kst_land[i], 1);
            mbar_init(&kst_free[i], 4);
        }
        for (int i = 0; i < kT8VSlots; ++i) {
            mbar_init(&v_land[i], 1);
            mbar_init(&v_full[i], 4);
            mbar_init(&v_free[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&k_full[i], 4);
            mbar_init(&k_free[i], 1);
            mbar_init(&pv_done[i], 1);
            mbar_init(&p_full[i], kT8SWarps);
        }
        for (int i = 0; i < 3; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&s_free[i], kT8SWarps);
        }
        mbar_init(o_final, 1);
        mbar_init(q_full, kT8SWarps);
        fence_mbar_init();
    }
    if (threadIdx.x < 64) m_run[threadIdx.x] = -INFINITY;
    if (warp == kT8WarpMma) {
        tmem_alloc(tmem_slot, 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    pdl_wait_primary();  // inputs may come from the previous kernel on the stream

    int64_t n_b = p.N_max;
    if (p.seqlens != nullptr) {
        n_b = p.seqlens[b];
        n_b = n_b < 0 ? 0 : (n_b > p.N_max ? p.N_max : n_b);
    }
    const int64_t key_lo = static_cast<int64_t>(split) * p.tiles_per_split * kT8Keys;
    int64_t key_hi = key_lo + static_cast<int64_t>(p.tiles_per_split) * kT8Keys;
    if (key_hi > n_b || split == p.splits - 1) key_hi = n_b;
    const int nc = key_hi > key_lo ? static_cast<int>((key_hi - key_lo + kT8Keys - 1) / kT8Keys) : 0;
    const int tail_valid = nc > 0 ? static_cast<int>(key_hi - (key_lo + static_cast<int64_t>(nc - 1) * kT8Keys)) : 0;
    float *o_base = p.o_out + static_cast<int64_t>(split) * p.o_split_stride;
    float *lse_base = p.lse_out + static_cast<int64_t>(split) * p.lse_split_stride;

    if (nc == 0) {  // empty split: sentinel rows
        for (int r = threadIdx.x; r < p.M; r += blockDim.x) {
            const int t = r / p.G, h = g * p.G + r % p.G;
            float4 *dst = reinterpret_cast<float4 *>(o_base + ((static_cast<int64_t>(b) * p.T + t) * p.H + h) * 128);
#pragma unroll
            for (int c = 0; c < 32; ++c) dst[c] = make_float4(0.f, 0.f, 0.f, 0.f);
            lse_base[(static_cast<int64_t>(b) * p.H + h) * p.T + t] = -INFINITY;
        }
    } else if (warp == kT8WarpTma) {
        // ================= TMA: lane 0 lands the E4M3 K tiles, lane 16 the V tiles (independent
        // rings: a K tile is never held back by a V slot that PV has not freed yet)
        if (lane == 0) {
            for (int j = 0; j < nc; ++j) {
                const int s = j % kT8Stages;
                mbar_wait(&kst_free[s], static_cast<uint32_t>(((j / kT8Stages) & 1) ^ 1));
                T8_TR(40, j);
                mbar_arrive_expect_tx(&kst_land[s], kT8StBytes);
                tma_load_4d(sKs + s * kT8StBytes, &tmap_k, &kst_land[s], 0, g, static_cast<int>(key_lo) + j * kT8Keys,
                            b, kT8KvPolicy);
                // the rings hold few tiles: stage the ones further ahead in L2 (HBM latency under
                // load is several times the tile period)
                if (j + kT8L2Ahead < nc)
                    tma_prefetch_l2_4d(&tmap_k, 0, g, static_cast<int>(key_lo) + (j + kT8L2Ahead) * kT8Keys, b);
            }
        } else if (lane == 16) {
            for (int j = 0; j < nc; ++j) {
                const int sv = j % kT8VSlots;
                mbar_wait(&v_free[sv], static_cast<uint32_t>(((j / kT8VSlots) & 1) ^ 1));
                T8_TR(41, j);
                mbar_arrive_expect_tx(&v_land[sv], kT8VBytes / 2);
                tma_load_4d(sV + sv * kT8VBytes + kT8VBytes / 2, &tmap_v, &v_land[sv], 0, g,
                            static_cast<int>(key_lo) + j * kT8Keys, b, kT8KvPolicy);
                if (j + kT8L2Ahead < nc)
                    tma_prefetch_l2_4d(&tmap_v, 0, g, static_cast<int>(key_lo) + (j + kT8L2Ahead) * kT8Keys, b);
            }
        }
        __syncwarp();
    } else if (warp >= kT8WarpKW && warp < kT8WarpKW + 4) {
        // ================= K widening: thread = key of lane quarter q; its 128-byte E4M3 row ->
        // 64 f16x2 words (column c = dims 2c, 2c+1) of the K buffer (A operand of S^T)
        const int q = warp & 3;
        const int key = 32 * q + lane;
        for (int j = 0; j < nc; ++j) {
            const int s = j % kT8Stages, kb = j & 1;
            mbar_wait(&kst_land[s], static_cast<uint32_t>((j / kT8Stages) & 1));
            T8_TR(42, j);
            if (j >= 2) mbar_wait(&k_free[kb], static_cast<uint32_t>(((j - 2) >> 1) & 1));
            T8_TR(43, j);
            tc_fence_after();
            const uint8_t *row = sKs + s * kT8StBytes + key * 128;
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                uint4 x[4];
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    x[c] = *reinterpret_cast<const uint4 *>(row + (((4 * hh + c) ^ (key & 7)) << 4));
                uint32_t w[32];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const uint32_t xs[4] = {x[c].x, x[c].y, x[c].z, x[c].w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        w[8 * c + 2 * e] = e4m3x2_to_f16x2(static_cast<uint16_t>(xs[e]));
                        w[8 * c + 2 * e + 1] = e4m3x2_to_f16x2(static_cast<uint16_t>(xs[e] >> 16));
                    }
                }
                t8_st32(tmem + (static_cast<uint32_t>(32 * q) << 16) + kT8KCol + kb * 64 + 32 * hh, w);
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&k_full[kb]);
                mbar_arrive(&kst_free[s]);
            }
            T8_TR(44, j);
        }
    } else if (warp >= kT8WarpVW && warp < kT8WarpVW + 4) {
        // ================= V widening: the E4M3 tile (128 keys x 128 B, unswizzled) sits in the
        // upper half of its f16 slot; warp `part` converts key rows [32 part, +32) in place into
        // the f16 SW128 layout [2 atoms][128 keys][128 B] (f16 row r's second atom is E4M3 row r:
        // rows are independent).  Rows past the end of the data (last tile) become zeros (Z13).
        const int part = warp - kT8WarpVW;
        for (int j = 0; j < nc; ++j) {
            const int sv = j % kT8VSlots;
            const int valid = j == nc - 1 ? tail_valid : kT8Keys;
            mbar_wait(&v_land[sv], static_cast<uint32_t>((j / kT8VSlots) & 1));
            T8_TR(45, j);
            uint8_t *slot = sV + sv * kT8VBytes;
            const uint8_t *src = slot + kT8VBytes / 2;
#pragma unroll
            for (int it0 = 0; it0 < 8; it0 += 4) {  // 32 rows x 8 chunks = 8 warp-iterations, 4 per batch
                uint4 x[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int idx = (8 * part + it0 + u) * 32 + lane;
                    x[u] = *reinterpret_cast<const uint4 *>(src + (idx >> 3) * 128 + (idx & 7) * 16);
                }
                __syncwarp();  // the batch's loads before any store over them
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int idx = (8 * part + it0 + u) * 32 + lane;
                    const int r = idx >> 3, c = idx & 7;  // E4M3 chunk c = dims 16c..16c+15
                    uint4 y0, y1;
                    y0.x = e4m3x2_to_f16x2(static_cast<uint16_t>(x[u].x));
                    y0.y = e4m3x2_to_f16x2(static_cast<uint16_t>(x[u].x >> 16));
                    y0.z = e4m3x2_to_f16x2(static_cast<uint16_t>(x[u].y));
                    y0.w = e4m3x2_to_f16x2(static_cast<uint16_t>(x[u].y >> 16));
                    y1.x = e4m3x2_to_f16x2(static_cast<uint16_t>(x[u].z));
                    y1.y = e4m3x2_to_f16x2(static_cast<uint16_t>(x[u].z >> 16));
                    y1.z = e4m3x2_to_f16x2(static_cast<uint16_t>(x[u].w));
                    y1.w = e4m3x2_to_f16x2(static_cast<uint16_t>(x[u].w >> 16));
                    if (r >= valid) y0 = y1 = make_uint4(0u, 0u, 0u, 0u);
                    const int ch = (c & 3) * 2;  // f16 chunk (8 dims) within the atom of dims 64*(c/4)..
                    uint8_t *row = slot + (c >> 2) * (kT8Keys * 128) + r * 128;
                    // the lanes of the second atom store their odd chunk first, so that each 8-lane
                    // phase of a 128-bit store hits 8 distinct bank groups
                    const bool sw = (c & 4) != 0;
                    *reinterpret_cast<uint4 *>(row + (((ch + (sw ? 1 : 0)) ^ (r & 7)) << 4)) = sw ? y1 : y0;
                    *reinterpret_cast<uint4 *>(row + (((ch + (sw ? 0 : 1)) ^ (r & 7)) << 4)) = sw ? y0 : y1;
                }
            }
            fence_proxy_async_smem();  // generic-proxy stores -> read by the tensor core
            __syncwarp();
            if (lane == 0) mbar_arrive(&v_full[sv]);
            T8_TR(47, j);
        }
    } else if (warp == kT8WarpMma) {
        // ================= MMA issuer (lane 0; the warp runs the loop converged).  Per tile j:
        // S^T_{j+3} (once the softmax has loaded S^T_j from its buffer), then PV_j.
        const uint32_t idesc_s = idesc_f16_f32(128, kT8Rows, 0);
        const uint32_t idesc_o = idesc_f16_f32(128, kT8Rows, 1) | (1u << 15);  // A (V^T) and B MN-major
        const uint64_t qd0 = sdesc_sw128(smem_u32(sQ), 16, 1024);
        const uint64_t pd0 = sdesc_sw128(smem_u32(sP), kT8PBytes, 1024);
        const uint64_t vd0 = sdesc_sw128(smem_u32(sV), kT8Keys * 128, 1024);  // atoms of 64 dims: 16 KB apart
        auto start_S = [&](int jj) {
            const int kb = jj & 1, sb = jj % 3;
            mbar_wait(&k_full[kb], static_cast<uint32_t>((jj >> 1) & 1));
            if (jj >= 3) mbar_wait(&s_free[sb], static_cast<uint32_t>((jj / 3 - 1) & 1));
            T8_TR(48, jj);
            tc_fence_after();
            if (lane == 0) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {  // 16 head-dim elements per step; Q atoms of 64 elements
                    const uint32_t qo = ((k / 4) * (kT8Rows * 128) + (k % 4) * 32) >> 4;
                    mma_bf16_ts(tmem + kT8SCol + sb * 64, tmem + kT8KCol + kb * 64 + k * 8, qd0 + qo, idesc_s,
                                k > 0 ? 1u : 0u);
                }
                tc_commit(&s_full[sb]);
                tc_commit(&k_free[kb]);
            }
            __syncwarp();
            T8_TR(55, jj);
        };
        mbar_wait(q_full, 0);
        for (int jj = 0; jj < 3 && jj < nc; ++jj) start_S(jj);
        for (int j = 0; j < nc; ++j) {
            if (j + 3 < nc) start_S(j + 3);
            const int vb = j & 1, sv = j % kT8VSlots;
            mbar_wait(&v_full[sv], static_cast<uint32_t>((j / kT8VSlots) & 1));
            mbar_wait(&p_full[vb], static_cast<uint32_t>((j >> 1) & 1));
            T8_TR(49, j);
            tc_fence_after();
            if (lane == 0) {
                const uint64_t pd = pd0 + static_cast<uint32_t>((vb * kT8PBytes) >> 4);
                const uint64_t vd = vd0 + static_cast<uint32_t>((sv * kT8VBytes) >> 4);
#pragma unroll
                for (int k = 0; k < 8; ++k)  // 16 keys per step: two 8-key groups = +2048 B (MN-major SW128)
                    mma_bf16_ss(tmem + kT8OCol, vd + static_cast<uint32_t>(k * 128), pd + static_cast<uint32_t>(k * 128),
                                idesc_o, (j > 0 || k > 0) ? 1u : 0u);
                tc_commit(&pv_done[vb]);
                tc_commit(&v_free[sv]);
            }
            __syncwarp();
            T8_TR(56, j);
        }
        if (lane == 0) tc_commit(o_final);
        __syncwarp();
    } else if (warp < kT8SWarps) {
        // ================= softmax: warp w holds key 32q + lane (q = w % 4) of every tile and the
        // kT8RW query rows [kT8RW*rq, +kT8RW) (rq = w / 4); the four warps of a row quarter share
        // their rows' maxima (named barrier 1 + rq).
        const int q = warp & 3, rq = warp >> 2;
        const int r0 = kT8RW * rq;
        const uint32_t bar_rq = 1u + static_cast<uint32_t>(rq);
        const int key = 32 * q + lane;
        // stage Q (bf16 -> f16, exact for |q| < 65504) into the K-major SW128 layout, rows >= M zero
        {
            const __nv_bfloat16 *qp = static_cast<const __nv_bfloat16 *>(p.q);
#pragma unroll
            for (int i = 0; i < 1024 / (32 * kT8SWarps); ++i) {
                const int idx = warp * 32 + lane + 32 * kT8SWarps * i;  // 64 rows x 16 chunks of 8 elements
                const int r = idx >> 4, ch = idx & 15;
                uint4 val = make_uint4(0u, 0u, 0u, 0u);
                if (r < p.M) {
                    const int t = r / p.G, hq = g * p.G + r % p.G;
                    val = __ldg(reinterpret_cast<const uint4 *>(qp + b * p.qs0 + t * p.qs1 + hq * p.qs2 + ch * 8));
                    uint32_t *wv = reinterpret_cast<uint32_t *>(&val);
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        wv[e] = pack_f16x2(__uint_as_float(wv[e] << 16), __uint_as_float(wv[e] & 0xFFFF0000u));
                }
                *reinterpret_cast<uint4 *>(sQ + (ch >> 3) * (kT8Rows * 128) + r * 128 + (((ch & 7) ^ (r & 7)) << 4)) =
                    val;
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(q_full);
        }
        const float c = p.scale_log2 * p.k_scale[g];  // K = k_scale[g] * E4M3
        const float *m_q = m_run + r0;
        const uint32_t lane_q = static_cast<uint32_t>(32 * q) << 16;
        float l[kT8RW];
#pragma unroll
        for (int i = 0; i < kT8RW; ++i) l[i] = 0.f;
        for (int j = 0; j < nc; ++j) {
            const int sb = j % 3, pb = j & 1;
            mbar_wait(&s_full[sb], static_cast<uint32_t>((j / 3) & 1));
            T8_TRS(0);
            tc_fence_after();
            float y[kT8RW];
            t8_ld16(tmem + lane_q + kT8SCol + sb * 64 + r0, y);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_free[sb]);
            // y = S * c (log2 units); keys past the split end -> -inf
            const bool kvalid = j < nc - 1 || key < tail_valid;
            bool ovf = false;
#pragma unroll
            for (int i4 = 0; i4 < kT8RW / 4; ++i4) {
                const float4 m4 = *reinterpret_cast<const float4 *>(m_q + 4 * i4);
                const float mm[4] = {m4.x, m4.y, m4.z, m4.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    float &v = y[4 * i4 + e];
                    v = kvalid ? v * c : -INFINITY;
                    ovf |= v > mm[e] + kT8Limit;
                }
            }
            T8_TRS(1);
            const bool any_ovf = bar_red_or(bar_rq, 128, ovf);
            T8_TRS(2);
            if (any_ovf) {
                // ---- rare: raise the running max of this quarter's rows to the tile's row maxima
                float t[kT8RW];
#pragma unroll
                for (int i = 0; i < kT8RW; ++i) t[i] = y[i];
                const float tmax = xreduce<true, kT8RW>(t, lane);  // row r0 + lane % kT8RW, this warp's keys
                if (lane < kT8RW) red[q * 64 + r0 + lane] = tmax;
                named_bar_sync(bar_rq, 128);
                if (q == 0 && lane < kT8RW) {
                    const float m_old = m_q[lane];
                    const float mx = fmaxf(fmaxf(red[r0 + lane], red[64 + r0 + lane]),
                                           fmaxf(red[128 + r0 + lane], red[192 + r0 + lane]));
                    const float m_new = fmaxf(m_old, mx);
                    fac[r0 + lane] = m_new == m_old ? 1.0f : exp2f(m_old - m_new);  // (m_old = -inf: 0)
                    m_run[r0 + lane] = m_new;
                }
                named_bar_sync(bar_rq, 128);
                bool any = false;
#pragma unroll
                for (int i = 0; i < kT8RW; ++i) {
                    const float f = fac[r0 + i];
                    l[i] *= f;
                    any |= f != 1.0f;
                }
                if (any && j > 0) {  // O^T columns of these rows: wait for PV_{j-1}, then rescale
                    mbar_wait(&pv_done[(j - 1) & 1], static_cast<uint32_t>(((j - 1) >> 1) & 1));
                    tc_fence_after();
                    float o[kT8RW];
                    const uint32_t oaddr = tmem + lane_q + kT8OCol + r0;
                    t8_ld16(oaddr, o);
#pragma unroll
                    for (int i = 0; i < kT8RW; ++i) o[i] *= fac[r0 + i];
                    t8_st16(oaddr, reinterpret_cast<const uint32_t *>(o));
                    tmem_st_wait();
                    tc_fence_before();
                }
            }
            // P^T_j = 2^(y - m) (f16) into buffer pb (free once PV_{j-2} is done); row sums
            if (j >= 2) mbar_wait(&pv_done[pb], static_cast<uint32_t>(((j - 2) >> 1) & 1));
            uint8_t *prow = sP + pb * kT8PBytes + key * 128;
#pragma unroll
            for (int c8 = 0; c8 < kT8RW / 8; ++c8) {  // rows r0 + 8*c8 .. +7: one 16-byte chunk
                const float4 ma = *reinterpret_cast<const float4 *>(m_q + 8 * c8);
                const float4 mb = *reinterpret_cast<const float4 *>(m_q + 8 * c8 + 4);
                const float mm[8] = {ma.x, ma.y, ma.z, ma.w, mb.x, mb.y, mb.z, mb.w};
                float pv[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    pv[e] = fast_exp2(y[8 * c8 + e] - mm[e]);  // (y = -inf: 0)
                    l[8 * c8 + e] += pv[e];
                }
                const uint4 wv = make_uint4(pack_f16x2(pv[0], pv[1]), pack_f16x2(pv[2], pv[3]), pack_f16x2(pv[4], pv[5]),
                                            pack_f16x2(pv[6], pv[7]));
                *reinterpret_cast<uint4 *>(prow + (((r0 / 8 + c8) ^ (key & 7)) << 4)) = wv;
            }
            fence_proxy_async_smem();  // generic-proxy stores -> read by the tensor core
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[pb]);
            T8_TRS(3);
            T8_TRFLUSH(j);
        }
        // ---- epilogue: row sums over the 128 keys (in-warp transposing sum, then the 4 warps of
        // the row quarter), O^T / l -> the split's partial (fp32, [B][T][H][d]), LSE (natural log)
        mbar_wait(o_final, 0);
        tc_fence_after();
        pdl_launch_dependents();
        const float lw = xreduce<false, kT8RW>(l, lane);  // row r0 + lane % kT8RW
        named_bar_sync(bar_rq, 128);  // (red is free: every overflow exchange has completed)
        if (lane < kT8RW) red[q * 64 + r0 + lane] = lw;
        named_bar_sync(bar_rq, 128);
        const int rl = r0 + lane % kT8RW;
        const float lsum = red[rl] + red[64 + rl] + red[128 + rl] + red[192 + rl];
        const float vs = p.v_scale[g];  // V = v_scale[g] * E4M3
        const float inv_lane = lsum > 0.f ? vs / lsum : 0.f;
        float o[kT8RW];
        t8_ld16(tmem + lane_q + kT8OCol + r0, o);
#pragma unroll
        for (int i = 0; i < kT8RW; ++i) {
            const int r = r0 + i;
            const float inv = __shfl_sync(0xffffffffu, inv_lane, i);
            if (r < p.M) {
                const int t = r / p.G, hq = g * p.G + r % p.G;
                o_base[((static_cast<int64_t>(b) * p.T + t) * p.H + hq) * 128 + key] = o[i] * inv;
            }
        }
        if (q == 0 && lane < kT8RW && rl < p.M) {
            const int t = rl / p.G, hq = g * p.G + rl % p.G;
            lse_base[(static_cast<int64_t>(b) * p.H + hq) * p.T + t] =
                lsum > 0.f ? (m_run[rl] + log2f(lsum)) * 0.69314718055994530942f : -INFINITY;
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == kT8WarpMma) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

}  // namespace

int prefix_t8_smem_bytes() { return kT8SmemBytes; }

cudaError_t launch_prefix_t8(const PrefixParams &p, const CUtensorMap &tk, const CUtensorMap &tv, cudaStream_t s) {
    if (!p.kv8 || p.d != 128 || p.M > kT8Rows || p.n_mgroups != 1 || p.tree_tiles != 0) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(prefix_t8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kT8SmemBytes);
    if (e != cudaSuccess) {
        fprintf(stderr, "hta: prefix_t8 shared-memory attribute (%d B): %s\n", kT8SmemBytes, cudaGetErrorString(e));
        return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.splits * p.H_kv * p.B);
    cfg.blockDim = dim3(kT8Threads);
    cfg.dynamicSmemBytes = kT8SmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, prefix_t8_kernel, tk, tv, p);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) fprintf(stderr, "hta: prefix_t8 launch failed: %s\n", cudaGetErrorString(e));
    return e;
}

}  // namespace hta

#endif  // HTA_T8
