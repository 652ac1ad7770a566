// hta_api.cu -- host side of the C ABI declared in include/hta.h: argument validation,
// work planning (split-KV schedule), TMA descriptor encoding and kernel launches.
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstring>
#include <cstdlib>
#include <mutex>

#include "hta_internal.h"

using namespace hta;

namespace {

constexpr int kDefaultSms = 148;

bool is_aligned(const void *p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

// Normalised copy of a shape with default strides filled in.
struct Shape {
    hta_shape_t s;
    int G;
    int64_t esize;
};

hta_status_t check_shape(const hta_shape_t *in, Shape *out) {
    if (in == nullptr) return HTA_ERR_INVALID_ARGUMENT;
    hta_shape_t s = *in;
    if (s.B < 1 || s.T < 1 || s.T > 256 || s.H < 1 || s.H_kv < 1 || s.H % s.H_kv != 0) return HTA_ERR_INVALID_ARGUMENT;
    if (s.N_max < 0 || s.N_max > (int64_t(1) << 31) - 1024) return HTA_ERR_INVALID_ARGUMENT;
    if (!(s.softmax_scale > 0.f) || !std::isfinite(s.softmax_scale)) return HTA_ERR_INVALID_ARGUMENT;
    if (s.dtype != HTA_BF16 && s.dtype != HTA_FP32) return HTA_ERR_INVALID_ARGUMENT;
    if (s.num_splits < 0 || s.max_seqlen < 0) return HTA_ERR_INVALID_ARGUMENT;
    if (s.d != 64 && s.d != 128) return HTA_ERR_UNSUPPORTED;
    const int64_t d = s.d;
    auto fill = [](int64_t *st, int64_t a, int64_t b, int64_t c) {
        if (st[0] == 0 && st[1] == 0 && st[2] == 0) {
            st[0] = a;
            st[1] = b;
            st[2] = c;
        }
    };
    fill(s.q_strides, int64_t(s.T) * s.H * d, int64_t(s.H) * d, d);
    fill(s.kv_strides, std::max<int64_t>(s.N_max, 1) * s.H_kv * d, int64_t(s.H_kv) * d, d);
    fill(s.tkv_strides, int64_t(s.T) * s.H_kv * d, int64_t(s.H_kv) * d, d);
    const int64_t esize = s.dtype == HTA_BF16 ? 2 : 4;
    const int64_t vec = 16 / esize;  // every row must start 16-byte aligned
    for (int i = 0; i < 3; ++i) {
        if (s.q_strides[i] <= 0 || s.kv_strides[i] <= 0 || s.tkv_strides[i] <= 0) return HTA_ERR_INVALID_ARGUMENT;
        if (s.q_strides[i] % vec || s.kv_strides[i] % vec || s.tkv_strides[i] % vec) return HTA_ERR_INVALID_ARGUMENT;
    }
    out->s = s;
    out->G = s.H / s.H_kv;
    out->esize = esize;
    return HTA_OK;
}

hta_status_t check_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return HTA_ERR_UNSUPPORTED;
    static std::atomic<int> cached_major[64];
    static std::atomic<int> cached_sms[64];
    if (dev < 0 || dev >= 64) return HTA_ERR_UNSUPPORTED;
    int major = cached_major[dev].load();
    if (major == 0) {
        int sms = 0;
        if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess)
            return HTA_ERR_UNSUPPORTED;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cached_sms[dev].store(sms);
        cached_major[dev].store(major);
    }
    return major == 10 ? HTA_OK : HTA_ERR_UNSUPPORTED;
}

int device_sms() {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return kDefaultSms;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
        return kDefaultSms;
    return sms;
}

// Makespan model of the split-KV schedule: waves(S) x (tiles per split + a fixed per-CTA cost of
// ~3 tiles for prologue and epilogue), with a 1%-per-split penalty for the partials each split
// adds (wave quantisation over the SMs, 1 CTA per SM).  Measured on B200: LongChat-16k is faster
// as one wave of 4 splits than as two waves of 9 (tools/split_sweep.py).  Returns the best S.
int best_splits(int ctas, int n_tiles, int num_sms, double *cost_out) {
    const int smax = std::max(1, std::min(n_tiles, 4 * num_sms / ctas + 1));
    double best = 1e30;
    int S = 1;
    for (int c = 1; c <= smax; ++c) {
        const int waves = (ctas * c + num_sms - 1) / num_sms;
        const int per = (n_tiles + c - 1) / c;
        const double cost = double(waves) * (per + 3) * (1.0 + 0.01 * c);
        if (cost < best - 1e-12) {
            best = cost;
            S = c;
        }
    }
    *cost_out = best;
    return S;
}

// Split-KV work plan.  tree_tiles: masked tree tiles the
// last split of every unit appends (fused tree pass of hta_forward); they are planned as tiles of
// the key range like the cache tiles, so the last split carries correspondingly fewer cache tiles.
PrefixPlan make_plan(const Shape &sh, int num_sms, int tree_tiles = 0) {
    const hta_shape_t &s = sh.s;
    PrefixPlan pl{};
    pl.G = sh.G;
    pl.M = s.T * sh.G;
    const int blk = s.dtype == HTA_BF16 ? kBlockN : kSimtBlock;
    // the filled length bound (max_seqlen) plans the schedule; the last split still runs to each
    // batch entry's own length
    const int64_t n_plan = (s.max_seqlen > 0 && s.max_seqlen < s.N_max) ? s.max_seqlen : s.N_max;
    pl.n_tiles = static_cast<int>((n_plan + blk - 1) / blk) + (s.dtype == HTA_BF16 ? tree_tiles : 0);
    int S = 1;
    if (s.dtype == HTA_BF16) {
        // More than 128 rows per KV head: CTA pairs (cta_group::2, 256 rows per pair), unless
        // single-CTA 128-row groups pack the rows tighter into a shorter schedule (G = 5, T = 64:
        // 320 rows = 2.5 x 128 fill 3 single groups at 83 % but 2 pair groups at 63 %).
        auto layout = [&](int nt, int *S_out) {
            const int mg = (pl.M + 128 * nt - 1) / (128 * nt);
#ifdef HTA_Q2
            const int ctas = s.B * s.H_kv * mg;  // experiment: one CTA holds both 128-row tiles
#else
            const int ctas = s.B * s.H_kv * mg * nt;  // CTAs per split (a pair is two CTAs, two SMs)
#endif
            double cost = 0.0;
            *S_out = s.num_splits > 0 ? s.num_splits : best_splits(ctas, std::max(pl.n_tiles, 1), num_sms, &cost);
            return cost;
        };
        int S1 = 1, S2 = 1;
        const double c1 = layout(1, &S1);
        pl.nt = 1;
        S = S1;
        if (pl.M > 128 && s.d == 128) {
            const double c2 = layout(2, &S2);
            if (s.num_splits > 0 || c2 <= c1) {
                pl.nt = 2;
                S = S2;
            }
        }
        pl.n_mgroups = (pl.M + 128 * pl.nt - 1) / (128 * pl.nt);
        pl.units = s.B * s.H_kv * pl.n_mgroups;
    } else {
        pl.nt = 1;
        pl.n_mgroups = 1;
        pl.units = (s.B * s.T * s.H + 3) / 4;  // SIMT: 4 rows per block
        S = s.num_splits > 0 ? s.num_splits : (4 * num_sms + pl.units - 1) / pl.units;
    }
    if (S < 1) S = 1;
    if (pl.n_tiles > 0 && S > pl.n_tiles) S = pl.n_tiles;
    if (pl.n_tiles == 0) S = 1;
    pl.tiles_per_split = pl.n_tiles > 0 ? (pl.n_tiles + S - 1) / S : 1;
    pl.splits = pl.n_tiles > 0 ? (pl.n_tiles + pl.tiles_per_split - 1) / pl.tiles_per_split : 1;
    return pl;
}

size_t part_floats(const hta_shape_t &s) {
    return size_t(s.B) * s.T * s.H * s.d + size_t(s.B) * s.H * s.T;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(ptr);
    });
    return fn;
}

// 4-D map over a [B, N, H_kv, d] (strided) bf16 cache: box = 64 x 1 x box_rows x 1, 128B swizzle.
hta_status_t make_kv_map(CUtensorMap *map, const void *base, const hta_shape_t &s, int box_rows) {
    EncodeTiledFn enc = encode_fn();
    if (enc == nullptr) return HTA_ERR_CUDA;
    cuuint64_t dims[4] = {cuuint64_t(s.d), cuuint64_t(s.H_kv), cuuint64_t(std::max<int64_t>(s.N_max, 1)),
                          cuuint64_t(s.B)};
    cuuint64_t strides[3] = {cuuint64_t(s.kv_strides[2] * 2), cuuint64_t(s.kv_strides[1] * 2),
                             cuuint64_t(s.kv_strides[0] * 2)};
    cuuint32_t box[4] = {64, 1, cuuint32_t(box_rows), 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? HTA_OK : HTA_ERR_INVALID_ARGUMENT;
}

// Q [B, T, H, d] viewed as 4-D (d, H, T, B): a box (64, G, 128/G, 1) at (kb*64, g*G, t0, b) is
// exactly 128 rows r = (t - t0)*G + (h - g*G) of a row tile, 128 B each, in the K-major
// SWIZZLE_128B layout the MMA reads; rows past M (t >= T) are zero-filled.  Needs G | 128 and
// 16-byte row strides; otherwise the kernel stages Q with plain loads.
bool make_q_map(CUtensorMap *map, const void *q, const hta_shape_t &s, int G) {
    if (128 % G != 0) return false;
    for (int i = 0; i < 3; ++i)
        if ((s.q_strides[i] * 2) % 16 != 0) return false;
    EncodeTiledFn enc = encode_fn();
    if (enc == nullptr) return false;
    cuuint64_t dims[4] = {cuuint64_t(s.d), cuuint64_t(s.H), cuuint64_t(s.T), cuuint64_t(s.B)};
    cuuint64_t strides[3] = {cuuint64_t(s.q_strides[2] * 2), cuuint64_t(s.q_strides[1] * 2),
                             cuuint64_t(s.q_strides[0] * 2)};
    cuuint32_t box[4] = {64, cuuint32_t(G), cuuint32_t(128 / G), 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(q), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Tree tiles of the fused tree pass (hta_forward, bf16, T <= 256): ceil(T / 128).
int fused_tree_tiles(const hta_shape_t &s) {
    return s.dtype == HTA_BF16 && s.T >= 1 && s.T <= 256 ? (s.T + kBlockN - 1) / kBlockN : 0;
}

// 4-D map over k_tree / v_tree [B, T, H_kv, d] (tkv_strides): box = 64 x 1 x box_rows x 1, 128B
// swizzle, rows past T zero-filled.  false when the strides are not 16-byte multiples (the tree
// pass then runs in the tree/merge kernel).
bool make_tree_map(CUtensorMap *map, const void *base, const hta_shape_t &s, int box_rows) {
    for (int i = 0; i < 3; ++i)
        if ((s.tkv_strides[i] * 2) % 16 != 0) return false;
    EncodeTiledFn enc = encode_fn();
    if (enc == nullptr) return false;
    cuuint64_t dims[4] = {cuuint64_t(s.d), cuuint64_t(s.H_kv), cuuint64_t(s.T), cuuint64_t(s.B)};
    cuuint64_t strides[3] = {cuuint64_t(s.tkv_strides[2] * 2), cuuint64_t(s.tkv_strides[1] * 2),
                             cuuint64_t(s.tkv_strides[0] * 2)};
    cuuint32_t box[4] = {64, 1, cuuint32_t(box_rows), 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Paged KV cache: a contiguous pool [num_pages, page_size, H_kv, d] and a
// block table [B][max_pages] of page indices.
struct PagedArgs {
    const int32_t *block_table;
    int32_t max_pages;
    int32_t page_size;
    int32_t num_pages;
};

// 4-D map over the page pool seen as [1, num_pages * page_size, H_kv, d]: 16-row boxes.
hta_status_t make_pool_map(CUtensorMap *map, const void *base, const hta_shape_t &s, const PagedArgs &pg) {
    EncodeTiledFn enc = encode_fn();
    if (enc == nullptr) return HTA_ERR_CUDA;
    const cuuint64_t rows = cuuint64_t(pg.num_pages) * cuuint64_t(pg.page_size);
    cuuint64_t dims[4] = {cuuint64_t(s.d), cuuint64_t(s.H_kv), rows, 1};
    const cuuint64_t row_bytes = cuuint64_t(s.H_kv) * s.d * 2;
    cuuint64_t strides[3] = {cuuint64_t(s.d) * 2, row_bytes, rows * row_bytes};
    cuuint32_t box[4] = {64, 1, 16, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? HTA_OK : HTA_ERR_INVALID_ARGUMENT;
}

// FP8 (E4M3) cache [B, N, H_kv, d] as bytes: box = box_cols x 1 x box_rows x 1, no swizzle (the
// kernel widens the landed tile into the 128B-swizzled f16 layout itself).
hta_status_t make_kv_map_fp8(CUtensorMap *map, const void *base, const hta_shape_t &s, int box_cols, int box_rows,
                             bool swizzle = false) {
    EncodeTiledFn enc = encode_fn();
    if (enc == nullptr) return HTA_ERR_CUDA;
    cuuint64_t dims[4] = {cuuint64_t(s.d), cuuint64_t(s.H_kv), cuuint64_t(std::max<int64_t>(s.N_max, 1)),
                          cuuint64_t(s.B)};
    cuuint64_t strides[3] = {cuuint64_t(s.kv_strides[2]), cuuint64_t(s.kv_strides[1]), cuuint64_t(s.kv_strides[0])};
    cuuint32_t box[4] = {cuuint32_t(box_cols), 1, cuuint32_t(box_rows), 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void *>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? HTA_OK : HTA_ERR_INVALID_ARGUMENT;
}

// FP8 cache arguments of the prefix pass (nullptr: the cache has the shape's dtype).
struct Fp8Args {
    const float *k_scale, *v_scale;
};

// Fused tree pass arguments of the prefix pass (tree_tiles = 0: none).
struct TreeArgs {
    int tree_tiles;
    const uint8_t *mask;
    int64_t mask_bs;
    const int32_t *parents;  // (mask == nullptr) visibility from the parent array
    int64_t par_bs;
    CUtensorMap tkt, tvt;
};

// Enqueue the prefix pass writing `splits` partials at (o_out, lse_out) with the given strides.
// FP8 cache: the transposed kernel (build option HTA_T8) takes single-CTA units of at most 64
// rows at d = 128
bool t8_eligible(const hta_shape_t &s, const PrefixPlan &pl) {
    return HTA_T8 && s.d == 128 && pl.nt == 1 && pl.n_mgroups == 1 && pl.M <= 64 && kBlockN == 128;
}

hta_status_t run_prefix(const Shape &sh, const PrefixPlan &pl, const void *q, const void *k, const void *v,
                        const int32_t *seqlens, float *o_out, float *lse_out, int64_t o_split_stride,
                        int64_t lse_split_stride, cudaStream_t st, const PagedArgs *pg = nullptr,
                        const Fp8Args *f8 = nullptr, const TreeArgs *tr = nullptr) {
    const hta_shape_t &s = sh.s;
    PrefixParams p{};
    if (f8 != nullptr) {
        p.kv8 = 1;
        p.k_scale = f8->k_scale;
        p.v_scale = f8->v_scale;
    }
    if (pg != nullptr) {
        p.block_table = pg->block_table;
        p.bt_stride = pg->max_pages;
        p.page_size = pg->page_size;
        p.max_pages = pg->max_pages;
    }
    p.q = q;
    p.qs0 = s.q_strides[0];
    p.qs1 = s.q_strides[1];
    p.qs2 = s.q_strides[2];
    p.k = k;
    p.v = v;
    p.ks0 = s.kv_strides[0];
    p.ks1 = s.kv_strides[1];
    p.ks2 = s.kv_strides[2];
    p.seqlens = seqlens;
    p.B = s.B;
    p.T = s.T;
    p.H = s.H;
    p.H_kv = s.H_kv;
    p.d = s.d;
    p.G = sh.G;
    p.M = pl.M;
    p.N_max = s.N_max;
    p.scale = s.softmax_scale;
    p.scale_log2 = s.softmax_scale * 1.4426950408889634f;
    p.nt = pl.nt;
    p.n_mgroups = pl.n_mgroups;
    p.splits = pl.splits;
    p.tiles_per_split = pl.tiles_per_split;
    p.o_out = o_out;
    p.lse_out = lse_out;
    p.o_split_stride = o_split_stride;
    p.lse_split_stride = lse_split_stride;
    cudaError_t e;
    if (s.dtype == HTA_BF16) {
        CUtensorMap tk, tv;
        hta_status_t r;
        if (f8 != nullptr && t8_eligible(s, pl)) {
            // units of at most 64 rows: the transposed kernel (K tiles 128-byte swizzled)
            if ((r = make_kv_map_fp8(&tk, k, s, 128, kBlockN, true)) != HTA_OK) return r;
            if ((r = make_kv_map_fp8(&tv, v, s, 128, kBlockN, false)) != HTA_OK) return r;  // (widened in place)
#if HTA_T8
            return launch_prefix_t8(p, tk, tv, st) == cudaSuccess ? HTA_OK : HTA_ERR_CUDA;
#endif
        }
        if (f8 != nullptr) {
            // a CTA of a pair loads half of each K tile (64 keys, all d) and half of each V tile
            // (64 columns, all 128 keys) -- the same halves as the bf16 cache
            // (d = 128, single CTAs: the E4M3 K tile is the MMA operand itself, landed 128-byte swizzled)
            if ((r = make_kv_map_fp8(&tk, k, s, s.d, pl.nt == 2 ? kBlockN / 2 : kBlockN,
                                     s.d == 128 && pl.nt == 1 && HTA_F8S)) !=
                HTA_OK)
                return r;
            // (d = 128, single CTAs of more than 64 rows, HTA_F8P: V is the MMA operand as landed,
            // 128-byte swizzled -- prefix_tc.cu launches the KV8 = 2 kernel for exactly these)
            if ((r = make_kv_map_fp8(&tv, v, s, pl.nt == 2 ? 64 : s.d, kBlockN,
                                     s.d == 128 && pl.nt == 1 && pl.M > 64 && HTA_F8S && HTA_F8P)) != HTA_OK)
                return r;
        } else if (pg != nullptr) {
            if ((r = make_pool_map(&tk, k, s, *pg)) != HTA_OK) return r;
            if ((r = make_pool_map(&tv, v, s, *pg)) != HTA_OK) return r;
        } else {
            // a CTA of a pair loads half of each K tile (64 keys) and half of each V tile (64 columns)
            if ((r = make_kv_map(&tk, k, s, pl.nt == 2 ? kBlockN / 2 : kBlockN)) != HTA_OK) return r;
            if ((r = make_kv_map(&tv, v, s, kBlockN)) != HTA_OK) return r;
        }
        CUtensorMap tq;
        std::memset(&tq, 0, sizeof(tq));
        // the FP8 variant stages Q with plain loads (converting it to f16 on the way)
        p.q_tma = f8 == nullptr && make_q_map(&tq, q, s, sh.G) ? 1 : 0;
        CUtensorMap none;
        std::memset(&none, 0, sizeof(none));
        if (tr != nullptr && tr->tree_tiles > 0) {
            p.tree_tiles = tr->tree_tiles;
            p.mask = tr->mask;
            p.mask_bs = tr->mask_bs;
            p.parents = tr->parents;
            p.par_bs = tr->par_bs;
        }
        const bool fused = p.tree_tiles > 0;
        e = launch_prefix_tc(p, tq, tk, tv, fused ? tr->tkt : none, fused ? tr->tvt : none,
                             prefix_tc_smem_bytes(s.d, pl.nt), st);
    } else {
        e = launch_prefix_simt(p, st);
    }
    return e == cudaSuccess ? HTA_OK : HTA_ERR_CUDA;
}

TreeMergeParams base_tm(const Shape &sh) {
    const hta_shape_t &s = sh.s;
    TreeMergeParams p{};
    p.B = s.B;
    p.T = s.T;
    p.H = s.H;
    p.H_kv = s.H_kv;
    p.G = sh.G;
    p.Hr = s.H;
    p.h0 = 0;
    p.qs0 = s.q_strides[0];
    p.qs1 = s.q_strides[1];
    p.qs2 = s.q_strides[2];
    p.ts0 = s.tkv_strides[0];
    p.ts1 = s.tkv_strides[1];
    p.ts2 = s.tkv_strides[2];
    p.scale = s.softmax_scale;
    p.out_hb = s.H;
    return p;
}

void set_out_contig_f32(TreeMergeParams &p, const hta_shape_t &s, float *o, float *lse) {
    p.o = o;
    p.os0 = int64_t(s.T) * s.H * s.d;
    p.os1 = int64_t(s.H) * s.d;
    p.os2 = s.d;
    p.lse = lse;
}

}  // namespace

// =============================================================================== ABI

extern "C" {

const char *hta_status_string(hta_status_t st) {
    switch (st) {
        case HTA_OK: return "HTA_OK";
        case HTA_ERR_INVALID_ARGUMENT: return "HTA_ERR_INVALID_ARGUMENT";
        case HTA_ERR_UNSUPPORTED: return "HTA_ERR_UNSUPPORTED";
        case HTA_ERR_INVALID_MASK: return "HTA_ERR_INVALID_MASK";
        case HTA_ERR_WORKSPACE: return "HTA_ERR_WORKSPACE";
        case HTA_ERR_CUDA: return "HTA_ERR_CUDA";
        case HTA_ERR_NCCL: return "HTA_ERR_NCCL";
    }
    return "HTA_ERR_UNKNOWN";
}

int32_t hta_version(void) { return 100; }

size_t hta_workspace_size(const hta_shape_t *shape, int32_t num_sms) {
    Shape sh;
    if (check_shape(shape, &sh) != HTA_OK) return size_t(-1);
    const int sms = num_sms > 0 ? num_sms : kDefaultSms;
    // the larger of the plans with and without the fused tree tiles (hta_forward uses the latter)
    const int splits = std::max(make_plan(sh, sms).splits, make_plan(sh, sms, fused_tree_tiles(sh.s)).splits);
    return size_t(splits) * part_floats(sh.s) * sizeof(float);
}

hta_status_t hta_prefix_attn(const hta_shape_t *shape, const void *q, const void *k_cache, const void *v_cache,
                             const int32_t *cache_seqlens, float *o_part, float *lse_part, void *ws, size_t ws_bytes,
                             hta_stream_t stream) {
    Shape sh;
    hta_status_t r = check_shape(shape, &sh);
    if (r != HTA_OK) return r;
    if (!q || !k_cache || !v_cache || !o_part || !lse_part) return HTA_ERR_INVALID_ARGUMENT;
    if (!is_aligned(q, 16) || !is_aligned(k_cache, 16) || !is_aligned(v_cache, 16) || !is_aligned(o_part, 16))
        return HTA_ERR_INVALID_ARGUMENT;
    if ((r = check_device()) != HTA_OK) return r;
    const hta_shape_t &s = sh.s;
    const PrefixPlan pl = make_plan(sh, device_sms());
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (pl.splits == 1)
        return run_prefix(sh, pl, q, k_cache, v_cache, cache_seqlens, o_part, lse_part, 0, 0, st);
    const size_t need = size_t(pl.splits) * part_floats(s) * sizeof(float);
    if (ws == nullptr || ws_bytes < need || !is_aligned(ws, 16)) return HTA_ERR_WORKSPACE;
    float *o_ws = static_cast<float *>(ws);
    const int64_t ostride = int64_t(s.B) * s.T * s.H * s.d;
    float *lse_ws = o_ws + size_t(pl.splits) * ostride;
    const int64_t lstride = int64_t(s.B) * s.H * s.T;
    r = run_prefix(sh, pl, q, k_cache, v_cache, cache_seqlens, o_ws, lse_ws, ostride, lstride, st);
    if (r != HTA_OK) return r;
    TreeMergeParams p = base_tm(sh);
    p.do_tree = 0;
    p.n_parts = pl.splits;
    p.o_parts = o_ws;
    p.lse_parts = lse_ws;
    p.o_part_stride = ostride;
    p.lse_part_stride = lstride;
    set_out_contig_f32(p, s, o_part, lse_part);
    return launch_tree_merge(p, s.d, s.dtype, HTA_FP32, true, st) == cudaSuccess ? HTA_OK : HTA_ERR_CUDA;
}

hta_status_t hta_tree_attn(const hta_shape_t *shape, const void *q, const void *k_tree, const void *v_tree,
                           const uint8_t *mask, int64_t mask_batch_stride, float *o_part, float *lse_part,
                           hta_stream_t stream) {
    Shape sh;
    hta_status_t r = check_shape(shape, &sh);
    if (r != HTA_OK) return r;
    const hta_shape_t &s = sh.s;
    if (!q || !k_tree || !v_tree || !mask || !o_part || !lse_part) return HTA_ERR_INVALID_ARGUMENT;
    if (mask_batch_stride != 0 && mask_batch_stride < int64_t(s.T) * s.T) return HTA_ERR_INVALID_ARGUMENT;
    if (!is_aligned(q, 16) || !is_aligned(k_tree, 16) || !is_aligned(v_tree, 16) || !is_aligned(o_part, 16))
        return HTA_ERR_INVALID_ARGUMENT;
    if ((r = check_device()) != HTA_OK) return r;
    TreeMergeParams p = base_tm(sh);
    p.q = q;
    p.kt = k_tree;
    p.vt = v_tree;
    p.mask = mask;
    p.mask_bs = mask_batch_stride;
    p.do_tree = 1;
    p.n_parts = 0;
    set_out_contig_f32(p, s, o_part, lse_part);
    return launch_tree_merge(p, s.d, s.dtype, HTA_FP32, false, reinterpret_cast<cudaStream_t>(stream)) == cudaSuccess
               ? HTA_OK
               : HTA_ERR_CUDA;
}

hta_status_t hta_merge_lse(const hta_shape_t *shape, int32_t n_parts, const float *o_parts, const float *lse_parts,
                           void *o, float *lse_out, hta_stream_t stream) {
    Shape sh;
    hta_status_t r = check_shape(shape, &sh);
    if (r != HTA_OK) return r;
    const hta_shape_t &s = sh.s;
    if (n_parts < 1 || !o_parts || !lse_parts || !o) return HTA_ERR_INVALID_ARGUMENT;
    if (!is_aligned(o_parts, 16) || !is_aligned(o, 16)) return HTA_ERR_INVALID_ARGUMENT;
    if ((r = check_device()) != HTA_OK) return r;
    TreeMergeParams p = base_tm(sh);
    p.do_tree = 0;
    p.n_parts = n_parts;
    p.o_parts = o_parts;
    p.lse_parts = lse_parts;
    p.o_part_stride = int64_t(s.B) * s.T * s.H * s.d;
    p.lse_part_stride = int64_t(s.B) * s.H * s.T;
    p.o = o;
    p.os0 = s.q_strides[0];
    p.os1 = s.q_strides[1];
    p.os2 = s.q_strides[2];
    p.lse = lse_out;
    return launch_tree_merge(p, s.d, s.dtype, s.dtype, false, reinterpret_cast<cudaStream_t>(stream)) == cudaSuccess
               ? HTA_OK
               : HTA_ERR_CUDA;
}

static hta_status_t forward_impl(const PagedArgs *pg, const hta_shape_t *shape, const void *q, const void *k_cache, const void *v_cache,
                               const int32_t *cache_seqlens, const void *k_tree, const void *v_tree,
                               const uint8_t *mask, int64_t mask_batch_stride, void *o, float *lse_out, void *ws,
                               size_t ws_bytes, hta_stream_t stream, void *ev_begin, void *ev_end,
                               const Fp8Args *f8 = nullptr, void *tree_ready = nullptr,
                               const int32_t *parents = nullptr, int64_t parents_bs = 0) {
    Shape sh;
    hta_status_t r = check_shape(shape, &sh);
    if (r != HTA_OK) return r;
    const hta_shape_t &s = sh.s;
    // the tree's visibility: the mask, or (hta_forward_tree) the parent array
    if (!q || !k_cache || !v_cache || !k_tree || !v_tree || (!mask && !parents) || !o) return HTA_ERR_INVALID_ARGUMENT;
    if (mask != nullptr && mask_batch_stride != 0 && mask_batch_stride < int64_t(s.T) * s.T)
        return HTA_ERR_INVALID_ARGUMENT;
    if (mask == nullptr && parents_bs != 0 && parents_bs < s.T) return HTA_ERR_INVALID_ARGUMENT;
    if (!is_aligned(q, 16) || !is_aligned(k_cache, 16) || !is_aligned(v_cache, 16) || !is_aligned(k_tree, 16) ||
        !is_aligned(v_tree, 16) || !is_aligned(o, 16))
        return HTA_ERR_INVALID_ARGUMENT;
    if ((r = check_device()) != HTA_OK) return r;
    // The tree pass runs inside the prefix kernel (masked tree tiles appended to the last split of
    // every unit) for single-CTA row groups; it stays in the tree/merge kernel
    // beside the merge for CTA pairs (there the tree tile costs the pair kernel more than the
    // separate tree pass costs the tail: Llama-8B-64k 71.1 vs 69.6 us, 128k 225.8 vs 219 us;
    // HTA_FUSE_PAIRS builds it),
    // for an FP8 cache, when the tree inputs arrive late on another stream (tree_ready), and when
    // k_tree / v_tree cannot be described by a tensor map.
    TreeArgs tr{};
    PrefixPlan pl = make_plan(sh, device_sms());
    if (f8 == nullptr && tree_ready == nullptr && fused_tree_tiles(s) > 0) {
        const PrefixPlan plt = make_plan(sh, device_sms(), fused_tree_tiles(s));
        // (a CTA of a pair loads its 64-key half of a tree K tile and a 64-column half of V)
        if ((plt.nt == 1 || HTA_FUSE_PAIRS) && make_tree_map(&tr.tkt, k_tree, s, plt.nt == 2 ? kBlockN / 2 : kBlockN) &&
            make_tree_map(&tr.tvt, v_tree, s, kBlockN)) {
            tr.tree_tiles = fused_tree_tiles(s);
            tr.mask = mask;
            tr.mask_bs = mask_batch_stride;
            tr.parents = mask == nullptr ? parents : nullptr;
            tr.par_bs = parents_bs;
            pl = plt;
        }
    }
    const size_t need = size_t(pl.splits) * part_floats(s) * sizeof(float);
    if (ws == nullptr || ws_bytes < need || !is_aligned(ws, 16)) return HTA_ERR_WORKSPACE;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    float *o_ws = static_cast<float *>(ws);
    const int64_t ostride = int64_t(s.B) * s.T * s.H * s.d;
    float *lse_ws = o_ws + size_t(pl.splits) * ostride;
    const int64_t lstride = int64_t(s.B) * s.H * s.T;
    if (ev_begin != nullptr && cudaEventRecord(static_cast<cudaEvent_t>(ev_begin), st) != cudaSuccess)
        return HTA_ERR_CUDA;
    r = run_prefix(sh, pl, q, k_cache, v_cache, cache_seqlens, o_ws, lse_ws, ostride, lstride, st, pg, f8, &tr);
    if (r != HTA_OK) return r;
    if (ev_end != nullptr && cudaEventRecord(static_cast<cudaEvent_t>(ev_end), st) != cudaSuccess)
        return HTA_ERR_CUDA;
    // the tree inputs (k_tree, v_tree, mask) may still be in flight on another stream: only the
    // tree/merge kernel waits for them, the prefix kernel above does not
    if (tree_ready != nullptr && cudaStreamWaitEvent(st, static_cast<cudaEvent_t>(tree_ready), 0) != cudaSuccess)
        return HTA_ERR_CUDA;
    TreeMergeParams p = base_tm(sh);
    p.q = q;
    p.kt = k_tree;
    p.vt = v_tree;
    p.mask = mask;
    p.mask_bs = mask_batch_stride;
    p.parents = mask == nullptr ? parents : nullptr;
    p.par_bs = parents_bs;
    p.do_tree = tr.tree_tiles > 0 ? 0 : 1;  // (fused: the partials already hold the tree part)
    p.n_parts = pl.splits;
    p.o_parts = o_ws;
    p.lse_parts = lse_ws;
    p.o_part_stride = ostride;
    p.lse_part_stride = lstride;
    p.o = o;
    p.os0 = s.q_strides[0];
    p.os1 = s.q_strides[1];
    p.os2 = s.q_strides[2];
    p.lse = lse_out;
    return launch_tree_merge(p, s.d, s.dtype, s.dtype, ev_end == nullptr, st) == cudaSuccess ? HTA_OK
                                                                                              : HTA_ERR_CUDA;
}

hta_status_t hta_forward_timed(const hta_shape_t *shape, const void *q, const void *k_cache, const void *v_cache,
                               const int32_t *cache_seqlens, const void *k_tree, const void *v_tree,
                               const uint8_t *mask, int64_t mask_batch_stride, void *o, float *lse_out, void *ws,
                               size_t ws_bytes, hta_stream_t stream, void *ev_begin, void *ev_end) {
    return forward_impl(nullptr, shape, q, k_cache, v_cache, cache_seqlens, k_tree, v_tree, mask, mask_batch_stride, o,
                        lse_out, ws, ws_bytes, stream, ev_begin, ev_end);
}

hta_status_t hta_forward_ex(const hta_shape_t *shape, const void *q, const void *k_cache, const void *v_cache,
                            const int32_t *cache_seqlens, const void *k_tree, const void *v_tree, const uint8_t *mask,
                            int64_t mask_batch_stride, void *o, float *lse_out, void *ws, size_t ws_bytes,
                            hta_stream_t stream, void *tree_inputs_ready) {
    return forward_impl(nullptr, shape, q, k_cache, v_cache, cache_seqlens, k_tree, v_tree, mask, mask_batch_stride, o,
                        lse_out, ws, ws_bytes, stream, nullptr, nullptr, nullptr, tree_inputs_ready);
}

hta_status_t hta_forward_paged(const hta_shape_t *shape, const void *q, const void *k_pool, const void *v_pool,
                               int32_t num_pages, int32_t page_size, const int32_t *block_table, int32_t max_pages,
                               const int32_t *cache_seqlens, const void *k_tree, const void *v_tree,
                               const uint8_t *mask, int64_t mask_batch_stride, void *o, float *lse_out, void *ws,
                               size_t ws_bytes, hta_stream_t stream) {
    if (shape == nullptr || block_table == nullptr || num_pages < 1 || max_pages < 1 || page_size < 16 ||
        page_size % 16 != 0)
        return HTA_ERR_INVALID_ARGUMENT;
    if (shape->dtype != HTA_BF16) return HTA_ERR_UNSUPPORTED;
    if (int64_t(num_pages) * page_size > (int64_t(1) << 31) - 1024) return HTA_ERR_INVALID_ARGUMENT;
    hta_shape_t s = *shape;
    s.N_max = int64_t(max_pages) * page_size;  // logical capacity of a batch entry
    s.kv_strides[0] = s.kv_strides[1] = s.kv_strides[2] = 0;  // (the pool is contiguous)
    const PagedArgs pg{block_table, max_pages, page_size, num_pages};
    return forward_impl(&pg, &s, q, k_pool, v_pool, cache_seqlens, k_tree, v_tree, mask, mask_batch_stride, o, lse_out,
                        ws, ws_bytes, stream, nullptr, nullptr);
}

hta_status_t hta_forward_tree(const hta_shape_t *shape, const void *q, const void *k_cache, const void *v_cache,
                              const int32_t *cache_seqlens, const void *k_tree, const void *v_tree,
                              const int32_t *parents, int64_t parents_batch_stride, void *o, float *lse_out, void *ws,
                              size_t ws_bytes, hta_stream_t stream, void *ev_prefix_begin, void *ev_prefix_end,
                              void *tree_inputs_ready) {
    if (parents == nullptr) return HTA_ERR_INVALID_ARGUMENT;
    return forward_impl(nullptr, shape, q, k_cache, v_cache, cache_seqlens, k_tree, v_tree, nullptr, 0, o, lse_out, ws,
                        ws_bytes, stream, ev_prefix_begin, ev_prefix_end, nullptr, tree_inputs_ready, parents,
                        parents_batch_stride);
}

hta_status_t hta_forward(const hta_shape_t *shape, const void *q, const void *k_cache, const void *v_cache,
                         const int32_t *cache_seqlens, const void *k_tree, const void *v_tree, const uint8_t *mask,
                         int64_t mask_batch_stride, void *o, float *lse_out, void *ws, size_t ws_bytes,
                         hta_stream_t stream) {
    return hta_forward_timed(shape, q, k_cache, v_cache, cache_seqlens, k_tree, v_tree, mask, mask_batch_stride, o,
                             lse_out, ws, ws_bytes, stream, nullptr, nullptr);
}

// Checks of the FP8-cache entry points: bf16 q / tree / o, d = 128 or 64, E4M3 rows 16-byte aligned.
static hta_status_t check_fp8(const hta_shape_t *shape, const void *k, const void *v, const float *ks,
                              const float *vs) {
    if (shape == nullptr || !k || !v || !ks || !vs) return HTA_ERR_INVALID_ARGUMENT;
    if (shape->dtype != HTA_BF16) return HTA_ERR_UNSUPPORTED;
    for (int i = 0; i < 3; ++i)
        if (shape->kv_strides[i] % 16 != 0) return HTA_ERR_INVALID_ARGUMENT;  // bytes: 16-byte rows
    if (!is_aligned(k, 16) || !is_aligned(v, 16) || !is_aligned(ks, 4) || !is_aligned(vs, 4))
        return HTA_ERR_INVALID_ARGUMENT;
    return HTA_OK;
}

hta_status_t hta_forward_fp8kv(const hta_shape_t *shape, const void *q, const void *k_cache, const void *v_cache,
                               const float *k_scale, const float *v_scale, const int32_t *cache_seqlens,
                               const void *k_tree, const void *v_tree, const uint8_t *mask,
                               int64_t mask_batch_stride, void *o, float *lse_out, void *ws, size_t ws_bytes,
                               hta_stream_t stream) {
    hta_status_t r = check_fp8(shape, k_cache, v_cache, k_scale, v_scale);
    if (r != HTA_OK) return r;
    const Fp8Args f8{k_scale, v_scale};
    return forward_impl(nullptr, shape, q, k_cache, v_cache, cache_seqlens, k_tree, v_tree, mask, mask_batch_stride, o,
                        lse_out, ws, ws_bytes, stream, nullptr, nullptr, &f8);
}

hta_status_t hta_prefix_attn_fp8kv(const hta_shape_t *shape, const void *q, const void *k_cache, const void *v_cache,
                                   const float *k_scale, const float *v_scale, const int32_t *cache_seqlens,
                                   float *o_part, float *lse_part, void *ws, size_t ws_bytes, hta_stream_t stream) {
    hta_status_t r = check_fp8(shape, k_cache, v_cache, k_scale, v_scale);
    if (r != HTA_OK) return r;
    Shape sh;
    if ((r = check_shape(shape, &sh)) != HTA_OK) return r;
    if (!q || !o_part || !lse_part || !is_aligned(q, 16) || !is_aligned(o_part, 16)) return HTA_ERR_INVALID_ARGUMENT;
    if ((r = check_device()) != HTA_OK) return r;
    const hta_shape_t &s = sh.s;
    const PrefixPlan pl = make_plan(sh, device_sms());
    const Fp8Args f8{k_scale, v_scale};
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (pl.splits == 1)
        return run_prefix(sh, pl, q, k_cache, v_cache, cache_seqlens, o_part, lse_part, 0, 0, st, nullptr, &f8);
    const size_t need = size_t(pl.splits) * part_floats(s) * sizeof(float);
    if (ws == nullptr || ws_bytes < need || !is_aligned(ws, 16)) return HTA_ERR_WORKSPACE;
    float *o_ws = static_cast<float *>(ws);
    const int64_t ostride = int64_t(s.B) * s.T * s.H * s.d;
    float *lse_ws = o_ws + size_t(pl.splits) * ostride;
    const int64_t lstride = int64_t(s.B) * s.H * s.T;
    r = run_prefix(sh, pl, q, k_cache, v_cache, cache_seqlens, o_ws, lse_ws, ostride, lstride, st, nullptr, &f8);
    if (r != HTA_OK) return r;
    TreeMergeParams p = base_tm(sh);
    p.do_tree = 0;
    p.n_parts = pl.splits;
    p.o_parts = o_ws;
    p.lse_parts = lse_ws;
    p.o_part_stride = ostride;
    p.lse_part_stride = lstride;
    set_out_contig_f32(p, s, o_part, lse_part);
    return launch_tree_merge(p, s.d, s.dtype, HTA_FP32, true, st) == cudaSuccess ? HTA_OK : HTA_ERR_CUDA;
}

hta_status_t hta_build_tree_mask(const int32_t *parents, int32_t T, uint8_t *mask, int32_t on_device,
                                 hta_stream_t stream) {
    if (T < 1 || T > 256 || parents == nullptr || mask == nullptr) return HTA_ERR_INVALID_ARGUMENT;
    if (!on_device) return host_build_mask(parents, T, mask) == 0 ? HTA_OK : HTA_ERR_INVALID_MASK;
    hta_status_t r = check_device();
    if (r != HTA_OK) return r;
    return launch_build_mask(parents, T, mask, reinterpret_cast<cudaStream_t>(stream)) == cudaSuccess ? HTA_OK
                                                                                                    : HTA_ERR_CUDA;
}

hta_status_t hta_tree_step(const int32_t *parents, int32_t T, uint8_t *mask, const int32_t *draft_tokens,
                           const int32_t *target_argmax, int32_t root, int32_t context_argmax, int32_t *path,
                           int32_t *path_len, int32_t *bonus, hta_stream_t stream) {
    if (T < 1 || T > 256 || root < -1 || root >= T) return HTA_ERR_INVALID_ARGUMENT;
    if (!parents || !draft_tokens || !target_argmax || !path || !path_len || !bonus) return HTA_ERR_INVALID_ARGUMENT;
    hta_status_t r = check_device();
    if (r != HTA_OK) return r;
    return launch_tree_step(parents, T, mask, draft_tokens, target_argmax, root, context_argmax, path, path_len,
                            bonus, reinterpret_cast<cudaStream_t>(stream)) == cudaSuccess
               ? HTA_OK
               : HTA_ERR_CUDA;
}

hta_status_t hta_validate_tree_mask(const uint8_t *mask, int32_t T) {
    if (mask == nullptr || T < 1 || T > 256) return HTA_ERR_INVALID_ARGUMENT;
    for (int i = 0; i < T; ++i) {
        const uint8_t *row = mask + int64_t(i) * T;
        if (row[i] != 1) return HTA_ERR_INVALID_MASK;
        int par = -1;
        for (int j = 0; j < T; ++j) {
            if (row[j] > 1) return HTA_ERR_INVALID_MASK;
            if (j > i && row[j]) return HTA_ERR_INVALID_MASK;
            if (j < i && row[j]) par = j;
        }
        // row i must equal row(par) + {i} (or {i} alone for a root)
        for (int j = 0; j < T; ++j) {
            const uint8_t want = (j == i) ? 1 : (par >= 0 ? mask[int64_t(par) * T + j] : 0);
            if (row[j] != want) return HTA_ERR_INVALID_MASK;
        }
    }
    return HTA_OK;
}

hta_status_t hta_commit_kv(const hta_shape_t *shape, const int32_t *path, int64_t path_stride,
                           const int32_t *path_len, const void *k_tree, const void *v_tree, void *k_cache,
                           void *v_cache, const int32_t *cache_seqlens, int32_t *seqlens_out, hta_stream_t stream) {
    Shape sh;
    hta_status_t r = check_shape(shape, &sh);
    if (r != HTA_OK) return r;
    const hta_shape_t &s = sh.s;
    if (!path || !path_len || !k_tree || !v_tree || !k_cache || !v_cache || !cache_seqlens || !seqlens_out)
        return HTA_ERR_INVALID_ARGUMENT;
    if (path_stride < s.T) return HTA_ERR_INVALID_ARGUMENT;
    if (!is_aligned(k_tree, 16) || !is_aligned(v_tree, 16) || !is_aligned(k_cache, 16) || !is_aligned(v_cache, 16))
        return HTA_ERR_INVALID_ARGUMENT;
    if ((r = check_device()) != HTA_OK) return r;
    CommitGeom gm;
    gm.T = s.T;
    gm.H_kv = s.H_kv;
    gm.esize = static_cast<int>(sh.esize);
    gm.row_bytes = static_cast<int>(s.d * sh.esize);
    gm.N_max = s.N_max;
    gm.ks0 = s.kv_strides[0];
    gm.ks1 = s.kv_strides[1];
    gm.ks2 = s.kv_strides[2];
    gm.ts0 = s.tkv_strides[0];
    gm.ts1 = s.tkv_strides[1];
    gm.ts2 = s.tkv_strides[2];
    return launch_commit_kv(path, path_stride, path_len, k_tree, v_tree, k_cache, v_cache, cache_seqlens, seqlens_out,
                            gm, s.B, reinterpret_cast<cudaStream_t>(stream)) == cudaSuccess
               ? HTA_OK
               : HTA_ERR_CUDA;
}

hta_status_t hta_accept_greedy(const int32_t *parents, const int32_t *draft_tokens, const int32_t *target_argmax,
                               int32_t T, int32_t root, int32_t context_argmax, int32_t *path, int32_t *path_len,
                               int32_t *bonus, int32_t on_device, hta_stream_t stream) {
    if (T < 1 || T > 256 || root < -1 || root >= T) return HTA_ERR_INVALID_ARGUMENT;
    if (!parents || !draft_tokens || !target_argmax || !path || !path_len || !bonus) return HTA_ERR_INVALID_ARGUMENT;
    if (!on_device)
        return host_accept(parents, draft_tokens, target_argmax, T, root, context_argmax, path, path_len, bonus) == 0
                   ? HTA_OK
                   : HTA_ERR_INVALID_MASK;
    hta_status_t r = check_device();
    if (r != HTA_OK) return r;
    return launch_accept(parents, draft_tokens, target_argmax, T, root, context_argmax, path, path_len, bonus,
                         reinterpret_cast<cudaStream_t>(stream)) == cudaSuccess
               ? HTA_OK
               : HTA_ERR_CUDA;
}

}  // extern "C"

// ======================================================================= seqpar helpers

namespace hta {

hta_status_t seqpar_local_parts(const hta_shape_t *shape, const void *q, const void *k, const void *v,
                                const int32_t *seqlens, float *parts_ws, size_t parts_bytes, float *sendb, int P,
                                cudaStream_t st, const P2pOut *p2p) {
    Shape sh;
    hta_status_t r = check_shape(shape, &sh);
    if (r != HTA_OK) return r;
    if ((r = check_device()) != HTA_OK) return r;
    const hta_shape_t &s = sh.s;
    const PrefixPlan pl = make_plan(sh, device_sms());
    const int64_t ostride = int64_t(s.B) * s.T * s.H * s.d;
    const int64_t lstride = int64_t(s.B) * s.H * s.T;
    if (size_t(pl.splits) * part_floats(s) * sizeof(float) > parts_bytes) return HTA_ERR_WORKSPACE;
    float *lse_ws = parts_ws + size_t(pl.splits) * ostride;
    r = run_prefix(sh, pl, q, k, v, seqlens, parts_ws, lse_ws, ostride, lstride, st);
    if (r != HTA_OK) return r;
    const int Hp = s.H / P;
    const int64_t blk = static_cast<int64_t>(seqpar_block_floats(s.B, s.T, Hp, s.d));
    TreeMergeParams p = base_tm(sh);
    p.do_tree = 0;
    p.n_parts = pl.splits;
    p.o_parts = parts_ws;
    p.lse_parts = lse_ws;
    p.o_part_stride = ostride;
    p.lse_part_stride = lstride;
    p.o = sendb;
    p.os0 = int64_t(s.T) * Hp * s.d;
    p.os1 = int64_t(Hp) * s.d;
    p.os2 = s.d;
    p.o_block_stride = blk;
    p.lse = sendb + int64_t(s.B) * s.T * Hp * s.d;
    p.lse_block_stride = blk;
    p.out_hb = Hp;
    if (p2p != nullptr) {  // straight into the peers' receive buffers
        if (P > kMaxP2pRanks) return HTA_ERR_INVALID_ARGUMENT;
        p.p2p_role = 1;
        p.p2p_epoch = p2p->epoch;
        p.p2p_parity = p2p->parity;
        p.p2p_lse_off = int64_t(s.B) * s.T * Hp * s.d;
        p.p2p_counter = p2p->counter;
        p.p2p_nranks = P;
        p.p2p_rank = p2p->rank;
        for (int i = 0; i < P; ++i) {
            p.p2p_dst[i] = p2p->dst[i];
            p.p2p_peer_flags[i] = p2p->peer_flags[i];
        }
    }
    return launch_tree_merge(p, s.d, s.dtype, HTA_FP32, true, st) == cudaSuccess ? HTA_OK : HTA_ERR_CUDA;
}

hta_status_t seqpar_final_merge(const hta_shape_t *shape, int P, int rank, const void *q, const void *kt,
                                const void *vt, const uint8_t *mask, int64_t mask_bs, const int32_t *parents,
                                int64_t par_bs, const float *recvb, size_t blk_floats, void *o, float *lse,
                                cudaStream_t st, const P2pIn *p2p) {
    Shape sh;
    hta_status_t r = check_shape(shape, &sh);
    if (r != HTA_OK) return r;
    const hta_shape_t &s = sh.s;
    if (mask == nullptr && parents == nullptr) return HTA_ERR_INVALID_ARGUMENT;
    if (mask != nullptr && mask_bs != 0 && mask_bs < int64_t(s.T) * s.T) return HTA_ERR_INVALID_ARGUMENT;
    if (mask == nullptr && par_bs != 0 && par_bs < s.T) return HTA_ERR_INVALID_ARGUMENT;
    const int Hp = s.H / P;
    TreeMergeParams p = base_tm(sh);
    p.Hr = Hp;
    p.h0 = rank * Hp;
    p.q = q;
    p.kt = kt;
    p.vt = vt;
    p.mask = mask;
    p.mask_bs = mask_bs;
    p.parents = mask == nullptr ? parents : nullptr;
    p.par_bs = par_bs;
    p.do_tree = 1;
    p.n_parts = P;
    p.o_parts = recvb;
    p.lse_parts = recvb + int64_t(s.B) * s.T * Hp * s.d;
    p.o_part_stride = int64_t(blk_floats);
    p.lse_part_stride = int64_t(blk_floats);
    p.o = o;
    p.os0 = int64_t(s.T) * Hp * s.d;
    p.os1 = int64_t(Hp) * s.d;
    p.os2 = s.d;
    p.lse = lse;
    p.out_hb = Hp;
    if (p2p != nullptr) {  // this step's half of the double-buffered receive blocks, once flagged
        p.p2p_role = 2;
        p.p2p_epoch = p2p->epoch;
        p.p2p_flags = p2p->flags;
        p.p2p_parity = p2p->parity;
    }
    return launch_tree_merge(p, s.d, s.dtype, s.dtype, false, st) == cudaSuccess ? HTA_OK : HTA_ERR_CUDA;
}

}  // namespace hta
