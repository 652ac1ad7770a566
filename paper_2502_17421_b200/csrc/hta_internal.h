// hta_internal.h -- parameter blocks and launchers shared by libhta's translation units.
// Not part of the ABI (include/hta.h is).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "../../include/hta.h"

namespace hta {

// Keys per KV tile of the prefix pass: TMEM holds 384 / kBlockN S/P buffers of kBlockN columns
// and the 128-column O accumulator (512 columns in all): three 128-key buffers (96-key tiles with
// four buffers measured slower: profiles/r02_experiments.md).
// Fused tree pass for CTA pairs too (build option; measured slower than the tree pass in the
// tree/merge kernel: Llama-8B-64k 71.1 vs 69.6 us, 128k/T=128 225.8 vs 219 us; profiles/
// r02_experiments.md).  Single-CTA row groups always fuse.
#ifndef HTA_FUSE_PAIRS
#define HTA_FUSE_PAIRS 0
#endif

// FP8 cache, d = 128: S = Q K^T on kind::f8f6f4 over the E4M3 K tile (q as two E4M3 terms); 0 =
// the K tile widened to f16 like V
#ifndef HTA_F8S
#define HTA_F8S 1
#endif

// ... and with it PV on kind::f8f6f4 (P as E4M3 + E5M2 terms in TMEM, V read as landed); 0 = V
// widened to f16, f16 P
#ifndef HTA_F8P
#define HTA_F8P 1
#endif

#ifndef HTA_BLOCK_N
#define HTA_BLOCK_N 128
#endif
constexpr int kBlockN = HTA_BLOCK_N;
static_assert(kBlockN == 96 || kBlockN == 128, "96-key tiles (four S/P buffers) or 128 (three)");
constexpr int kSimtBlock = 16;   // key block (split granularity) of the fp32 SIMT prefix pass
constexpr int kRowsPerTile = 128;  // rows of one tcgen05 M=128 tile

// Work decomposition of the prefix pass.
struct PrefixPlan {
    int G;            // H / H_kv
    int M;            // rows per (b, kv-head) = T * G   (t-major, then the G heads)
    int nt;           // M tiles (of 128 rows) per CTA: 1 or 2
    int n_mgroups;    // ceil(M / (128 * nt))
    int units;        // B * H_kv * n_mgroups
    int n_tiles;      // ceil(N_max / kBlockN) (bf16) or ceil(N_max / kSimtBlock) (fp32)
    int tiles_per_split;
    int splits;       // S
};

struct PrefixParams {
    const void *q;                    // [B,T,H,d] dtype
    int64_t qs0, qs1, qs2;            // element strides of q
    const void *k, *v;                // SIMT path only (the tcgen05 path reads via TMA)
    int64_t ks0, ks1, ks2;
    const int32_t *seqlens;           // [B] or nullptr
    int B, T, H, H_kv, d, G, M;
    int64_t N_max;
    float scale;                      // softmax scale
    float scale_log2;                 // scale * log2(e)
    int nt, n_mgroups, splits, tiles_per_split;
    int q_tma;                                  // Q rows of a tile come from tmap_q (G divides 128)
    // Paged KV (page_size > 0): the K/V maps cover a pool of pages seen as
    // one [rows, H_kv, d] tensor; logical key k of batch b sits at pool row
    // block_table[b * bt_stride + k / page_size] * page_size + k % page_size.  TMA boxes are 16
    // rows (page_size % 16 == 0).
    const int32_t *block_table;
    int64_t bt_stride;
    int page_size;
    int max_pages;                              // entries per block-table row (clamp)
    // FP8 cache (kv8 = 1): k/v are E4M3 bytes, K = k_scale[g] * E4M3 and
    // V = v_scale[g] * E4M3 per KV head g (device float [H_kv]); the maps load E4M3 tiles.
    int kv8;
    const float *k_scale, *v_scale;
    // Fused tree pass (hta_forward, bf16 cache): the last split of every unit appends tree_tiles
    // (= ceil(T / 128)) masked tiles of the tree keys (tmap_kt / tmap_vt over k_tree / v_tree) to
    // its cache tiles, so its partial already holds the tree part (the Appendix C merge applied
    // inside the online softmax).  Row r of token t sees tree key s iff mask[b*mask_bs + t*T + s].
    int tree_tiles;
    const uint8_t *mask;
    int64_t mask_bs;
    const int32_t *parents;           // hta_forward_tree: visibility from parents [b*par_bs + t] instead of mask
    int64_t par_bs;
    float *o_out;                     // [S][B][T][H][d] fp32, normalised partials
    float *lse_out;                   // [S][B][H][T] natural-log LSE
    int64_t o_split_stride, lse_split_stride;  // elements between splits
};

constexpr int kMaxP2pRanks = 8;  // ranks of the peer-memory exchange (one NVSwitch node)

struct TreeMergeParams {
    // Row space: (b, t, hl) with hl in [0, Hr); the global query head is h = h0 + hl.
    int B, T, H, H_kv, G, Hr, h0;
    const void *q;                    // [B,T,H,d] (tree pass only)
    int64_t qs0, qs1, qs2;
    const void *kt, *vt;              // [B,T,H_kv,d]
    int64_t ts0, ts1, ts2;
    const uint8_t *mask;              // [B,T,T]
    int64_t mask_bs;                  // batch stride (0 = shared)
    const int32_t *parents;           // or (mask == nullptr) the parent array [B,T] (visibility = ancestors)
    int64_t par_bs;                   // batch stride of parents (0 = shared)
    float scale;
    int do_tree;                      // run the masked tree pass
    int n_parts;                      // prefix partials to merge (0 = none)
    const float *o_parts;             // [n][B][T][Hr][d]
    const float *lse_parts;           // [n][B][Hr][T]
    int64_t o_part_stride, lse_part_stride;
    // Output: head hl goes to block hl / out_hb at local head hl % out_hb:
    //   o   + (hl/out_hb)*o_block_stride   + b*os0 + t*os1 + (hl%out_hb)*os2
    //   lse + (hl/out_hb)*lse_block_stride + (b*out_hb + hl%out_hb)*T + t
    void *o;
    int64_t os0, os1, os2, o_block_stride;
    float *lse;                       // may be nullptr
    int64_t lse_block_stride;
    int out_hb;
    // Peer-memory exchange of the sequence-parallel step (p2p_role != 0):
    //  role 1 (split combine): block blk goes to p2p_dst[blk] + ((*p2p_epoch) & 1) * p2p_parity
    //         (O) and + p2p_lse_off (LSE), i.e. straight into rank blk's receive buffer, followed by
    //         a system-scope fence;
    //  role 2 (final merge): the partials are read at o_parts + (((*p2p_epoch) - 1) & 1) *
    //         p2p_parity after every p2p_flags[q], q < n_parts, has reached *p2p_epoch.
    //  role 1 also signals: its last block (p2p_counter, a step-long block counter) raises flag
    //  p2p_rank in every p2p_peer_flags[q], q < p2p_nranks, to the new step and advances *p2p_epoch.
    int p2p_role;
    const uint32_t *p2p_epoch;
    const uint32_t *p2p_flags;
    int64_t p2p_parity, p2p_lse_off;
    float *p2p_dst[kMaxP2pRanks];
    uint32_t *p2p_counter;
    uint32_t *p2p_peer_flags[kMaxP2pRanks];
    int p2p_nranks, p2p_rank;
};

// Launchers (return cudaGetLastError() of the launch).
cudaError_t launch_prefix_tc(const PrefixParams &p, const CUtensorMap &tmap_q, const CUtensorMap &tmap_k,
                             const CUtensorMap &tmap_v, const CUtensorMap &tmap_kt, const CUtensorMap &tmap_vt,
                             int smem_bytes, cudaStream_t s);
int prefix_tc_smem_bytes(int d, int nt);
// FP8 cache, units of at most 64 rows, d = 128: the transposed kernel (prefix_t8.cu); tk / tv are
// E4M3 maps with 128 x 128-byte boxes, tk with 128-byte swizzle, tv without.  A build option
// (-DHTA_T8=1): correct, but not faster than prefix_tc.cu's widening warps on LongChat-16k
// (63.5 vs 61.5 us; profiles/r02_experiments.md), so the default library does not contain it.
#ifndef HTA_T8
#define HTA_T8 0
#endif
cudaError_t launch_prefix_t8(const PrefixParams &p, const CUtensorMap &tk, const CUtensorMap &tv, cudaStream_t s);
cudaError_t launch_prefix_simt(const PrefixParams &p, cudaStream_t s);
cudaError_t launch_tree_merge(const TreeMergeParams &p, int d, hta_dtype_t in_dtype, hta_dtype_t out_dtype,
                              bool pdl, cudaStream_t s);

// Geometry of hta_commit_kv (element strides; esize bytes per element).
struct CommitGeom {
    int T, H_kv, row_bytes, esize;
    int64_t N_max;
    int64_t ks0, ks1, ks2;  // cache [B, N, H_kv]
    int64_t ts0, ts1, ts2;  // tree  [B, T, H_kv]
};
cudaError_t launch_commit_kv(const int32_t *path, int64_t path_stride, const int32_t *path_len, const void *kt,
                             const void *vt, void *kc, void *vc, const int32_t *seqlens, int32_t *seqlens_out,
                             const CommitGeom &gm, int B, cudaStream_t s);
cudaError_t launch_build_mask(const int32_t *parents, int T, uint8_t *mask, cudaStream_t s);
// Mask (if mask != nullptr) and greedy accepted path (if draft != nullptr) in one launch.
cudaError_t launch_tree_step(const int32_t *parents, int T, uint8_t *mask, const int32_t *draft, const int32_t *tgt,
                             int root, int ctx, int32_t *path, int32_t *path_len, int32_t *bonus, cudaStream_t s);
cudaError_t launch_accept(const int32_t *parents, const int32_t *draft, const int32_t *tgt, int T, int root,
                          int ctx, int32_t *path, int32_t *path_len, int32_t *bonus, cudaStream_t s);

// Host reference-free implementations of the tree utilities (shared by the host ABI paths).
int host_build_mask(const int32_t *parents, int T, uint8_t *mask);  // 0 ok, -1 invalid
int host_accept(const int32_t *parents, const int32_t *draft, const int32_t *tgt, int T, int root, int ctx,
                int32_t *path, int32_t *path_len, int32_t *bonus);  // 0 ok, -1 invalid

// Floats of one destination-major exchange block of the sequence-parallel step: O [B][T][Hp][d]
// then LSE [B][Hp][T], rounded up to a multiple of 4 floats so that every block (and the
// vectorised O rows in it) stays 16-byte aligned.
inline size_t seqpar_block_floats(int B, int T, int Hp, int d) {
    const size_t n = size_t(B) * T * Hp * d + size_t(B) * Hp * T;
    return (n + 3) & ~size_t(3);
}

// Sequence-parallel building blocks (implemented in hta_api.cu, used by seqpar.cu).
// Local prefix pass over this rank's KV slice, combined into one partial per row laid out
// destination-major: block p (for rank p) = O [B][T][H/P][d] then LSE [B][H/P][T].
// Peer-memory exchange: the split combine of rank r writes block q into
// dst[q] + (epoch & 1) * parity (rank r's slot of rank q's double-buffered receive buffer); the
// final merge reads its receive buffer's half ((epoch - 1) & 1) once flags[q] >= epoch for all q.
struct P2pOut {
    float *dst[kMaxP2pRanks];
    uint32_t *epoch;        // this rank's step counter
    uint32_t *counter;      // this rank's block counter of the split combine
    uint32_t *peer_flags[kMaxP2pRanks];
    int rank;
    int64_t parity;
};
struct P2pIn {
    const uint32_t *epoch;
    const uint32_t *flags;
    int64_t parity;
};
hta_status_t seqpar_local_parts(const hta_shape_t *s, const void *q, const void *k, const void *v,
                                const int32_t *seqlens, float *parts_ws, size_t parts_bytes, float *sendb, int P,
                                cudaStream_t st, const P2pOut *p2p = nullptr);
// Merge the P received partials (blocks of `blk_floats`) with the tree pass of heads
// [r*H/P, (r+1)*H/P) into o [B,T,H/P,d] (dtype) and lse [B,H/P,T] (optional).
// The tree's visibility is the mask, or (mask == nullptr) the parent array (ancestor walk).
hta_status_t seqpar_final_merge(const hta_shape_t *s, int P, int r, const void *q, const void *kt, const void *vt,
                                const uint8_t *mask, int64_t mask_bs, const int32_t *parents, int64_t par_bs,
                                const float *recvb, size_t blk_floats, void *o, float *lse, cudaStream_t st,
                                const P2pIn *p2p = nullptr);

}  // namespace hta
