/*
 * hta.h -- C ABI of libhta, a B200-native (sm_100a) implementation of the verification-step
 * attention of LongSpec (arXiv 2502.17421): Hybrid Tree Attention.
 *
 * Citations "P:n" are lines of the paper's text (reference PAPER.md), "S:n" lines of the
 * reference SPEC.md, "Zk" the readings listed in DESIGN.md.
 *
 * The method (Appendix C).  T tree ("speculative") tokens, each with H
 * query heads of size d, attend to
 *   (a) the target model's KV cache of N tokens -- "the queries and the cached key-value
 *       pairs {K_cache, V_cache} do not require additional masks", and
 *   (b) the T speculative keys/values {K_specs, V_specs} under the T x T tree mask
 *       ("only ... the current speculative tokens need masking").
 * Each part yields a normalised output O and its row log-sum-exp LSE;
 * the parts are merged exactly:
 *   LSE = log(exp(LSE_cache) + exp(LSE_specs)),
 *   O   = O_cache exp(LSE_cache - LSE) + O_specs exp(LSE_specs - LSE).
 *
 * Conventions (all entry points):
 *  - Tensor pointers are DEVICE pointers owned by the caller (e.g. PyTorch tensors) unless an
 *    argument says "host"; they must stay valid until the enqueued work on `stream` finishes.
 *    The library never allocates device memory in a compute call (only hta_comm_create does).
 *  - Calls validate their arguments on the host, enqueue kernels on `stream` and return
 *    without synchronising.  Host-checkable errors return a status before any launch.  A
 *    failed launch returns HTA_ERR_CUDA.  Asynchronous faults surface at the caller's next
 *    synchronisation.  No exceptions cross the ABI; the library never calls exit().
 *  - Functions are stateless and re-entrant; concurrent calls on different streams are legal.
 *  - LSE is the NATURAL log of the sum of exp of the SCALED logits, z = scale * q.k
 *    (reading Z1), as returned by flash_attn's softmax_lse (the paper's prefix
 *    call, P:108 footnote).  LSE tensors are float32 [B, H, T].
 *  - Partial outputs (O parts) are float32 [B, T, H, d], contiguous, each normalised by its own
 *    sum of exp.  An empty part (no visible key) is the sentinel O = 0, LSE = -inf
 *    (reading Z10), which is the identity of the merge; no NaN is produced for it.
 *  - GQA: query head h reads KV head h / (H / H_kv) (reading Z8).
 *  - No CPU fallback: compute entry points require an sm_100 device; on any other device they
 *    return HTA_ERR_UNSUPPORTED.
 */
#ifndef HTA_H_
#define HTA_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#pragma GCC visibility push(default) /* the ABI symbols are exported even with -fvisibility=hidden */
#endif
#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *hta_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
    HTA_OK = 0,
    HTA_ERR_INVALID_ARGUMENT = 1, /* shape, stride, alignment, range or NULL-pointer error   */
    HTA_ERR_UNSUPPORTED = 2,      /* valid request this build cannot run (device, d, dtype)  */
    HTA_ERR_INVALID_MASK = 3,     /* tree mask / parent array is not an ancestor-closed tree */
    HTA_ERR_WORKSPACE = 4,        /* workspace NULL or smaller than hta_workspace_size()     */
    HTA_ERR_CUDA = 5,             /* a CUDA runtime / driver call or kernel launch failed    */
    HTA_ERR_NCCL = 6              /* NCCL unavailable or an NCCL call failed                 */
} hta_status_t;

typedef enum { HTA_BF16 = 0, HTA_FP32 = 1 } hta_dtype_t;

/* Problem shape and memory layout.  Strides are in ELEMENTS; the innermost dimension (d) is
 * always contiguous.  A stride triple of all zeros selects the contiguous default. */
typedef struct {
    int32_t B;            /* batch size, >= 1                                               */
    int32_t T;            /* tree tokens (queries and speculative keys), 1 <= T <= 256      */
    int32_t H;            /* query heads, H % H_kv == 0                                     */
    int32_t H_kv;         /* key/value heads                                                */
    int32_t d;            /* head dim: 64 or 128                                            */
    int64_t N_max;        /* cache capacity = sequence extent of k_cache / v_cache, >= 0    */
    float softmax_scale;  /* multiplies q.k; normally 1/sqrt(d)                     */
    hta_dtype_t dtype;    /* element type of q, k_*, v_* and o                              */
    int64_t q_strides[3];   /* [B, T, H]    of q and o; default {T*H*d, H*d, d}             */
    int64_t kv_strides[3];  /* [B, N, H_kv] of k_cache, v_cache; default {N*H_kv*d, H_kv*d, d} */
    int64_t tkv_strides[3]; /* [B, T, H_kv] of k_tree, v_tree; default {T*H_kv*d, H_kv*d, d} */
    int32_t num_splits;   /* KV splits of the prefix pass per (b, kv-head, row tile);
                             0 = chosen by the library from the SM count                    */
    int32_t max_seqlen;   /* optional upper bound on cache_seqlens (0 = N_max), used only to
                             plan the split-KV schedule when the cache capacity is much larger
                             than the filled length; a batch entry longer than the bound is
                             still computed exactly (the last split runs to its length)     */
} hta_shape_t;

/* Human-readable name of a status (static string, never NULL). */
const char *hta_status_string(hta_status_t status);

/* Library version as major*10000 + minor*100 + patch. */
int32_t hta_version(void);

/* Bytes of device workspace hta_prefix_attn / hta_forward need for `shape` on a device with
 * `num_sms` SMs (pass the device's multiProcessorCount; <= 0 means 148, one B200).  The
 * workspace holds the split-KV partials: num_splits x (B*T*H*d + B*H*T) floats (at least one
 * split).  Returns (size_t)-1 for an invalid shape.  Host-only; never touches the GPU. */
size_t hta_workspace_size(const hta_shape_t *shape, int32_t num_sms);

/* attend_cache: UNMASKED attention of every tree query over the KV cache -- the
 * paper's FlashAttention/FlashDecoding prefix call.
 *   q            [B, T, H, d] dtype (q_strides)
 *   k_cache      [B, N_max, H_kv, d] dtype (kv_strides); v_cache likewise
 *   cache_seqlens device int32 [B] valid prefix length per batch (<= N_max), or NULL (= N_max).
 *                Rows j >= cache_seqlens[b] are never read into the softmax (reading Z13).
 *   o_part       float32 [B, T, H, d] contiguous (output);  lse_part float32 [B, H, T] (output)
 *   ws, ws_bytes device workspace of at least hta_workspace_size(shape) bytes (may be NULL
 *                when that size is 0).
 * A batch with cache_seqlens[b] == 0 yields the sentinel.  bf16 runs on the tcgen05
 * tensor cores (fp32 accumulation, P rounded to bf16 for P.V); fp32 runs on FFMA. */
hta_status_t hta_prefix_attn(const hta_shape_t *shape, const void *q, const void *k_cache,
                             const void *v_cache, const int32_t *cache_seqlens, float *o_part,
                             float *lse_part, void *ws, size_t ws_bytes, hta_stream_t stream);

/* attend_specs: MASKED attention of every tree query over the T speculative keys
 * (the paper's fused_mask_attn).
 *   k_tree, v_tree [B, T, H_kv, d] dtype (tkv_strides)
 *   mask         device uint8 [B, T, T] row-major, mask[b][i][j] != 0 <=> key j visible to
 *                query i; mask_batch_stride = elements between batches (0 = one mask shared
 *                by all b, otherwise >= T*T).
 *   o_part, lse_part as in hta_prefix_attn.
 * Any 0/1 pattern is accepted; an all-zero row yields the sentinel (deviation from S:386,
 * which raises: use hta_validate_tree_mask to reject malformed trees). */
hta_status_t hta_tree_attn(const hta_shape_t *shape, const void *q, const void *k_tree,
                           const void *v_tree, const uint8_t *mask, int64_t mask_batch_stride,
                           float *o_part, float *lse_part, hta_stream_t stream);

/* merge_attention, n-ary form of the aggregation P:207-218 (max-shifted, reading Z11):
 *   o_parts   float32 [n_parts, B, T, H, d] contiguous; lse_parts float32 [n_parts, B, H, T]
 *   o         [B, T, H, d] in shape->dtype with q_strides (output, round-to-nearest)
 *   lse_out   float32 [B, H, T] (output) or NULL.
 * n_parts >= 1.  Rows whose parts are all sentinels give O = 0, LSE = -inf. */
hta_status_t hta_merge_lse(const hta_shape_t *shape, int32_t n_parts, const float *o_parts,
                           const float *lse_parts, void *o, float *lse_out, hta_stream_t stream);

/* hybrid_tree_attention: prefix pass + tree pass + merge, i.e. the full
 * verification-step attention of one layer.  Two kernels: the split-KV prefix kernel, then
 * one kernel that merges the split partials.  The tree pass runs in the prefix kernel (masked
 * tree tiles appended to each unit's last split) for bf16 caches whose row groups are single
 * CTAs (T*H/H_kv rows packing into 128-row tiles; MHA, G = 5, d = 64), else in the second kernel
 * beside the merge; the result is the same up to rounding.  Arguments as above; o in
 * shape->dtype with q_strides; lse_out optional (NULL). */
hta_status_t hta_forward(const hta_shape_t *shape, const void *q, const void *k_cache,
                         const void *v_cache, const int32_t *cache_seqlens, const void *k_tree,
                         const void *v_tree, const uint8_t *mask, int64_t mask_batch_stride,
                         void *o, float *lse_out, void *ws, size_t ws_bytes,
                         hta_stream_t stream);

/* hta_forward with instrumentation for benchmarks: when non-NULL, `ev_prefix_begin` and
 * `ev_prefix_end` (cudaEvent_t) are recorded on `stream` immediately before and after the
 * prefix-pass kernel, so its duration can be timed with cudaEventElapsedTime.  Otherwise
 * identical to hta_forward (the events cost the programmatic-launch overlap of the second
 * kernel, so time steps with hta_forward and kernels with this call). */
hta_status_t hta_forward_timed(const hta_shape_t *shape, const void *q, const void *k_cache,
                               const void *v_cache, const int32_t *cache_seqlens,
                               const void *k_tree, const void *v_tree, const uint8_t *mask,
                               int64_t mask_batch_stride, void *o, float *lse_out, void *ws,
                               size_t ws_bytes, hta_stream_t stream, void *ev_prefix_begin,
                               void *ev_prefix_end);

/* hta_forward whose tree inputs arrive late: `tree_inputs_ready` (a cudaEvent_t, or NULL) is
 * waited for on `stream` after the prefix kernel is enqueued and before the tree/merge kernel, so
 * k_tree, v_tree and mask may still be in flight (e.g. copied from the host on another stream)
 * while the prefix pass streams the cache -- only q and the cache gate the prefix.  Otherwise
 * identical to hta_forward. */
hta_status_t hta_forward_ex(const hta_shape_t *shape, const void *q, const void *k_cache,
                            const void *v_cache, const int32_t *cache_seqlens, const void *k_tree,
                            const void *v_tree, const uint8_t *mask, int64_t mask_batch_stride,
                            void *o, float *lse_out, void *ws, size_t ws_bytes,
                            hta_stream_t stream, void *tree_inputs_ready);

/* hta_forward with the tree given by its parent array instead of a mask (
 * reading Z4): row t sees tree key s iff s == t or s is an ancestor of t, derived inside the
 * kernels by walking the parent links -- the same rows hta_build_tree_mask writes (a chain
 * through an invalid entry, parents[a] < -1 or >= a, hides the whole row).  The mask build (a0)
 * is then off the attention's critical path: a verification step can build the mask it keeps
 * (hta_tree_step) on another stream while this runs.
 *   parents    device int32 [B][T] (parents_batch_stride elements apart; 0 = one tree shared
 *              by the batch), parents[t] in [-1, t)
 *   ev_prefix_begin / ev_prefix_end  optional cudaEvent_t recorded around the prefix kernel,
 *              as in hta_forward_timed (NULL: none)
 *   tree_inputs_ready  optional cudaEvent_t: k_tree, v_tree and parents may still be in flight
 *              (e.g. copied from the host on another stream); only the kernel after the prefix
 *              pass waits for it, as in hta_forward_ex (the tree pass then runs there)
 * Other arguments, layout, ownership and errors as hta_forward. */
hta_status_t hta_forward_tree(const hta_shape_t *shape, const void *q, const void *k_cache,
                              const void *v_cache, const int32_t *cache_seqlens,
                              const void *k_tree, const void *v_tree, const int32_t *parents,
                              int64_t parents_batch_stride, void *o, float *lse_out, void *ws,
                              size_t ws_bytes, hta_stream_t stream, void *ev_prefix_begin,
                              void *ev_prefix_end, void *tree_inputs_ready);

/* hybrid_tree_attention over a PAGED KV cache (the block-table layout of
 * flash_attn_with_kvcache, for batched serving): as hta_forward (bf16 only), with
 *   k_pool, v_pool  bf16 [num_pages, page_size, H_kv, d] contiguous (the pages of all batches)
 *   page_size       a multiple of 16 (16-row TMA boxes)
 *   block_table     device int32 [B, max_pages]: logical key k of batch b lives in page
 *                   block_table[b][k / page_size], row k % page_size.  Entries past the pages a
 *                   batch uses are not read for valid keys (negative ones read page 0, masked).
 *   shape->N_max    ignored (the logical capacity is max_pages * page_size); kv_strides ignored.
 * The result equals hta_forward on the gathered contiguous cache (the same tiles in the same
 * order: bit-identical). */
hta_status_t hta_forward_paged(const hta_shape_t *shape, const void *q, const void *k_pool,
                               const void *v_pool, int32_t num_pages, int32_t page_size,
                               const int32_t *block_table, int32_t max_pages,
                               const int32_t *cache_seqlens, const void *k_tree, const void *v_tree,
                               const uint8_t *mask, int64_t mask_batch_stride, void *o,
                               float *lse_out, void *ws, size_t ws_bytes, hta_stream_t stream);

/* hybrid_tree_attention over an FP8 (E4M3) KV cache (beyond the paper, which
 * runs fp16 only): as hta_forward with
 *   k_cache, v_cache  E4M3 bytes [B, N_max, H_kv, d] (kv_strides in ELEMENTS = bytes, multiples of
 *                     16; 16-byte aligned rows), holding K8, V8 with
 *                     K = k_scale[g] * K8,  V = v_scale[g] * V8  for KV head g
 *   k_scale, v_scale  device float32 [H_kv]
 *   q, k_tree, v_tree, o   bf16 (shape->dtype must be HTA_BF16; d 64 or 128)
 * The HBM traffic of the cache is halved.  The prefix contraction runs on the tensor cores with
 * fp32 accumulation: for one-CTA row groups with d = 128, S = q K^T on the FP8
 * tensor path straight from the E4M3 K tile with q split into two E4M3 terms at a power-of-two
 * scale per row (bf16 q reproduced to within 2^-17 of its row maximum), and, when a group has
 * more than 64 rows, P V on the FP8 path too with P as an E4M3 + E5M2 pair (about bf16's
 * precision; P below 2^-22 of the running maximum dropped); otherwise the E4M3 tiles are widened
 * to f16 in shared memory (exact), q is converted to f16 and P rounded to f16.  The result
 * matches hybrid tree attention over the decoded cache within the bf16 tolerances.  Workspace and
 * errors as hta_forward; HTA_ERR_UNSUPPORTED for dtype fp32. */
hta_status_t hta_forward_fp8kv(const hta_shape_t *shape, const void *q, const void *k_cache,
                               const void *v_cache, const float *k_scale, const float *v_scale,
                               const int32_t *cache_seqlens, const void *k_tree,
                               const void *v_tree, const uint8_t *mask,
                               int64_t mask_batch_stride, void *o, float *lse_out, void *ws,
                               size_t ws_bytes, hta_stream_t stream);

/* The prefix pass alone over an FP8 cache (as hta_prefix_attn; arguments as hta_forward_fp8kv). */
hta_status_t hta_prefix_attn_fp8kv(const hta_shape_t *shape, const void *q, const void *k_cache,
                                   const void *v_cache, const float *k_scale,
                                   const float *v_scale, const int32_t *cache_seqlens,
                                   float *o_part, float *lse_part, void *ws, size_t ws_bytes,
                                   hta_stream_t stream);

/* Tree mask from a parent array ("attention masks derived from prefix trees"; reading
 * Z4: mask[i][j] = 1 iff j == i or j is an ancestor of i).
 *   parents  int32 [T], parents[i] in [-1, i) (-1 = child of the committed context; reading Z6)
 *   mask     uint8 [T, T] row-major (output)
 *   on_device 0: parents and mask are HOST pointers, the call is synchronous, and an invalid
 *                parent array returns HTA_ERR_INVALID_MASK;
 *             1: DEVICE pointers, enqueued on `stream`; an invalid entry parents[i] makes row
 *                i all-zero (detectable by hta_validate_tree_mask). */
hta_status_t hta_build_tree_mask(const int32_t *parents, int32_t T, uint8_t *mask, int32_t on_device,
                                 hta_stream_t stream);

/* Host check that a HOST uint8 [T, T] mask is a tree mask: reflexive (diagonal 1), only
 * earlier nodes visible (j <= i), and ancestor-closed (row i = row p(i) + {i} where p(i) is
 * the largest j < i visible to i).  HTA_OK or HTA_ERR_INVALID_MASK. */
hta_status_t hta_validate_tree_mask(const uint8_t *mask, int32_t T);

/* Greedy accepted path (lossless verification at temperature 0, P:190, P:239, P:449;
 * reading Z12): the LONGEST root-anchored path in which every node's draft token equals the
 * target's argmax at its parent; among equally long paths the lexicographically smallest
 * node-index sequence; bonus = target argmax at the path's last node.
 *   parents, draft_tokens, target_argmax  int32 [T]  (target_argmax[u] = target's greedy
 *                token after the prefix ending at node u)
 *   root >= 0  : the path starts at node `root` (path[0] = root, normally 0 = pending token);
 *   root == -1 : forest; nodes with parents == -1 are matched against context_argmax (the
 *                target's token after the committed context); the path may be empty, in which
 *                case bonus = context_argmax.
 *   path int32 [T] (output, first *path_len entries valid), path_len int32 [1], bonus int32 [1].
 * Emitted tokens = draft tokens of the path (excluding a root node) + bonus.
 * on_device 0: host pointers, synchronous, invalid input -> HTA_ERR_INVALID_MASK;
 *           1: device pointers enqueued on `stream` (invalid input -> path_len = -1). */
hta_status_t hta_accept_greedy(const int32_t *parents, const int32_t *draft_tokens,
                               const int32_t *target_argmax, int32_t T, int32_t root,
                               int32_t context_argmax, int32_t *path, int32_t *path_len,
                               int32_t *bonus, int32_t on_device, hta_stream_t stream);

/* The per-step tree work of a verification step in ONE launch on `stream` (device pointers):
 * the tree mask of `parents` (as hta_build_tree_mask with on_device = 1; mask may be NULL to skip
 * it) and the greedy accepted path (as hta_accept_greedy with on_device = 1).  Invalid parent
 * entries give all-zero mask rows and path_len = -1.  The kernel lets the next kernel on the
 * stream start its prologue at once (programmatic dependent launch), so a following hta_forward,
 * which needs the mask only in its tree pass, is barely delayed by it. */
hta_status_t hta_tree_step(const int32_t *parents, int32_t T, uint8_t *mask,
                           const int32_t *draft_tokens, const int32_t *target_argmax, int32_t root,
                           int32_t context_argmax, int32_t *path, int32_t *path_len,
                           int32_t *bonus, hta_stream_t stream);

/* commit_kv ("the large model only updates its KV cache upon
 * verification completion"): append the accepted tree nodes' K/V rows to the cache, in path
 * order, on the device (no host round trip between acceptance and the next step).
 *   shape        B, T, H_kv, d, N_max, dtype, kv_strides (cache), tkv_strides (tree) as above
 *   path         device int32 [B][path_stride]: accepted node indices (rows of k_tree / v_tree)
 *                in path order, e.g. hta_accept_greedy's `path` (path_stride = T)
 *   path_len     device int32 [B]: accepted nodes of batch b (<= 0: nothing to commit)
 *   k_tree, v_tree  [B, T, H_kv, d] (read);  k_cache, v_cache [B, N_max, H_kv, d] (written at
 *                rows cache_seqlens[b] ... cache_seqlens[b] + path_len[b] - 1 only)
 *   cache_seqlens   device int32 [B]: committed length n_b before the call (read; a negative
 *                value counts as 0)
 *   seqlens_out     device int32 [B]: n_b + the rows written (may be cache_seqlens itself: the
 *                update is made after the copies).  Rows that would land at or beyond N_max, and
 *                everything from the first node index outside [0, T) on, are not written and not
 *                counted (reading Z18).
 * k_tree / v_tree must not overlap the cache rows being written (the copies run in parallel).
 * Enqueued on `stream`; one CTA per batch entry.  Host-checkable errors as for hta_forward. */
hta_status_t hta_commit_kv(const hta_shape_t *shape, const int32_t *path, int64_t path_stride,
                           const int32_t *path_len, const void *k_tree, const void *v_tree,
                           void *k_cache, void *v_cache, const int32_t *cache_seqlens,
                           int32_t *seqlens_out, hta_stream_t stream);

/* ---------------------------------------------------------------- sequence parallel
 * The prefix KV is split contiguously along the sequence across P ranks (one process per
 * GPU); rank r holds KV[:, r*N/P : (r+1)*N/P].  Each rank runs the prefix pass on its slice,
 * the partials are exchanged with one NCCL all-to-all of head slices over NVLink, and each
 * rank merges the P prefix partials with the tree partial for its H/P heads.  Exactness is
 * the Appendix C identity applied P+1 ways.  The paper itself runs on one GPU
 * (P:890); this exchange is an addition of this build. */
typedef struct hta_comm_s *hta_comm_t;

/* Fill the 128-byte NCCL unique id (host buffer) on one rank; the caller broadcasts it to the
 * other ranks (e.g. with torch.distributed) before hta_comm_create. */
hta_status_t hta_comm_unique_id(void *unique_id_128);
/* Create the communicator for `nranks` ranks on the current CUDA device. Collective. */
hta_status_t hta_comm_create(const void *unique_id_128, int32_t nranks, int32_t rank,
                             hta_comm_t *comm);
hta_status_t hta_comm_destroy(hta_comm_t comm);

/* Loopback communicator: `nranks` VIRTUAL ranks held by this one process on the current device
 * (no NCCL).  It drives hta_forward_seqpar_loopback, which runs every rank's phases of the
 * sequence-parallel step (local prefix pass into destination-major blocks, the all-to-all of
 * head slices -- here device-to-device copies --, the P-way merge with the tree pass at rank r's
 * head offset r*H/P, the optional all-gather) on one GPU.  It exists so that the P > 1 data
 * path can be checked against the oracle where only one GPU is available.  1 <= nranks <= 64. */
hta_status_t hta_comm_create_loopback(int32_t nranks, hta_comm_t *comm);

/* HTA_OK, or HTA_ERR_NCCL if NCCL reported an asynchronous error on this communicator
 * (ncclCommGetAsyncError; e.g. a peer failed during an earlier step).  hta_forward_seqpar checks
 * it before enqueueing.  A loopback communicator always returns HTA_OK. */
hta_status_t hta_comm_async_error(hta_comm_t comm);

/* Peer-memory exchange for the sequence-parallel step (the fused compute +
 * collective path over NVLink / NVSwitch).  Instead of the NCCL all-to-all, the split-combine
 * kernel of rank r writes head block q of its prefix partial straight into rank q's receive
 * buffer (P2P stores over NVLink to an IPC-mapped allocation), one signal kernel fences at system
 * scope and raises rank r's flag in every peer's flag array, and the final merge waits for all P
 * flags of its step.  Receive buffers are double-buffered by a device-side step counter, so the
 * step can be captured in a CUDA graph and replayed.  Used by hta_forward_seqpar[_tree] (and the
 * loopback forward) whenever it is enabled, gather_output is 0 and the step's block fits the
 * capacity; otherwise the NCCL path runs.
 *   hta_comm_p2p_alloc: allocate this rank's buffers on the current device for blocks of at most
 *     block_capacity_floats floats (B*T*(H/P)*d + B*(H/P)*T for the shapes to be run), and write
 *     its two CUDA IPC handles (receive buffer, flags; 64 bytes each) to ipc_handles_128.  For a
 *     loopback communicator it allocates every virtual rank's buffers, wires them to each other
 *     and enables the exchange at once (the handles are zeroed).
 *   hta_comm_p2p_open: ipc_handles_all = the nranks ranks' 128-byte handles in rank order (e.g.
 *     all-gathered over the process group); opens the peers' buffers and enables the exchange.
 * At most 8 ranks (one NVSwitch node): HTA_ERR_UNSUPPORTED beyond.  Errors leave the exchange
 * disabled (HTA_ERR_CUDA: an allocation, IPC export or IPC open failed). */
hta_status_t hta_comm_p2p_alloc(hta_comm_t comm, size_t block_capacity_floats, void *ipc_handles_128);
hta_status_t hta_comm_p2p_open(hta_comm_t comm, const void *ipc_handles_all);
/* Switch an allocated and opened peer-memory exchange off (0: the NCCL exchange runs) or on. */
hta_status_t hta_comm_p2p_set(hta_comm_t comm, int32_t enabled);
/* HTA_OK, or HTA_ERR_CUDA once a final merge gave up waiting (100 ms) for a peer's flag (a peer
 * that never signals must not hang the step; that step's output is garbage).  Synchronous (reads
 * a device word). */
hta_status_t hta_comm_p2p_error(hta_comm_t comm);

/* Workspace for hta_forward_seqpar: split partials + send/receive buffers. */
size_t hta_workspace_size_seqpar(const hta_shape_t *shape_local, int32_t num_sms,
                                 int32_t nranks);

/* One verification-attention step with the prefix sharded over the communicator's ranks.
 *   shape_local         N_max = this rank's KV-slice capacity; H must be divisible by nranks
 *   k_cache_local, v_cache_local, cache_seqlens_local   this rank's slice and its valid length
 *   q, k_tree, v_tree, mask   replicated on every rank
 *   o   [B, T, H/P, d] (heads [r*H/P, (r+1)*H/P)) when gather_output == 0, else [B, T, H, d];
 *       contiguous, shape->dtype.  lse_out optional, same head extent, float32 [B, Hx, T].
 * Collective: every rank must call it with the same shape, on its own stream. */
hta_status_t hta_forward_seqpar(hta_comm_t comm, const hta_shape_t *shape_local, const void *q,
                                const void *k_cache_local, const void *v_cache_local,
                                const int32_t *cache_seqlens_local, const void *k_tree,
                                const void *v_tree, const uint8_t *mask,
                                int64_t mask_batch_stride, void *o, float *lse_out,
                                int32_t gather_output, void *ws, size_t ws_bytes,
                                hta_stream_t stream);

/* hta_forward_seqpar with the tree given by its parent array instead of a mask (as
 * hta_forward_tree: each row's visible tree keys derived in the final merge by walking the
 * parent links, bit-identical to the mask hta_build_tree_mask writes), so the mask build can
 * run beside the step.  parents: device int32 [B][T] (parents_batch_stride apart; 0 = shared).
 * Other arguments, layout, ownership and errors as hta_forward_seqpar. */
hta_status_t hta_forward_seqpar_tree(hta_comm_t comm, const hta_shape_t *shape_local, const void *q,
                                     const void *k_cache_local, const void *v_cache_local,
                                     const int32_t *cache_seqlens_local, const void *k_tree,
                                     const void *v_tree, const int32_t *parents,
                                     int64_t parents_batch_stride, void *o, float *lse_out,
                                     int32_t gather_output, void *ws, size_t ws_bytes,
                                     hta_stream_t stream);

/* hta_forward_seqpar for all ranks of a loopback communicator at once, on `stream` of the
 * current device.  Per-rank arguments are HOST arrays of `nranks` DEVICE pointers:
 *   k_cache_local[r], v_cache_local[r], cache_seqlens_local[r] (the array itself may be NULL:
 *   full slices)   rank r's KV slice, as for hta_forward_seqpar on rank r
 *   o[r], lse_out[r] (lse_out may be NULL)   rank r's outputs (head slice r, or all heads when
 *   gather_output)
 *   ws, ws_bytes   nranks x the 16-byte rounded hta_workspace_size_seqpar(shape_local, ...)
 * q, k_tree, v_tree and mask are shared by the ranks (they are replicated in the real step).
 * The per-rank computation is the same code as hta_forward_seqpar's; only the exchange is a
 * local copy instead of NCCL.  Errors: as hta_forward_seqpar; HTA_ERR_INVALID_ARGUMENT for an
 * NCCL communicator. */
hta_status_t hta_forward_seqpar_loopback(hta_comm_t comm, const hta_shape_t *shape_local,
                                         const void *q, const void *const *k_cache_local,
                                         const void *const *v_cache_local,
                                         const int32_t *const *cache_seqlens_local,
                                         const void *k_tree, const void *v_tree,
                                         const uint8_t *mask, int64_t mask_batch_stride,
                                         void *const *o, float *const *lse_out,
                                         int32_t gather_output, void *ws, size_t ws_bytes,
                                         hta_stream_t stream);

#ifdef __cplusplus
}
#endif
#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#endif /* HTA_H_ */
