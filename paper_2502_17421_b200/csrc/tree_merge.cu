// tree_merge.cu -- the tree pass and the LSE merge as a kernel of their own (one warp per
// output row): hta_tree_attn, hta_merge_lse, the sequence-parallel final merge, and the second
// kernel of hta_forward.  The row-level
// device functions are in tree_pass.cuh.
#include "tree_pass.cuh"

namespace hta {

constexpr uint64_t kP2pTimeoutNs = 100000000ull;  // 100 ms: a step takes well under 1 ms


#ifndef HTA_TM_WARPS
#define HTA_TM_WARPS 1
#endif
constexpr int kTmWarps = HTA_TM_WARPS;  // warps (= rows) per block
// One warp per row; small blocks of at most 128 registers per thread, so that blocks fit beside
// the prefix kernel's CTAs and start (programmatic dependent launch) during its epilogue.
template <typename Tin, typename Tout, int D>
__global__ void __launch_bounds__(32 * kTmWarps, 16 / kTmWarps) tree_merge_kernel(const TreeMergeParams p) {
    constexpr int E = D / 32;
    const int row = blockIdx.x * kTmWarps + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= p.B * p.T * p.Hr) return;
    const int hl = row % p.Hr, t = (row / p.Hr) % p.T, b = row / (p.Hr * p.T);
    // tree pass: before griddepcontrol.wait, so it overlaps the tail of the prefix kernel
    float ot[E];
    float lse_t = -INFINITY;
#pragma unroll
    for (int e = 0; e < E; ++e) ot[e] = 0.f;
    if (p.do_tree) lse_t = tree_row<Tin, D>(p, b, t, p.h0 + hl, lane, ot);
    if (p.n_parts > 0) pdl_wait_primary();  // the partials come from the preceding prefix kernel
    if (p.p2p_role == 2) {
        // peer-memory exchange: every rank's block of this step has landed in the receive buffer
        // once its flag reached this rank's step counter; lane q acquires flag q (all at once), the
        // warp barrier then orders every lane's loads below after those acquires
        const uint32_t e = *p.p2p_epoch;
        if (lane < p.n_parts) {
            // a peer that never signals (a broken peer mapping) must not hang the step: after
            // kP2pTimeoutNs the wait gives up and records the failure in the error word
            // (hta_comm_p2p_error; the result of that step is garbage)
            const uint64_t t0 = global_ns();
            while (ld_acquire_sys(p.p2p_flags + lane) < e)
                if (global_ns() - t0 > kP2pTimeoutNs) {
                    atomicExch(const_cast<uint32_t *>(p.p2p_flags) + p.n_parts + 2, 1u);
                    break;
                }
        }
        __syncwarp();
    }
    const bool signal = p.p2p_role == 1;
    const uint32_t e0 = signal ? *p.p2p_epoch : 0u;  // (read before any block can advance it)
    merge_row<Tout, D, false>(p, b, t, hl, lane, ot, lse_t);
    if (signal) {
        // peer-memory exchange, split combine: the block that finishes last (the block counter
        // reaches the grid size) fences at system scope, raises this rank's flag in every rank's
        // flag array, advances the step counter and re-arms the block counter for the next step;
        // the warp barrier and the counter's atomics order every block's stores before that fence
        __syncwarp();
        if (lane == 0) {
            __threadfence();
            if (atomicAdd(p.p2p_counter, 1u) + 1u == gridDim.x) {
                __threadfence_system();
                for (int q = 0; q < p.p2p_nranks; ++q) st_release_sys(p.p2p_peer_flags[q] + p.p2p_rank, e0 + 1u);
                atomicExch(const_cast<uint32_t *>(p.p2p_epoch), e0 + 1u);
                atomicExch(p.p2p_counter, 0u);
            }
        }
    }
}

template <typename Tin, typename Tout, int D>
static cudaError_t launch_tm_d(const TreeMergeParams &p, bool pdl, cudaStream_t s) {
    const int rows = p.B * p.T * p.Hr;
    if (rows == 0) return cudaSuccess;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((rows + kTmWarps - 1) / kTmWarps);
    cfg.blockDim = dim3(32 * kTmWarps);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, tree_merge_kernel<Tin, Tout, D>, p);
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

