// mma_rate.cu -- diagnostics: sustained tcgen05.mma throughput for the instruction shapes the
// prefix kernel issues (kind::f16 bf16 -> fp32, M = 128 or 256 (pair), N = 128, K = 16), with
// A from smem (SS) or TMEM (TS), and a commit every `per_commit` instructions.  Operands are
// whatever sits in smem/TMEM (timing only).  Build & run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude tools/mma_rate.cu -o /tmp/mma_rate
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "ptx_extra.cuh"

using namespace hta;

template <bool PAIR, bool TS, int N, bool W = false, int PW = 0>
__global__ void __launch_bounds__(320, 1) mma_kernel(int iters, int per_commit, int b_mn_major, unsigned long long *cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 65536);
    uint64_t *fin = bar + 1;
    uint32_t *tslot = reinterpret_cast<uint32_t *>(bar + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_init(fin, 1);
        fence_mbar_init();
    }
    if (warp == 1) {
        if (PAIR) {
            tmem_alloc2(tslot, 512);
            tmem_relinquish2();
        } else {
            tmem_alloc(tslot, 512);
            tmem_relinquish();
        }
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    volatile __shared__ int stop_flag;
    if (threadIdx.x == 0) stop_flag = 0;
    __syncthreads();
    if (PW > 0 && warp >= 2 && warp < 2 + PW) {
        // TMEM pressure: S-like loads of 64 columns per thread + P-like stores, as the softmax does
        const int q = warp & 3;
        const uint32_t lane_off = static_cast<uint32_t>(q * 32 + ((warp - 2) >> 2) * 16) << 16;
        float acc = 0.f;
        for (int it = 0; it < 4000 && !stop_flag; ++it) {
            float v[64];
            tmem_ld_16x64_split64(tmem + lane_off + 256, v);
            uint32_t pk[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) pk[i] = __float_as_uint(v[2 * i] + v[2 * i + 1] + acc);
            tmem_st_16x32_split<32>(tmem + lane_off + 320, pk);
            acc += v[5];
        }
        if (acc == 1.2345f) cycles[1] = 1;
    }
    if (W && warp == 0 && rank == 0) {
        // warp-converged issue with descriptors precomputed once and bumped by constants
        const uint32_t base = smem_u32(smem);
        const uint32_t idesc = idesc_bf16_f32(PAIR ? 256 : 128, N, b_mn_major);
        const uint64_t bd0 = sdesc_sw128(base + 32768, b_mn_major ? 16384 : 16, 1024);
        const uint64_t ad0 = sdesc_sw128(base, 16, 1024);
        const unsigned long long t0 = clock64();
        for (int i = 0; i < iters; i += 8) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint64_t bd = bd0 + 2u * k;  // +32 bytes (>> 4) along K inside the swizzle atom
                if (TS) {
                    if (PAIR)
                        mma2_bf16_ts_elect(tmem + (N == 256 ? 256 : 384), tmem + k * 8, bd, idesc, 1u);
                    else
                        mma_bf16_ts_elect(tmem + (N == 256 ? 256 : 384), tmem + k * 8, bd, idesc, 1u);
                } else {
                    if (PAIR)
                        mma2_bf16_ss_elect(tmem + (N == 256 ? 0 : 128 * (k & 1)), ad0 + 2u * k, bd, idesc, 1u);
                    else
                        mma_bf16_ss_elect(tmem + (N == 256 ? 0 : 128 * (k & 1)), ad0 + 2u * k, bd, idesc, 1u);
                }
            }
            if (per_commit <= 8 || ((i / 8) % (per_commit / 8)) == 0) {
                if (PAIR)
                    tc_commit2_mc_elect(bar);
                else
                    tc_commit_elect(bar);
            }
        }
        if (PAIR)
            tc_commit2_mc_elect(fin);
        else
            tc_commit_elect(fin);
        mbar_wait(fin, 0);
        const unsigned long long t1 = clock64();
        if (lane == 0) cycles[blockIdx.x * 2] = t1 - t0;
        stop_flag = 1;
    } else if (!W && warp == 0 && rank == 0 && lane == 0) {
        const uint32_t base = smem_u32(smem);
        const uint32_t idesc = idesc_bf16_f32(PAIR ? 256 : 128, N, b_mn_major);
        const unsigned long long t0 = clock64();
        uint32_t phase = 0;
        int since = 0;
        for (int i = 0; i < iters; ++i) {
            const int k = i & 7;
            const uint64_t bd = sdesc_sw128(base + 32768 + k * 32, b_mn_major ? 16384 : 16, 1024);
            if (TS) {
                if (PAIR)
                    mma2_bf16_ts(tmem + (N == 256 ? 256 : 384), tmem + k * 8, bd, idesc, 1u);
                else
                    mma_bf16_ts(tmem + (N == 256 ? 256 : 384), tmem + k * 8, bd, idesc, 1u);
            } else {
                const uint64_t ad = sdesc_sw128(base + k * 32, 16, 1024);
                if (PAIR)
                    mma2_bf16_ss(tmem + (N == 256 ? 0 : 128 * (i % 3 == 0 ? 0 : 1)), ad, bd, idesc, 1u);
                else
                    mma_bf16_ss(tmem + (N == 256 ? 0 : 128 * (i % 3 == 0 ? 0 : 1)), ad, bd, idesc, 1u);
            }
            if (++since == per_commit) {
                since = 0;
                if (PAIR)
                    tc_commit2_mc(bar);
                else
                    tc_commit(bar);
                // keep at most ~4 groups in flight (like the kernel's barriers would)
            }
        }
        if (PAIR)
            tc_commit2_mc(fin);
        else
            tc_commit(fin);
        (void)phase;
        mbar_wait(fin, 0);  // all MMAs done
        const unsigned long long t1 = clock64();
        cycles[blockIdx.x * 2] = t1 - t0;
    }
    if (PAIR && rank == 1 && threadIdx.x == 0) mbar_wait(fin, 0);  // multicast commit reached us too
    __syncthreads();
    if (PAIR) cluster_sync();
    if (warp == 1) {
        if (PAIR)
            tmem_dealloc2(tmem, 512);
        else
            tmem_dealloc(tmem, 512);
    }
}

template <bool PAIR, bool TS, int N = 128, bool W = false, int PW = 0>
void run(const char *name, int per_commit, int mn) {
    auto kern = mma_kernel<PAIR, TS, N, W, PW>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
    unsigned long long *cyc;
    cudaMalloc(&cyc, 148 * 2 * 8);
    const int iters = 8 * 2000;
    const int grid = 148;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(320);
    cfg.dynamicSmemBytes = 65536 + 1024;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = PAIR ? 2 : 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9;
    for (int it = 0; it < 4; ++it) {
        cudaEventRecord(e0);
        cudaLaunchKernelEx(&cfg, kern, iters, per_commit, mn, cyc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it > 0 && ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    // FLOPs: per SM, each instruction is 128 x 128 x 16 MACs
    const double flops = 2.0 * 128 * N * 16 * double(iters) * grid;
    unsigned long long c0;
    cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-34s N%-3d commit/%-3d %8.1f us %7.1f TFLOP/s  %6.1f SM-cycles/instr  (implied clock %.2f GHz)%s\n", name, N,
           per_commit, best * 1e3, flops / (best * 1e-3) / 1e12, double(c0) / iters, double(c0) / (best * 1e-3) / 1e9,
           err == cudaSuccess ? "" : cudaGetErrorString(err));
}


// The prefix kernel's exact MMA stream for one pair: per tile S (SS, 8 x K16 into buffer j%3)
// then PV (TS, 8 x K16 reading P from buffer (j-2)%3, into O), four commits per tile, no waits.
template <bool PAIR>
__global__ void __launch_bounds__(64, 1) seq_kernel(int tiles, unsigned long long *cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 65536 + 65536);
    uint64_t *fin = bar + 8;
    uint32_t *tslot = reinterpret_cast<uint32_t *>(bar + 9);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 9; ++i) mbar_init(&bar[i], 1);
        fence_mbar_init();
    }
    if (warp == 1) {
        if (PAIR) { tmem_alloc2(tslot, 512); tmem_relinquish2(); } else { tmem_alloc(tslot, 512); tmem_relinquish(); }
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    if (warp == 0 && rank == 0) {
        const uint32_t base = smem_u32(smem);
        const uint32_t idesc_qk = idesc_bf16_f32(PAIR ? 256 : 128, 128, 0);
        const uint32_t idesc_pv = idesc_bf16_f32(PAIR ? 256 : 128, 128, 1);
        const uint64_t qd0 = sdesc_sw128(base, 16, 1024);
        const uint64_t kd0 = sdesc_sw128(base + 32768, 16, 1024);
        const uint64_t vd0 = sdesc_sw128(base + 65536, 128 * 128, 1024);
        const unsigned long long t0 = clock64();
        for (int j = 0; j < tiles; ++j) {
            const int buf = j % 3;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t qo = ((k / 4) * 16384 + (k % 4) * 32) >> 4;
                const uint32_t ko = ((k / 4) * 8192 + (k % 4) * 32) >> 4;
                if (PAIR) mma2_bf16_ss_elect(tmem + 128 * buf, qd0 + qo, kd0 + ko, idesc_qk, k > 0);
                else mma_bf16_ss_elect(tmem + 128 * buf, qd0 + qo, kd0 + ko, idesc_qk, k > 0);
            }
            if (PAIR) { tc_commit2_mc_elect(&bar[buf]); tc_commit2_mc_elect(&bar[3]); }
            else { tc_commit_elect(&bar[buf]); tc_commit_elect(&bar[3]); }
            const int pb = (j + 1) % 3;  // PV of tile j-2
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (PAIR) mma2_bf16_ts_elect(tmem + 384, tmem + 128 * pb + k * 8, vd0 + k * 128, idesc_pv, 1u);
                else mma_bf16_ts_elect(tmem + 384, tmem + 128 * pb + k * 8, vd0 + k * 128, idesc_pv, 1u);
            }
            if (PAIR) { tc_commit2_mc_elect(&bar[4 + pb]); tc_commit2_mc_elect(&bar[7]); }
            else { tc_commit_elect(&bar[4 + pb]); tc_commit_elect(&bar[7]); }
        }
        if (PAIR) tc_commit2_mc_elect(fin); else tc_commit_elect(fin);
        mbar_wait(fin, 0);
        const unsigned long long t1 = clock64();
        if (lane == 0) cycles[0] = t1 - t0;
    }
    if (PAIR && rank == 1 && threadIdx.x == 0) mbar_wait(fin, 0);
    __syncthreads();
    if (PAIR) cluster_sync();
    if (warp == 1) { if (PAIR) tmem_dealloc2(tmem, 512); else tmem_dealloc(tmem, 512); }
}

template <bool PAIR>
void run_seq(const char *name) {
    auto kern = seq_kernel<PAIR>;
    const int smem = 65536 * 2 + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long *cyc;
    cudaMalloc(&cyc, 64);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(64);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = PAIR ? 2 : 1; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr; cfg.numAttrs = 1;
    const int tiles = 1000;
    for (int it = 0; it < 3; ++it) cudaLaunchKernelEx(&cfg, kern, tiles, cyc);
    cudaDeviceSynchronize();
    unsigned long long c0;
    cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-40s %7.1f SM-cycles per tile (S + PV; 1024 = full rate) %s\n", name, double(c0) / tiles,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    run_seq<true>("kernel MMA sequence, pair");
    run_seq<false>("kernel MMA sequence, single");
    run<true, false, 128, true, 0>("WARP pair SS M256, no pressure", 8, 0);
    run<true, true, 128, true, 0>("WARP pair TS M256, no pressure", 8, 1);
    run<true, false, 128, true, 8>("WARP pair SS M256, 8 TMEM warps", 8, 0);
    run<true, true, 128, true, 8>("WARP pair TS M256, 8 TMEM warps", 8, 1);
    run<true, true, 128, true, 4>("WARP pair TS M256, 4 TMEM warps", 8, 1);
    run<false, true, 128, true, 8>("WARP single TS M128, 8 TMEM warps", 8, 1);
    // the transposed FP8 kernel's shapes (prefix_t8.cu): N = 64 query rows
    run<false, false, 64, true, 0>("WARP single SS M128 N64", 8, 0);
    run<false, false, 64, true, 0>("WARP single SS M128 N64 B MN-major", 8, 1);
    run<false, true, 64, true, 0>("WARP single TS M128 N64", 8, 0);
    run<false, false, 128, true, 0>("WARP single SS M128 N128", 8, 0);
    run<false, true, 128, true, 0>("WARP single TS M128 N128", 8, 0);
    run<false, false, 256, true, 0>("WARP single SS M128 N256", 8, 0);
    return 0;
}
