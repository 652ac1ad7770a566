// sync_lat.cu -- diagnostics: latency of the synchronisation paths the prefix kernel relies on:
// (1) tcgen05.mma x8 + tcgen05.commit -> mbarrier wait observed by another warp (single CTA and
// CTA pair with multicast commit), (2) remote mbarrier arrive from the peer CTA -> leader wait.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude tools/sync_lat.cu -o /tmp/sync_lat
#include <cuda_runtime.h>

#include <cstdio>

#include "ptx_extra.cuh"

using namespace hta;

template <bool PAIR, int NMMA>
__global__ void __launch_bounds__(128, 1) lat_kernel(int reps, long long *out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 65536);
    uint64_t *back = bar + 1;
    uint32_t *tslot = reinterpret_cast<uint32_t *>(bar + 2);
    volatile long long *stamp = reinterpret_cast<volatile long long *>(bar + 4);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_init(back, PAIR ? 2 : 1);
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
    const uint32_t back0 = PAIR ? mapa_shared(smem_u32(back), 0) : smem_u32(back);
    long long sum_commit = 0, sum_round = 0;
    if (warp == 0 && rank == 0) {
        const uint32_t base = smem_u32(smem);
        const uint32_t idesc = idesc_bf16_f32(PAIR ? 256 : 128, 128, 0);
        const uint64_t ad = sdesc_sw128(base, 16, 1024), bd = sdesc_sw128(base + 32768, 16, 1024);
        for (int i = 0; i < reps; ++i) {
            const long long t0 = clock64();
            for (int k = 0; k < NMMA; ++k) {
                if (PAIR) mma2_bf16_ss_elect(tmem, ad + 2 * k, bd + 2 * k, idesc, 1u);
                else mma_bf16_ss_elect(tmem, ad + 2 * k, bd + 2 * k, idesc, 1u);
            }
            if (PAIR) tc_commit2_mc_elect(bar); else tc_commit_elect(bar);
            if (lane == 0) stamp[0] = t0;
            // the "consumer" warps observe the commit and answer on `back`
            mbar_wait(back, i & 1);
            const long long t2 = clock64();
            sum_round += t2 - t0;
        }
        if (lane == 0) {
            out[blockIdx.x * 4 + 0] = sum_round / reps;
        }
    } else if (warp == 2) {
        // consumer in each CTA: wait for the MMA commit, then arrive on the leader's `back`
        for (int i = 0; i < reps; ++i) {
            mbar_wait(bar, i & 1);
            const long long t1 = clock64();
            if (rank == 0) sum_commit += t1 - stamp[0];
            tc_fence_after();
            __syncwarp();
            if (lane == 0) {
                if (PAIR) mbar_arrive_remote(back0); else mbar_arrive(back);
            }
        }
        if (lane == 0 && rank == 0) out[blockIdx.x * 4 + 1] = sum_commit / reps;
    }
    __syncthreads();
    if (PAIR) cluster_sync();
    if (warp == 1) { if (PAIR) tmem_dealloc2(tmem, 512); else tmem_dealloc(tmem, 512); }
}

template <bool PAIR, int NMMA>
void run(const char *name) {
    auto kern = lat_kernel<PAIR, NMMA>;
    const int smem = 65536 + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    long long *out;
    cudaMalloc(&out, 148 * 4 * 8);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(PAIR ? 2 : 1);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = PAIR ? 2 : 1; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, 200, out);
    cudaDeviceSynchronize();
    long long h[4];
    cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
    printf("%-28s %d MMA: issue->commit observed %lld cyc, full round trip (MMA, commit, consumer arrive, wait) %lld cyc %s\n",
           name, NMMA, h[1], h[0], cudaGetErrorString(cudaGetLastError()));
}

int main() {
    run<false, 1>("single");
    run<false, 8>("single");
    run<true, 1>("pair (multicast commit)");
    run<true, 8>("pair (multicast commit)");
    return 0;
}
