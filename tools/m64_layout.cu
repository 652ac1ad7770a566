// m64_layout.cu -- diagnostics: where the rows of a tcgen05.mma.cta_group::1 accumulator land in
// TMEM for M = 64 (and M = 128 for reference), and whether an M = 64 "TS" MMA (A from TMEM) reads
// its A rows from the same lanes.  A[r][0] = r + 1 (bf16, K-major SWIZZLE_128B), B[n][0] = 1, so
// D[r][n] = r + 1; every warp then reads column 0 of its lane quarter.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/m64_layout.cu -o /tmp/m64 && /tmp/m64
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2502_17421_b200/csrc/ptx_sm100.cuh"

using namespace hta;

__device__ __forceinline__ uint32_t tmem_ld1(uint32_t taddr) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n\ttcgen05.wait::ld.sync.aligned;"
                 : "=r"(v)
                 : "r"(taddr)
                 : "memory");
    return v;
}

template <int M>
__global__ void layout_kernel(float *out, float *out_ts) {
    __shared__ __align__(1024) uint8_t sA[128 * 128];
    __shared__ __align__(1024) uint8_t sB[32 * 128];
    __shared__ __align__(1024) uint8_t sI[64 * 128];  // 64 x 64 identity (B of the TS check)
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 128 * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sA)[i] = 0u;
    for (int i = tid; i < 32 * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sB)[i] = 0u;
    for (int i = tid; i < 64 * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sI)[i] = 0u;
    __syncthreads();
    // element (row, k) of a K-major SW128 tile with 64 bf16 per row: row*128 + ((k/8) ^ (row%8))*16 + (k%8)*2
    auto at = [](uint8_t *base, int row, int k) {
        return reinterpret_cast<__nv_bfloat16 *>(base + row * 128 + (((k / 8) ^ (row % 8)) << 4) + (k % 8) * 2);
    };
    if (tid < M) *at(sA, tid, 0) = __float2bfloat16(static_cast<float>(tid + 1));
    if (tid < 32) *at(sB, tid, 0) = __float2bfloat16(1.0f);
    if (tid < 64) *at(sI, tid, tid) = __float2bfloat16(1.0f);  // identity: I[n][k] = (n == k)
    fence_proxy_async_smem();
    if (warp == 0) {
        tmem_alloc(&tslot, 128);
        tmem_relinquish();
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (tid == 0) {
        const uint64_t ad = sdesc_sw128(smem_u32(sA), 16, 1024);
        const uint64_t bd = sdesc_sw128(smem_u32(sB), 16, 1024);
        mma_bf16_ss(tmem, ad, bd, idesc_bf16_f32(M, 32, 0), 0u);
        tc_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    // column 0 of this warp's lane quarter
    out[warp * 32 + lane] = __uint_as_float(tmem_ld1(tmem + (static_cast<uint32_t>(warp * 32) << 16)));
    // TS check: A = the D just computed, packed to bf16 pairs at column 96 by its own lanes (col
    // 96 + i holds keys 2i, 2i+1: key 0 = r + 1, others 0), times B = identity (N = 64 keys as K)
    // -> E[r][n] = A[r][n]; E[r][0] = r + 1 if the TS MMA reads A rows from the D lanes
    {
        float v = __uint_as_float(tmem_ld1(tmem + (static_cast<uint32_t>(warp * 32) << 16)));
        uint32_t w[8] = {pack_bf16x2(v, 0.f), 0u, 0u, 0u, 0u, 0u, 0u, 0u};
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n\ttcgen05.wait::st.sync.aligned;" ::"r"(
                tmem + (static_cast<uint32_t>(warp * 32) << 16) + 96u),
            "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
            : "memory");
        for (int c = 1; c < 4; ++c) {  // columns 104.. of the A tile (keys 16..63): zero
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};\n\ttcgen05.wait::st.sync.aligned;" ::"r"(
                    tmem + (static_cast<uint32_t>(warp * 32) << 16) + 96u + 8u * c),
                "r"(0u)
                : "memory");
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
        const uint64_t id = sdesc_sw128(smem_u32(sI), 16, 1024);
        for (int k = 0; k < 4; ++k)  // K = 64 keys in 4 steps of 16 (A from TMEM: 8 columns per step)
            mma_bf16_ts(tmem + 32u, tmem + 96u + 8u * k, id + static_cast<uint32_t>((k * 32) >> 4),
                        idesc_bf16_f32(M, 64, 0), k > 0 ? 1u : 0u);
        tc_commit(&bar);
    }
    mbar_wait(&bar, 1);
    tc_fence_after();
    out_ts[warp * 32 + lane] = __uint_as_float(tmem_ld1(tmem + (static_cast<uint32_t>(warp * 32) << 16) + 32u));
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 128);
    }
}

template <int M>
void run() {
    float *d, *d2, h[128], h2[128];
    cudaMalloc(&d, 512);
    cudaMalloc(&d2, 512);
    layout_kernel<M><<<1, 128>>>(d, d2);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 512, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2, d2, 512, cudaMemcpyDeviceToHost);
    printf("M = %d (%s): TMEM lane -> accumulator row (0 = none)\n", M, cudaGetErrorString(e));
    for (int q = 0; q < 4; ++q) {
        printf("  lanes %3d..%3d:", 32 * q, 32 * q + 31);
        for (int l = 0; l < 32; ++l) printf(" %g", h[32 * q + l] - 1.0f + 1.0f > 0 ? h[32 * q + l] - 1 : -1.0f);
        printf("\n");
    }
    printf("  TS MMA (A from these lanes) -> row + 1 read back:");
    for (int l = 0; l < 128; ++l) printf(" %g", h2[l]);
    printf("\n");
}

int main() {
    run<64>();
    run<128>();
    return 0;
}
