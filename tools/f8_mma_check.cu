// f8_mma_check.cu -- diagnostics: one tcgen05.mma kind::f8f6f4 chain (M = 128, N = 128, K = 128 as
// four K = 32 steps) over E4M3 A and B tiles in the K-major SWIZZLE_128B layout (128-byte rows),
// as the FP8-cache prefix kernel issues S = q K^T; the TMEM result is compared with the exact
// product on the host.  Small-integer operands, so every product and sum is exact in fp32.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/f8_mma_check.cu -o /tmp/f8c && /tmp/f8c
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <vector>

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

__host__ __device__ inline int aval(int r, int k) { return (r * 7 + k * 3) % 5 - 2; }
__host__ __device__ inline int bval(int n, int k) { return (n * 5 + k) % 3 - 1; }

__global__ void check_kernel(float *out, int *status, int pair_layout) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *sA = sm;              // 128 rows x 128 B
    uint8_t *sB = sm + 128 * 128;  // 128 rows x 128 B
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5;
    // element (row, k) of a K-major SW128 tile with 128 E4M3 per row: row*128 + ((k/16) ^ (row%8))*16 + k%16
    for (int i = tid; i < 128 * 128; i += blockDim.x) {
        const int r = i / 128, k = i % 128;
        const int off = r * 128 + (((k / 16) ^ (r % 8)) << 4) + k % 16;
        sA[off] = static_cast<uint8_t>(f32x2_to_e4m3x2(static_cast<float>(aval(r, k)), 0.f) & 0xFF);
        sB[off] = static_cast<uint8_t>(f32x2_to_e4m3x2(static_cast<float>(bval(r, k)), 0.f) & 0xFF);
    }
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
        for (int k = 0; k < 4; ++k)
            mma_e4m3_ss(tmem, ad + ((k * 32) >> 4), bd + ((k * 32) >> 4), idesc_e4m3_f32(128, 128), k > 0 ? 1u : 0u);
        tc_commit(&bar);
    }
    // bounded wait: report a hang instead of trapping
    const long long t0 = clock64();
    bool ok = false;
    while (clock64() - t0 < 2000000000LL) {
        if (mbar_try_wait(smem_u32(&bar), 0)) {
            ok = true;
            break;
        }
    }
    if (!ok) {
        if (tid == 0) *status = 1;
        return;
    }
    tc_fence_after();
    const int row = warp * 32 + (tid & 31);
    for (int n = 0; n < 128; ++n)
        out[row * 128 + n] = __uint_as_float(tmem_ld1(tmem + (static_cast<uint32_t>(warp * 32) << 16) + n));
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 128);
}

int main() {
    float *d_out;
    int *d_st;
    cudaMalloc(&d_out, 128 * 128 * 4);
    cudaMalloc(&d_st, 4);
    cudaMemset(d_st, 0, 4);
    cudaFuncSetAttribute(check_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 128 * 128);
    check_kernel<<<1, 128, 2 * 128 * 128>>>(d_out, d_st, 0);
    cudaError_t e = cudaDeviceSynchronize();
    int st = -1;
    cudaMemcpy(&st, d_st, 4, cudaMemcpyDeviceToHost);
    std::vector<float> h(128 * 128);
    cudaMemcpy(h.data(), d_out, h.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    double maxerr = 0;
    for (int r = 0; r < 128; ++r)
        for (int n = 0; n < 128; ++n) {
            int ref = 0;
            for (int k = 0; k < 128; ++k) ref += aval(r, k) * bval(n, k);
            const double err = std::fabs(h[r * 128 + n] - ref);
            maxerr = err > maxerr ? err : maxerr;
            if (err > 0 && bad++ < 5) std::printf("  D[%d][%d] = %g, want %d\n", r, n, h[r * 128 + n], ref);
        }
    std::printf("f8f6f4 E4M3 M128 N128 K128: %s, status %d (1 = hang), %d wrong, max err %g\n", cudaGetErrorString(e),
                st, bad, maxerr);
    return bad == 0 && st == 0 && e == cudaSuccess ? 0 : 1;
}
