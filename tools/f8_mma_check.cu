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

// TS form as the FP8 PV step would issue it: A = P (128 rows x 128 keys, 8-bit, format AF) in
// TMEM (4 keys per 32-bit column, row r in lane r), B = V (128 keys x 128 columns, E4M3) MN-major
// SWIZZLE_128B in shared memory (the layout TMA lands a [keys][128 B] box in), four K = 32 steps.
__host__ __device__ inline int pval(int r, int k) { return (r + 3 * k) % 4; }        // 0..3
__host__ __device__ inline int vval(int k, int n) { return (k * 5 + n * 3) % 5 - 2; }  // -2..2

__global__ void ts_kernel(float *out, int *status, int a_fmt) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *sV = sm;  // 128 keys x 128 B
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 128 * 128; i += blockDim.x) {
        const int k = i / 128, n = i % 128;
        sV[k * 128 + (((n / 16) ^ (k % 8)) << 4) + n % 16] =
            static_cast<uint8_t>(f32x2_to_e4m3x2(static_cast<float>(vval(k, n)), 0.f) & 0xFF);
    }
    fence_proxy_async_smem();
    if (warp == 0) {
        tmem_alloc(&tslot, 256);
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
    // P row tid -> TMEM lane tid, columns 128..159 (4 keys per column, key 4c + byte)
    {
        uint32_t w[32];
        for (int c = 0; c < 32; ++c) {
            uint32_t x = 0;
            for (int bb = 0; bb < 4; ++bb) {
                const float v = static_cast<float>(pval(tid, 4 * c + bb));
                uint16_t e;
                if (a_fmt == 0) {
                    e = f32x2_to_e4m3x2(v, 0.f);
                } else {
                    asm("cvt.rn.satfinite.e5m2x2.f32 %0, %1, %2;" : "=h"(e) : "f"(0.f), "f"(v));
                }
                x |= static_cast<uint32_t>(e & 0xFF) << (8 * bb);
            }
            w[c] = x;
        }
        const uint32_t ta = tmem + (static_cast<uint32_t>(warp * 32) << 16) + 128;
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
            "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
            "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]),
            "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]), "r"(w[16]),
            "r"(w[17]), "r"(w[18]), "r"(w[19]), "r"(w[20]), "r"(w[21]), "r"(w[22]), "r"(w[23]), "r"(w[24]),
            "r"(w[25]), "r"(w[26]), "r"(w[27]), "r"(w[28]), "r"(w[29]), "r"(w[30]), "r"(w[31])
            : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
        const uint64_t vd = sdesc_sw128(smem_u32(sV), 128 * 128, 1024);
        const uint32_t idesc = (1u << 4) | (static_cast<uint32_t>(a_fmt) << 7) | (1u << 16) | ((128u >> 3) << 17) |
                               ((128u >> 4) << 24);
        for (int k = 0; k < 4; ++k) {
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                "r"(tmem + 128 + k * 8), "l"(vd + ((k * 4096) >> 4)), "r"(idesc), "r"(k > 0 ? 1u : 0u)
                : "memory");
        }
        tc_commit(&bar);
    }
    const long long t0 = clock64();
    bool ok = false;
    while (clock64() - t0 < 2000000000LL)
        if (mbar_try_wait(smem_u32(&bar), 0)) {
            ok = true;
            break;
        }
    if (!ok) {
        if (tid == 0) *status = 1;
        return;
    }
    tc_fence_after();
    for (int n = 0; n < 128; ++n)
        out[tid * 128 + n] = __uint_as_float(tmem_ld1(tmem + (static_cast<uint32_t>(warp * 32) << 16) + n));
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 256);
}

int ts_check(int a_fmt) {
    float *d_out;
    int *d_st;
    cudaMalloc(&d_out, 128 * 128 * 4);
    cudaMalloc(&d_st, 4);
    cudaMemset(d_st, 0, 4);
    cudaFuncSetAttribute(ts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 128);
    ts_kernel<<<1, 128, 128 * 128>>>(d_out, d_st, a_fmt);
    cudaError_t e = cudaDeviceSynchronize();
    int st = -1;
    cudaMemcpy(&st, d_st, 4, cudaMemcpyDeviceToHost);
    std::vector<float> h(128 * 128);
    cudaMemcpy(h.data(), d_out, h.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int r = 0; r < 128; ++r)
        for (int n = 0; n < 128; ++n) {
            int ref = 0;
            for (int k = 0; k < 128; ++k) ref += pval(r, k) * vval(k, n);
            if (h[r * 128 + n] != ref && bad++ < 5) std::printf("  D[%d][%d] = %g, want %d\n", r, n, h[r * 128 + n], ref);
        }
    std::printf("f8f6f4 TS A=%s(TMEM) B=E4M3 MN-major M128 N128 K128: %s, status %d, %d wrong\n",
                a_fmt == 0 ? "E4M3" : "E5M2", cudaGetErrorString(e), st, bad);
    return bad == 0 && st == 0 && e == cudaSuccess ? 0 : 1;
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
    const int rc_ss = bad == 0 && st == 0 && e == cudaSuccess ? 0 : 1;
    return rc_ss | ts_check(0) | ts_check(1);
}
