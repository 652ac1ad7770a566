// cvt_rate.cu -- diagnostics: issue cost (SM-sub-partition cycles per warp instruction) of the
// E4M3 -> f16 widening options of the FP8 KV cache path, registers only, W warps per sub-partition.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/cvt_rate.cu -o /tmp/cvt_rate
//   /tmp/cvt_rate
// Modes (per 32-bit E4M3 word -> two f16x2 words):
//   0  cvt.rn.f16x2.e4m3x2 x2 (F2FP unpack)
//   1  bit relocation (x 2^-8): prmt, lop3, iadd, shl per output word
//   2  bit relocation with imad: prmt, lop3, imad (t + m) * 128 via two imads
//   3  half the words by F2FP, half by relocation (two pipes)
//   4  F2FP + hmul2 (x 2^-8) per output word
//   5  cvt.rn.bf16x2.f32 (the softmax's P packing) for reference
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t f2fp(uint16_t x) {
    uint32_t r;
    asm volatile("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(r) : "h"(x));
    return r;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t sel) {
    uint32_t r;
    asm volatile("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(a), "r"(sel));
    return r;
}
// two E4M3 bytes (selected by sel: 0x4140 = bytes 0,1; 0x4342 = bytes 2,3) -> f16x2 x 2^-8
__device__ __forceinline__ uint32_t reloc(uint32_t x, uint32_t sel) {
    const uint32_t t = prmt(x, sel);    // [0 b1 0 b0]
    const uint32_t m = t & 0x00800080u;  // the sign bits
    return (t + m) << 7;                 // the sign carries into bit 8 -> bit 15
}
__device__ __forceinline__ uint32_t hmul2(uint32_t a, uint32_t b) {
    uint32_t r;
    asm volatile("mul.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t packbf(float lo, float hi) {
    uint32_t r;
    asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

template <int MODE>
__global__ void rate(int iters, uint32_t seed, uint32_t *out, long long *cyc) {
    uint32_t x[8], acc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = seed * (threadIdx.x + 1) + i * 0x01010101u;
    const uint32_t s8 = 0x1C001C00u;  // f16x2 (2^-8, 2^-8)
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            uint32_t a, b;
            if (MODE == 0) {
                a = f2fp(static_cast<uint16_t>(x[i]));
                b = f2fp(static_cast<uint16_t>(x[i] >> 16));
            } else if (MODE == 1 || MODE == 2) {
                a = reloc(x[i], 0x4140u);
                b = reloc(x[i], 0x4342u);
            } else if (MODE == 3) {
                if (i & 1) {
                    a = hmul2(f2fp(static_cast<uint16_t>(x[i])), s8);
                    b = hmul2(f2fp(static_cast<uint16_t>(x[i] >> 16)), s8);
                } else {
                    a = reloc(x[i], 0x4140u);
                    b = reloc(x[i], 0x4342u);
                }
            } else if (MODE == 4) {
                a = hmul2(f2fp(static_cast<uint16_t>(x[i])), s8);
                b = hmul2(f2fp(static_cast<uint16_t>(x[i] >> 16)), s8);
            } else {
                a = packbf(__uint_as_float(x[i]), __uint_as_float(x[i] ^ 0x5555u));
                b = packbf(__uint_as_float(x[i] >> 1), __uint_as_float(x[i] + 3u));
            }
            acc ^= a + b;
            x[i] += 0x01030507u;
        }
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// relocation == F2FP x 2^-8 for every pair of E4M3 bytes except the NaN codes (0x7F, 0xFF)
__global__ void check(int *bad) {
    const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;  // two bytes
    if (v >= 65536u) return;
    const uint32_t b0 = v & 0xFF, b1 = v >> 8;
    if ((b0 & 0x7F) == 0x7F || (b1 & 0x7F) == 0x7F) return;
    const uint32_t want = hmul2(f2fp(static_cast<uint16_t>(v)), 0x1C001C00u);
    if (reloc(v, 0x4140u) != want || reloc(v << 16, 0x4342u) != want) atomicAdd(bad, 1);
}

template <int MODE>
void run(const char *name, int warps_per_smsp) {
    const int iters = 4096, blocks = 148, threads = 128 * warps_per_smsp;
    uint32_t *out;
    long long *cyc;
    cudaMalloc(&out, blocks * threads * 4);
    cudaMalloc(&cyc, blocks * 8);
    rate<MODE><<<blocks, threads>>>(16, 1u, out, cyc);
    rate<MODE><<<blocks, threads>>>(iters, 1u, out, cyc);
    cudaDeviceSynchronize();
    long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    // output words converted per sub-partition: warps_per_smsp x iters x 16 (per lane: 8 x 2)
    const double words = double(warps_per_smsp) * iters * 16;
    printf("%-44s W=%d: %.2f cycles per 32 output words per sub-partition\n", name, warps_per_smsp, c / words);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    int *bad, nbad = -1;
    cudaMalloc(&bad, 4);
    cudaMemset(bad, 0, 4);
    check<<<256, 256>>>(bad);
    cudaMemcpy(&nbad, bad, 4, cudaMemcpyDeviceToHost);
    printf("relocation vs F2FP x 2^-8: %d mismatches over 65536 byte pairs (NaN codes skipped)\n", nbad);
    for (int w : {1, 2, 4}) {
        run<0>("F2FP e4m3x2 unpack", w);
        run<1>("relocation (prmt, lop3, iadd, shl)", w);
        run<3>("half F2FP+hmul2, half relocation", w);
        run<4>("F2FP + hmul2", w);
        run<5>("cvt.rn.bf16x2.f32 (reference)", w);
    }
    return 0;
}
