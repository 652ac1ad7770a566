// softmax_rate.cu -- diagnostics: throughput of the prefix kernel's softmax inner loop (per row:
// scale, exp2, row sum, pack to bf16) for different fractions of FMA-pipe polynomial exp2, with
// 8 softmax warps per SM as in the kernel.  Registers only (no TMEM).  Build & run on the box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude tools/softmax_rate.cu -o /tmp/sm_rate
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2502_17421_b200/csrc/ptx_sm100.cuh"

using namespace hta;

// EMU8: number of column pairs out of every 8 computed by the polynomial; SPREAD: poly pairs
// spread evenly (i % 8 in {0, 3, 6}) instead of clustered ({0, 1, 2})
// EMU8 = -1: exp2 of a pair as one MUFU ex2.approx.f16x2 (fp16 in/out), unpacked to fp32 for the
// row sum and repacked to bf16; EMU8 = -2: same but the row sum is accumulated in f16x2.
__device__ __forceinline__ uint32_t ex2_f16x2(uint32_t x) {
    uint32_t y;
    asm("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}
// (pack_f16x2: from ptx_sm100.cuh)
// PACK: 0 = cvt.rn.bf16x2.f32 (the kernel's), 1 = truncation by one byte permute (the row sum then
// adds the truncated values: one AND per element)
template <int EMU8, bool SPREAD = false, int PACK = 0>
__global__ void __launch_bounds__(256, 1) softmax_loop(int iters, float c, float *out) {
    float s[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) s[i] = (threadIdx.x * 0.001f) - i * 0.01f;
    float m = 0.5f, acc_all = 0.f;
    uint32_t sink = 0;
    for (int it = 0; it < iters; ++it) {
        const float2 c2 = make_float2(c, c), neg2 = make_float2(-m, -m);
        float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
        const float2 *s2 = reinterpret_cast<const float2 *>(s);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            const float2 x = __ffma2_rn(s2[i], c2, neg2);
            float2 pp;
            if (EMU8 < 0) {
                const uint32_t e = ex2_f16x2(pack_f16x2(x.x, x.y));
                __half2 h = *reinterpret_cast<const __half2 *>(&e);
                if (EMU8 == -2) {
                    __half2 a = *reinterpret_cast<__half2 *>(&sink);
                    a = __hadd2(a, h);
                    pp = __half22float2(h);
                    sink ^= pack_bf16x2(pp.x, pp.y) + *reinterpret_cast<uint32_t *>(&a);
                    continue;
                }
                pp = __half22float2(h);
                if (i & 1)
                    acc1 = __fadd2_rn(acc1, pp);
                else
                    acc0 = __fadd2_rn(acc0, pp);
                sink ^= pack_bf16x2(pp.x, pp.y);
                continue;
            }
            const bool poly = SPREAD ? (EMU8 == 3 && ((i & 7) == 0 || (i & 7) == 3 || (i & 7) == 6))
                                     : ((i & 7) < EMU8);
            if (poly) {
                pp = exp2_poly2(x);
            } else {
                pp.x = fast_exp2(x.x);
                pp.y = fast_exp2(x.y);
            }
            if (PACK == 1) {
                const uint32_t ux = __float_as_uint(pp.x) & 0xFFFF0000u, uy = __float_as_uint(pp.y) & 0xFFFF0000u;
                pp = make_float2(__uint_as_float(ux), __uint_as_float(uy));
                sink ^= __byte_perm(ux, uy, 0x7632);
            }
            if (i & 1)
                acc1 = __fadd2_rn(acc1, pp);
            else
                acc0 = __fadd2_rn(acc0, pp);
            if (PACK == 0) sink ^= pack_bf16x2(pp.x, pp.y);
        }
        acc_all += (acc0.x + acc1.x) + (acc0.y + acc1.y);
        m += 1e-7f;  // loop-carried so the compiler cannot hoist the exps
    }
    if (sink == 0x12345 || acc_all == 1.2345f) out[threadIdx.x] = acc_all;
}

template <int EMU8, bool SPREAD = false, int PACK = 0>
void run(int threads = 256) {
    float *out;
    cudaMalloc(&out, 4096);
    const int iters = 20000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9;
    for (int r = 0; r < 4; ++r) {
        cudaEventRecord(e0);
        softmax_loop<EMU8, SPREAD, PACK><<<148, threads>>>(iters, 0.12f, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;
    }
    // per SMSP: threads/128 warps x 64 elements x iters
    const double elems_per_smsp = threads / 128.0 * 64 * iters;
    printf("mode %d/8%s%s, %d warps/SMSP: %8.1f us  -> %.2f cycles per 32-wide element slot per SMSP @1.9GHz\n",
           EMU8, SPREAD ? " spread" : "", PACK ? " trunc-pack" : "", threads / 128, best * 1e3,
           best * 1e-3 * 1.9e9 / elems_per_smsp);
}

int main() {
    for (int t : {256, 512}) {
        run<-1>(t);
        run<-2>(t);
        run<0>(t);
        run<2>(t);
        run<3>(t);
        run<3, true>(t);
        run<4>(t);
        run<8>(t);
        run<2, false, 1>(t);
        run<3, false, 1>(t);
        run<0, false, 1>(t);
    }
    return 0;
}
