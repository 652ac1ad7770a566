// tma_bw.cu -- diagnostics: TMA streaming bandwidth of a KV cache in the layouts / boxes the
// prefix kernel uses (no compute).  Build & run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude tools/tma_bw.cu -o /tmp/tma_bw -lcuda
//   /tmp/tma_bw
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "../paper_2502_17421_b200/csrc/ptx_sm100.cuh"

using namespace hta;

constexpr int kRing = 196608;  // bytes of smem ring (as in the prefix kernel)

// Each CTA streams `tiles` tiles; one tile = `nbox` TMA boxes of `box_bytes` each into a slot.
__global__ void __launch_bounds__(64) stream_kernel(const __grid_constant__ CUtensorMap map,
                                                   const __grid_constant__ CUtensorMap map2, int two, int tiles, int nbox,
                                                   int box_bytes, int rows_per_box, int heads, int keys_per_cta,
                                                   int head_major, int ring, uint64_t policy) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int slot_bytes = nbox * box_bytes * (two ? 2 : 1);
    const int kSlots = ring / slot_bytes;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + ring);
    uint64_t *empty = full + kSlots;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kSlots; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    // CTA c reads head (c % heads), key range [(c / heads) * keys_per_cta, +keys_per_cta)
    const int head = blockIdx.x % heads;
    const int k0 = (blockIdx.x / heads) * keys_per_cta;
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < tiles; ++i) {
            const int s = i % kSlots;
            mbar_wait(&empty[s], ((i / kSlots) & 1) ^ 1);
            mbar_arrive_expect_tx(&full[s], slot_bytes);
            for (int m = 0; m < (two ? 2 : 1); ++m)
            for (int b = 0; b < nbox; ++b) {
                // boxes walk the d halves (b & 1) and consecutive key blocks (b >> 1)
                const int n = k0 + (i * (nbox / 2 > 0 ? nbox / 2 : 1) + (b >> 1)) * rows_per_box;
                tma_load_4d(smem + s * slot_bytes + (m * nbox + b) * box_bytes, m ? &map2 : &map, &full[s], (b & 1) * 64,
                            head_major ? n : head, head_major ? head : n, 0, policy);
            }
        }
    } else if (warp == 1 && lane == 0) {
        for (int i = 0; i < tiles; ++i) {
            const int s = i % kSlots;
            mbar_wait(&full[s], (i / kSlots) & 1);
            mbar_arrive(&empty[s]);
        }
    }
}

__global__ void __launch_bounds__(512) ldg_kernel(const int4 *__restrict__ src, size_t n16, int4 *sink) {
    int4 acc = make_int4(0, 0, 0, 0);
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x * 4) {
        int4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const size_t k = i + size_t(u) * gridDim.x * blockDim.x;
            v[u] = k < n16 ? __ldcs(src + k) : make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc.x ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    if (acc.x == 0x12345678) sink[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static void read_flush(const void *flush, int4 *sink) {
    ldg_kernel<<<148 * 8, 512>>>(static_cast<const int4 *>(flush), (size_t(512) << 20) / 16, sink);
}

int main(int argc, char **argv) {
    const int H = 8, D = 128;
    EncodeFn enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void **>(&enc), cudaEnableDefault, &q);
    void *flush;
    cudaMalloc(&flush, size_t(512) << 20);
    cudaMemset(flush, 1, size_t(512) << 20);
    int4 *sink;
    cudaMalloc(&sink, 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int N : {65536, 262144}) {
        const size_t bytes = size_t(N) * H * D * 2;  // one of K / V
        void *buf;
        cudaMalloc(&buf, bytes * 2);
        cudaMemset(buf, 1, bytes * 2);
        for (int grid : {148 * 4, 148 * 8}) {
            float best = 1e9;
            for (int it = 0; it < 5; ++it) {
                read_flush(flush, sink);
                cudaEventRecord(e0);
                ldg_kernel<<<grid, 512>>>(static_cast<const int4 *>(buf), bytes * 2 / 16, sink);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (it > 0 && ms < best) best = ms;
            }
            printf("N=%6d LDG.128 K+V %4d x 512                          %8.1f us  %7.0f GB/s\n", N, grid, best * 1e3,
                   2 * bytes / (best * 1e-3) / 1e9);
        }
        struct Cfg {
            const char *name;
            int head_major, rows, ctas, ring;
        } cfgs[] = {
            {"K+V [N,Hkv,d] 64x96 x2, 144 CTA, ring 48K", 0, 96, 144, 49152},
            {"K+V [N,Hkv,d] 64x96 x2, 144 CTA, ring 96K", 0, 96, 144, 98304},
            {"K+V [N,Hkv,d] 64x96 x2, 144 CTA, ring 144K", 0, 96, 144, 147456},
            {"K+V [N,Hkv,d] 64x96 x2, 144 CTA, ring 192K", 0, 96, 144, 196608},
            {"K+V [N,Hkv,d] 64x64 x2, 144 CTA, ring 96K", 0, 64, 144, 98304},
            {"K+V [N,Hkv,d] 64x96 x2, 288 CTA, ring 48K", 0, 96, 288, 49152},
            {"K+V [Hkv,N,d] 64x96 x2, 144 CTA, ring 96K", 1, 96, 144, 98304},
            {"K+V [Hkv,N,d] 64x96 x2, 144 CTA, ring 192K", 1, 96, 144, 196608},
        };
        for (auto &c : cfgs) {
            CUtensorMap map, map2;
            cuuint64_t dims[4], strides[3];
            if (!c.head_major) {
                dims[0] = D; dims[1] = H; dims[2] = N; dims[3] = 1;
                strides[0] = D * 2; strides[1] = size_t(H) * D * 2; strides[2] = bytes;
            } else {
                dims[0] = D; dims[1] = N; dims[2] = H; dims[3] = 1;
                strides[0] = D * 2; strides[1] = size_t(N) * D * 2; strides[2] = bytes;
            }
            cuuint32_t box[4] = {64, c.head_major ? (cuuint32_t)c.rows : 1u, c.head_major ? 1u : (cuuint32_t)c.rows, 1};
            cuuint32_t es[4] = {1, 1, 1, 1};
            enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            enc(&map2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, static_cast<char *>(buf) + bytes, dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            const int keys_per_cta = N / (c.ctas / H);
            const int tiles = keys_per_cta / c.rows;
            const int box_bytes = 64 * c.rows * 2;
            float best = 1e9;
            for (int it = 0; it < 5; ++it) {
                read_flush(flush, sink);
                cudaEventRecord(e0);
                stream_kernel<<<c.ctas, 64, c.ring + 1024>>>(map, map2, 1, tiles, 2, box_bytes, c.rows, H, keys_per_cta,
                                                            c.head_major, c.ring, kPolicyEvictFirst);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (it > 0 && ms < best) best = ms;
            }
            cudaError_t err = cudaGetLastError();
            printf("N=%6d %-50s %8.1f us  %7.0f GB/s  %s\n", N, c.name, best * 1e3, 2 * bytes / (best * 1e-3) / 1e9,
                   err == cudaSuccess ? "" : cudaGetErrorString(err));
        }
        cudaFree(buf);
    }
    return 0;
}
