// sort_kernels.cuh -- spatial binning of a sample batch (an execution-order
// optimisation; the encode results do not depend on it beyond fp summation
// order).  Samples are counting-sorted by a 16-bit Morton code of their bin
// on a grid of 2^bits[a] bins per axis over [0,1]^4 (KeySpec, chosen per
// encoder so that bins are about cubic in cells of its finest level), so a
// run of consecutive sorted samples covers a compact region: the tiled
// encode (tiled_kernels.cuh) stages that region of each level in shared
// memory.
#pragma once
#include <stdint.h>

#include "encode_params.h"

namespace fh {
namespace sortk {

constexpr int kKeyBits = 16;
constexpr int kBins = 1 << kKeyBits;           // 65536

// bin of p on an axis with 2^b bins (NaN -> 0 as R2; 1.0 -> last bin)
__device__ __forceinline__ uint32_t qbin(float p, uint32_t b) {
    const float pc = (p >= 0.f) ? fminf(p, 1.f) : 0.f;
    const uint32_t nb = 1u << b;
    const uint32_t v = (uint32_t)(pc * (float)nb);
    return min(v, nb - 1u);
}

__device__ __forceinline__ uint32_t morton_key(float4 p, const KeySpec &K) {
    const uint32_t a[4] = {qbin(p.x, K.bits[0]), qbin(p.y, K.bits[1]), qbin(p.z, K.bits[2]), qbin(p.w, K.bits[3])};
    uint32_t k = 0;
#pragma unroll
    for (int ax = 0; ax < 4; ax++)
#pragma unroll
        for (int j = 0; j < kKeyBits; j++)
            if (j < (int)K.bits[ax]) k |= ((a[ax] >> j) & 1u) << K.pos[ax][j];
    return k;
}

__global__ void __launch_bounds__(256) key_hist_kernel(const __grid_constant__ KeySpec K,
                                                       const float4 *__restrict__ coords, int64_t N,
                                                       uint16_t *__restrict__ keys, uint32_t *__restrict__ hist) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = morton_key(__ldg(coords + i), K);
        keys[i] = (uint16_t)k;
        atomicAdd(hist + k, 1u);
    }
}

// Exclusive scan of the kBins counters in two levels: kScanBlocks CTAs each
// scan 1024 counters in place (block-local exclusive prefix) and write their
// total to sums[b]; the scatter kernel adds the prefix of those totals.
constexpr int kScanBlocks = kBins / 1024;   // 64

__global__ void __launch_bounds__(1024) scan_blocks_kernel(uint32_t *__restrict__ hist, uint32_t *__restrict__ sums) {
    __shared__ uint32_t wsum[32];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    uint32_t *h = hist + blockIdx.x * 1024;
    const uint32_t x = h[t];
    uint32_t v = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    if (lane == 31) wsum[w] = v;
    __syncthreads();
    if (w == 0) {
        uint32_t s = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        wsum[lane] = s;  // inclusive prefix of warp totals
    }
    __syncthreads();
    h[t] = v - x + (w > 0 ? wsum[w - 1] : 0u);
    if (t == 1023) sums[blockIdx.x] = wsum[31];
}

__global__ void __launch_bounds__(256) scatter_kernel(const uint16_t *__restrict__ keys, int64_t N,
                                                      uint32_t *__restrict__ offs, const uint32_t *__restrict__ sums,
                                                      uint32_t *__restrict__ perm) {
    __shared__ uint32_t pre[kScanBlocks];
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        uint32_t a = sums[2 * lane], b = sums[2 * lane + 1];
        uint32_t s = a + b;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        const uint32_t ex = s - a - b;  // exclusive prefix of this lane's pair
        pre[2 * lane] = ex;
        pre[2 * lane + 1] = ex + a;
    }
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = keys[i];
        const uint32_t pos = atomicAdd(offs + k, 1u) + pre[k >> 10];
        perm[pos] = (uint32_t)i;
    }
}

}  // namespace sortk
}  // namespace fh
