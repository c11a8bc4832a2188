// sort_kernels.cuh -- spatial binning of a sample batch (an execution-order
// optimisation; the encode results do not depend on it beyond fp summation
// order).  Samples are counting-sorted by the 16-bit Morton code of their
// cell on a 16^4 grid over [0,1]^4, so consecutive threads (and the warps
// resident on one SM) touch nearby table entries: coarse-level corners hit
// in L1 in the forward and reductions to the same entry arrive together in
// the backward.
#pragma once
#include <stdint.h>

namespace fh {
namespace sortk {

constexpr int kBits = 4;                       // per axis
constexpr int kBins = 1 << (4 * kBits);        // 65536

__device__ __forceinline__ uint32_t q4(float p) {
    const float pc = (p >= 0.f) ? fminf(p, 1.f) : 0.f;   // NaN -> 0 (as R2)
    int v = (int)(pc * 16.f);
    return (uint32_t)min(v, 15);
}

__device__ __forceinline__ uint32_t morton4(float4 p) {
    const uint32_t a[4] = {q4(p.x), q4(p.y), q4(p.z), q4(p.w)};
    uint32_t k = 0;
#pragma unroll
    for (int b = 0; b < kBits; b++)
#pragma unroll
        for (int ax = 0; ax < 4; ax++) k |= ((a[ax] >> b) & 1u) << (4 * b + ax);
    return k;
}

__global__ void __launch_bounds__(256) key_hist_kernel(const float4 *__restrict__ coords, int64_t N,
                                                       uint16_t *__restrict__ keys, uint32_t *__restrict__ hist) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = morton4(__ldg(coords + i));
        keys[i] = (uint16_t)k;
        atomicAdd(hist + k, 1u);
    }
}

// Exclusive scan of kBins counters in place, one CTA of 1024 threads.
__global__ void __launch_bounds__(1024) scan_kernel(uint32_t *__restrict__ hist) {
    __shared__ uint32_t part[1024];
    constexpr int per = kBins / 1024;
    const int t = threadIdx.x;
    uint32_t loc[per];
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < per; i++) { loc[i] = hist[t * per + i]; s += loc[i]; }
    part[t] = s;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
        const uint32_t v = t >= off ? part[t - off] : 0u;
        __syncthreads();
        part[t] += v;
        __syncthreads();
    }
    uint32_t run = part[t] - s;  // exclusive prefix of this thread's chunk
#pragma unroll
    for (int i = 0; i < per; i++) { hist[t * per + i] = run; run += loc[i]; }
}

__global__ void __launch_bounds__(256) scatter_kernel(const uint16_t *__restrict__ keys, int64_t N,
                                                      uint32_t *__restrict__ offs, uint32_t *__restrict__ perm) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t pos = atomicAdd(offs + keys[i], 1u);
        perm[pos] = (uint32_t)i;
    }
}

}  // namespace sortk
}  // namespace fh
