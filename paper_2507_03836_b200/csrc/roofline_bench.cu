// roofline_bench.cu -- measurement kernels (include/fhash_bench.h): the
// gather / red ceilings for the encode's access shape.  Not the method.
#include <cuda_runtime.h>

#include <cstdio>

#include "../../include/fhash_bench.h"

namespace {

__device__ __forceinline__ uint32_t mix32(uint32_t x) {  // murmur3 finalizer
    x ^= x >> 16; x *= 0x85ebca6bu; x ^= x >> 13; x *= 0xc2b2ae35u; x ^= x >> 16;
    return x;
}

__device__ __forceinline__ uint32_t rand_index(uint64_t tid, int k, uint32_t seed, uint32_t range) {
    const uint32_t h = mix32((uint32_t)tid * 0x9E3779B9u ^ mix32((uint32_t)(tid >> 32) + seed * 16u + k));
    return (uint32_t)(((uint64_t)h * range) >> 32);
}

template <typename V>
__device__ __forceinline__ float vsum(V v);
template <> __device__ __forceinline__ float vsum<float>(float v) { return v; }
template <> __device__ __forceinline__ float vsum<float2>(float2 v) { return v.x + v.y; }
template <> __device__ __forceinline__ float vsum<float4>(float4 v) { return v.x + v.y + v.z + v.w; }

// mode 0 ("split"): the two entries of a pair are two loads of entry width.
// mode 1 ("ideal"): the pair is ONE aligned load of twice the entry width --
// the minimum-sector access of SURVEY.md §8(d) (x-pairs share a sector).
template <typename V, typename V2, int P, int MODE>
__global__ void __launch_bounds__(256) gather_kernel(const V *__restrict__ buf, uint32_t range, int64_t n,
                                                     uint32_t seed, float *__restrict__ sink) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    float s = 0.f;
    if constexpr (MODE == 0) {
        V a[P], b[P];
#pragma unroll
        for (int k = 0; k < P; k++) {
            const uint32_t i = rand_index(t, k, seed, range);
            a[k] = __ldg(buf + i);
            b[k] = __ldg(buf + i + 1);
        }
#pragma unroll
        for (int k = 0; k < P; k++) s += vsum(a[k]) + vsum(b[k]);
    } else {
        V2 a[P];
        const V2 *b2 = reinterpret_cast<const V2 *>(buf);
#pragma unroll
        for (int k = 0; k < P; k++) a[k] = __ldg(b2 + rand_index(t, k, seed, range / 2));
#pragma unroll
        for (int k = 0; k < P; k++) s += vsum(a[k]);
    }
    sink[t] = s;
}

template <int W>
__device__ __forceinline__ void red_w(float *p, float v) {
    if constexpr (W == 1) atomicAdd(p, v);
    else if constexpr (W == 2) atomicAdd(reinterpret_cast<float2 *>(p), make_float2(v, v));
    else atomicAdd(reinterpret_cast<float4 *>(p), make_float4(v, v, v, v));
}

template <int W, int P, int MODE>
__global__ void __launch_bounds__(256) red_kernel(float *__restrict__ buf, uint32_t range, int64_t n,
                                                  uint32_t seed) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const float v = 1e-7f * (float)(t & 7);
#pragma unroll
    for (int k = 0; k < P; k++) {
        if constexpr (MODE == 0 || W >= 4) {
            const uint32_t i = rand_index(t, k, seed, range);
            red_w<W>(buf + (size_t)i * W, v);
            red_w<W>(buf + (size_t)(i + 1) * W, v);
        } else {  // one aligned red of twice the entry width per pair
            const uint32_t j = rand_index(t, k, seed, range / 2);
            red_w<2 * W>(buf + (size_t)j * 2 * W, v);
        }
    }
}

// Level-mix shape of the encode: thread t = (sample t / L, level t % L),
// level fastest as in fwd_kernel / bwd_kernel; its 8 x-pairs are ONE aligned
// access of two entries each at uniform positions inside the level's range
// of the packed table (the "ideal" pair of mode 1).  16-byte entries: two
// entry accesses per pair (no 32-byte red exists).
struct LevelRanges {
    int L;
    uint32_t off[32];    // first entry of level l
    uint32_t pairs[32];  // floor(T_l / 2) aligned pairs inside the level
};

__device__ __forceinline__ uint32_t level_pair(const LevelRanges &R, int l, uint64_t t, int k, uint32_t seed) {
    // chunk of two entries (global index) fully inside level l
    const uint32_t o = R.off[l];
    const uint32_t j = rand_index(t, k, seed, R.pairs[l]);
    return ((o + 1u) >> 1) + j;   // first whole chunk at or after o
}

template <typename V2>
__global__ void __launch_bounds__(256) gather_levels_kernel(const V2 *__restrict__ buf, const __grid_constant__ LevelRanges R,
                                                            int64_t n, uint32_t seed, float *__restrict__ sink) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int l = (int)(t % R.L);
    V2 a[8];
#pragma unroll
    for (int k = 0; k < 8; k++) a[k] = __ldg(buf + level_pair(R, l, t, k, seed));
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; k++) s += vsum(a[k]);
    sink[t] = s;
}

template <int W>
__global__ void __launch_bounds__(256) red_levels_kernel(float *__restrict__ buf, const __grid_constant__ LevelRanges R,
                                                         int64_t n, uint32_t seed) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int l = (int)(t % R.L);
    const float v = 1e-7f * (float)(t & 7);
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const uint32_t c = level_pair(R, l, t, k, seed);
        if constexpr (W >= 4) {
            red_w<W>(buf + (size_t)c * 2 * W, v);
            red_w<W>(buf + (size_t)c * 2 * W + W, v);
        } else {
            red_w<2 * W>(buf + (size_t)c * 2 * W, v);
        }
    }
}

__global__ void __launch_bounds__(256) copy_kernel(const int4 *__restrict__ src, int4 *__restrict__ dst, int64_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) dst[i] = __ldcs(src + i);
}

thread_local char g_berr[256];

fh_status launch_ok(const char *who) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        snprintf(g_berr, sizeof g_berr, "%s: %s", who, cudaGetErrorString(e));
        fprintf(stderr, "%s\n", g_berr);
        return FH_E_CUDA;
    }
    return FH_OK;
}

}  // namespace

extern "C" {

fh_status fh_bench_gather(const void *buf, uint64_t n_entries, int entry_bytes, int64_t n_threads, int pairs,
                          int mode, uint32_t seed, float *sink, fh_stream stream) {
    if (!buf || !sink || n_entries < 4 || n_entries > 0xFFFFFFFFull || n_threads <= 0 || pairs != 8 ||
        (mode != 0 && mode != 1))
        return FH_E_ARG;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const dim3 g((unsigned)((n_threads + 255) / 256));
    const uint32_t range = (uint32_t)(n_entries - 1);
#define FH_G(V, V2) \
    (mode ? gather_kernel<V, V2, 8, 1><<<g, 256, 0, s>>>((const V *)buf, range, n_threads, seed, sink) \
          : gather_kernel<V, V2, 8, 0><<<g, 256, 0, s>>>((const V *)buf, range, n_threads, seed, sink))
    switch (entry_bytes) {
        case 4: FH_G(float, float2); break;
        case 8: FH_G(float2, float4); break;
        case 16: FH_G(float4, float4); break;
        default: return FH_E_ARG;
    }
#undef FH_G
    return launch_ok("fh_bench_gather");
}

fh_status fh_bench_red(float *buf, uint64_t n_entries, int entry_bytes, int64_t n_threads, int pairs, int mode,
                       uint32_t seed, fh_stream stream) {
    if (!buf || n_entries < 4 || n_entries > 0xFFFFFFFFull || n_threads <= 0 || pairs != 8 ||
        (mode != 0 && mode != 1))
        return FH_E_ARG;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const dim3 g((unsigned)((n_threads + 255) / 256));
    const uint32_t range = (uint32_t)(n_entries - 1);
#define FH_R(W) \
    (mode ? red_kernel<W, 8, 1><<<g, 256, 0, s>>>(buf, range, n_threads, seed) \
          : red_kernel<W, 8, 0><<<g, 256, 0, s>>>(buf, range, n_threads, seed))
    switch (entry_bytes) {
        case 4: FH_R(1); break;
        case 8: FH_R(2); break;
        case 16: FH_R(4); break;
        default: return FH_E_ARG;
    }
#undef FH_R
    return launch_ok("fh_bench_red");
}

static fh_status make_ranges(const uint64_t *off, const uint64_t *size, int L, LevelRanges &R) {
    if (!off || !size || L < 1 || L > 32) return FH_E_ARG;
    R.L = L;
    for (int l = 0; l < L; l++) {
        if (off[l] + size[l] > 0xFFFFFFFFull || size[l] < 4) return FH_E_ARG;
        R.off[l] = (uint32_t)off[l];
        R.pairs[l] = (uint32_t)((size[l] - (off[l] & 1)) / 2);
    }
    return FH_OK;
}

fh_status fh_bench_gather_levels(const void *buf, const uint64_t *level_off, const uint64_t *level_size, int L,
                                 int entry_bytes, int64_t n_samples, uint32_t seed, float *sink, fh_stream stream) {
    LevelRanges R;
    if (!buf || !sink || n_samples <= 0 || make_ranges(level_off, level_size, L, R) != FH_OK) return FH_E_ARG;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int64_t n = n_samples * L;
    const dim3 g((unsigned)((n + 255) / 256));
    switch (entry_bytes) {
        case 4: gather_levels_kernel<float2><<<g, 256, 0, s>>>((const float2 *)buf, R, n, seed, sink); break;
        case 8: gather_levels_kernel<float4><<<g, 256, 0, s>>>((const float4 *)buf, R, n, seed, sink); break;
        default: return FH_E_ARG;
    }
    return launch_ok("fh_bench_gather_levels");
}

fh_status fh_bench_red_levels(float *buf, const uint64_t *level_off, const uint64_t *level_size, int L,
                              int entry_bytes, int64_t n_samples, uint32_t seed, fh_stream stream) {
    LevelRanges R;
    if (!buf || n_samples <= 0 || make_ranges(level_off, level_size, L, R) != FH_OK) return FH_E_ARG;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int64_t n = n_samples * L;
    const dim3 g((unsigned)((n + 255) / 256));
    switch (entry_bytes) {
        case 4: red_levels_kernel<1><<<g, 256, 0, s>>>(buf, R, n, seed); break;
        case 8: red_levels_kernel<2><<<g, 256, 0, s>>>(buf, R, n, seed); break;
        case 16: red_levels_kernel<4><<<g, 256, 0, s>>>(buf, R, n, seed); break;
        default: return FH_E_ARG;
    }
    return launch_ok("fh_bench_red_levels");
}

fh_status fh_bench_copy(void *dst, const void *src, uint64_t bytes, fh_stream stream) {
    if (!dst || !src || (bytes % 16) != 0) return FH_E_ARG;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    copy_kernel<<<148 * 8, 256, 0, s>>>((const int4 *)src, (int4 *)dst, (int64_t)(bytes / 16));
    return launch_ok("fh_bench_copy");
}

}  // extern "C"
