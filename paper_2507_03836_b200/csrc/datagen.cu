// datagen.cu -- synthetic fields and the voxel sampler (include/fhash_data.h).
// Harness code: stands in for the paper's datasets; not part of the method.
#include <cuda_runtime.h>

#include <cfloat>
#include <cmath>
#include <cstring>

#include "internal.h"
#include "../../include/fhash_data.h"

using fh::cuda_check;
using fh::fail;

namespace {

constexpr int kMaxBlobs = 32;
struct Blobs {
    int n;
    float p[kMaxBlobs][7];
};

__global__ void blobs_kernel(float *field, int S, int T, const Blobs B) {
    const int64_t n = (int64_t)S * S * S * T;
    const float inv = 1.0f / (float)(S - 1);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(i % S), y = (int)((i / S) % S), z = (int)((i / ((int64_t)S * S)) % S);
        const int t = (int)(i / ((int64_t)S * S * S));
        const float px = x * inv, py = y * inv, pz = z * inv;
        const float tau = T > 1 ? (float)t / (float)(T - 1) : 0.f;
        float v = 0.1f * sinpif(8.f * px) * sinpif(8.f * py);
        for (int b = 0; b < B.n; b++) {
            const float *q = B.p[b];
            const float cx = q[1] + q[4] * tau, cy = q[2] + q[5] * tau, cz = q[3] + q[6] * tau;
            const float d2 = (px - cx) * (px - cx) + (py - cy) * (py - cy) + (pz - cz) * (pz - cz);
            v += expf(-d2 / (2.f * q[0] * q[0]));
        }
        field[i] = v;
    }
}

__device__ __forceinline__ uint32_t hash4(uint32_t x, uint32_t y, uint32_t z, uint32_t t, uint32_t seed) {
    uint32_t h = seed * 0x9E3779B9u;
    h ^= x * 0x85EBCA6Bu; h = (h << 13) | (h >> 19); h = h * 5u + 0xE6546B64u;
    h ^= y * 0xC2B2AE35u; h = (h << 13) | (h >> 19); h = h * 5u + 0xE6546B64u;
    h ^= z * 0x27D4EB2Fu; h = (h << 13) | (h >> 19); h = h * 5u + 0xE6546B64u;
    h ^= t * 0x165667B1u; h = (h << 13) | (h >> 19); h = h * 5u + 0xE6546B64u;
    h ^= h >> 16; h *= 0x85EBCA6Bu; h ^= h >> 13; h *= 0xC2B2AE35u; h ^= h >> 16;
    return h;
}

__device__ __forceinline__ float fade(float u) { return u * u * u * (u * (u * 6.f - 15.f) + 10.f); }

__device__ float value_noise4(float x, float y, float z, float t, uint32_t seed) {
    const float fx = floorf(x), fy = floorf(y), fz = floorf(z), ft = floorf(t);
    const uint32_t ix = (uint32_t)(int)fx, iy = (uint32_t)(int)fy, iz = (uint32_t)(int)fz, it = (uint32_t)(int)ft;
    const float u[4] = {fade(x - fx), fade(y - fy), fade(z - fz), fade(t - ft)};
    float acc = 0.f;
#pragma unroll
    for (int c = 0; c < 16; c++) {
        const uint32_t bx = c & 1, by = (c >> 1) & 1, bz = (c >> 2) & 1, bt = (c >> 3) & 1;
        const float w = (bx ? u[0] : 1.f - u[0]) * (by ? u[1] : 1.f - u[1]) * (bz ? u[2] : 1.f - u[2]) *
                        (bt ? u[3] : 1.f - u[3]);
        const float val = (float)(hash4(ix + bx, iy + by, iz + bz, it + bt, seed) >> 8) * (1.f / 16777216.f);
        acc += w * val;
    }
    return acc;
}

__global__ void noise_kernel(float *field, int Sx, int Sy, int Sz, int T, uint32_t seed) {
    const int64_t n = (int64_t)Sx * Sy * Sz * T;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(i % Sx);
        const int y = (int)((i / Sx) % Sy);
        const int z = (int)((i / ((int64_t)Sx * Sy)) % Sz);
        const int t = (int)(i / ((int64_t)Sx * Sy * Sz));
        const float px = (float)x / (float)(Sx - 1), py = (float)y / (float)(Sy - 1);
        const float pz = (float)z / (float)(Sz - 1), pt = T > 1 ? (float)t / (float)(T - 1) : 0.f;
        float v = 0.f, freq = 4.f, amp = 1.f;
        for (int o = 0; o < 3; o++) {
            v += amp * value_noise4(px * freq, py * freq, pz * freq, pt * freq, seed + 7919u * o);
            freq *= 2.f;
            amp *= 0.5f;
        }
        field[i] = v;
    }
}

__device__ __forceinline__ void atomic_min_f(float *a, float v) {
    if (v >= 0.f) atomicMin(reinterpret_cast<int *>(a), __float_as_int(v));
    else atomicMax(reinterpret_cast<unsigned int *>(a), __float_as_uint(v));
}
__device__ __forceinline__ void atomic_max_f(float *a, float v) {
    if (v >= 0.f) atomicMax(reinterpret_cast<int *>(a), __float_as_int(v));
    else atomicMin(reinterpret_cast<unsigned int *>(a), __float_as_uint(v));
}

__global__ void minmax_kernel(const float *f, int64_t n, float *mm) {
    float lo = FLT_MAX, hi = -FLT_MAX;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float v = f[i];
        lo = fminf(lo, v);
        hi = fmaxf(hi, v);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomic_min_f(mm, lo);
        atomic_max_f(mm + 1, hi);
    }
}

__global__ void affine_kernel(float *f, int64_t n, const float *mm, float band) {
    const float lo = mm[0], scale = 1.f / fmaxf(mm[1] - mm[0], 1e-30f);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float v = (f[i] - lo) * scale;
        if (band > 0.f) {
            const float d = (v - 0.5f) / band;
            v = 0.5f * v + 0.5f * expf(-d * d);
        }
        f[i] = v;
    }
}

__global__ void init_mm(float *mm) { mm[0] = FLT_MAX; mm[1] = -FLT_MAX; }

// Philox4x32-10 (Salmon et al. 2011).
__device__ __forceinline__ uint4 philox(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; r++) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}

__global__ void sample_kernel(const float *field, int Sx, int Sy, int Sz, int T, int64_t N, uint2 key, uint32_t sub,
                              uint32_t off, float4 *coords, float *target) {
    const int64_t n_vox = (int64_t)Sx * Sy * Sz * T;
    const float ix = 1.f / (float)(Sx - 1), iy = 1.f / (float)(Sy - 1), iz = 1.f / (float)(Sz - 1);
    const float it = T > 1 ? 1.f / (float)(T - 1) : 0.f;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const uint4 r = philox(make_uint4((uint32_t)i, (uint32_t)(i >> 32), sub, off), key);
        const uint64_t u = ((uint64_t)r.x << 32) | r.y;
        const int64_t v = (int64_t)(u % (uint64_t)n_vox);
        const int x = (int)(v % Sx), y = (int)((v / Sx) % Sy), z = (int)((v / ((int64_t)Sx * Sy)) % Sz);
        const int t = (int)(v / ((int64_t)Sx * Sy * Sz));
        coords[i] = make_float4(x * ix, y * iy, z * iz, t * it);
        target[i] = __ldg(field + v);
    }
}

int grid_for(int64_t n) {
    int64_t g = (n + 255) / 256;
    if (g > 148 * 32) g = 148 * 32;
    return (int)(g < 1 ? 1 : g);
}

}  // namespace

extern "C" {

fh_status fh_data_gaussian_blobs(float *field, int S, int T, int n_blobs, const float *blobs, fh_stream stream) {
    fh::g_err[0] = 0;
    if (!field || !blobs || S < 2 || T < 1 || n_blobs < 0 || n_blobs > kMaxBlobs)
        return fail(FH_E_ARG, "fh_data_gaussian_blobs: bad arguments");
    Blobs B;
    B.n = n_blobs;
    memcpy(B.p, blobs, sizeof(float) * 7 * n_blobs);
    const int64_t n = (int64_t)S * S * S * T;
    blobs_kernel<<<grid_for(n), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(field, S, T, B);
    return cuda_check(cudaGetLastError(), "blobs_kernel");
}

fh_status fh_data_value_noise(float *field, int Sx, int Sy, int Sz, int T, uint32_t seed, fh_stream stream) {
    fh::g_err[0] = 0;
    if (!field || Sx < 2 || Sy < 2 || Sz < 2 || T < 1) return fail(FH_E_ARG, "fh_data_value_noise: bad arguments");
    const int64_t n = (int64_t)Sx * Sy * Sz * T;
    noise_kernel<<<grid_for(n), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(field, Sx, Sy, Sz, T, seed);
    return cuda_check(cudaGetLastError(), "noise_kernel");
}

fh_status fh_data_normalize(float *field, int64_t n, float band, void *scratch, fh_stream stream) {
    fh::g_err[0] = 0;
    if (!field || !scratch || n < 1) return fail(FH_E_ARG, "fh_data_normalize: bad arguments");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    float *mm = reinterpret_cast<float *>(scratch);
    for (int pass = 0; pass < (band > 0.f ? 2 : 1); pass++) {
        init_mm<<<1, 1, 0, s>>>(mm);
        minmax_kernel<<<grid_for(n), 256, 0, s>>>(field, n, mm);
        affine_kernel<<<grid_for(n), 256, 0, s>>>(field, n, mm, pass == 0 ? band : 0.f);
    }
    fh_status st = cuda_check(cudaGetLastError(), "normalize kernels");
    if (st != FH_OK) return st;
    return cuda_check(cudaStreamSynchronize(s), "normalize sync");
}

fh_status fh_data_sample_voxels(const float *field, int Sx, int Sy, int Sz, int T, int64_t N, uint64_t seed,
                                uint32_t sub, uint32_t off, float *coords, float *target, fh_stream stream) {
    fh::g_err[0] = 0;
    if (!field || !coords || !target || N < 0 || Sx < 2 || Sy < 2 || Sz < 2 || T < 1)
        return fail(FH_E_ARG, "fh_data_sample_voxels: bad arguments");
    if (N == 0) return FH_OK;
    const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    sample_kernel<<<grid_for(N), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        field, Sx, Sy, Sz, T, N, key, sub, off, reinterpret_cast<float4 *>(coords), target);
    return cuda_check(cudaGetLastError(), "sample_kernel");
}

}  // extern "C"
