// mhe_kernels.cuh -- NEXT-3: the MHE baseline encoder on the same
// machinery (the comparison system of P:378 / Fig. 4; SPEC
// baseline_encode S:321-329): one 3D multi-resolution hash encoder per key
// frame, a fixed table of T entries per level and frame, direct indexing
// when R^3 <= T else the spatial hash (x*1 ^ y*2654435761 ^ z*805459861)
// mod T, trilinear blend of 8 corners (4 x-pairs).  The sample's frame is
// the nearest key frame of its t (reading R20).
//
// Level fields reused: res[0..2] = R, res[3] = n_frames, scale[3] =
// n_frames - 1, sy = R, sz = R*R, st = T (frame stride), mask = T - 1,
// hashed = (R^3 > T), offset = first entry of the level.
#pragma once
#include "encode_kernels.cuh"

namespace fh {
namespace mhe {

struct Cell8 {
    uint32_t idx[8];
    float w[3];
};

__device__ __forceinline__ bool cell_of(const Level &lv, float4 p, Cell8 &c) {
    uint32_t ix, iy, iz;
    bool bad = false;
    locate(p.x, lv.scale[0], lv.res[0], ix, c.w[0], bad);
    locate(p.y, lv.scale[1], lv.res[1], iy, c.w[1], bad);
    locate(p.z, lv.scale[2], lv.res[2], iz, c.w[2], bad);
    // nearest key frame (R20): s = fp32(t (n-1)), k = floor(s) + (frac >= 0.5)
    float pt = p.w;
    if (!(pt >= 0.0f)) { pt = 0.0f; bad = true; }
    else if (pt > 1.0f) { pt = 1.0f; bad = true; }
    const float s = __fmul_rn(pt, lv.scale[3]);
    const float fl = floorf(s);
    int k = (int)fl + ((__fsub_rn(s, fl) >= 0.5f) ? 1 : 0);
    k = min(max(k, 0), (int)lv.res[3] - 1);
    const uint32_t base = lv.offset + (uint32_t)k * lv.st;
    if (!lv.hashed) {
        const uint32_t b0 = base + ix + iy * lv.sy + iz * lv.sz;
#pragma unroll
        for (int q = 0; q < 8; q++) c.idx[q] = b0 + (q & 1) + ((q >> 1) & 1) * lv.sy + ((q >> 2) & 1) * lv.sz;
    } else {
        const uint32_t hy0 = iy * kPy, hy1 = (iy + 1) * kPy, hz0 = iz * kPz, hz1 = (iz + 1) * kPz;
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const uint32_t h = ((q & 1) ? ix + 1 : ix) ^ (((q >> 1) & 1) ? hy1 : hy0) ^ (((q >> 2) & 1) ? hz1 : hz0);
            c.idx[q] = base + (h & lv.mask);
        }
    }
    return bad;
}

template <int F, typename T, typename O>
__global__ void __launch_bounds__(256) fwd_kernel(const __grid_constant__ Params P, const float4 *__restrict__ coords,
                                                  int64_t N, const T *__restrict__ table, O *__restrict__ out,
                                                  int *__restrict__ flag, int l0, int lc) {
    __shared__ LevelSmem slv;
    load_levels(P, slv);
    const int L = P.L;
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n = gid / lc;
    if (n >= N) return;
    const int l = l0 + (int)(gid - n * lc);
    Cell8 c;
    const bool bad = cell_of(slv.get(l), __ldg(coords + n), c);
    if (bad && l == l0) atomicOr(flag, 1);
    float e[8][F];
#pragma unroll
    for (int q = 0; q < 8; q++) Gather<F, T>::load(table, c.idx[q], e[q]);
    float v[F];
#pragma unroll
    for (int f = 0; f < F; f++) {
        const float x00 = lerp(e[0][f], e[1][f], c.w[0]);
        const float x10 = lerp(e[2][f], e[3][f], c.w[0]);
        const float x01 = lerp(e[4][f], e[5][f], c.w[0]);
        const float x11 = lerp(e[6][f], e[7][f], c.w[0]);
        v[f] = lerp(lerp(x00, x10, c.w[1]), lerp(x01, x11, c.w[1]), c.w[2]);
    }
    Store<F, O>::store(out + n * (int64_t)(L * F) + l * F, v);
}

template <int F>
__global__ void __launch_bounds__(256) bwd_kernel(const __grid_constant__ Params P, const float4 *__restrict__ coords,
                                                  int64_t N, const float *__restrict__ dout,
                                                  float *__restrict__ dtable, int *__restrict__ flag, int l0, int lc) {
    __shared__ LevelSmem slv;
    load_levels(P, slv);
    const int L = P.L;
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n = gid / lc;
    if (n >= N) return;
    const int l = l0 + (int)(gid - n * lc);
    Cell8 c;
    const bool bad = cell_of(slv.get(l), __ldg(coords + n), c);
    if (bad && l == l0) atomicOr(flag, 1);
    float g[F];
    const float *gp = dout + n * (int64_t)(L * F) + l * F;
#pragma unroll
    for (int f = 0; f < F; f++) g[f] = __ldg(gp + f);
    const float wx[2] = {__fsub_rn(1.0f, c.w[0]), c.w[0]}, wy[2] = {__fsub_rn(1.0f, c.w[1]), c.w[1]};
    const float wz[2] = {__fsub_rn(1.0f, c.w[2]), c.w[2]};
#pragma unroll
    for (int q = 0; q < 8; q += 2) {
        const float Wyz = wy[(q >> 1) & 1] * wz[(q >> 2) & 1];
        const float W0 = wx[0] * Wyz, W1 = wx[1] * Wyz;
        float v0[F], v1[F];
#pragma unroll
        for (int f = 0; f < F; f++) { v0[f] = W0 * g[f]; v1[f] = W1 * g[f]; }
        red_pair<F>(dtable, nullptr, c.idx[q], c.idx[q + 1], v0, v1);
    }
}

__global__ void __launch_bounds__(256) indices_kernel(const __grid_constant__ Params P,
                                                      const float4 *__restrict__ coords, int64_t N,
                                                      uint32_t *__restrict__ idx, float *__restrict__ wout,
                                                      int *__restrict__ flag) {
    __shared__ LevelSmem slv;
    load_levels(P, slv);
    const int L = P.L;
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n = gid / L;
    if (n >= N) return;
    const int l = (int)(gid - n * L);
    Cell8 c;
    const bool bad = cell_of(slv.get(l), __ldg(coords + n), c);
    if (bad && l == 0) atomicOr(flag, 1);
#pragma unroll
    for (int q = 0; q < 8; q++) idx[gid * 8 + q] = c.idx[q];
    if (wout) {
        const float wx[2] = {1.0f - c.w[0], c.w[0]}, wy[2] = {1.0f - c.w[1], c.w[1]};
        const float wz[2] = {1.0f - c.w[2], c.w[2]};
#pragma unroll
        for (int q = 0; q < 8; q++) wout[gid * 8 + q] = wx[q & 1] * wy[(q >> 1) & 1] * wz[(q >> 2) & 1];
    }
}

}  // namespace mhe
}  // namespace fh
