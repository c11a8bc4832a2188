// encode_device.cuh -- device functions of the F-Hash Tesseract encode
// (cell location, MPHF / hash indices, the pair gathers, the quadrilinear
// blend), shared by the encode kernels (encode_kernels.cuh) and the fused
// inference kernel (infer_kernels.cuh) so both compute bit-identical values.
//
// Paper: §3.2.4 "Input Encoding", steps 1-4, Eq. 9 F-Hash
// (P:170), Eqs. 10-12 quadrilinear interpolation; readings
// R2 (cell location), R3 (corner order), R5 (capped hash), R6 (Eq. 12).
//
// Thread mapping: one thread per (sample n, level l), l fastest, so the
// L threads of a sample are adjacent lanes: the coordinate load is one
// broadcast per sample, the output row [n][L*F] is written contiguously by
// adjacent lanes, and each thread keeps its 16 corner gathers in flight
// together (16 independent loads per thread).  Level metadata is staged in
// shared memory because lanes of a warp read different levels.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "encode_params.h"

namespace fh {

// R5 hash primes (Teschner et al. spatial hash; the t prime is
// this build's choice).
constexpr uint32_t kPy = 2654435761u;
constexpr uint32_t kPz = 805459861u;
constexpr uint32_t kPt = 2246822519u;

// R5: a capped level's bucket of vertex (X, Y, Z, T) is
//   (X + (Y kPy ^ Z kPz ^ T kPt)) mod 2^32 mod T_l
// -- x enters additively, so x-neighbours stay adjacent entries as in Eq. 9
// (the pair layout of DESIGN.md §8.1 then covers every x-pair).
#ifndef FH_HASH_XADD
#define FH_HASH_XADD 1
#endif
__device__ __forceinline__ uint32_t hash_x(uint32_t X, uint32_t yzt) {
#if FH_HASH_XADD
    return X + yzt;
#else
    return X ^ yzt;
#endif
}

// Steps 1-2 on one axis (R2): clamp to [0,1] (NaN -> 0), one IEEE fp32
// multiply s = p*(R-1), i = clamp(floor s, 0, R-2), w = s - i (exact).
__device__ __forceinline__ void locate(float p, float scale, uint32_t R, uint32_t &i, float &w,
                                       bool &bad) {
    float pc = p;
    if (!(p >= 0.0f)) { pc = 0.0f; bad = true; }
    else if (p > 1.0f) { pc = 1.0f; bad = true; }
    const float s = __fmul_rn(pc, scale);
    int ii = __float2int_rd(s);
    ii = min(ii, (int)R - 2);
    ii = max(ii, 0);
    i = (uint32_t)ii;
    w = __fsub_rn(s, __int2float_rn(ii));
}

// NEXT-2 ("Other linearizations like Morton and Z-order can also be
// used to construct F-Hash with preserved locality"; reading R21): brick
// order of a bijective level -- 2x2x2x2-vertex bricks (clipped to e_a = 1 at
// an odd grid edge) enumerated row-major, vertices row-major inside a brick.
// With b = v >> 1, i = v & 1, e = min(2, R - 2b) per axis:
//   idx = 2 b_t RxRyRz + 2 b_z RxRy e_t + 2 b_y Rx e_z e_t + 2 b_x e_y e_z e_t
//       + ((i_t e_z + i_z) e_y + i_y) e_x + i_x
// The 16 corners of a cell at even coordinates are one brick, i.e. 16
// consecutive entries (one 128-byte line at 8-byte entries).
__device__ __forceinline__ uint32_t brick_index(const Level &lv, uint32_t X, uint32_t Y, uint32_t Z, uint32_t T) {
    const uint32_t bx = X >> 1, by = Y >> 1, bz = Z >> 1, bt = T >> 1;
    const uint32_t ex = min(2u, lv.res[0] - 2u * bx), ey = min(2u, lv.res[1] - 2u * by);
    const uint32_t ez = min(2u, lv.res[2] - 2u * bz), et = min(2u, lv.res[3] - 2u * bt);
    return 2u * bt * lv.st + 2u * bz * lv.sz * et + 2u * by * lv.sy * ez * et + 2u * bx * ey * ez * et +
           (((T & 1u) * ez + (Z & 1u)) * ey + (Y & 1u)) * ex + (X & 1u);
}

// Entry of lattice vertex (X, Y, Z, T) of a level: Eq. 9, the brick order
// (R21) or the R5 hash -- the per-vertex form of cell_of's corner indices
// (used by encoding_stats, stats.cuh).
__device__ __forceinline__ uint32_t vertex_entry(const Level &lv, uint32_t X, uint32_t Y, uint32_t Z, uint32_t Tt) {
    if (lv.hashed == 0) return lv.offset + X + Y * lv.sy + Z * lv.sz + Tt * lv.st;
    if (lv.hashed == 2) return lv.offset + brick_index(lv, X, Y, Z, Tt);
    return lv.offset + (hash_x(X, (Y * kPy) ^ (Z * kPz) ^ (Tt * kPt)) & lv.mask);
}

// Cell of one (sample, level): base indices and fractions.
struct Cell {
    uint32_t idx[16];
    float w[4];
};

// Step 3: the 16 corner entries.  Bijective levels: Eq. 9 at the cell
// origin, each corner adds bx + by*Rx + bz*Rx*Ry + bt*Rx*Ry*Rz ("a single
// look-up ... through simple shifting").  Hashed levels: R5.
__device__ __forceinline__ bool cell_of(const Level &lv, float4 p, Cell &c) {
    uint32_t ix, iy, iz, it;
    bool bad = false;
    locate(p.x, lv.scale[0], lv.res[0], ix, c.w[0], bad);
    locate(p.y, lv.scale[1], lv.res[1], iy, c.w[1], bad);
    locate(p.z, lv.scale[2], lv.res[2], iz, c.w[2], bad);
    locate(p.w, lv.scale[3], lv.res[3], it, c.w[3], bad);
    if (lv.hashed == 0) {
        const uint32_t base = lv.offset + ix + iy * lv.sy + iz * lv.sz + it * lv.st;
#pragma unroll
        for (int k = 0; k < 16; k++)
            c.idx[k] = base + (k & 1) + ((k >> 1) & 1) * lv.sy + ((k >> 2) & 1) * lv.sz +
                       ((k >> 3) & 1) * lv.st;
    } else if (lv.hashed == 2) {
#pragma unroll
        for (int k = 0; k < 16; k++)
            c.idx[k] = lv.offset + brick_index(lv, ix + (k & 1), iy + ((k >> 1) & 1), iz + ((k >> 2) & 1),
                                               it + ((k >> 3) & 1));
    } else {
        const uint32_t hx0 = ix, hx1 = ix + 1;
        const uint32_t hy0 = iy * kPy, hy1 = (iy + 1) * kPy;
        const uint32_t hz0 = iz * kPz, hz1 = (iz + 1) * kPz;
        const uint32_t ht0 = it * kPt, ht1 = (it + 1) * kPt;
#pragma unroll
        for (int k = 0; k < 16; k++) {
            const uint32_t h = hash_x(((k & 1) ? hx1 : hx0), (((k >> 1) & 1) ? hy1 : hy0) ^
                                                                 (((k >> 2) & 1) ? hz1 : hz0) ^ (((k >> 3) & 1) ? ht1 : ht0));
            c.idx[k] = lv.offset + (h & lv.mask);
        }
    }
    return bad;
}

// ------------------------------------------------------------ gathers
// Load the F features of one entry as floats.  F*sizeof(T) <= 16 bytes is
// one vector load through the read-only path.
template <int F, typename T> struct Gather;

template <> struct Gather<1, float> {
    static __device__ __forceinline__ void load(const float *t, uint32_t i, float *o) { o[0] = __ldg(t + i); }
};
template <> struct Gather<2, float> {
    static __device__ __forceinline__ void load(const float *t, uint32_t i, float *o) {
        const float2 v = __ldg(reinterpret_cast<const float2 *>(t) + i);
        o[0] = v.x; o[1] = v.y;
    }
};
template <> struct Gather<4, float> {
    static __device__ __forceinline__ void load(const float *t, uint32_t i, float *o) {
        const float4 v = __ldg(reinterpret_cast<const float4 *>(t) + i);
        o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    }
};
template <> struct Gather<8, float> {
    static __device__ __forceinline__ void load(const float *t, uint32_t i, float *o) {
        const float4 a = __ldg(reinterpret_cast<const float4 *>(t) + 2 * (size_t)i);
        const float4 b = __ldg(reinterpret_cast<const float4 *>(t) + 2 * (size_t)i + 1);
        o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w; o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
    }
};
template <> struct Gather<1, __half> {
    static __device__ __forceinline__ void load(const __half *t, uint32_t i, float *o) {
        o[0] = __half2float(__ldg(t + i));
    }
};
template <> struct Gather<2, __half> {
    static __device__ __forceinline__ void load(const __half *t, uint32_t i, float *o) {
        const __half2 v = __ldg(reinterpret_cast<const __half2 *>(t) + i);
        const float2 f = __half22float2(v);
        o[0] = f.x; o[1] = f.y;
    }
};
template <> struct Gather<4, __half> {
    static __device__ __forceinline__ void load(const __half *t, uint32_t i, float *o) {
        const uint2 v = __ldg(reinterpret_cast<const uint2 *>(t) + i);
        const float2 a = __half22float2(*reinterpret_cast<const __half2 *>(&v.x));
        const float2 b = __half22float2(*reinterpret_cast<const __half2 *>(&v.y));
        o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
    }
};
template <> struct Gather<8, __half> {
    static __device__ __forceinline__ void load(const __half *t, uint32_t i, float *o) {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(t) + i);
        const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const float2 f = __half22float2(*reinterpret_cast<const __half2 *>(&u[k]));
            o[2 * k] = f.x; o[2 * k + 1] = f.y;
        }
    }
};

// ------------------------------------------------------------ stores
// The output rows and the coords / dout rows are streamed once per pass:
// evict-first (st.global.cs / ld.global.cs) so they do not push the level
// group's tables (forward) or gradients (backward) out of the L2.
template <int F, typename O> struct Store;
template <int F> struct Store<F, float> {
    static __device__ __forceinline__ void store(float *o, const float *v) {
        if constexpr (F == 1) __stcs(o, v[0]);
        else if constexpr (F == 2) __stcs(reinterpret_cast<float2 *>(o), make_float2(v[0], v[1]));
        else {
#pragma unroll
            for (int k = 0; k < F; k += 4)
                __stcs(reinterpret_cast<float4 *>(o + k), make_float4(v[k], v[k + 1], v[k + 2], v[k + 3]));
        }
    }
};
template <int F> struct Store<F, __nv_bfloat16> {
    static __device__ __forceinline__ void store(__nv_bfloat16 *o, const float *v) {
        if constexpr (F == 1) o[0] = __float2bfloat16_rn(v[0]);
        else if constexpr (F == 2) {
            __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]);
            __stcs(reinterpret_cast<unsigned int *>(o), *reinterpret_cast<unsigned int *>(&a));
        } else if constexpr (F == 4) {
            __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]), b = __floats2bfloat162_rn(v[2], v[3]);
            uint2 u;
            u.x = *reinterpret_cast<uint32_t *>(&a);
            u.y = *reinterpret_cast<uint32_t *>(&b);
            __stcs(reinterpret_cast<uint2 *>(o), u);
        } else {
            uint4 u;
            uint32_t *pu = reinterpret_cast<uint32_t *>(&u);
#pragma unroll
            for (int k = 0; k < 4; k++) {
                __nv_bfloat162 a = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
                pu[k] = *reinterpret_cast<uint32_t *>(&a);
            }
            __stcs(reinterpret_cast<uint4 *>(o), u);
        }
    }
};

// lerp (1-w) a + w b as fma(w, b, (1-w)*a): each rounding is relative to
// (1-w)|a| + w|b|, so four nested levels stay within ~12 u * sum_c W_c|E_c|
// (u = 2^-24), inside the 1e-6 forward bar.  The form
// a + w (b - a) is NOT used: at w ~ 1 it leaves an error of ulp(a) against
// a result of size |b|.
__device__ __forceinline__ float lerp(float a, float b, float w) {
    return fmaf(w, b, __fmul_rn(__fsub_rn(1.0f, w), a));
}

__device__ __forceinline__ void load_levels(const Params &P, Level *s) {
    const int n = P.L * (int)(sizeof(Level) / 4);
    const uint32_t *src = reinterpret_cast<const uint32_t *>(P.lv);
    uint32_t *dst = reinterpret_cast<uint32_t *>(s);
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
    __syncthreads();
}

// Level table in shared memory, transposed in 16-byte quarters: quarter q of
// level l at g[q][l].  The lanes of a warp read up to 16 different levels
// (l fastest in the thread mapping); with the 64-byte Level stride an
// LDS.128 of 16 levels hit only two bank groups (8 wavefronts; ncu showed
// 34 M shared wavefronts, 30 % of the forward's LSU data pipe), transposed
// it is 256 contiguous bytes (2 wavefronts).
struct LevelSmem {
    uint4 g[4][kMaxLevels];
    __device__ __forceinline__ Level get(int l) const {
        Level v;
        uint4 *d = reinterpret_cast<uint4 *>(&v);
#pragma unroll
        for (int q = 0; q < 4; q++) d[q] = g[q][l];
        return v;
    }
};
static_assert(sizeof(Level) == 64, "Level is four 16-byte quarters");

__device__ __forceinline__ void load_levels(const Params &P, LevelSmem &s) {
    const uint4 *src = reinterpret_cast<const uint4 *>(P.lv);
    for (int i = threadIdx.x; i < 4 * P.L; i += blockDim.x) s.g[i & 3][i >> 2] = src[i];
    __syncthreads();
}

// ------------------------------------------------------------ pair gather
// The 16 corners are 8 x-adjacent pairs.  Eq. 9 puts a pair at entries
// (i, i+1); the R5 hash puts it at (h, h') with h' = h^1 when X is even.
// When the two entries form one aligned 2-entry chunk (i1 == i0 ^ 1, about
// half the pairs) they are fetched with one load of twice the entry width
// (wider 32-byte block loads measured slower).
template <typename T, int F> struct EntryTraits {
    static constexpr int kBytes = F * (int)sizeof(T);
    static constexpr int kWords = kBytes >= 4 ? kBytes / 4 : 1;        // 32-bit words per entry
};

struct Block32 { uint32_t w[8]; };

__device__ __forceinline__ Block32 ld_block(const void *base, uint32_t b) {
    Block32 r;
    const char *p = reinterpret_cast<const char *>(base) + (size_t)b * 32;
    asm("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]), "=r"(r.w[6]),
          "=r"(r.w[7])
        : "l"(p));
    return r;
}

// Raw loads for the pair gather: one entry (W words) or an aligned pair of
// entries (2W words) through the read-only path.
template <int W>
__device__ __forceinline__ void ld_entry(const void *table, uint32_t i, uint32_t *o) {
    if constexpr (W == 1) {
        o[0] = __ldg(reinterpret_cast<const uint32_t *>(table) + i);
    } else if constexpr (W == 2) {
        const uint2 v = __ldg(reinterpret_cast<const uint2 *>(table) + i);
        o[0] = v.x; o[1] = v.y;
    } else {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(table) + i);
        o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    }
}
template <int W>
__device__ __forceinline__ void ld_pair(const void *table, uint32_t chunk, uint32_t *o) {
    if constexpr (W == 1) {
        const uint2 v = __ldg(reinterpret_cast<const uint2 *>(table) + chunk);
        o[0] = v.x; o[1] = v.y;
    } else if constexpr (W == 2) {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(table) + chunk);
        o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    } else {
        const Block32 b = ld_block(table, chunk);
#pragma unroll
        for (int j = 0; j < 8; j++) o[j] = b.w[j];
    }
}
// F features of type T packed in 32-bit words -> floats.
template <typename T, int F>
__device__ __forceinline__ void words_to_float(const uint32_t *w, float *o) {
    if constexpr (sizeof(T) == 4) {
#pragma unroll
        for (int j = 0; j < F; j++) o[j] = __uint_as_float(w[j]);
    } else {
#pragma unroll
        for (int j = 0; j < F / 2; j++) {
            const float2 f = __half22float2(*reinterpret_cast<const __half2 *>(&w[j]));
            o[2 * j] = f.x; o[2 * j + 1] = f.y;
        }
    }
}

// Gather the 16 corner entries of one (sample, level) into e[16][F].
// (full_blocks, the number of complete 32-byte blocks of the table, is not
// needed by the pair loads, which never leave the two entries' chunk.)
template <typename T, int F>
__device__ __forceinline__ void gather16(const T *__restrict__ table, const T *__restrict__ tsh,
                                         const uint32_t (&idx)[16], float (&e)[16][F]) {
    using Tr = EntryTraits<T, F>;
    if constexpr (Tr::kBytes == 4 || Tr::kBytes == 8 || Tr::kBytes == 16) {
        // x-pair in ONE load of the aligned 2-entry chunk when both entries
        // share it (i1 == i0 ^ 1: about half the pairs on Eq. 9 and on the R5
        // hash, whose x-neighbours differ in the low bits), else two entry
        // loads into the same registers.  1.5 L1 requests per pair instead of
        // 2, no extra registers.  Measured on B200: cfg2 fwd 0.763 -> 0.738
        // ms, cfg4 fwd 3.017 -> 2.841 ms.
        constexpr int W = Tr::kWords;          // 32-bit words per entry (1, 2, 4)
        uint32_t r[8][2 * W];
#pragma unroll
        for (int k = 0; k < 8; k++) {
            const uint32_t i0 = idx[2 * k], i1 = idx[2 * k + 1];
            if (tsh && i1 == i0 + 1u && (i0 & 1u)) {
                ld_pair<W>(tsh, i0 >> 1, r[k]);      // odd-aligned pair: the shifted copy's chunk
            } else if ((i0 ^ i1) == 1u) {
                ld_pair<W>(table, i0 >> 1, r[k]);
            } else {
                ld_entry<W>(table, i0, r[k]);
                ld_entry<W>(table, i1, r[k] + W);
            }
        }
#pragma unroll
        for (int k = 0; k < 8; k++) {
            const uint32_t i0 = idx[2 * k], i1 = idx[2 * k + 1];
            const bool swap = ((i0 ^ i1) == 1u) && (i0 & 1u);  // the chunk holds (i1, i0)
            uint32_t wa[W], wb[W];
#pragma unroll
            for (int j = 0; j < W; j++) {
                wa[j] = swap ? r[k][W + j] : r[k][j];
                wb[j] = swap ? r[k][j] : r[k][W + j];
            }
            words_to_float<T, F>(wa, e[2 * k]);
            words_to_float<T, F>(wb, e[2 * k + 1]);
        }
    } else {   // 2- and 32-byte entries: one load per corner
#pragma unroll
        for (int k = 0; k < 16; k++) Gather<F, T>::load(table, idx[k], e[k]);
    }
}

// Step 4 (Eqs. 10-12) on the 16 gathered corners e[c][f] (c = bx + 2 by +
// 4 bz + 8 bt, R3): trilinear per time slice (8 x-lerps -> 4 y -> 2 z),
// then the temporal lerp (R6), per feature.
template <int F>
__device__ __forceinline__ void blend16(const float (&e)[16][F], const float (&w)[4], float (&v)[F]) {
#pragma unroll
    for (int f = 0; f < F; f++) {
        float s[2];
#pragma unroll
        for (int bt = 0; bt < 2; bt++) {
            const int o = bt * 8;
            const float x00 = lerp(e[o + 0][f], e[o + 1][f], w[0]);
            const float x10 = lerp(e[o + 2][f], e[o + 3][f], w[0]);
            const float x01 = lerp(e[o + 4][f], e[o + 5][f], w[0]);
            const float x11 = lerp(e[o + 6][f], e[o + 7][f], w[0]);
            const float y0 = lerp(x00, x10, w[1]);
            const float y1 = lerp(x01, x11, w[1]);
            s[bt] = lerp(y0, y1, w[2]);
        }
        v[f] = lerp(s[0], s[1], w[3]);
    }
}

}  // namespace fh
