// tiled_kernels.cuh -- the encode of coarse and mid levels over a SPATIALLY
// SORTED batch, with each level's working set staged in shared memory.
//
// Same method as encode_kernels.cuh (steps 1-4 of §3.2.4; Eq. 9,
// P:170; Eqs. 10-12; readings R2-R6); only the memory path
// differs.  A CTA takes a tile of S consecutive samples of a Morton-sorted
// order (fh_spatial_sort), so the tile covers a compact region of [0,1]^4.
// Cell location is monotone in each coordinate (R2: clamp, one rounded
// multiply, floor, clamp), so the cells the tile touches on level l lie in
// the box [cell(min p), cell(max p) + 1] per axis, computed once per tile
// from the per-axis min / max of its coordinates.  When that box of
// vertices fits in shared memory:
//   forward   the box's table entries are copied in once (coalesced rows
//             along x for Eq.-9 levels; one gather per vertex for hashed
//             levels), and the 16 corner reads of every sample come from
//             shared memory;
//   backward  see bwd_agg_kernel below (warp-aggregated reductions; the
//             backward does not stage boxes).
// Otherwise the tile falls back to the direct global path for that level.
// Results are those of the direct kernels: the forward is bit-identical
// (same values, same lerp tree), the backward differs only in fp32
// summation order.
#pragma once
#include "encode_kernels.cuh"

namespace fh {
namespace tiled {

constexpr int kThreads = 512;
constexpr int kMaxPer = 4;                     // samples per thread
constexpr int kMaxTile = kThreads * kMaxPer;   // 2048 samples per tile
constexpr int kWarps = kThreads / 32;

struct TileSet {
    int n;                  // number of tiled levels
    int id[kMaxLevels];     // their level ids
    int S;                  // samples per tile (<= kMaxTile)
    int box_bytes;          // dynamic shared memory for one level's box
};

__device__ __forceinline__ float clamp01(float p) { return (p >= 0.0f) ? fminf(p, 1.0f) : 0.0f; }

__device__ __forceinline__ bool out_of_domain(float4 p) {
    return !(p.x >= 0.f && p.x <= 1.f && p.y >= 0.f && p.y <= 1.f && p.z >= 0.f && p.z <= 1.f && p.w >= 0.f &&
             p.w <= 1.f);
}

// The tile's samples, held in registers: thread t owns sorted positions
// j0 + q * kThreads + t (q < kMaxPer), so lane-adjacent samples are
// neighbours in the sorted order.
struct Tile {
    float4 p[kMaxPer];      // clamped coordinates
    uint32_t n[kMaxPer];    // original sample index
    bool v[kMaxPer];
    float lo[4], hi[4];     // per-axis min / max of the clamped coordinates
};

__device__ __forceinline__ void load_tile(Tile &tl, const float4 *__restrict__ coords, const uint32_t *__restrict__ perm,
                                          int64_t j0, int64_t j1, int *flag, float (*red)[8]) {
    float mn[4] = {2.f, 2.f, 2.f, 2.f}, mx[4] = {-1.f, -1.f, -1.f, -1.f};
    bool bad = false;
#pragma unroll
    for (int q = 0; q < kMaxPer; q++) {
        const int64_t j = j0 + (int64_t)q * kThreads + threadIdx.x;
        tl.v[q] = j < j1;
        tl.n[q] = 0;
        tl.p[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (tl.v[q]) {
            const uint32_t n = perm ? __ldg(perm + j) : (uint32_t)j;
            const float4 p = __ldg(coords + n);
            bad |= out_of_domain(p);
            const float4 c = make_float4(clamp01(p.x), clamp01(p.y), clamp01(p.z), clamp01(p.w));
            tl.n[q] = n;
            tl.p[q] = c;
            mn[0] = fminf(mn[0], c.x); mx[0] = fmaxf(mx[0], c.x);
            mn[1] = fminf(mn[1], c.y); mx[1] = fmaxf(mx[1], c.y);
            mn[2] = fminf(mn[2], c.z); mx[2] = fmaxf(mx[2], c.z);
            mn[3] = fminf(mn[3], c.w); mx[3] = fmaxf(mx[3], c.w);
        }
    }
    if (bad) atomicOr(flag, 1);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int a = 0; a < 4; a++) {
            mn[a] = fminf(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
            mx[a] = fmaxf(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
        }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0)
#pragma unroll
        for (int a = 0; a < 4; a++) { red[w][a] = mn[a]; red[w][4 + a] = mx[a]; }
    __syncthreads();
#pragma unroll
    for (int a = 0; a < 4; a++) { tl.lo[a] = 2.f; tl.hi[a] = -1.f; }
    for (int k = 0; k < kWarps; k++)
#pragma unroll
        for (int a = 0; a < 4; a++) { tl.lo[a] = fminf(tl.lo[a], red[k][a]); tl.hi[a] = fmaxf(tl.hi[a], red[k][4 + a]); }
}

// The box of vertices the tile touches on one level.
struct Box {
    uint32_t lo[4];   // first vertex per axis
    uint32_t B[4];    // vertices per axis
    uint32_t V;       // total vertices (valid when fits)
    bool fits;
};

__device__ __forceinline__ Box box_of(const Level &lv, const Tile &tl, uint32_t max_vertices) {
    Box b;
    uint64_t V = 1;
#pragma unroll
    for (int a = 0; a < 4; a++) {
        uint32_t i0, i1;
        float w;
        bool bad = false;
        locate(tl.lo[a], lv.scale[a], lv.res[a], i0, w, bad);
        locate(tl.hi[a], lv.scale[a], lv.res[a], i1, w, bad);
        b.lo[a] = i0;
        b.B[a] = i1 - i0 + 2;
        V *= b.B[a];
    }
    b.fits = V <= (uint64_t)max_vertices;
    b.V = b.fits ? (uint32_t)V : 0u;
    return b;
}

// Global entry of vertex (X, Y, Z, Tt) of a level: Eq. 9, the brick order (R21) or the R5 hash
// (the same arithmetic as cell_of's corner loop).
__device__ __forceinline__ uint32_t vertex_entry(const Level &lv, uint32_t X, uint32_t Y, uint32_t Z, uint32_t Tt) {
    if (lv.hashed == 0) return lv.offset + X + Y * lv.sy + Z * lv.sz + Tt * lv.st;
    if (lv.hashed == 2) return lv.offset + brick_index(lv, X, Y, Z, Tt);
    return lv.offset + (hash_x(X, (Y * kPy) ^ (Z * kPz) ^ (Tt * kPt)) & lv.mask);
}

// Box vertex v (x fastest) -> global entry.
__device__ __forceinline__ uint32_t box_vertex_entry(const Level &lv, const Box &b, uint32_t v) {
    const uint32_t x = v % b.B[0];
    uint32_t r = v / b.B[0];
    const uint32_t y = r % b.B[1];
    r /= b.B[1];
    const uint32_t z = r % b.B[2];
    const uint32_t t = r / b.B[2];
    return vertex_entry(lv, b.lo[0] + x, b.lo[1] + y, b.lo[2] + z, b.lo[3] + t);
}

// Raw storage of one table entry (F features of type T).
template <int EB> struct RawT;
template <> struct RawT<2> { using type = unsigned short; };
template <> struct RawT<4> { using type = uint32_t; };
template <> struct RawT<8> { using type = uint2; };
template <> struct RawT<16> { using type = uint4; };
struct Raw32 { uint4 a, b; };
template <> struct RawT<32> { using type = Raw32; };

template <typename T, int F> using RawOf = typename RawT<F * (int)sizeof(T)>::type;

template <typename T, int F>
__device__ __forceinline__ RawOf<T, F> ld_raw_global(const T *__restrict__ table, uint32_t i) {
    using R = RawOf<T, F>;
    const R *p = reinterpret_cast<const R *>(table) + i;
    if constexpr (sizeof(R) == 32) {
        Raw32 r;
        r.a = __ldg(reinterpret_cast<const uint4 *>(p));
        r.b = __ldg(reinterpret_cast<const uint4 *>(p) + 1);
        return r;
    } else {
        return __ldg(p);
    }
}

template <typename T, int F>
__device__ __forceinline__ void raw_to_float(const RawOf<T, F> &r, float *o) {
    const T *e = reinterpret_cast<const T *>(&r);
#pragma unroll
    for (int f = 0; f < F; f++) {
        if constexpr (sizeof(T) == 4) o[f] = e[f];
        else o[f] = __half2float(e[f]);
    }
}

// Offsets of the 16 corners inside a box (R3 corner order).
__device__ __forceinline__ uint32_t corner_delta(int k, uint32_t Bx, uint32_t Bxy, uint32_t Bxyz) {
    return (uint32_t)(k & 1) + ((k >> 1) & 1) * Bx + ((k >> 2) & 1) * Bxy + ((k >> 3) & 1) * Bxyz;
}

// ------------------------------------------------------------ async copy
__device__ __forceinline__ void cp_async(void *smem_dst, const void *gmem_src, int bytes) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
    if (bytes == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem_src) : "memory");
    else if (bytes == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gmem_src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Copy the box's table entries into shared memory without waiting
// (cp.async: every thread issues all its copies back to back, so the
// gathers of hashed levels are all in flight at once).
template <typename T, int F>
__device__ __forceinline__ void fill_box(RawOf<T, F> *box, const Level &lv, const Box &b, const T *__restrict__ table) {
    using R = RawOf<T, F>;
    constexpr int EB = (int)sizeof(R);
    for (uint32_t v = threadIdx.x; v < b.V; v += kThreads) {
        const R *src = reinterpret_cast<const R *>(table) + box_vertex_entry(lv, b, v);
        if constexpr (EB == 2) {
            box[v] = *src;  // no 2-byte cp.async: plain copy
        } else if constexpr (EB == 32) {
            cp_async(&box[v], src, 16);
            cp_async(reinterpret_cast<char *>(&box[v]) + 16, reinterpret_cast<const char *>(src) + 16, 16);
        } else {
            cp_async(&box[v], src, EB);
        }
    }
    cp_async_commit();
}

// Largest box (vertices) a tile stages, relative to its sample count: above
// this the staged copy costs about as much as the direct corner gathers.
constexpr uint32_t kMaxBoxPerSample = 6;

// ------------------------------------------------------------ forward
// Levels are processed in TS order with two box buffers: while the tile
// blends level li from one buffer, the copies of level li+1's box land in
// the other.
template <int F, typename T, typename O>
__global__ void __launch_bounds__(kThreads, 1)
    fwd_tiled_kernel(const __grid_constant__ Params P, const __grid_constant__ TileSet TS,
                     const float4 *__restrict__ coords, int64_t N, const uint32_t *__restrict__ perm,
                     const T *__restrict__ table, uint32_t full_blocks, O *__restrict__ out, int *__restrict__ flag) {
    using R = RawOf<T, F>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t half = (uint32_t)(TS.box_bytes / 2 / (int)sizeof(R));  // vertices per buffer
    R *buf[2] = {reinterpret_cast<R *>(smem_raw), reinterpret_cast<R *>(smem_raw) + half};
    __shared__ Level slv[kMaxLevels];
    __shared__ float red[kWarps][8];
    load_levels(P, slv);
    const int64_t j0 = (int64_t)blockIdx.x * TS.S;
    const int64_t j1 = min(j0 + (int64_t)TS.S, N);
    Tile tl;
    load_tile(tl, coords, perm, j0, j1, flag, red);
    const int LF = P.L * F;
    const uint32_t maxv = min(half, kMaxBoxPerSample * (uint32_t)(j1 - j0));
    Box nb = box_of(slv[TS.id[0]], tl, maxv);
    if (nb.fits) fill_box<T, F>(buf[0], slv[TS.id[0]], nb, table);
    for (int li = 0; li < TS.n; li++) {
        const int l = TS.id[li];
        const Level &lv = slv[l];
        const Box b = nb;
        R *box = buf[li & 1];
        cp_async_wait_all();
        __syncthreads();  // box li landed; every thread is done with level li-1's buffer
        if (li + 1 < TS.n) {
            nb = box_of(slv[TS.id[li + 1]], tl, maxv);
            if (nb.fits) fill_box<T, F>(buf[(li + 1) & 1], slv[TS.id[li + 1]], nb, table);
        }
        const uint32_t Bxy = b.B[0] * b.B[1], Bxyz = Bxy * b.B[2];
#pragma unroll
        for (int q = 0; q < kMaxPer; q++) {
            if (!tl.v[q]) continue;
            float e[16][F];
            float w[4];
            if (b.fits) {
                uint32_t i[4];
                bool bad = false;
                locate(tl.p[q].x, lv.scale[0], lv.res[0], i[0], w[0], bad);
                locate(tl.p[q].y, lv.scale[1], lv.res[1], i[1], w[1], bad);
                locate(tl.p[q].z, lv.scale[2], lv.res[2], i[2], w[2], bad);
                locate(tl.p[q].w, lv.scale[3], lv.res[3], i[3], w[3], bad);
                const uint32_t base = (i[0] - b.lo[0]) + (i[1] - b.lo[1]) * b.B[0] + (i[2] - b.lo[2]) * Bxy +
                                      (i[3] - b.lo[3]) * Bxyz;
#pragma unroll
                for (int k = 0; k < 16; k++) raw_to_float<T, F>(box[base + corner_delta(k, b.B[0], Bxy, Bxyz)], e[k]);
            } else {
                Cell c;
                cell_of(lv, tl.p[q], c);
#pragma unroll
                for (int a = 0; a < 4; a++) w[a] = c.w[a];
                gather16<T, F>(table, nullptr, c.idx, e);
            }
            float val[F];
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
                val[f] = lerp(s[0], s[1], w[3]);
            }
            Store<F, O>::store(out + (int64_t)tl.n[q] * LF + l * F, val);
        }
    }
}

// ------------------------------------------------------------ backward
// Warp-aggregated reductions over a SORTED batch (the coarse levels, where
// many samples share a cell).  A warp takes 32 consecutive samples of the
// order at one level; lanes whose samples lie in the same cell (match on the
// 64-bit cell id) form a group with identical 16 corner entries.  Every lane
// stages its 16 F contributions W_c g in a per-warp shared-memory scratch,
// then the lanes of a group split the 16 corners among themselves, sum each
// corner over the group's members and issue ONE global reduction per
// (group, corner): reductions drop by the group size, and every lane reads
// about 16 contributions whatever the group size.  Warps whose lanes are all
// in distinct cells skip the scratch and reduce directly.  Shared-memory
// fp32 atomics are not used (they are CAS loops on sm_100).
constexpr int kAggThreads = 256;
constexpr int kAggWarps = kAggThreads / 32;

template <int F> struct AggLayout {
    static constexpr int kRow = 16 * F + (F >= 4 ? 4 : F);   // floats per lane (padded: bank spread)
    static constexpr int kWarpFloats = 32 * kRow;
};

template <int F>
__global__ void __launch_bounds__(kAggThreads)
    bwd_agg_kernel(const __grid_constant__ Params P, const __grid_constant__ LevelList LL,
                   const float4 *__restrict__ coords, int64_t N, const uint32_t *__restrict__ perm,
                   const float *__restrict__ dout, float *__restrict__ dtable, int *__restrict__ flag) {
    using A = AggLayout<F>;
    extern __shared__ __align__(16) float scratch[];   // kAggWarps * A::kWarpFloats (dynamic)
    __shared__ Level slv[kMaxLevels];
    load_levels(P, slv);
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * kAggThreads + threadIdx.x) >> 5;  // global warp
    const int li = (int)(gw % LL.n);
    const int64_t j = (gw / LL.n) * 32 + lane;
    if ((gw / LL.n) * 32 >= N) return;  // warp-uniform
    const int l = LL.id[li];
    const Level &lv = slv[l];
    const bool valid = j < N;
    Cell c;
    float g[F];
    unsigned long long key = ~0ull;
    if (valid) {
        const uint32_t n = __ldg(perm + j);
        const float4 p = __ldg(coords + n);
        if (cell_of(lv, p, c) && li == 0) atomicOr(flag, 1);
#pragma unroll
        for (int f = 0; f < F; f++) g[f] = __ldg(dout + (int64_t)n * (P.L * F) + l * F + f);
        // the cell's linear id (64-bit: unique on hashed levels too)
        uint32_t i[4];
        float w;
        bool bad = false;
        locate(fminf(fmaxf(p.x, 0.f), 1.f), lv.scale[0], lv.res[0], i[0], w, bad);
        locate(fminf(fmaxf(p.y, 0.f), 1.f), lv.scale[1], lv.res[1], i[1], w, bad);
        locate(fminf(fmaxf(p.z, 0.f), 1.f), lv.scale[2], lv.res[2], i[2], w, bad);
        locate(fminf(fmaxf(p.w, 0.f), 1.f), lv.scale[3], lv.res[3], i[3], w, bad);
        key = (((unsigned long long)i[3] * lv.res[2] + i[2]) * lv.res[1] + i[1]) * (unsigned long long)lv.res[0] + i[0];
    } else {
#pragma unroll
        for (int f = 0; f < F; f++) g[f] = 0.f;
#pragma unroll
        for (int k = 0; k < 16; k++) c.idx[k] = 0;
#pragma unroll
        for (int a = 0; a < 4; a++) c.w[a] = 0.f;
    }
    const uint32_t peers = __match_any_sync(0xffffffffu, key);
    const float wx[2] = {__fsub_rn(1.0f, c.w[0]), c.w[0]}, wy[2] = {__fsub_rn(1.0f, c.w[1]), c.w[1]};
    const float wz[2] = {__fsub_rn(1.0f, c.w[2]), c.w[2]}, wt[2] = {__fsub_rn(1.0f, c.w[3]), c.w[3]};
    if (__all_sync(0xffffffffu, __popc(peers) == 1)) {
        if (!valid) return;
#pragma unroll
        for (int k = 0; k < 16; k += 2) {
            const float Wyzt = wy[(k >> 1) & 1] * wz[(k >> 2) & 1] * wt[(k >> 3) & 1];
            const float W0 = wx[0] * Wyzt, W1 = wx[1] * Wyzt;
            float v0[F], v1[F];
#pragma unroll
            for (int f = 0; f < F; f++) { v0[f] = W0 * g[f]; v1[f] = W1 * g[f]; }
            red_pair<F>(dtable, nullptr, c.idx[k], c.idx[k + 1], v0, v1);
        }
        return;
    }
    float *S = scratch + (threadIdx.x >> 5) * A::kWarpFloats;
    float *row = S + lane * A::kRow;
#pragma unroll
    for (int k = 0; k < 16; k++) {
        const float W = wx[k & 1] * (wy[(k >> 1) & 1] * wz[(k >> 2) & 1] * wt[(k >> 3) & 1]);
        if constexpr (F >= 4) {
#pragma unroll
            for (int f = 0; f < F; f += 4)
                *reinterpret_cast<float4 *>(row + k * F + f) = make_float4(W * g[f], W * g[f + 1], W * g[f + 2], W * g[f + 3]);
        } else if constexpr (F == 2) {
            *reinterpret_cast<float2 *>(row + k * F) = make_float2(W * g[0], W * g[1]);
        } else {
            row[k] = W * g[0];
        }
    }
    __syncwarp();
    if (!valid) return;
    const int gs = __popc(peers);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    for (int k = rank; k < 16; k += gs) {
        float acc[F];
#pragma unroll
        for (int f = 0; f < F; f++) acc[f] = 0.f;
        uint32_t mm = peers;
        while (mm) {
            const int m = __ffs(mm) - 1;
            mm &= mm - 1;
            const float *src = S + m * A::kRow + k * F;
#pragma unroll
            for (int f = 0; f < F; f++) acc[f] += src[f];
        }
        red_entry<F>(dtable, c.idx[k], acc);
    }
}

}  // namespace tiled
}  // namespace fh
