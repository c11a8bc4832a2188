// encode_kernels.cuh -- sm_100a kernels of the F-Hash Tesseract encode.
//
// Paper: §3.2.4 "Input Encoding", steps 1-4, Eq. 9 F-Hash
// (P:170), Eqs. 10-12 quadrilinear interpolation; readings
// R2 (cell location), R3 (corner order), R5 (capped hash), R6 (Eq. 12).
// The per-(sample, level) arithmetic is in encode_device.cuh.
#pragma once
#include "encode_device.cuh"

namespace fh {

// ------------------------------------------------------------ forward
// Step 4 (Eqs. 10-12): trilinear per time slice (8 x-lerps -> 4 y -> 2 z),
// then the temporal lerp (R6), per feature.
// Occupancy: the gathers are latency-bound at the L1->L2 request port, so
// resident warps matter.  F <= 2 fits 64 registers (4 CTAs of 256 per SM;
// cfg2 fwd 0.633 -> 0.605 ms); wider entries keep 2 (their 16 corners need
// the registers: cfg4 2.97 -> 3.17 ms when capped at 64).
template <int F>
struct FwdMinBlocks { static constexpr int value = F <= 2 ? 4 : 2; };

template <int F, typename T, typename O>
__global__ void __launch_bounds__(256, FwdMinBlocks<F>::value) fwd_kernel(const __grid_constant__ Params P,
                                                  const float4 *__restrict__ coords, int64_t N,
                                                  const T *__restrict__ table, const T *__restrict__ tsh,
                                                  O *__restrict__ out, int *__restrict__ flag,
                                                  const __grid_constant__ LevelList LL) {
    // the levels LL.id[0..LL.n) of every sample (a level group: see DESIGN.md §8)
    __shared__ LevelSmem slv;
    load_levels(P, slv);
    const int L = P.L;
    const int lc = LL.n;
    // F >= 4: a capped, grid-stride grid (FwdGrid) -- each CTA sets up its
    // level table once and works through many (sample, level) items; F <= 2
    // keeps one item per thread (its 64-register budget would spill the loop)
    constexpr bool kLoop = F >= 4;
    const int64_t total = N * lc, stride = kLoop ? (int64_t)gridDim.x * blockDim.x : total;
#pragma unroll 1
    for (int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gid < total; gid += stride) {
        const int64_t j = gid / lc;
        const int li = (int)(gid - j * lc);
        const int l = LL.id[li];
        const int64_t n = j;
        const Level lv = slv.get(l);
        const float4 p = __ldcs(coords + n);
        Cell c;
        const bool bad = cell_of(lv, p, c);
        if (bad && li == 0) atomicOr(flag, 1);
        float e[16][F];
        gather16<T, F>(table, lv.tshift ? tsh : nullptr, c.idx, e);
        float v[F];
        blend16<F>(e, c.w, v);
        Store<F, O>::store(out + n * (int64_t)(L * F) + l * F, v);
        if constexpr (!kLoop) break;
    }
}

// ------------------------------------------------------------ backward
// dtable[idx_c] += W_c * g (adjoint of the forward), W_c = prod of the four
// per-axis factors (bx ? wx : 1-wx) ... in fp32.  Vector reductions carry the
// F features of an entry in one op (REDG.E.ADD.F32x2/x4); for F <= 2 an
// x-pair that falls in one 16-byte chunk is ONE red.v4 (zeros in unused
// lanes are exact no-ops), so a pair costs 1.5 reduction ops on average.
__device__ __forceinline__ void red4(float *p, float a, float b, float c, float d) {
    atomicAdd(reinterpret_cast<float4 *>(p), make_float4(a, b, c, d));
}

template <int F>
__device__ __forceinline__ void red_entry(float *dtable, uint32_t i, const float *v) {
    if constexpr (F == 1) atomicAdd(dtable + i, v[0]);
    else if constexpr (F == 2) atomicAdd(reinterpret_cast<float2 *>(dtable) + i, make_float2(v[0], v[1]));
    else {
#pragma unroll
        for (int k = 0; k < F; k += 4) red4(dtable + (size_t)i * F + k, v[k], v[k + 1], v[k + 2], v[k + 3]);
    }
}

template <int F>
__device__ __forceinline__ void red_pair(float *dtable, float *gsh, uint32_t i0, uint32_t i1, const float *v0,
                                         const float *v1) {
    // gsh (optional): the shifted gradient scratch, holding entry j at float
    // offset j*F - 2 (kShiftFloats), so that an x-pair (i, i+1) straddling a
    // 16-byte chunk of dtable lies in ONE 16-byte chunk of gsh; merged back
    // by merge_shift_kernel.
    if constexpr (F == 2) {
        if ((i0 >> 1) == (i1 >> 1)) {  // both entries in one 16-byte chunk
            float *p = dtable + (size_t)(i0 & ~1u) * 2;
            if (i0 & 1) red4(p, v1[0], v1[1], v0[0], v0[1]);
            else red4(p, v0[0], v0[1], v1[0], v1[1]);
            return;
        }
        if (gsh && i1 == i0 + 1u) {    // i0 odd: chunk (i0, i0+1) of gsh
            red4(gsh + (size_t)i0 * 2 - 2, v0[0], v0[1], v1[0], v1[1]);
            return;
        }
    } else if constexpr (F == 1) {
        if (gsh && i1 == i0 + 1u && (i0 & 3u) == 3u) {   // gsh chunk (i0-1 .. i0+2)
            red4(gsh + (size_t)i0 - 3, 0.f, v0[0], v1[0], 0.f);
            return;
        }
        if ((i0 >> 2) == (i1 >> 2)) {
            const uint32_t a = i0 & 3, b = i1 & 3;
            float q[4];
#pragma unroll
            for (int j = 0; j < 4; j++) q[j] = (a == (uint32_t)j ? v0[0] : 0.f) + (b == (uint32_t)j ? v1[0] : 0.f);
            red4(dtable + (i0 & ~3u), q[0], q[1], q[2], q[3]);
            return;
        }
    }
    red_entry<F>(dtable, i0, v0);
    red_entry<F>(dtable, i1, v1);
}

// dtable[m + 2] += gsh[m] over float range [m0, m1) of the shifted scratch
// (m0 even), by threads t0, t0 + nt, ...: the merge of the pair layout
// (merge_shift_kernel, or the first CTAs of the next group's bwd_kernel).
__device__ __forceinline__ void merge_shift_range(float *__restrict__ dtable, float *__restrict__ gsh, int64_t m0,
                                                  int64_t m1, int64_t t0, int64_t nt) {
    const int64_t q0 = m0 >> 1, q1 = (m1 + 1) >> 1;
    float2 *g2 = reinterpret_cast<float2 *>(gsh);
    float2 *d2 = reinterpret_cast<float2 *>(dtable) + 1;
    for (int64_t q = q0 + t0; q < q1; q += nt) {
        const float2 v = g2[q];
        if (v.x != 0.f || v.y != 0.f) {
            float2 d = d2[q];
            d.x += v.x;
            d.y += v.y;
            d2[q] = d;
        }
    }
}

// A merge carried by the first `ctas` CTAs of a backward launch: the
// previous level group's shifted partial sums, folded while this group's
// reductions run (its ranges are disjoint from this group's).
struct MergeJob {
    float *gsh;
    int64_t m0, m1;
    int ctas;
};

// RANGED: only corners whose entry lies in [lo, lo + span) are reduced --
// one of several passes over a level whose gradients exceed the L2 budget,
// each pass's range staying L2-resident (the index math and dout are
// repeated per pass, the reductions are not).
template <int F, bool RANGED = false>
__global__ void __launch_bounds__(256) bwd_kernel(const __grid_constant__ Params P,
                                                  const float4 *__restrict__ coords, int64_t N,
                                                  const float *__restrict__ dout, const DoutLayout dl,
                                                  float *__restrict__ dtable, float *__restrict__ gsh,
                                                  int *__restrict__ flag, const __grid_constant__ LevelList LL,
                                                  uint32_t lo = 0,
                                                  uint32_t span = 0, uint32_t rep_n = 0, int64_t rep_stride = 0,
                                                  const MergeJob mj = MergeJob{nullptr, 0, 0, 0},
                                                  const RepSpec rs = RepSpec{0, {}, {}, {}, {}}) {
    if ((int)blockIdx.x < mj.ctas) {   // the previous group's merge (see MergeJob)
        merge_shift_range(dtable, mj.gsh, mj.m0, mj.m1, (int64_t)blockIdx.x * blockDim.x + threadIdx.x,
                          (int64_t)mj.ctas * blockDim.x);
        return;
    }
    __shared__ LevelSmem slv;
    load_levels(P, slv);
    const int lc = LL.n;
    const int64_t bid = (int64_t)blockIdx.x - mj.ctas;
    const int64_t gid = bid * blockDim.x + threadIdx.x;
    // replicated pass (one contended level): CTA b reduces into copy b % rep_n
    if (rep_n > 1) dtable += (int64_t)(bid % rep_n) * rep_stride;
    const int64_t j = gid / lc;
    if (j >= N) return;
    const int li = (int)(gid - j * lc);
    const int l = LL.id[li];
    const int64_t n = j;
    const Level lv = slv.get(l);
    const float4 p = __ldcs(coords + n);
    Cell c;
    const bool bad = cell_of(lv, p, c);
    if (bad && li == 0) atomicOr(flag, 1);
    float g[F];
    const float *gp = dout + n * dl.ns + l * dl.ls;
    if constexpr (F == 2) {
        const float2 q = __ldcs(reinterpret_cast<const float2 *>(gp));
        g[0] = q.x; g[1] = q.y;
    } else if constexpr (F % 4 == 0) {
#pragma unroll
        for (int f = 0; f < F; f += 4) {
            const float4 q = __ldcs(reinterpret_cast<const float4 *>(gp + f));
            g[f] = q.x; g[f + 1] = q.y; g[f + 2] = q.z; g[f + 3] = q.w;
        }
    } else {
#pragma unroll
        for (int f = 0; f < F; f++) g[f] = __ldcs(gp + f);
    }
    const float wx[2] = {__fsub_rn(1.0f, c.w[0]), c.w[0]}, wy[2] = {__fsub_rn(1.0f, c.w[1]), c.w[1]};
    const float wz[2] = {__fsub_rn(1.0f, c.w[2]), c.w[2]}, wt[2] = {__fsub_rn(1.0f, c.w[3]), c.w[3]};
    float *dt = dtable;   // or this CTA's replicated copy of a contended level (RepSpec)
#pragma unroll
    for (int q = 0; q < kMaxInRep; q++)   // constant indices: the spec stays in parameter space
        if (q < rs.n && l == rs.lvl[q]) dt = rs.base[q] + (int64_t)((uint32_t)bid % (uint32_t)rs.R[q]) * rs.stride[q];
#pragma unroll
    for (int k = 0; k < 16; k += 2) {
        const float Wyzt = wy[(k >> 1) & 1] * wz[(k >> 2) & 1] * wt[(k >> 3) & 1];
        const float W0 = wx[0] * Wyzt, W1 = wx[1] * Wyzt;
        float v0[F], v1[F];
#pragma unroll
        for (int f = 0; f < F; f++) { v0[f] = W0 * g[f]; v1[f] = W1 * g[f]; }
        if constexpr (RANGED) {
            const bool in0 = c.idx[k] - lo < span, in1 = c.idx[k + 1] - lo < span;
            if (in0 && in1) {
                red_pair<F>(dt, gsh, c.idx[k], c.idx[k + 1], v0, v1);
            } else {
                if (in0) red_entry<F>(dt, c.idx[k], v0);
                if (in1) red_entry<F>(dt, c.idx[k + 1], v1);
            }
        } else {
            red_pair<F>(dt, gsh, c.idx[k], c.idx[k + 1], v0, v1);
        }
    }
}

// ------------------------------------------------------------ shifted scratch
// The pair layout of DESIGN.md §8.1: an x-pair of entries (i, i+1) with i
// odd (F = 2; i = 3 mod 4 for F = 1) straddles a 16-byte chunk of the table.
// The forward reads it from a copy of the table shifted by one entry; the
// backward reduces it into a scratch gsh shifted by two floats
// (kShiftFloats), which this kernel adds back, dtable[m + 2] += gsh[m], over
// float range [m0, m1) of gsh (m0 even; the host zeroes that range right
// before the group's backward launch).
constexpr int kShiftFloats = 2;

__global__ void __launch_bounds__(256) merge_shift_kernel(float *__restrict__ dtable, float *__restrict__ gsh,
                                                          int64_t m0, int64_t m1) {
    merge_shift_range(dtable, gsh, m0, m1, (int64_t)blockIdx.x * blockDim.x + threadIdx.x,
                      (int64_t)gridDim.x * blockDim.x);
}

// Sum of the replicated copies of one level into dtable (the replicated
// backward pass): dst[i] += sum_r src[r * stride + i], i < count.
__global__ void __launch_bounds__(256) rep_reduce_kernel(float *__restrict__ dst, const float *__restrict__ src,
                                                         int R, int64_t stride, int64_t count) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        float v = 0.f;
        for (int r = 0; r < R; r++) v += src[r * stride + i];
        if (v != 0.f) dst[i] += v;
    }
}

// ------------------------------------------------------------ small levels
// The fold schedule (Eqs. 4-8) ends in tiny levels (down to 2x2x2x2 = 16
// entries) that receive ~16 N contributions: global reductions to the same
// few addresses serialise in the L2 atomic units.  These levels are
// accumulated per CTA in shared memory instead (CTA-private copies; the
// shared-memory fp32 atomics are CAS loops on sm_100a), the tiniest (<= 64
// floats) in one private copy per LANE updated with plain read-add-write,
// and flushed with one global reduction per entry per CTA.
template <int F>
__global__ void __launch_bounds__(256) bwd_small_kernel(const __grid_constant__ Params P,
                                                        const __grid_constant__ SmallSet S,
                                                        const float4 *__restrict__ coords, int64_t N,
                                                        const float *__restrict__ dout, const DoutLayout dl,
                                                        float *__restrict__ dtable, int *__restrict__ flag) {
    extern __shared__ float acc[];
    __shared__ LevelSmem slv;
    load_levels(P, slv);
    // lane-private blocks of the tiny levels: [warp][slot][lane] after acc
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // S.copies = 1: one block per CTA; = warps: one block per warp
    const int ncopy = S.copies > 1 ? S.copies : 1;
    float *blk = acc + (ncopy > 1 ? warp * S.total : 0);
    float *lp = acc + ncopy * S.total + warp * S.ttotal * 32 + lane;
    for (int i = threadIdx.x; i < ncopy * S.total + (int)(blockDim.x >> 5) * S.ttotal * 32; i += blockDim.x) acc[i] = 0.f;
    __syncthreads();
    const int64_t items = N * S.n;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // one item ahead: the next item's coordinates and upstream gradient are
    // in flight while this one accumulates (the lane-private launches run
    // few warps per SM, so the loads' latency is not hidden by occupancy)
    auto fetch = [&](int64_t gid, float4 &pc, float (&gg)[F]) {
        const int64_t j = gid / S.n;
        const int li = (int)(gid - j * S.n);
        const int64_t n = j;
        pc = __ldg(coords + n);
#pragma unroll
        for (int f = 0; f < F; f++) gg[f] = __ldg(dout + n * dl.ns + S.id[li] * dl.ls + f);
    };
    float4 p_nxt = make_float4(0.f, 0.f, 0.f, 0.f);
    float g_nxt[F];
    int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid < items) fetch(gid, p_nxt, g_nxt);
    for (; gid < items; gid += stride) {
        const int64_t j = gid / S.n;
        const int li = (int)(gid - j * S.n);
        const int l = S.id[li];
        const Level lv = slv.get(l);
        const float4 pcur = p_nxt;
        float g[F];
#pragma unroll
        for (int f = 0; f < F; f++) g[f] = g_nxt[f];
        if (gid + stride < items) fetch(gid + stride, p_nxt, g_nxt);
        Cell c;
        if (cell_of(lv, pcur, c) && li == 0) atomicOr(flag, 1);
        const float wx[2] = {__fsub_rn(1.0f, c.w[0]), c.w[0]}, wy[2] = {__fsub_rn(1.0f, c.w[1]), c.w[1]};
        const float wz[2] = {__fsub_rn(1.0f, c.w[2]), c.w[2]}, wt[2] = {__fsub_rn(1.0f, c.w[3]), c.w[3]};
        if (S.toff[li] >= 0) {
            // tiny level: every lane owns a private copy (column `lane` of its
            // warp's block, conflict-free): plain read-add-write, no atomics
            // (indices local to the level: entry - offset, no 32-bit overflow
            // for levels placed near the top of the 2^32 parameter range)
            float *t = lp + S.toff[li] * 32;
#pragma unroll
            for (int k = 0; k < 16; k += 2) {
                const float Wyzt = wy[(k >> 1) & 1] * wz[(k >> 2) & 1] * wt[(k >> 3) & 1];
                const float W0 = wx[0] * Wyzt, W1 = wx[1] * Wyzt;
                const uint32_t e0 = c.idx[k] - lv.offset, e1 = c.idx[k + 1] - lv.offset;
#pragma unroll
                for (int f = 0; f < F; f++) {
                    t[(e0 * F + f) * 32] += W0 * g[f];
                    t[(e1 * F + f) * 32] += W1 * g[f];
                }
            }
            continue;
        }
        float *a = blk + S.soff[li];
#pragma unroll
        for (int k = 0; k < 16; k += 2) {
            const float Wyzt = wy[(k >> 1) & 1] * wz[(k >> 2) & 1] * wt[(k >> 3) & 1];
            const float W0 = wx[0] * Wyzt, W1 = wx[1] * Wyzt;
            const uint32_t e0 = c.idx[k] - lv.offset, e1 = c.idx[k + 1] - lv.offset;
#pragma unroll
            for (int f = 0; f < F; f++) {
                atomicAdd(a + e0 * F + f, W0 * g[f]);
                atomicAdd(a + e1 * F + f, W1 * g[f]);
            }
        }
    }
    __syncwarp();
    // fold the lane-private blocks into the CTA copy: lane l sums slot s over
    // the warp's 32 lanes (rotated start: conflict-free), then one CTA atomic
    if (S.ttotal > 0) {
        const float *wb = acc + ncopy * S.total + warp * S.ttotal * 32;
        for (int slot = lane; slot < S.ttotal; slot += 32) {
            float v = 0.f;
            for (int m = 0; m < 32; m++) v += wb[slot * 32 + ((m + lane) & 31)];
            if (v != 0.f) atomicAdd(acc + S.tmap[slot], v);
        }
    }
    __syncthreads();
    // flush this CTA's partial sums
    for (int li = 0; li < S.n; li++) {
        const Level lv = slv.get(S.id[li]);
        const int cnt = (li + 1 < S.n ? S.soff[li + 1] : S.total) - S.soff[li];
        float *dst = dtable + (size_t)lv.offset * F;
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
            float v = 0.f;
            for (int w = 0; w < ncopy; w++) v += acc[w * S.total + S.soff[li] + i];
            if (v != 0.f) atomicAdd(dst + i, v);
        }
    }
}

// ------------------------------------------------------------ indices
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
    const float4 p = __ldg(coords + n);
    Cell c;
    const bool bad = cell_of(slv.get(l), p, c);
    if (bad && l == 0) atomicOr(flag, 1);
    uint4 *o = reinterpret_cast<uint4 *>(idx + gid * 16);
#pragma unroll
    for (int k = 0; k < 16; k += 4) o[k / 4] = make_uint4(c.idx[k], c.idx[k + 1], c.idx[k + 2], c.idx[k + 3]);
    if (wout) {
        const float wx[2] = {1.0f - c.w[0], c.w[0]}, wy[2] = {1.0f - c.w[1], c.w[1]};
        const float wz[2] = {1.0f - c.w[2], c.w[2]}, wt[2] = {1.0f - c.w[3], c.w[3]};
        float4 *ow = reinterpret_cast<float4 *>(wout + gid * 16);
#pragma unroll
        for (int k = 0; k < 16; k += 4) {
            float q[4];
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const int kk = k + j;
                q[j] = wx[kk & 1] * wy[(kk >> 1) & 1] * wz[(kk >> 2) & 1] * wt[(kk >> 3) & 1];
            }
            ow[k / 4] = make_float4(q[0], q[1], q[2], q[3]);
        }
    }
}

}  // namespace fh
