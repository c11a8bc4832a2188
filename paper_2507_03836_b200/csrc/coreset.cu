// coreset.cu -- NEXT-4: feature-based coreset selection on the GPU
// (include/fhash_coreset.h; §3.1, Eqs. 1-3; readings
// R22-R26 in DESIGN.md §3).
//
// The paper builds d_k with a hash-based dictionary on the CPU.  Here
// the masks are BIT ROWS: one uint32 word holds 32 x-consecutive vertices of
// one (frame, z, y) row, so every step after the feature test is word-wide
// integer work on a mask 32x smaller than the volume:
//   feature_kernel   warp per word: lane i tests vertex x0+i (one coalesced
//                    load, the only pass over the fp32 volume) and the
//                    ballot is the word; the isosurface adds the corners of
//                    straddling cells (straddle_kernel, one bit per cell)
//   dilate_kernel    thread per word: d = OR over the 3x3 neighbouring rows
//                    of (w | w<<1 | w>>1 | carries) -- the 26-neighbourhood;
//                    per-frame bounding box from ffs/clz; per-CTA popcounts
//   cellrow_kernel   cell-row bits = (OR of the 4 corner rows) | >> 1
//   occupancy_kernel thread per 32-bit word of the Morton-ordered cell
//                    bitmap: its 32 cells are a fixed pattern of offsets
//                    from one decoded base, each one cell-row bit
//   emit_kernel      CTA per 256 mask words: block scan of popcounts, then
//                    each warp writes its words' set bits as samples
//                    (Eqs. 1-3), 32 consecutive samples per store
// Order of samples = word order then bit order = frame-major row-major (R26).
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "internal.h"
#include "../../include/fhash_coreset.h"

using fh::aligned;
using fh::cuda_check;
using fh::fail;
using fh::g_err;

namespace fh {
namespace coreset {

constexpr int kThreads = 256;   // also the mask words per emit / count chunk

struct Dims {
    uint32_t X, Y, Z;
    uint64_t V;     // X*Y*Z
    int n;
    uint32_t Wx;    // mask words per vertex row  = ceil(X / 32)
    uint32_t Wc;    // mask words per cell row    = ceil((X-1) / 32)
};

// R24 Morton layout of the cell grid (cells_a = dims_a - 1).
struct Morton {
    uint32_t bits[3];
    int nbits;
    uint8_t axis[64];
    uint8_t bit[64];
    uint8_t lo_off[32][3];   // cell offsets of the 32 codes of one word (low 5 code bits)
    int nrows;               // distinct (dy, dz) among them
    bool std5;               // low 5 code bits are x0 y0 z0 x1 y1 (every axis has >= 2 bits)
    bool cube8;              // std5 and code bits 5..7 are z1 x2 y2 (every axis has >= 3 bits)
    uint8_t row_dy[32], row_dz[32], row_of[32];
};

__host__ __device__ inline uint32_t bits_for(uint32_t cells) {
    uint32_t b = 0;
    while (b < 32 && (1ull << b) < cells) b++;
    return b;
}

static Morton make_morton(uint32_t X, uint32_t Y, uint32_t Z) {
    Morton m{};
    const uint32_t c[3] = {X - 1, Y - 1, Z - 1};
    for (int a = 0; a < 3; a++) m.bits[a] = bits_for(c[a]);
    int pos = 0;
    for (uint32_t j = 0; j < 32; j++)
        for (int a = 0; a < 3; a++)
            if (m.bits[a] > j) {
                m.axis[pos] = (uint8_t)a;
                m.bit[pos] = (uint8_t)j;
                pos++;
            }
    m.nbits = pos;
    m.std5 = m.bits[0] >= 2 && m.bits[1] >= 2 && m.bits[2] >= 2;
    m.cube8 = m.std5 && m.nbits >= 8 && m.axis[5] == 2 && m.bit[5] == 1 && m.axis[6] == 0 && m.bit[6] == 2 &&
              m.axis[7] == 1 && m.bit[7] == 2;
    m.nrows = 0;
    for (int i = 0; i < 32; i++) {
        m.lo_off[i][0] = m.lo_off[i][1] = m.lo_off[i][2] = 0;
        for (int p = 0; p < 5 && p < m.nbits; p++)
            if ((i >> p) & 1) m.lo_off[i][m.axis[p]] |= (uint8_t)(1u << m.bit[p]);
        int r = 0;
        while (r < m.nrows && !(m.row_dy[r] == m.lo_off[i][1] && m.row_dz[r] == m.lo_off[i][2])) r++;
        if (r == m.nrows) {
            m.row_dy[r] = m.lo_off[i][1];
            m.row_dz[r] = m.lo_off[i][2];
            m.nrows++;
        }
        m.row_of[i] = (uint8_t)r;
    }
    return m;
}

__device__ __forceinline__ uint32_t last_word_mask(uint32_t width, uint32_t w, uint32_t nwords) {
    const uint32_t r = width & 31u;
    return (w + 1 == nwords && r) ? ((1u << r) - 1u) : 0xFFFFFFFFu;
}

// ------------------------------------------------------------ isosurface cells
// s bit of cell (cx, cy, cz) of frame k: min <= iso <= max over its 8
// corners.  Warp per cell-row word: lane i reads column x0+i of the 4 corner
// rows (coalesced), takes column x0+i+1 from lane i+1, and the ballot is the
// word.
__global__ void __launch_bounds__(kThreads) straddle_kernel(const float *__restrict__ vol, Dims d, float iso,
                                                           uint32_t *__restrict__ sbits) {
    // 32-bit index math throughout: n X Y Z < 2^32 (make_dims)
    const uint32_t total = (uint32_t)d.n * (d.Z - 1) * (d.Y - 1) * d.Wc;
    const int lane = threadIdx.x & 31;
    for (uint32_t g = (blockIdx.x * kThreads + threadIdx.x) >> 5; g < total; g += (gridDim.x * kThreads) >> 5) {
        const uint32_t row = g / d.Wc;
        const uint32_t w = g - row * d.Wc;
        const uint32_t cy = row % (d.Y - 1), cz = (row / (d.Y - 1)) % (d.Z - 1);
        const uint32_t k = row / ((d.Y - 1) * (d.Z - 1));
        const uint32_t x = w * 32 + lane;
        float mn = INFINITY, mx = -INFINITY, mn1 = INFINITY, mx1 = -INFINITY;
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const float *r = vol + (uint64_t)k * d.V + ((uint64_t)(cz + (q >> 1)) * d.Y + (cy + (q & 1))) * d.X;
            if (x < d.X) {
                const float u = __ldg(r + x);
                mn = fminf(mn, u);
                mx = fmaxf(mx, u);
            }
            if (lane == 31 && x + 1 < d.X) {   // the column after the word
                const float u = __ldg(r + x + 1);
                mn1 = fminf(mn1, u);
                mx1 = fmaxf(mx1, u);
            }
        }
        const float nmn = __shfl_down_sync(0xffffffffu, mn, 1), nmx = __shfl_down_sync(0xffffffffu, mx, 1);
        if (lane < 31) { mn1 = nmn; mx1 = nmx; }
        const bool in = x + 1 < d.X && fminf(mn, mn1) <= iso && iso <= fmaxf(mx, mx1);
        const uint32_t bits = __ballot_sync(0xffffffffu, in);
        if (lane == 0) sbits[g] = bits;
    }
}

// ------------------------------------------------------------ feature
// Warp per mask word: lane i tests vertex x0+i (one coalesced 128-byte load
// per warp -- the only pass over the fp32 volume); the ballot is the word.
__device__ __forceinline__ bool feature_test(float v, const fh_feature_spec &s) {
    if (s.kind == FH_FEAT_INTERVAL) return (s.p0 <= v) && (v <= s.p1);
    if (s.kind == FH_FEAT_SEGMENTATION) return v >= s.p0;
    return fabs((double)v - (double)s.p0) <= (double)s.p1;  // exact: fp32 operands
}

constexpr int kFeatUnroll = 8;   // words (independent 128-byte loads) in flight per warp
#ifndef FH_FEAT_UNITS
#define FH_FEAT_UNITS 8   // 128-vertex units per warp in flight (the X % 128 == 0 fast path)
#endif

// Warp per vertex ROW (grid-stride over the n Z Y rows): the row's
// (frame, z, y) is derived once, then lane i tests vertex 32 w + i of each
// word w of the row, kFeatUnroll loads in flight; the ballot is the word.
__global__ void __launch_bounds__(kThreads) feature_kernel(const float *__restrict__ vol, Dims d, fh_feature_spec s,
                                                          const uint32_t *__restrict__ sbits,
                                                          uint32_t *__restrict__ f) {
    const uint32_t rows = (uint32_t)d.n * d.Z * d.Y;   // < 2^32 (make_dims)
    const int lane = threadIdx.x & 31;
    const uint32_t G = (gridDim.x * kThreads) >> 5;   // warps in the grid
    if (s.kind != FH_FEAT_ISOSURFACE && (d.X & 127u) == 0) {
        // rows of whole 128-vertex groups: the (row, group) units of the
        // volume flattened, kUnits per warp in flight (memory-level
        // parallelism: one unit is only 512 B per warp).  Lane i loads
        // vertex 32 j + i of word j (four coalesced 128-byte loads per unit),
        // so each ballot IS a mask word: no bit spreading (the float4 form
        // spent ~100 warp instructions per unit spreading ballot bytes and was
        // issue-bound, 121 us for 8 x 256^3).
        constexpr int kUnits = FH_FEAT_UNITS;
        // both kinds here are one interval test, hoisted out of the ballots:
        // segmentation v >= p0 == p0 <= v <= +inf (NaN fails both forms)
        const float lo = s.p0, hi = s.kind == FH_FEAT_INTERVAL ? s.p1 : INFINITY;
        const uint32_t groups = d.X / 128;
        const uint64_t units = (uint64_t)rows * groups;
        const uint64_t warp0 = (blockIdx.x * kThreads + threadIdx.x) >> 5;
        for (uint64_t u0 = warp0 * kUnits; u0 < units; u0 += (uint64_t)G * kUnits) {
            float v[kUnits][4];
#pragma unroll
            for (int u = 0; u < kUnits; u++)
#pragma unroll
                for (int j = 0; j < 4; j++)
                    v[u][j] = u0 + u < units ? __ldcs(vol + (u0 + u) * 128 + j * 32 + lane) : 0.f;
#pragma unroll
            for (int u = 0; u < kUnits; u++) {
                if (u0 + u >= units) break;   // warp-uniform
                const uint32_t b0 = __ballot_sync(0xffffffffu, lo <= v[u][0] && v[u][0] <= hi);
                const uint32_t b1 = __ballot_sync(0xffffffffu, lo <= v[u][1] && v[u][1] <= hi);
                const uint32_t b2 = __ballot_sync(0xffffffffu, lo <= v[u][2] && v[u][2] <= hi);
                const uint32_t b3 = __ballot_sync(0xffffffffu, lo <= v[u][3] && v[u][3] <= hi);
                // unit (row, q) -> words 4 q .. 4 q + 3 of the row (Wx = 4 groups)
                if (lane < 4) f[(u0 + u) * 4 + lane] = lane == 0 ? b0 : lane == 1 ? b1 : lane == 2 ? b2 : b3;
            }
        }
        return;
    }
    for (uint32_t row = (blockIdx.x * kThreads + threadIdx.x) >> 5; row < rows; row += G) {
        const float *r = vol + (uint64_t)row * d.X;   // rows of [n][Z][Y][X] are contiguous
        uint32_t *frow = f + (uint64_t)row * d.Wx;
        const uint32_t y = row % d.Y, z = (row / d.Y) % d.Z, k = row / (d.Y * d.Z);
        uint32_t w_begin = 0;
        if (s.kind != FH_FEAT_ISOSURFACE && (d.X & 3u) == 0 && (reinterpret_cast<uintptr_t>(vol) & 15u) == 0) {
            // 128 vertices (4 words) per step: lane l loads vertices 4l .. 4l+3
            // as one float4; ballot j has bit l = vertex 4l + j, so word w
            // takes byte w of the four ballots, spread to bits 4i + j.
            const uint32_t groups = d.X / 128;
            const float4 *r4 = reinterpret_cast<const float4 *>(r);
            for (uint32_t q0 = 0; q0 < groups; q0 += 2) {
                float4 v[2];
#pragma unroll
                for (int u = 0; u < 2; u++)
                    v[u] = q0 + u < groups ? __ldg(r4 + (q0 + u) * 32 + lane) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int u = 0; u < 2; u++) {
                    if (q0 + u >= groups) break;   // warp-uniform
                    const uint32_t b0 = __ballot_sync(0xffffffffu, feature_test(v[u].x, s));
                    const uint32_t b1 = __ballot_sync(0xffffffffu, feature_test(v[u].y, s));
                    const uint32_t b2 = __ballot_sync(0xffffffffu, feature_test(v[u].z, s));
                    const uint32_t b3 = __ballot_sync(0xffffffffu, feature_test(v[u].w, s));
                    if (lane < 4) {
                        auto spread = [](uint32_t x) {   // bit i -> bit 4 i (i < 8)
                            x = (x | (x << 12)) & 0x000F000Fu;
                            x = (x | (x << 6)) & 0x03030303u;
                            return (x | (x << 3)) & 0x11111111u;
                        };
                        const uint32_t sh = 8u * lane;
                        frow[(q0 + u) * 4 + lane] = spread((b0 >> sh) & 0xFFu) | (spread((b1 >> sh) & 0xFFu) << 1) |
                                                    (spread((b2 >> sh) & 0xFFu) << 2) | (spread((b3 >> sh) & 0xFFu) << 3);
                    }
                }
            }
            w_begin = groups * 4;
        }
        for (uint32_t w0 = w_begin; w0 < d.Wx; w0 += kFeatUnroll) {
            float v[kFeatUnroll];
#pragma unroll
            for (int u = 0; u < kFeatUnroll; u++) {
                const uint32_t x = (w0 + u) * 32 + lane;
                v[u] = x < d.X ? __ldg(r + x) : 0.f;
            }
#pragma unroll
            for (int u = 0; u < kFeatUnroll; u++) {
                const uint32_t w = w0 + u;
                if (w >= d.Wx) break;   // warp-uniform
                uint32_t bits = __ballot_sync(0xffffffffu, (w * 32 + lane < d.X) && feature_test(v[u], s));
                if (lane == 0) {
                    if (s.kind == FH_FEAT_ISOSURFACE) {
                        // corners of straddling cells: vertex (x, y, z) is a corner of
                        // the cells (x-1..x, y-1..y, z-1..z); cell x -> vertices x, x+1
                        for (int dz = 0; dz < 2; dz++)
                            for (int dy = 0; dy < 2; dy++) {
                                const int cy = (int)y - dy, cz = (int)z - dz;
                                if (cy < 0 || cz < 0 || cy >= (int)d.Y - 1 || cz >= (int)d.Z - 1) continue;
                                const uint32_t *sr = sbits + ((k * (d.Z - 1) + cz) * (d.Y - 1) + cy) * d.Wc;
                                const uint32_t cw = w < d.Wc ? sr[w] : 0u;
                                const uint32_t cprev = w > 0 ? sr[w - 1] : 0u;
                                bits |= cw | (cw << 1) | (cprev >> 31);
                            }
                        bits &= last_word_mask(d.X, w, d.Wx);
                    }
                    frow[w] = bits;
                }
            }
        }
    }
}

// ------------------------------------------------------------ dilation
// d = 26-neighbourhood of f (clamped); per-frame bounding box; per-CTA
// chunk popcounts (the counts of the compaction, chunk = 256 words).  A thread
// owns kDW consecutive words of one row (when Wx % kDW == 0; otherwise one
// word each, the generic path), so a neighbour row costs kDW + 2 loads for
// kDW outputs instead of 3 kDW, and the box / count reductions run once per
// kDW words (was 61 M warp instructions, 73 us for 8 x 256^3).
constexpr int kDW = 4;

__device__ __forceinline__ void box_add(int bb[6], uint32_t acc, uint32_t w, uint32_t y, uint32_t z) {
    if (acc) {
        bb[0] = min(bb[0], (int)(w * 32 + __ffs(acc) - 1));
        bb[3] = max(bb[3], (int)(w * 32 + 31 - __clz(acc)));
        bb[1] = min(bb[1], (int)y);
        bb[4] = max(bb[4], (int)y);
        bb[2] = min(bb[2], (int)z);
        bb[5] = max(bb[5], (int)z);
    }
}

__global__ void __launch_bounds__(kThreads) dilate_kernel(const uint32_t *__restrict__ f, Dims d,
                                                         uint32_t *__restrict__ dm, int *__restrict__ boxes,
                                                         uint32_t *__restrict__ counts) {
    __shared__ uint32_t wcnt[kThreads / 32];
    const uint32_t total = (uint32_t)d.n * d.Z * d.Y * d.Wx;
    const bool vec = (d.Wx % kDW) == 0;
    const int per = vec ? kDW : 1;            // words per thread; the CTA covers `per` chunks
    int bb[6] = {INT_MAX, INT_MAX, INT_MAX, -1, -1, -1};
    uint32_t cnt = 0;
    int frame = -1;
    {
        const uint32_t g0 = (blockIdx.x * kThreads + threadIdx.x) * per;
        if (g0 < total) {
            const uint32_t row = g0 / d.Wx;
            const uint32_t w0 = g0 - row * d.Wx;
            const uint32_t y = row % d.Y, z = (row / d.Y) % d.Z;
            const uint32_t k = row / (d.Y * d.Z);
            frame = (int)k;
            uint32_t acc[kDW] = {0, 0, 0, 0};
            for (int dz = -1; dz <= 1; dz++) {
                const int zz = (int)z + dz;
                if (zz < 0 || zz >= (int)d.Z) continue;
                for (int dy = -1; dy <= 1; dy++) {
                    const int yy = (int)y + dy;
                    if (yy < 0 || yy >= (int)d.Y) continue;
                    const uint32_t *r = f + ((k * d.Z + zz) * d.Y + yy) * d.Wx;
                    const uint32_t lft = w0 > 0 ? __ldg(r + w0 - 1) : 0u;
                    if (vec) {
                        const uint4 c4 = __ldg(reinterpret_cast<const uint4 *>(r + w0));
                        const uint32_t rgt = w0 + kDW < d.Wx ? __ldg(r + w0 + kDW) : 0u;
                        const uint32_t c[kDW] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
                        for (int i = 0; i < kDW; i++) {
                            const uint32_t l = i > 0 ? c[i - 1] : lft, rr = i + 1 < kDW ? c[i + 1] : rgt;
                            acc[i] |= c[i] | (c[i] << 1) | (c[i] >> 1) | (l >> 31) | (rr << 31);
                        }
                    } else {
                        const uint32_t c = __ldg(r + w0);
                        const uint32_t rgt = w0 + 1 < d.Wx ? __ldg(r + w0 + 1) : 0u;
                        acc[0] |= c | (c << 1) | (c >> 1) | (lft >> 31) | (rgt << 31);
                    }
                }
            }
            if (vec) {
#pragma unroll
                for (int i = 0; i < kDW; i++) {
                    acc[i] &= last_word_mask(d.X, w0 + i, d.Wx);
                    cnt += __popc(acc[i]);
                    box_add(bb, acc[i], w0 + i, y, z);
                }
                *reinterpret_cast<uint4 *>(dm + g0) = make_uint4(acc[0], acc[1], acc[2], acc[3]);
            } else {
                acc[0] &= last_word_mask(d.X, w0, d.Wx);
                cnt = __popc(acc[0]);
                box_add(bb, acc[0], w0, y, z);
                dm[g0] = acc[0];
            }
        }
    }
    // boxes are per frame: reduce over the warp when its lanes share the frame
    const int f0 = __shfl_sync(0xffffffffu, frame, 0);
    const bool same = __all_sync(0xffffffffu, frame == f0 || frame < 0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (same) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int a = 0; a < 3; a++) {
                bb[a] = min(bb[a], __shfl_xor_sync(0xffffffffu, bb[a], o));
                bb[3 + a] = max(bb[3 + a], __shfl_xor_sync(0xffffffffu, bb[3 + a], o));
            }
        if ((threadIdx.x & 31) == 0 && bb[3] >= 0 && f0 >= 0) {
            int *b = boxes + 6 * f0;
            for (int a = 0; a < 3; a++) {
                atomicMin(b + a, bb[a]);
                atomicMax(b + 3 + a, bb[3 + a]);
            }
        }
    } else if (bb[3] >= 0) {   // rare: a warp straddling two frames
        int *b = boxes + 6 * frame;
        for (int a = 0; a < 3; a++) {
            atomicMin(b + a, bb[a]);
            atomicMax(b + 3 + a, bb[3 + a]);
        }
    }
    if ((threadIdx.x & 31) == 0) wcnt[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if ((int)threadIdx.x < per) {   // chunk c of this CTA = its warps [c w, (c + 1) w), w = 8 / per
        const int wpc = (kThreads / 32) / per;
        const uint64_t c = (uint64_t)blockIdx.x * per + threadIdx.x;
        uint32_t s = 0;
        for (int i = 0; i < wpc; i++) s += wcnt[threadIdx.x * wpc + i];
        if (c * kThreads < total) counts[c] = s;
    }
}

__global__ void init_boxes_kernel(int *boxes, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < 6 * n) boxes[i] = (i % 6) < 3 ? INT_MAX : -1;
}

// ------------------------------------------------------------ occupancy
// Cell-row mask: cell x of row (cy, cz) is touched iff vertex x or x+1 of
// one of its 4 corner rows is in d_k.  kDW words of one cell row per thread
// when Wc % kDW == 0 (one index decode and 4 (kDW + 1) loads per kDW words),
// else one word per thread.
__global__ void __launch_bounds__(kThreads) cellrow_kernel(const uint32_t *__restrict__ dm, Dims d,
                                                          uint32_t *__restrict__ cm) {
    const uint32_t total = (uint32_t)d.n * (d.Z - 1) * (d.Y - 1) * d.Wc;
    const bool vec = (d.Wc % kDW) == 0;
    const uint32_t per = vec ? kDW : 1;
    for (uint32_t g = (blockIdx.x * kThreads + threadIdx.x) * per; g < total; g += gridDim.x * kThreads * per) {
        const uint32_t row = g / d.Wc;
        const uint32_t w = g - row * d.Wc;
        const uint32_t cy = row % (d.Y - 1), cz = (row / (d.Y - 1)) % (d.Z - 1);
        const uint32_t k = row / ((d.Y - 1) * (d.Z - 1));
        if (vec) {
            uint32_t c[kDW] = {0, 0, 0, 0};
            uint32_t nx = 0;
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const uint32_t *r = dm + ((k * d.Z + cz + (q >> 1)) * d.Y + cy + (q & 1)) * d.Wx;
#pragma unroll
                for (int i = 0; i < kDW; i++) c[i] |= __ldg(r + w + i);   // Wx >= Wc: w + kDW - 1 < Wx
                if (w + kDW < d.Wx) nx |= __ldg(r + w + kDW);
            }
            uint32_t o[kDW];
#pragma unroll
            for (int i = 0; i < kDW; i++) {
                const uint32_t next = i + 1 < kDW ? c[i + 1] : nx;
                o[i] = (c[i] | (c[i] >> 1) | (next << 31)) & last_word_mask(d.X - 1, w + i, d.Wc);
            }
            *reinterpret_cast<uint4 *>(cm + g) = make_uint4(o[0], o[1], o[2], o[3]);
        } else {
            uint32_t c = 0, nx = 0;
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const uint32_t *r = dm + ((k * d.Z + cz + (q >> 1)) * d.Y + cy + (q & 1)) * d.Wx;
                c |= __ldg(r + w);
                if (w + 1 < d.Wx) nx |= __ldg(r + w + 1);
            }
            cm[g] = (c | (c >> 1) | (nx << 31)) & last_word_mask(d.X - 1, w, d.Wc);
        }
    }
}

// kOW consecutive 32-bit words of the Morton-ordered bitmap per thread: the
// base cell of the first word is decoded once (the code bits above the
// thread's block); the kOW - 1 others differ from it only in code bits
// 5 .. 5 + log2(kOW) - 1.  Each word's 32 cells are fixed offsets (lo_off)
// from its base that lie in m.nrows distinct cell rows (<= 8 on a cube: a
// 4x4x2 block), each read once -- the x offsets stay inside one 32-bit word
// because the base x is a multiple of the x extent of the pattern.  (One
// word per thread decoded all nbits code bits per word: 80 M warp
// instructions, 95 us for 8 x 255^3 cells.)
constexpr int kOW = 8, kOWBits = 3;

__device__ __forceinline__ uint32_t occupancy_word(const uint32_t *__restrict__ fr, const Dims &d, const Morton &m,
                                                   const uint32_t base[3]) {
    const int ncodes = 1 << (m.nbits < 5 ? m.nbits : 5);
    const uint32_t Yc = d.Y - 1, Zc = d.Z - 1, Xc = d.X - 1;
    uint32_t word = 0;
    if (base[0] >= Xc) return 0u;
    if (m.std5) {
        // low code bits (x0, y0, z0, x1, y1): row (y, z) contributes the 4 x
        // bits (base x .. base x + 3) at code positions off(y, z) + {0, 1, 8, 9}
#pragma unroll
        for (int zz = 0; zz < 2; zz++)
#pragma unroll
            for (int yy = 0; yy < 4; yy++) {
                const uint32_t cy = base[1] + yy, cz = base[2] + zz;
                if (cy >= Yc || cz >= Zc) continue;
                const uint32_t rw = __ldg(fr + (cz * Yc + cy) * d.Wc + (base[0] >> 5));
                const uint32_t nib = (rw >> (base[0] & 31)) & 0xFu;   // bits past the grid are 0
                const uint32_t spread = (nib & 3u) | ((nib & 12u) << 6);
                word |= spread << ((yy & 1) * 2 + zz * 4 + (yy >> 1) * 16);
            }
    } else if (m.nrows <= 8) {
        uint32_t rows[8];
#pragma unroll
        for (int r = 0; r < 8; r++) {
            const uint32_t cy = base[1] + m.row_dy[r], cz = base[2] + m.row_dz[r];
            rows[r] = (r < m.nrows && cy < Yc && cz < Zc) ? __ldg(fr + (cz * Yc + cy) * d.Wc + (base[0] >> 5)) : 0u;
        }
#pragma unroll
        for (int i = 0; i < 32; i++) {
            if (i >= ncodes) break;
            const int ri = m.row_of[i];
            uint32_t rw = rows[0];
#pragma unroll
            for (int r = 1; r < 8; r++) rw = ri == r ? rows[r] : rw;   // register select, no local memory
            // bits past the grid are 0 in the cell-row mask (last_word_mask)
            word |= ((rw >> ((base[0] + m.lo_off[i][0]) & 31)) & 1u) << i;
        }
    } else {   // degenerate shapes (an axis of one cell): one load per code
        for (int i = 0; i < ncodes; i++) {
            const uint32_t cx = base[0] + m.lo_off[i][0], cy = base[1] + m.lo_off[i][1], cz = base[2] + m.lo_off[i][2];
            if (cx >= Xc || cy >= Yc || cz >= Zc) continue;
            word |= ((__ldg(fr + (cz * Yc + cy) * d.Wc + (cx >> 5)) >> (cx & 31)) & 1u) << i;
        }
    }
    return word;
}

__global__ void __launch_bounds__(kThreads) occupancy_kernel(const uint32_t *__restrict__ cm, Dims d, Morton m,
                                                            uint64_t words, uint32_t *__restrict__ occ) {
    const uint64_t k = blockIdx.y;   // frame
    const uint32_t *fr = cm + k * (uint64_t)(d.Z - 1) * (d.Y - 1) * d.Wc;   // a frame's offsets fit 32 bits
    const bool vec = (words % 4) == 0 && (reinterpret_cast<uintptr_t>(occ) & 15) == 0;
    for (uint64_t wi0 = ((uint64_t)blockIdx.x * kThreads + threadIdx.x) * kOW; wi0 < words;
         wi0 += (uint64_t)gridDim.x * kThreads * kOW) {
        uint32_t base0[3] = {0, 0, 0};
        for (int p = 5 + kOWBits; p < m.nbits; p++) {   // selects, not a dynamically indexed array
            const uint32_t b = (uint32_t)((wi0 >> (p - 5)) & 1) << m.bit[p];
            const int a = m.axis[p];
            base0[0] |= a == 0 ? b : 0u;
            base0[1] |= a == 1 ? b : 0u;
            base0[2] |= a == 2 ? b : 0u;
        }
        uint32_t out[kOW];
        if (m.cube8) {
            // the kOW = 8 words (code bits 5..7 = z1 x2 y2) cover cells
            // x0 .. x0+7 (one cell-row word: x0 % 8 == 0), y0 .. y0+7,
            // z0 .. z0+3: each of those 32 rows is loaded once (was 8 per word)
            const uint32_t Yc = d.Y - 1, Zc = d.Z - 1, x0 = base0[0];
            uint32_t rw[4][8];
#pragma unroll
            for (int zz = 0; zz < 4; zz++)
#pragma unroll
                for (int yy = 0; yy < 8; yy++) {
                    const uint32_t cy = base0[1] + yy, cz = base0[2] + zz;
                    rw[zz][yy] = (x0 < d.X - 1 && cy < Yc && cz < Zc)
                                     ? __ldg(fr + (cz * Yc + cy) * d.Wc + (x0 >> 5)) : 0u;
                }
#pragma unroll
            for (int j = 0; j < kOW; j++) {
                const int zo = (j & 1) * 2, xo = ((j >> 1) & 1) * 4, yo = ((j >> 2) & 1) * 4;
                uint32_t word = 0;
#pragma unroll
                for (int zz = 0; zz < 2; zz++)
#pragma unroll
                    for (int yy = 0; yy < 4; yy++) {
                        // bits past the grid are 0 in the cell-row mask (last_word_mask)
                        const uint32_t nib = (rw[zo + zz][yo + yy] >> ((x0 + xo) & 31)) & 0xFu;
                        const uint32_t spread = (nib & 3u) | ((nib & 12u) << 6);
                        word |= spread << ((yy & 1) * 2 + zz * 4 + (yy >> 1) * 16);
                    }
                out[j] = wi0 + j < words ? word : 0u;
            }
        } else
#pragma unroll
        for (int j = 0; j < kOW; j++) {
            uint32_t base[3] = {base0[0], base0[1], base0[2]};
#pragma unroll
            for (int i = 0; i < kOWBits; i++) {
                const int p = 5 + i;
                const uint32_t b = (p < m.nbits) ? (uint32_t)((j >> i) & 1) << m.bit[p] : 0u;
                const int a = m.axis[p];
                base[0] |= a == 0 ? b : 0u;
                base[1] |= a == 1 ? b : 0u;
                base[2] |= a == 2 ? b : 0u;
            }
            out[j] = wi0 + j < words ? occupancy_word(fr, d, m, base) : 0u;
        }
        uint32_t *o = occ + k * words + wi0;
        if (vec && wi0 + kOW <= words) {
#pragma unroll
            for (int j = 0; j < kOW; j += 4)
                *reinterpret_cast<uint4 *>(o + j) = make_uint4(out[j], out[j + 1], out[j + 2], out[j + 3]);
        } else {
#pragma unroll
            for (int j = 0; j < kOW; j++)
                if (wi0 + j < words) o[j] = out[j];
        }
    }
}

// ------------------------------------------------------------ compaction
// In-place exclusive scan of 1024-element blocks; block totals to sums.
__global__ void __launch_bounds__(1024) scan_block_kernel(uint32_t *__restrict__ a, uint64_t n,
                                                         uint32_t *__restrict__ sums) {
    __shared__ uint32_t wsum[32];
    const uint64_t i = (uint64_t)blockIdx.x * 1024 + threadIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t x = i < n ? a[i] : 0u;
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
        wsum[lane] = s;
    }
    __syncthreads();
    if (i < n) a[i] = v - x + (w > 0 ? wsum[w - 1] : 0u);
    if (threadIdx.x == 1023 && sums) sums[blockIdx.x] = wsum[31];
}

__global__ void add_block_offsets_kernel(uint32_t *__restrict__ a, uint64_t n, const uint32_t *__restrict__ sums) {
    const uint64_t i = (uint64_t)blockIdx.x * 1024 + threadIdx.x;
    if (i < n) a[i] += sums[blockIdx.x];
}

// FBB = fusion of the per-frame boxes, single-vertex axes padded
// (R25); count = total of the chunk counts.
__global__ void fbb_kernel(const int *__restrict__ boxes, int n, Dims d, const uint32_t *__restrict__ offs,
                           const uint32_t *__restrict__ counts, uint64_t nchunks, int *__restrict__ fbb_out,
                           int *__restrict__ fbb_ws, uint64_t *__restrict__ count) {
    int lo[3] = {INT_MAX, INT_MAX, INT_MAX}, hi[3] = {-1, -1, -1};
    for (int k = 0; k < n; k++) {
        if (boxes[6 * k + 3] < 0) continue;
        for (int a = 0; a < 3; a++) {
            lo[a] = min(lo[a], boxes[6 * k + a]);
            hi[a] = max(hi[a], boxes[6 * k + 3 + a]);
        }
    }
    const uint32_t D[3] = {d.X, d.Y, d.Z};
    if (hi[0] >= 0)
        for (int a = 0; a < 3; a++)
            if (hi[a] == lo[a]) {
                if ((uint32_t)hi[a] + 1 < D[a]) hi[a]++;
                else lo[a]--;
            }
    for (int a = 0; a < 3; a++) {
        fbb_ws[a] = lo[a];
        fbb_ws[3 + a] = hi[a];
        if (fbb_out) { fbb_out[a] = lo[a]; fbb_out[3 + a] = hi[a]; }
    }
    *count = nchunks ? (uint64_t)offs[nchunks - 1] + counts[nchunks - 1] : 0ull;
}

// Position of the r-th (0-based) set bit of m (r < popc(m)).
__device__ __forceinline__ uint32_t nth_set_bit(uint32_t m, uint32_t r) {
    uint32_t pos = 0;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        const uint32_t low = __popc(m & ((1u << s) - 1u));
        if (r >= low) {
            r -= low;
            m >>= s;
            pos += s;
        }
    }
    return pos;
}

// Warp-cooperative: the warp's 32 words own the output slots [base, base +
// Cw); slot j = j0 + lane finds its word (the last lane whose exclusive
// count is <= j: a 5-step shuffle binary search) and its bit (the r-th set
// bit of that word), so every store instruction writes 32 consecutive
// samples (512 B of coords, 128 B of values).  (A lane per word writing its
// own samples serially made each store touch 32 lines: 40 us at 2^21 samples.)
__global__ void __launch_bounds__(kThreads) emit_kernel(const uint32_t *__restrict__ dm, const float *__restrict__ vol,
                                                       Dims d, const uint32_t *__restrict__ offs,
                                                       const uint32_t *__restrict__ counts,
                                                       const int *__restrict__ fbb, float4 *__restrict__ coords,
                                                       float *__restrict__ values, uint64_t capacity) {
    __shared__ uint32_t ws[kThreads / 32];
    // empty chunk (most of a sparse coreset's volume): its count is known
    // from the dilation, so skip the mask read and the scan (CTA-uniform)
    if (counts[blockIdx.x] == 0) return;
    const uint32_t total = (uint32_t)d.n * d.Z * d.Y * d.Wx;
    const uint32_t g = blockIdx.x * kThreads + threadIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t bits = g < total ? dm[g] : 0u;
    const uint32_t c = __popc(bits);
    uint32_t v = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    if (lane == 31) ws[w] = v;
    __syncthreads();
    const uint32_t Cw = __shfl_sync(0xffffffffu, v, 31);
    if (Cw == 0) return;   // warp-uniform
    uint32_t base = offs[blockIdx.x];
    for (int i = 0; i < w; i++) base += ws[i];
    const uint32_t excl = v - c;
    // this lane's word: row, x word, and the (y, z, t) coordinates of its samples
    const uint32_t gg = g < total ? g : 0u;
    const uint32_t row = gg / d.Wx;
    const uint32_t wx = gg - row * d.Wx;
    const uint32_t y = row % d.Y, z = (row / d.Y) % d.Z;
    const uint32_t k = row / (d.Y * d.Z);
    const int lo0 = fbb[0];
    const float span0 = (float)(fbb[3] - fbb[0]);
    // Eqs. 1-2 then (q+1)/2 (R2, R25): (i - lo) / (hi - lo), one rounding
    const float fy = __fdiv_rn((float)((int)y - fbb[1]), (float)(fbb[4] - fbb[1]));
    const float fz = __fdiv_rn((float)((int)z - fbb[2]), (float)(fbb[5] - fbb[2]));
    const float ft = d.n > 1 ? __fdiv_rn((float)k, (float)(d.n - 1)) : 0.5f;   // n = 1: t = 0 in [-1,1]
    for (uint32_t j0 = 0; j0 < Cw; j0 += 32) {
        const uint32_t j = j0 + lane;
        int L = 0;
#pragma unroll
        for (int st = 16; st > 0; st >>= 1)
            if (__shfl_sync(0xffffffffu, excl, L + st) <= j) L += st;
        const uint32_t wb = __shfl_sync(0xffffffffu, bits, L);
        const uint32_t r = j - __shfl_sync(0xffffffffu, excl, L);
        const uint32_t rowL = __shfl_sync(0xffffffffu, row, L), wxL = __shfl_sync(0xffffffffu, wx, L);
        const float fyL = __shfl_sync(0xffffffffu, fy, L), fzL = __shfl_sync(0xffffffffu, fz, L),
                    ftL = __shfl_sync(0xffffffffu, ft, L);
        const uint64_t pos = (uint64_t)base + j;
        if (j < Cw && pos < capacity) {
            const uint32_t x = wxL * 32 + nth_set_bit(wb, r);
            coords[pos] = make_float4(__fdiv_rn((float)((int)x - lo0), span0), fyL, fzL, ftL);
            values[pos] = __ldg(vol + (uint64_t)rowL * d.X + x);
        }
    }
}

// ------------------------------------------------------------ host helpers
struct Layout {
    size_t f, dm, sb, boxes, fbb, total, counts, offs, scratch, bytes;
    uint64_t words, nchunks, swords;
};

static size_t up(size_t v) { return (v + 255) / 256 * 256; }

static bool make_dims(const uint32_t dims[3], int n, Dims &d) {
    if (!dims || n < 1 || dims[0] < 2 || dims[1] < 2 || dims[2] < 2) return false;
    d.X = dims[0];
    d.Y = dims[1];
    d.Z = dims[2];
    d.V = (uint64_t)d.X * d.Y * d.Z;
    d.n = n;
    d.Wx = (d.X + 31) / 32;
    d.Wc = (d.X - 1 + 31) / 32;
    return d.V * (uint64_t)n < (1ull << 32);
}

static Layout layout(const Dims &d) {
    Layout L{};
    L.words = (uint64_t)d.n * d.Z * d.Y * d.Wx;
    L.swords = (uint64_t)d.n * (d.Z - 1) * (d.Y - 1) * d.Wc;
    L.nchunks = (L.words + kThreads - 1) / kThreads;
    size_t o = 0;
    L.f = o; o += up(4 * L.words);
    L.dm = o; o += up(4 * L.words);
    L.sb = o; o += up(4 * L.swords);
    L.boxes = o; o += up(24 * (size_t)d.n);
    L.fbb = o; o += 256;
    L.total = o; o += 256;
    L.counts = o; o += up(4 * L.nchunks);
    L.offs = o; o += up(4 * L.nchunks);
    L.scratch = o;   // block sums of every level of the recursive scan
    uint64_t m = L.nchunks;
    while (m > 1) {
        m = (m + 1023) / 1024;
        o += up(4 * m);
    }
    L.bytes = o + 256;
    return L;
}

// Exclusive scan of a[0..n) in place (recursive over 1024-element blocks).
static void scan_u32(uint32_t *a, uint64_t n, uint32_t *scratch, cudaStream_t s) {
    if (n == 0) return;
    const uint64_t blocks = (n + 1023) / 1024;
    { scan_block_kernel<<<(unsigned)blocks, 1024, 0, s>>>(a, n, blocks > 1 ? scratch : nullptr); fh::count_launch(); }
    if (blocks > 1) {
        scan_u32(scratch, blocks, scratch + up(4 * blocks) / 4, s);
        { add_block_offsets_kernel<<<(unsigned)blocks, 1024, 0, s>>>(a, n, scratch); fh::count_launch(); }
    }
}

static unsigned grid_for(uint64_t items) {
    uint64_t g = (items + kThreads - 1) / kThreads;
    return (unsigned)(g < 148ull * 64 ? (g ? g : 1) : 148ull * 64);
}

}  // namespace coreset
}  // namespace fh

using namespace fh::coreset;

extern "C" {

size_t fh_coreset_workspace_size(const uint32_t dims_xyz[3], int n_frames) {
    Dims d;
    if (!make_dims(dims_xyz, n_frames, d)) return 0;
    return layout(d).bytes;
}

uint64_t fh_occupancy_words(const uint32_t dims_xyz[3]) {
    if (!dims_xyz || dims_xyz[0] < 2 || dims_xyz[1] < 2 || dims_xyz[2] < 2) return 0;
    uint32_t b = 0;
    for (int a = 0; a < 3; a++) b += bits_for(dims_xyz[a] - 1);
    return ((1ull << b) + 31) / 32;
}

uint64_t fh_morton_cell(const uint32_t dims_xyz[3], uint32_t x, uint32_t y, uint32_t z) {
    if (!dims_xyz || dims_xyz[0] < 2 || dims_xyz[1] < 2 || dims_xyz[2] < 2) return UINT64_MAX;
    if (x >= dims_xyz[0] - 1 || y >= dims_xyz[1] - 1 || z >= dims_xyz[2] - 1) return UINT64_MAX;
    const Morton m = make_morton(dims_xyz[0], dims_xyz[1], dims_xyz[2]);
    const uint32_t c[3] = {x, y, z};
    uint64_t code = 0;
    for (int p = 0; p < m.nbits; p++) code |= (uint64_t)((c[m.axis[p]] >> m.bit[p]) & 1u) << p;
    return code;
}

fh_status fh_coreset_build(const float *vol, const uint32_t dims_xyz[3], int n_frames, const fh_feature_spec *spec,
                           void *workspace, size_t workspace_bytes, uint32_t *occupancy, int32_t *fbb,
                           uint64_t *count, fh_stream stream) {
    g_err[0] = 0;
    Dims d;
    if (!dims_xyz || n_frames < 1 || dims_xyz[0] < 2 || dims_xyz[1] < 2 || dims_xyz[2] < 2)
        return fail(FH_E_ARG, "fh_coreset_build: need n_frames >= 1 and every dim >= 2");
    if (!make_dims(dims_xyz, n_frames, d)) return fail(FH_E_RANGE, "fh_coreset_build: n X Y Z >= 2^32");
    if (!spec || spec->kind < FH_FEAT_INTERVAL || spec->kind > FH_FEAT_SEGMENTATION)
        return fail(FH_E_ARG, "fh_coreset_build: bad feature spec");
    if (!vol || !aligned(vol, 4) || !workspace || !aligned(workspace, 16) || !count || !aligned(count, 8))
        return fail(FH_E_ARG, "fh_coreset_build: NULL or misaligned pointer");
    const Layout L = layout(d);
    if (workspace_bytes < L.bytes) return fail(FH_E_ARG, "fh_coreset_build: workspace too small");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    char *w = reinterpret_cast<char *>(workspace);
    uint32_t *f = reinterpret_cast<uint32_t *>(w + L.f);
    uint32_t *dm = reinterpret_cast<uint32_t *>(w + L.dm);
    uint32_t *sb = reinterpret_cast<uint32_t *>(w + L.sb);
    int *boxes = reinterpret_cast<int *>(w + L.boxes);
    uint32_t *counts = reinterpret_cast<uint32_t *>(w + L.counts);
    uint32_t *offs = reinterpret_cast<uint32_t *>(w + L.offs);
    if (spec->kind == FH_FEAT_ISOSURFACE)
        { straddle_kernel<<<grid_for(32 * L.swords), kThreads, 0, s>>>(vol, d, spec->p0, sb); fh::count_launch(); }
    { feature_kernel<<<grid_for(32ull * d.n * d.Z * d.Y), kThreads, 0, s>>>(vol, d, *spec, sb, f); fh::count_launch(); }
    { init_boxes_kernel<<<(6 * n_frames + 255) / 256, 256, 0, s>>>(boxes, n_frames); fh::count_launch(); }
    {
        const uint64_t per = d.Wx % kDW == 0 ? kDW : 1;
        dilate_kernel<<<(unsigned)((L.nchunks + per - 1) / per), kThreads, 0, s>>>(f, d, dm, boxes, counts);
        fh::count_launch();
    }
    if (occupancy) {
        // the cell-row mask reuses the straddle bit buffer (same shape)
        { cellrow_kernel<<<grid_for(d.Wc % kDW == 0 ? L.swords / kDW : L.swords), kThreads, 0, s>>>(dm, d, sb);
          fh::count_launch(); }
        const uint64_t words = fh_occupancy_words(dims_xyz);
        const dim3 og(grid_for((words + kOW - 1) / kOW), (unsigned)d.n);
        { occupancy_kernel<<<og, kThreads, 0, s>>>(sb, d, make_morton(d.X, d.Y, d.Z), words, occupancy); fh::count_launch(); }
    }
    cudaMemcpyAsync(offs, counts, 4 * L.nchunks, cudaMemcpyDeviceToDevice, s);
    scan_u32(offs, L.nchunks, reinterpret_cast<uint32_t *>(w + L.scratch), s);
    { fbb_kernel<<<1, 1, 0, s>>>(boxes, n_frames, d, offs, counts, L.nchunks, fbb, reinterpret_cast<int *>(w + L.fbb),
                               count); fh::count_launch(); }
    return cuda_check(cudaGetLastError(), "fh_coreset_build launch");
}

fh_status fh_coreset_emit(const float *vol, const uint32_t dims_xyz[3], int n_frames, const void *workspace,
                          size_t workspace_bytes, float *coords, float *values, uint64_t capacity, fh_stream stream) {
    g_err[0] = 0;
    Dims d;
    if (!dims_xyz || n_frames < 1 || dims_xyz[0] < 2 || dims_xyz[1] < 2 || dims_xyz[2] < 2)
        return fail(FH_E_ARG, "fh_coreset_emit: need n_frames >= 1 and every dim >= 2");
    if (!make_dims(dims_xyz, n_frames, d)) return fail(FH_E_RANGE, "fh_coreset_emit: n X Y Z >= 2^32");
    if (!vol || !workspace || !aligned(workspace, 16) || (capacity > 0 && (!coords || !aligned(coords, 16) || !values)))
        return fail(FH_E_ARG, "fh_coreset_emit: NULL or misaligned pointer");
    const Layout L = layout(d);
    if (workspace_bytes < L.bytes) return fail(FH_E_ARG, "fh_coreset_emit: workspace too small");
    if (capacity == 0) return FH_OK;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const char *w = reinterpret_cast<const char *>(workspace);
    { emit_kernel<<<(unsigned)L.nchunks, kThreads, 0, s>>>(
        reinterpret_cast<const uint32_t *>(w + L.dm), vol, d, reinterpret_cast<const uint32_t *>(w + L.offs),
        reinterpret_cast<const uint32_t *>(w + L.counts), reinterpret_cast<const int *>(w + L.fbb), reinterpret_cast<float4 *>(coords), values, capacity); fh::count_launch(); }
    return cuda_check(cudaGetLastError(), "fh_coreset_emit launch");
}

}  // extern "C"
