// encode_params.h -- per-level launch parameters of the encode kernels.
#pragma once
#include <stdint.h>

namespace fh {

// 64 bytes per level; kernel parameters carry up to FH_MAX_LEVELS of them.
struct __align__(16) Level {
    uint32_t res[4];     // Rx, Ry, Rz, Rt (vertices)
    float scale[4];      // fp32(R - 1) per axis (R2)
    uint32_t sy, sz, st; // Eq. 9 strides: Rx, Rx*Ry, Rx*Ry*Rz
    uint32_t hashed;     // 0: Eq. 9 (row-major); 1: capped level, R5 hash; 2: brick order (NEXT-2, R21)
    uint32_t mask;       // T_l - 1 for hashed levels (T_l power of two)
    uint32_t offset;     // first entry of the level in the packed table
    uint32_t tshift;     // forward: x-pairs at odd entries read the shifted table copy (set per launch)
    uint32_t pad;
};

constexpr int kMaxLevels = 32;

struct Params {
    int L;
    int F;
    Level lv[kMaxLevels];
};

// Levels whose fp32 grads are accumulated in shared memory in the backward
// (see bwd_small_kernel).
struct SmallSet {
    int n;                    // number of small levels
    int id[kMaxLevels];       // level ids
    int soff[kMaxLevels];     // float offset of each level's block in shared memory
    int total;                // floats in shared memory
    // tiny levels (T_l F <= 64, e.g. the 2x2x2x2 end of a fold schedule):
    // lane-private accumulators, toff[i] = float offset of small level i in
    // every lane's private block (-1: not tiny); ttotal floats per lane
    int toff[kMaxLevels];
    int ttotal;
    int tmap[320];            // tiny slot -> float offset of the same element in the CTA block
    int copies;               // blocks of `total` floats: 1 per CTA, or one per warp (= warps per CTA)
};
constexpr int kMaxTinyFloats = 320;   // lane-private floats per lane (all tiny levels together)
constexpr int kMaxTinyLevel = 256;    // a level of at most this many floats (T_l F) is tiny

// A set of levels one direct encode launch processes (thread = (sample,
// list entry), list entry fastest).
struct LevelList {
    int n;
    int id[kMaxLevels];
};

// Layout of the backward's upstream gradient: level l of sample n starts at
// dout + n * ns + l * ls (floats).  Row-major [N][L][F] (the ABI default):
// ns = L F, ls = F.  Level-major [L][N][F] (FH_BWD_DOUT_LEVEL_MAJOR, the
// trainer's dL/d(enc) for F >= 4): ns = F, ls = N F -- a level pass then
// reads contiguous F-float rows instead of F of every L F floats.
struct DoutLayout {
    int64_t ns, ls;
};

// In-pass replicated copies (F >= 4): the contended coarse levels of a
// level-group launch reduce into R copies in the scratch (CTA b -> copy
// b % R) instead of dtable, so same-address reductions, which serialise in
// the L2, spread over R addresses; rep_reduce_kernel adds the copies into
// dtable after the launch.  base[q] is the copies' start minus the level's
// entry offset times F, so base[q] + idx * F addresses copy 0 directly.
constexpr int kMaxInRep = 4;
struct RepSpec {
    int n;
    int lvl[kMaxInRep];
    int R[kMaxInRep];
    float *base[kMaxInRep];
    int64_t stride[kMaxInRep];   // floats between copies
};

}  // namespace fh
