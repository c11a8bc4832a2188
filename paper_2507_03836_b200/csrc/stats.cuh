// stats.cu -- encoding_stats on the GPU (the collision /
// bucket-waste contrast of Fig. 4): for one
// level, every lattice vertex is mapped to its bucket exactly as the encode
// kernels map corners (Eq. 9, the brick order R21, the capped hash R5, or
// the MHE direct / spatial hash for one key frame), a T-bit bitmap records
// the buckets hit, and a popcount gives the distinct buckets.  collisions =
// vertices - distinct, utilisation = distinct / T.  Diagnostic (exhaustive:
// up to ~10^10 vertices), not on the train path.
// Included by fhash_api.cu (the encode kernels are defined in one TU).
#pragma once

namespace fh_stats {
using fh::cuda_check;
using fh::fail;
using fh::g_err;

// vertex v (x fastest) of the level's lattice -> bucket in [0, T)
__global__ void __launch_bounds__(256) stats_mark_kernel(const fh::Level lv, int kind, uint64_t C, uint64_t T,
                                                         uint32_t *__restrict__ bits) {
    const uint64_t nx = lv.res[0], ny = lv.res[1], nz = lv.res[2];
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < C; v += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t x = (uint32_t)(v % nx);
        uint64_t r = v / nx;
        const uint32_t y = (uint32_t)(r % ny);
        r /= ny;
        const uint32_t z = (uint32_t)(r % nz);
        const uint32_t t = (uint32_t)(r / nz);
        uint64_t b;
        if (kind == 1) {   // MHE, one key frame: direct when R^3 <= T, else the 3D spatial hash
            b = lv.hashed ? (uint64_t)((x ^ (y * fh::kPy) ^ (z * fh::kPz)) & lv.mask)
                          : (uint64_t)x + (uint64_t)y * lv.sy + (uint64_t)z * lv.sz;
        } else {
            b = (uint64_t)(fh::vertex_entry(lv, x, y, z, t) - lv.offset);
        }
        if (b < T) atomicOr(bits + (b >> 5), 1u << (b & 31));
    }
}

__global__ void __launch_bounds__(256) stats_count_kernel(const uint32_t *__restrict__ bits, uint64_t words,
                                                          unsigned long long *__restrict__ out) {
    uint32_t c = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words; i += (uint64_t)gridDim.x * blockDim.x)
        c += __popc(bits[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

// (vertices C, buckets T) of a level; the MHE counts one key frame
void level_shape(fh_encoder e, int l, uint64_t &C, uint64_t &T) {
    const fh_level_info &I = e->info[l];
    if (e->kind == 1) {
        C = (uint64_t)I.res[0] * I.res[1] * I.res[2];
        T = e->cap;
    } else {
        C = I.corners;
        T = I.table_size;
    }
}

}  // namespace fh_stats

extern "C" {

size_t fh_level_stats_workspace_size(fh_encoder e, int level) {
    if (!e || level < 0 || level >= e->L) return 0;
    uint64_t C, T;
    fh_stats::level_shape(e, level, C, T);
    return (size_t)((T + 31) / 32) * 4 + 256;
}

fh_status fh_level_stats(fh_encoder e, int level, void *workspace, size_t workspace_bytes, uint64_t *out,
                         fh_stream stream) {
    fh::g_err[0] = 0;
    if (!e || !workspace || !out) return fh::fail(FH_E_ARG, "fh_level_stats: NULL argument");
    if (level < 0 || level >= e->L) return fh::fail(FH_E_ARG, "fh_level_stats: level %d out of range", level);
    if (!fh::aligned(workspace, 16) || !fh::aligned(out, 8)) return fh::fail(FH_E_ARG, "fh_level_stats: misaligned");
    if (workspace_bytes < fh_level_stats_workspace_size(e, level))
        return fh::fail(FH_E_ARG, "fh_level_stats: workspace too small");
    uint64_t C, T;
    fh_stats::level_shape(e, level, C, T);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    uint32_t *bits = reinterpret_cast<uint32_t *>(workspace);
    const uint64_t words = (T + 31) / 32;
    fh_status st = fh::cuda_check(cudaMemsetAsync(bits, 0, words * 4, s), "fh_level_stats memset");
    if (st != FH_OK) return st;
    st = fh::cuda_check(cudaMemsetAsync(out, 0, 8, s), "fh_level_stats memset out");
    if (st != FH_OK) return st;
    uint64_t g = (C + 255) / 256;
    if (g > 148ull * 64) g = 148ull * 64;
    { fh_stats::stats_mark_kernel<<<(unsigned)(g ? g : 1), 256, 0, s>>>(e->params.lv[level], e->kind, C, T, bits); fh::count_launch(); }
    uint64_t g2 = (words + 255) / 256;
    if (g2 > 148ull * 16) g2 = 148ull * 16;
    { fh_stats::stats_count_kernel<<<(unsigned)(g2 ? g2 : 1), 256, 0, s>>>(bits, words,
                                                                reinterpret_cast<unsigned long long *>(out)); fh::count_launch(); }
    return fh::cuda_check(cudaGetLastError(), "fh_level_stats launch");
}

}  // extern "C"
