/*
 * fhash_coreset.h -- NEXT-4: the feature-based coreset selection that feeds
 * the F-Hash encoder (§3.1 "Feature-Based Coreset Selection",
 * P:58-84, Fig. 1, Eqs. 1-3), on the GPU.  Same conventions as fhash.h:
 * plain pointers and sizes, caller-owned device buffers, stream-ordered,
 * no synchronisation, errors returned synchronously for bad arguments.
 * Readings R22-R26 are in DESIGN.md §3 (and oracle/coreset.py).
 */
#ifndef FHASH_CORESET_H_
#define FHASH_CORESET_H_

#include "fhash.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Feature of interest (R22).  The thresholds are float32 and every
 * predicate is evaluated exactly on the float32 values:
 *   FH_FEAT_INTERVAL      lo <= v <= hi                       (p0 = lo, p1 = hi)
 *   FH_FEAT_ISOSURFACE    |v - iso| <= eps, plus the 8 corners of every cell
 *                         whose corner values satisfy min <= iso <= max
 *                                                             (p0 = iso, p1 = eps)
 *   FH_FEAT_SEGMENTATION  v >= threshold (components of any size)  (p0)   */
typedef enum { FH_FEAT_INTERVAL = 0, FH_FEAT_ISOSURFACE = 1, FH_FEAT_SEGMENTATION = 2 } fh_feature_kind;
typedef struct { int kind; float p0, p1; } fh_feature_spec;

/* Bytes of workspace fh_coreset_build needs for n key frames of X*Y*Z
 * vertices; 0 if n X Y Z >= 2^32 or any dim < 2. */
size_t fh_coreset_workspace_size(const uint32_t dims_xyz[3], int n_frames);

/* Words (uint32) of one frame's occupancy bitmap: 2^(bx+by+bz) bits rounded
 * up to words, b_a = ceil(log2(cells_a)), cells_a = dims_a - 1 (R24). */
uint64_t  fh_occupancy_words(const uint32_t dims_xyz[3]);

/* The R24 Morton index of cell (x, y, z) of a grid of dims_xyz vertices:
 * bit j of x, y, z interleaved from bit 0 upwards while the axis has more
 * than j bits (the standard x-in-bit-0 interleave on cubic grids).  Host
 * function (for tests and callers).  Returns UINT64_MAX out of range. */
uint64_t  fh_morton_cell(const uint32_t dims_xyz[3], uint32_t x, uint32_t y, uint32_t z);

/* fh_coreset_build -- steps 1-3 of §3.1 for the n key frames in vol
 * ([n][Z][Y][X] float32, device, normalised values):
 *   feature extraction f_k, dilation d_k = f_k plus its
 *   26-neighbourhood, clamped (R23), the occupancy bitmap of the cells
 *   d_k touches (R24; occupancy = [n][fh_occupancy_words] uint32,
 *   device, may be NULL), the per-frame bounding boxes b_k and their fusion,
 *   the FBB (an axis of one vertex is padded to two, R25), and the
 *   coreset size M = sum_k |d_k| (Eq. 3).
 * fbb (device, 6 int32: lo x,y,z, hi x,y,z; lo = INT_MAX if no frame has
 * the feature) and count (device, 1 uint64 = M) receive the results.
 * workspace: fh_coreset_workspace_size bytes (device, 16-byte aligned); it
 * carries the masks to fh_coreset_emit and must stay untouched in between.
 * Errors: FH_E_ARG (dims, n, kind, pointers), FH_E_RANGE (n X Y Z >= 2^32),
 * FH_E_CUDA. */
fh_status fh_coreset_build(const float *vol, const uint32_t dims_xyz[3], int n_frames,
                           const fh_feature_spec *spec, void *workspace, size_t workspace_bytes,
                           uint32_t *occupancy, int32_t *fbb, uint64_t *count, fh_stream stream);

/* fh_coreset_emit -- steps 4-5 (Eqs. 1-3) from the workspace of the last
 * fh_coreset_build with the same arguments: for every key frame k and every
 * vertex of d_k, in frame-major row-major order (R26), one training sample
 *   coords[i] = (x, y, z, t) float32 in the encoder domain [0,1]: Eqs. 1-2
 *               put the vertex in the FBB's [-1,1] frame (translate by the
 *               FBB centroid, scale by 2 / Size^FBB), mapped by (q+1)/2 (R2),
 *               i.e. (i_a - lo_a) / (hi_a - lo_a) rounded once; t = k/(n-1)
 *               (the key frame's [-1,1] time -1 + 2k/(n-1), R25, mapped the
 *               same way; 0.5 when n = 1)
 *   values[i] = vol[k][z][y][x].
 * Writes min(M, capacity) samples (coords [capacity][4], values [capacity],
 * device).  If no frame has the feature nothing is written (the caller sees
 * lo = INT_MAX in fbb: the paper's feature-not-found case).
 * Errors: FH_E_ARG, FH_E_CUDA. */
fh_status fh_coreset_emit(const float *vol, const uint32_t dims_xyz[3], int n_frames, const void *workspace,
                          size_t workspace_bytes, float *coords, float *values, uint64_t capacity,
                          fh_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* FHASH_CORESET_H_ */
