/*
 * fhash_data.h -- synthetic data generation on the device (HARNESS, not the
 * method): the time-varying scalar fields that stand in for the paper's
 * datasets (Combustion, Argon Bubble, Supernova; PAPER.md Table
 * tab:datasets, not available here) and the voxel sampler that
 * draws training batches ([t,x,y,z], v) samples, Eq. 3) from them.
 * Recipes: BASELINE.json configs[2] / configs[3]; values
 * min-max normalised to [0,1].  Field layout [t][z][y][x] fp32.
 */
#ifndef FHASH_DATA_H_
#define FHASH_DATA_H_

#include "fhash.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Sum of n_blobs Gaussian blobs moving linearly in time plus
 * 0.1 sin(8 pi x) sin(8 pi y) (unnormalised).  blobs: HOST array [n][7] =
 * (sigma, c0x, c0y, c0z, vx, vy, vz); blob centre at tau = t/(T-1) is
 * c0 + v tau; coordinates x = i/(S-1).  field: device [T][S][S][S]. */
fh_status fh_data_gaussian_blobs(float *field, int S, int T, int n_blobs, const float *blobs, fh_stream stream);

/* 3 octaves of 4D value noise (integer-hash lattice values U(0,1), quintic
 * fade, frequencies 4/8/16 per unit, amplitudes 1/0.5/0.25), unnormalised.
 * field: device [T][Sz][Sy][Sx]. */
fh_status fh_data_value_noise(float *field, int Sx, int Sy, int Sz, int T, uint32_t seed, fh_stream stream);

/* In place: v <- (v - min) / (max - min).  If band_width > 0, then also
 * v <- 0.5 v + 0.5 exp(-((v - 0.5) / band_width)^2) followed by a second
 * min-max normalisation (the "sharp isosurface band" of configs[3]).
 * scratch: device, >= 64 bytes.  Synchronous on `stream` (reads min/max). */
fh_status fh_data_normalize(float *field, int64_t n, float band_width, void *scratch, fh_stream stream);

/* N random voxels (uniform over the T*Sz*Sy*Sx grid) drawn with
 * Philox4x32-10 (key = seed, counter = (sample, subsequence, offset)):
 * coords [N][4] = (x/(Sx-1), y/(Sy-1), z/(Sz-1), t/(T-1)) f32, target [N] =
 * field value.  Same (seed, subsequence, offset) -> same batch. */
fh_status fh_data_sample_voxels(const float *field, int Sx, int Sy, int Sz, int T, int64_t N, uint64_t seed,
                                uint32_t subsequence, uint32_t offset, float *coords, float *target,
                                fh_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* FHASH_DATA_H_ */
