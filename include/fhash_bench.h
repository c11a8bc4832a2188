/*
 * fhash_bench.h -- roofline microbenchmarks exported by libfhash.so.
 *
 * These are MEASUREMENT kernels, not part of the method: they reproduce the
 * memory access shape of the encode (SURVEY.md §8(d) "Roofline
 * definition") so bench.py can state the measured gather / reduction
 * ceiling of the hot path on the box it runs on:
 *   - each thread issues `pairs` independent x-adjacent pairs of entry-sized
 *     accesses (entry i and i+1; the encode's 16 corners are 8 such pairs,
 *     P:166 "single look-up ... simple shifting" makes x-neighbours
 *     adjacent in Eq. 9), at pseudo-random i uniform over [0, n_entries-1);
 *   - gather: 8/16-byte loads through the read-only path (as fh_encode_fwd);
 *   - red: vector red.global.add.f32 of entry width (as fh_encode_bwd).
 * Buffers are caller-owned device memory; entry_bytes in {4, 8, 16}.
 * Errors: FH_E_ARG (NULL, entry_bytes, sizes), FH_E_CUDA.
 */
#ifndef FHASH_BENCH_H_
#define FHASH_BENCH_H_

#include "fhash.h"

#ifdef __cplusplus
extern "C" {
#endif

/* mode 0 ("split"): the two entries of a pair are two accesses of entry
 * width (2 L1/L2 requests per pair).  mode 1 ("ideal"): each pair is ONE
 * aligned access of twice the entry width (1 request / 1 sector per pair:
 * the minimum-sector shape).  pairs must be 8.
 * sink [n_threads] f32 receives one value per thread (defeats DCE). */
fh_status fh_bench_gather(const void *buf, uint64_t n_entries, int entry_bytes, int64_t n_threads,
                          int pairs, int mode, uint32_t seed, float *sink, fh_stream stream);

/* buf [n_entries] entries of f32 accumulated into (+= small values). */
fh_status fh_bench_red(float *buf, uint64_t n_entries, int entry_bytes, int64_t n_threads, int pairs,
                       int mode, uint32_t seed, fh_stream stream);

/* Level-mix variants (the encode's own shape): thread t is
 * (sample t / L, level t % L) as in the encode kernels, and issues 8 x-pairs,
 * each ONE aligned access of two entries (the ideal pair of mode 1) at a
 * uniform position inside level l's range [level_off[l], level_off[l] +
 * level_size[l]) of the packed buffer (host arrays, L <= 32, sizes >= 4).
 * n_samples * L threads; sink [n_samples * L].  gather: entry_bytes 4 or 8;
 * red: 4, 8 or 16 (16-byte entries: two reductions per pair). */
fh_status fh_bench_gather_levels(const void *buf, const uint64_t *level_off, const uint64_t *level_size, int L,
                                 int entry_bytes, int64_t n_samples, uint32_t seed, float *sink, fh_stream stream);
fh_status fh_bench_red_levels(float *buf, const uint64_t *level_off, const uint64_t *level_size, int L,
                              int entry_bytes, int64_t n_samples, uint32_t seed, fh_stream stream);

/* Streaming copy dst[i] = src[i] over `bytes` (16-byte aligned): the HBM
 * ceiling measured with the library's own kernel. */
fh_status fh_bench_copy(void *dst, const void *src, uint64_t bytes, fh_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* FHASH_BENCH_H_ */
