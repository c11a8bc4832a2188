/*
 * fhash.h -- C ABI of libfhash.so, the B200 (sm_100a) hot path of F-Hash
 * (arXiv 2507.03836): the multi-resolution Tesseract (x,y,z,t) embedding
 * encode through the paper's minimal perfect hash, forward and backward, and
 * the small-MLP train step that uses it.
 *
 * Citations: "P:n" = the paper text line n with its section /
 * equation; "S:n" = SPEC.md line n.  Readings R1..R18 of ambiguous passages
 * are listed in DESIGN.md §3.
 *
 * Conventions shared by every entry point
 *   - Plain pointers and sizes only.  "device" pointers are CUDA global
 *     memory on the current device, allocated and OWNED BY THE CALLER; the
 *     library owns only the opaque host handles it returns and one 16-byte
 *     status word per encoder (made by fh_build_levels / fh_build_mhe on
 *     the current device).  No stream-ordered call allocates device memory.
 *   - Every call that takes a stream is stream-ordered on it and does NOT
 *     synchronise (except fh_status_sync).  stream may be NULL (legacy
 *     default stream).
 *   - Errors: host-side validation returns synchronously (FH_E_ARG,
 *     FH_E_RANGE, FH_E_STATE); launch failures return FH_E_CUDA.  Nothing
 *     aborts and nothing throws across the ABI.  fh_last_error() returns a
 *     thread-local message for the last failing call on the calling thread.
 *   - Coordinates: [N][4] float32 = (x, y, z, t) in the ABI domain [0,1]
 *     (R2: a caller in the paper's [-1,1] domain, maps q -> (q+1)/2).
 *     16-byte aligned.  Out-of-domain or NaN coordinates are clamped to
 *     [0,1] (NaN -> 0) and set a sticky per-encoder device flag that
 *     fh_status_sync reports as FH_E_DOMAIN; they never fault.
 *   - Tables: one packed buffer [sum_l T_l][F], level-major in the order
 *     given to fh_build_levels, the F features of an entry contiguous.
 */
#ifndef FHASH_H_
#define FHASH_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    FH_OK = 0,
    FH_E_ARG = -1,       /* bad argument: null/misaligned pointer, L, R, F, dtype */
    FH_E_RANGE = -2,     /* sizes overflow the supported range */
    FH_E_DOMAIN = -3,    /* a kernel saw out-of-domain / NaN coordinates (clamped) */
    FH_E_CUDA = -4,      /* CUDA launch or runtime error */
    FH_E_DIVERGED = -5,  /* non-finite loss in a train step */
    FH_E_STATE = -6      /* handle in the wrong state / wrong device */
} fh_status;

typedef enum { FH_F32 = 0, FH_F16 = 1, FH_BF16 = 2 } fh_dtype;

/* Opaque CUDA stream (binary-compatible with cudaStream_t). */
typedef struct CUstream_st *fh_stream;

#define FH_MAX_LEVELS 32

/* Vertices per axis of one level, order (x, y, z, t); each >= 2.
 * R1: "Res" is the VERTEX count -- Eq. 9 is bijective only when
 * 0 <= x < Res_x; confirmed by the Table-3 parameter counts. */
typedef struct { uint32_t res[4]; } fh_level_res;

typedef struct {
    uint32_t res[4];      /* x, y, z, t vertex counts */
    uint64_t corners;     /* C_l = prod res (64-bit) */
    uint64_t table_size;  /* T_l: = C_l (bijective, Eq. 9) or the cap (hashed, R5) */
    uint32_t hashed;      /* 1 if C_l > cap */
    uint32_t reserved;    /* linearization of a bijective level: FH_LIN_EQ9 or FH_LIN_BRICK (0 if hashed) */
    uint64_t offset;      /* first entry of this level in the packed table */
} fh_level_info;

typedef struct fh_encoder_s *fh_encoder;

/* ---------------------------------------------------------------- a1 ---
 * fh_fold_schedule -- Eqs. 4-8 (§3.2.1) and the temporal
 * analogue (§3.2.2).
 *   Level 1 = native (S_x, S_y, S_z, n_t) (Eq. 4); per-axis level count
 *   L_a = ceil(log_fold S_a) (Eq. 5, integer: least L with fold^L >= S_a);
 *   L_s = max over the four axes (Eq. 6, R9); Res^l = ceil(Res^{l-1}/fold)
 *   while Res^{l-1} > fold, else Tail = 2, for l = 2..L_s (Eqs. 7-8, R8).
 * out: caller array of *L_inout entries; on success *L_inout = L_s and out
 * holds the levels in PAPER ORDER (finest first).
 * Errors: FH_E_ARG if any S < 2, n_t < 2, fold < 2 or a NULL pointer;
 * FH_E_RANGE if L_s exceeds the capacity *L_inout (which is set to L_s). */
fh_status fh_fold_schedule(const uint32_t S_xyz[3], uint32_t n_t, uint32_t fold,
                           fh_level_res *out, int *L_inout);

/* ---------------------------------------------------------------- a1 ---
 * fh_build_levels -- the per-level tables (D1/D2: "hash tables ... scaling
 * their sizes proportionally with the embedding grid size").
 *   res[L] (1 <= L <= 32): levels in OUTPUT order (R11: the concatenation
 *   order of the encoded vector).  F in {1,2,4,8} features per entry.
 *   table_dtype: FH_F32 or FH_F16 (the dtype of the table passed to the
 *   encode calls).  cap: 0 = uncapped (pure MPHF); otherwise a power
 *   of two; a level with C_l > cap becomes a hashed level of T_l = cap
 *   entries (R5; the paper never caps).
 * Errors: FH_E_ARG (L, F, R < 2, cap not a power of two, dtype);
 * FH_E_RANGE if sum_l T_l * F >= 2^32; FH_E_CUDA if the status word
 * cannot be made.  On success *out owns a host handle, bound to the
 * current device: its launch plan (L2-sized level groups, few-cell and
 * replicated backward levels) is fixed here from the device's L2 size and
 * SM count, and a 16-byte status word is allocated there (synchronously:
 * this is set-up, not a stream-ordered call).  Built with no CUDA device
 * present, the handle answers the host queries (level info, scratch size)
 * and every device call returns FH_E_STATE; calls from another device
 * also return FH_E_STATE. */
fh_status fh_build_levels(const fh_level_res *res, int L, int F, fh_dtype table_dtype,
                          uint64_t cap, fh_encoder *out);

/* ---------------------------------------------------------- NEXT-2 ---
 * fh_build_levels_lin -- fh_build_levels with a choice of the bijective
 * linearization ("Other linearizations like Morton and Z-order can also be
 * used to construct F-Hash with preserved locality", §3.2.3):
 *   FH_LIN_EQ9    Eq. 9 row-major, x fastest -- fh_build_levels;
 *   FH_LIN_BRICK  brick order (reading R21): 2x2x2x2-vertex bricks (clipped
 *                 at odd grid edges) in row-major order, vertices row-major
 *                 inside a brick; with b = v>>1, i = v&1, e = min(2, R-2b):
 *                 idx = 2 b_t RxRyRz + 2 b_z RxRy e_t + 2 b_y Rx e_z e_t
 *                     + 2 b_x e_y e_z e_t + ((i_t e_z + i_z) e_y + i_y) e_x + i_x.
 *                 Still a bijection onto [0, C_l) (minimal perfect hash); the
 *                 16 corners of a cell at even coordinates are 16 consecutive
 *                 entries.  Hashed (capped) levels are unaffected.
 * Table size, packing and every encode call are as for fh_build_levels.
 * Errors: as fh_build_levels, FH_E_ARG for another linearization value. */
enum { FH_LIN_EQ9 = 0, FH_LIN_BRICK = 1 };
fh_status fh_build_levels_lin(const fh_level_res *res, int L, int F, fh_dtype table_dtype,
                              uint64_t cap, int linearization, fh_encoder *out);

/* ---------------------------------------------------------- NEXT-3 ---
 * fh_build_mhe -- the MHE baseline the paper compares against (
 * Fig. 4; SPEC baseline_encode S:321-329), on the same kernels:
 * one 3D multi-resolution hash encoder per key frame.  res[L]: vertices per
 * spatial axis per level; every level and frame has a FIXED table of T
 * entries (power of two): direct index x + y R + z R^2 when R^3 <= T (the
 * rest of the T buckets are wasted), else (x*1 ^ y*2654435761 ^ z*805459861)
 * mod T (uint32).  A sample's frame is the key frame nearest to its t:
 * s = fp32(t (n_frames-1)), k = floor(s) + (s - floor(s) >= 0.5) (R20);
 * trilinear blend of the 8 corners of its (x,y,z) cell.  Table: level l,
 * frame k at entries offset_l + k T + [0, T); params = L n_frames T F.
 * The fh_encode_* calls accept the returned handle (fh_encode_indices then
 * writes [N][L][8]); the trainer does not.
 * Errors: FH_E_ARG, FH_E_RANGE. */
fh_status fh_build_mhe(const uint32_t *res, int L, int F, fh_dtype table_dtype, uint64_t T,
                       uint32_t n_frames, fh_encoder *out);
/* 0 = F-Hash Tesseract encoder, 1 = MHE baseline. */
int       fh_encoder_kind(fh_encoder enc);

fh_status fh_level_info_get(fh_encoder enc, int l, fh_level_info *out);
int       fh_num_levels(fh_encoder enc);
int       fh_feature_dim(fh_encoder enc);
uint64_t  fh_table_entries(fh_encoder enc);   /* sum_l T_l */
uint64_t  fh_param_count(fh_encoder enc);     /* sum_l T_l * F */
void      fh_encoder_destroy(fh_encoder enc);

/* ------------------------------------------------------------ a2..a7 ---
 * fh_encode_fwd -- steps 1-4 of §3.2.4 for every sample and
 * level, concatenated:
 *   per axis s = fp32(p * (R-1)), i = clamp(floor s, 0, R-2), w = s - i
 *   (R2; steps 1-2); the 16 corners c = bx+2by+4bz+8bt (R3)
 *   map through Eq. 9 ("a single look-up ... through simple
 *   shifting") or the capped hash (R5) to entries of the level's
 *   table; out = quadrilinear blend, trilinear per time slice (Eqs. 10-11)
 *   then linear in t (Eq. 12, R6).
 * coords [N][4] f32 (device); table [sum T][F] of the encoder's table_dtype
 * (device, 32-byte aligned: x-pairs of corners are fetched as aligned
 * 2-entry chunks); out [N][L*F] of out_dtype FH_F32 or FH_BF16 (device),
 * row n = (level 0 features, level 1 features, ...).
 * Scratch: large passes use the caller-owned scratch attached to the
 * calling stream (fh_encoder_attach_scratch; the table
 * shifted by one entry, and in fh_encode_bwd a shifted gradient scratch);
 * a stream without one runs without the shifted pairs (same results).
 * Calls of one encoder are safe concurrently on different streams, each
 * with its own scratch; do not run two passes of one encoder concurrently
 * on the SAME stream's scratch (e.g. a replayed graph and a live call).
 * N = 0 is a no-op.  Errors: FH_E_ARG (NULL/misaligned, dtype),
 * FH_E_STATE (no device state / wrong device), FH_E_CUDA. */
fh_status fh_encode_fwd(fh_encoder enc, const float *coords, int64_t N, const void *table,
                        void *out, fh_dtype out_dtype, fh_stream stream);

/* ---------------------------------------------------------------- a10 --
 * fh_encode_bwd -- adjoint of fh_encode_fwd ("gradient
 * computation ... during backpropagation"):
 *   dtable[idx_c][f] += W_c * dout[n][l*F+f]  for every n, l, corner c,
 * with W_c the quadrilinear weight of corner c.  dout [N][L*F] f32 (device);
 * dtable [sum T][F] f32 (device), ACCUMULATED INTO (the caller zeroes it).
 * Order of the floating-point sums is unspecified (atomics).
 * Errors: FH_E_ARG, FH_E_CUDA. */
fh_status fh_encode_bwd(fh_encoder enc, const float *coords, int64_t N, const float *dout,
                        float *dtable, fh_stream stream);

/* fh_encode_bwd_ex -- fh_encode_bwd with flags.  FH_BWD_OVERWRITE: dtable
 * is OVERWRITTEN with the gradient instead of accumulated into; the library
 * zeroes it level group by level group right before the launch that
 * reduces into that group (so the zeroed lines are still L2-resident when
 * the reductions arrive; a separate fh_zero_grad before the forward has
 * them evicted by the forward's traffic).  Unknown flags: FH_E_ARG. */
#define FH_BWD_OVERWRITE 1u
/* FH_BWD_DOUT_LEVEL_MAJOR: dout is level-major, [L][N][F] f32 (level l's
 * gradient rows at dout + l N F), instead of the row-major [N][L F] of
 * fh_encode_bwd; same values, same result.  A level pass then reads
 * contiguous F-float rows (cfg4, F = 4: bwd 6.11 -> 5.51 ms; F = 2:
 * neutral).  The trainer's dL/d(enc) for F >= 4 is in this layout.
 * F-Hash encoders only (MHE: FH_E_ARG). */
#define FH_BWD_DOUT_LEVEL_MAJOR 2u
fh_status fh_encode_bwd_ex(fh_encoder enc, const float *coords, int64_t N, const float *dout,
                           float *dtable, unsigned flags, fh_stream stream);

/* ---------------------------------------------------------------- a4 ---
 * fh_encode_indices -- the corner indices alone (steps 1-3), for parity:
 * idx [N][L][16] uint32 global entry indices (level offset included),
 * corner order R3; w [N][L][16] f32 corner weights (may be NULL). */
fh_status fh_encode_indices(fh_encoder enc, const float *coords, int64_t N, uint32_t *idx,
                            float *w, fh_stream stream);

/* fh_zero_grad -- dtable [sum T][F] f32 (device) := 0, stream-ordered
 * (cudaMemsetAsync).  Errors: FH_E_ARG (NULL), FH_E_CUDA. */
fh_status fh_zero_grad(fh_encoder enc, float *dtable, fh_stream stream);

/* fh_encode_fwd_bwd -- one encode step on device buffers, the unit
 * bench.py times for BASELINE.json configs[1]: fh_encode_fwd (out,
 * out_dtype), then fh_encode_bwd_ex (dout -> dtable; FH_BWD_OVERWRITE when
 * zero_dtable, i.e. dtable = the gradient, else dtable += it).  Arguments
 * and errors as those calls. */
fh_status fh_encode_fwd_bwd(fh_encoder enc, const float *coords, int64_t N, const void *table,
                            void *out, fh_dtype out_dtype, const float *dout, float *dtable,
                            int zero_dtable, fh_stream stream);

/* fh_encode_step_host -- one encode fwd+bwd step from HOST buffers (the
 * end-to-end form used by bench.py's "e2e" figure): copies coords_h
 * [N][4] and dout_h [N][L*F] (pinned host memory for asynchrony) into the
 * caller's device buffers coords_d / dout_d, runs fh_encode_fwd (out_d,
 * f32) and fh_encode_bwd_ex (FH_BWD_OVERWRITE: dtable_d = the gradient), and
 * copies out_d -> out_h and dtable_d -> dtable_h.  All on `stream`; returns
 * without waiting.  Stream-ordered, so a caller pipelines consecutive steps
 * by rotating over several streams with their own device buffers and host
 * outputs: step k+1's H2D then overlaps step k's kernels and step k-1's D2H
 * (bench.py's e2e uses three), each stream with its own attached scratch.
 * Errors: as the calls it makes. */
fh_status fh_encode_step_host(fh_encoder enc, const float *coords_h, const float *dout_h,
                              int64_t N, const void *table_d, float *coords_d, float *dout_d,
                              float *out_d, float *dtable_d, float *out_h, float *dtable_h,
                              fh_stream stream);

/* fh_status_sync -- synchronise `stream`, then report and clear the
 * encoder's sticky domain flag: FH_E_DOMAIN if any kernel of this encoder
 * clamped an out-of-domain / NaN coordinate since the last call, else FH_OK
 * (or FH_E_CUDA if the stream reported an error). */
fh_status fh_status_sync(fh_encoder enc, fh_stream stream);

/* ============================================================ train step
 * The INR train step around the encoder (§3(4) of SURVEY; the paper trains
 * "the INRs with input encoding ... Adam ... learning rate of 0.01", P:489,
 * on the "shallow network" of P:233, "2 layers x 64 neurons"):
 *   a2-a7 encode fwd (fp16 table shadow -> bf16 encoding, R13)
 *   a8    MLP n_in -> 64 -> 64 -> 1, ReLU, biases (R15) on tcgen05 tensor
 *         cores, forward and backward, bf16 operands / fp32 accumulation
 *   a9    MSE over the GLOBAL batch: loss = sum (y - t)^2 / N_global,
 *         dL/dy = 2 (y - t) / N_global (R12)
 *   a10   encode bwd (fp32 dL/d(enc) scattered into fp32 table grads)
 *   a11   dense bias-corrected Adam (lr, beta1, beta2, eps; R12) on fp32
 *         masters of every parameter; rewrites the low-precision shadows and
 *         zeroes the grads.
 * Data parallel: fh_train_fwd_bwd leaves the complete local gradients in
 * the caller's grad buffers; the caller all-reduces (SUM) them across ranks
 * (e.g. torch.distributed over NCCL) and then calls fh_train_apply.  The
 * loss is already scaled by 1/N_global, so summed gradients are exact. */
typedef struct fh_trainer_s *fh_trainer;

typedef struct {
    int n_in;             /* MLP input width; must equal L*F; one of 16, 32, 48, 64 */
    int n_hidden;         /* must be 64 */
    int n_hidden_layers;  /* must be 2 */
} fh_mlp_desc;

/* Every buffer is caller-owned device memory (16-byte aligned).
 * Table buffers have fh_table_entries(enc) * F elements; MLP buffers have
 * fh_mlp_param_count() elements in the flat order
 *   W1[64][n_in], b1[64], W2[64][64], b2[64], w3[64], b3
 * (weights [out][in] row-major).  table_shadow has the encoder's table
 * dtype (FH_F16: Adam writes it; FH_F32: pass NULL, the master is read
 * directly); mlp_shadow is bf16.  The grad buffers need no initialisation:
 * every fh_train_fwd_bwd overwrites them with the step's gradient. */
typedef struct {
    float *table_master;
    void *table_shadow;
    float *table_grad;
    float *table_m;
    float *table_v;
    float *mlp_master;
    void *mlp_shadow;
    float *mlp_grad;
    float *mlp_m;
    float *mlp_v;
    void *workspace;          /* fh_train_workspace_size bytes */
    size_t workspace_bytes;
} fh_train_buffers;

/* Adam hyper-parameters in double: 1 - beta is formed in double and rounded
 * once to fp32 (fp32 1 - 0.999f is 1.3e-5 relative off 0.001). */
typedef struct { double lr, beta1, beta2, eps; } fh_adam;

uint64_t  fh_mlp_param_count(const fh_mlp_desc *mlp);
size_t    fh_train_workspace_size(fh_encoder enc, const fh_mlp_desc *mlp, int64_t max_batch);

/* Errors: FH_E_ARG (shape, NULL/misaligned buffer, small workspace),
 * FH_E_CUDA.  The trainer keeps a reference to enc (caller keeps it alive). */
fh_status fh_trainer_create(fh_encoder enc, const fh_mlp_desc *mlp, const fh_train_buffers *buf,
                            const fh_adam *adam, int64_t max_batch, fh_trainer *out);

/* Forward + loss + backward for N_local samples (coords [N][4] f32,
 * target [N] f32, device).  loss_dev (device f32, may be NULL) receives
 * sum_local (y - t)^2 / N_global.  The grad buffers are OVERWRITTEN with
 * this call's gradient (table grads zeroed level group by level group right
 * before the reductions, FH_BWD_OVERWRITE; MLP grads zeroed first), so the
 * optimiser never has to clear them.  N_local <= max_batch, N_global >=
 * N_local. */
fh_status fh_train_fwd_bwd(fh_trainer tr, const float *coords, const float *target, int64_t N_local,
                           int64_t N_global, float *loss_dev, fh_stream stream);

/* fh_train_dx_layout -- the layout of the trainer's dL/d(enc) workspace
 * (the MLP kernel's dX, the encode backward's dout): 0 = row-major
 * [N][L F]; F (>= 4) = level-major [L][N][F] (FH_BWD_DOUT_LEVEL_MAJOR),
 * chosen at fh_trainer_create for F >= 4 unless FH_DX_ROW_MAJOR is set in
 * the environment.  -1: NULL trainer.  Host only. */
int       fh_train_dx_layout(fh_trainer tr);

/* One Adam step on all parameters (step counter += 1). */
fh_status fh_train_apply(fh_trainer tr, fh_stream stream);

/* Sharded Adam (data parallel, ZeRO-1 style): Adam on the
 * table parameters [begin, end) of the flat table space [0, entries*F),
 * reading their (already reduce-scattered) gradients from grad_shard
 * (device f32, end - begin values), plus the full MLP segment from the
 * trainer's mlp_grad (already all-reduced).  Updates masters, moments and
 * shadows in the range only.  begin must be a multiple of 4.  The caller
 * then all-gathers the shadow (or, for FH_F32 tables, the master). */
fh_status fh_train_apply_sharded(fh_trainer tr, int64_t begin, int64_t end, const float *grad_shard,
                                 fh_stream stream);

/* ---- overlapping the gradient reduction with the backward
 * The encode backward of fh_train_fwd_bwd runs as a few launches (the
 * shared-memory pass over the tiny levels, then level groups sized to the
 * L2); once launch i has run, the table gradients of its ranges are final,
 * so a data-parallel caller can reduce them while later launches run.
 * fh_train_bwd_launches: number of backward launches (-1 on error).
 * fh_train_bwd_ranges: the flat table element ranges [r[2k], r[2k+1]) that
 *   launch i finalises (k < *n_ranges); FH_E_RANGE if more than max_ranges.
 * fh_train_set_bwd_events: from now on fh_train_fwd_bwd records events[i]
 *   (caller-owned cudaEvent_t, created by the caller) on its stream right
 *   after the launch that completes backward group i (a group's last step,
 *   the merge of the shifted scratch, may ride in the next group's launch);
 *   n = fh_train_bwd_launches, or 0 to stop.
 * fh_train_apply_ranges: one Adam step (step counter += 1) over the table
 *   element ranges [begin_i, end_i) (disjoint) reading grad_i[0 .. end_i -
 *   begin_i) (device f32, e.g. this rank's reduce-scattered chunks), plus the
 *   whole MLP segment from the trainer's mlp_grad; rewrites the shadows of
 *   those ranges.  At most
 *   63 ranges; ranges whose pointers are not 16-byte aligned take a scalar
 *   path.  Errors: FH_E_ARG. */
int       fh_train_bwd_launches(fh_trainer tr);
fh_status fh_train_bwd_ranges(fh_trainer tr, int launch, int64_t *ranges, int max_ranges, int *n_ranges);
fh_status fh_train_set_bwd_events(fh_trainer tr, void *const *events, int n);
fh_status fh_train_apply_ranges(fh_trainer tr, int n, const int64_t *begin, const int64_t *end,
                                const float *const *grad, fh_stream stream);

/* ---- fused reduce-scatter + Adam + all-gather over peer memory (§8(e) 3)
 * fh_train_apply_peers: ONE kernel per call, for a data-parallel group of W
 * ranks (1 <= W <= 8) whose gradient and shadow buffers are mapped into
 * this process (e.g. torch symmetric memory over NVLink / NVSwitch).  For
 * every table element range [begin_i, end_i) it reads the gradient as the
 * SUM over ranks r = 0..W-1 (in that order) of peer_table_grad[r][e], runs
 * Adam on this trainer's fp32 master / moments, and stores the fp16 value
 * into peer_table_shadow[r][e] of EVERY rank (broadcast[i] = 1: this rank's
 * chunk) or only into its own shadow (broadcast[i] = 0: a range every rank
 * updates identically).  with_mlp = 1 also updates the MLP from the sum of
 * peer_mlp_grad[r].  new_step = 1 on the first call of a step (step
 * counter += 1; later calls of the same step pass 0).  Does NOT zero any
 * gradient (peers may still be reading them): the caller zeroes its local
 * grads once every rank is done, and orders the call after every rank's
 * backward (e.g. a symmetric-memory barrier).  Pointers: device-accessible
 * (peer) addresses of each rank's flat table grad [entries*F] f32, fp16
 * shadow, and MLP grad.  Errors: FH_E_ARG, FH_E_STATE (no fp16 shadow). */
fh_status fh_train_apply_peers(fh_trainer tr, int W, const float *const *peer_table_grad,
                               void *const *peer_table_shadow, const float *const *peer_mlp_grad, int n,
                               const int64_t *begin, const int64_t *end, const int *broadcast, int with_mlp,
                               int new_step, fh_stream stream);

/* fh_train_apply_multicast: the same step through an NVLS multicast object
 * ("multimem.ld_reduce of a shard from an NVLS
 * multicast buffer, Adam in registers, then multimem.st of the fp16 shard
 * to all peers").  mc_table_grad, mc_table_shadow, mc_mlp_grad are the
 * MULTICAST addresses of the group's flat table grad buffer [entries*F]
 * f32, fp16 table shadow and MLP grad buffer (a multicast object bound to
 * the same buffer on every rank: torch symmetric memory's multicast
 * pointer, or cuMulticastCreate + cuMulticastBindMem; 16-byte aligned
 * grads, 8-byte aligned shadow).  Each element's gradient is ONE
 * multimem.ld_reduce (.add.f32: the sum over the ranks, formed by the
 * NVSwitch); broadcast ranges store the fp16 shadow with ONE multimem.st
 * into every rank's shadow (in f16x2 pairs: broadcast ranges have even
 * begin and end), replicated ranges (and the MLP) store locally
 * -- replicas stay identical when every rank receives the same reduced
 * value.  Same range / broadcast / with_mlp / new_step / ordering contract
 * as fh_train_apply_peers (the caller orders the call after every rank's
 * backward and zeroes nothing).  Errors: FH_E_ARG (NULL / misaligned
 * address, bad ranges), FH_E_STATE (no fp16 shadow, first call without
 * new_step). */
fh_status fh_train_apply_multicast(fh_trainer tr, const float *mc_table_grad, void *mc_table_shadow,
                                   const float *mc_mlp_grad, int n, const int64_t *begin, const int64_t *end,
                                   const int *broadcast, int with_mlp, int new_step, fh_stream stream);

/* ---- the fused data-parallel form (SURVEY.md §8(b) "nccl_comm", §8(e))
 * The library drives the gradient exchange itself with NCCL: the
 * libnccl.so.2 the process already loaded (torch's; resolved with dlopen
 * RTLD_NOLOAD, else a plain dlopen), so the library shares torch's NCCL.
 * fh_nccl_unique_id: 128 bytes of ncclUniqueId into id (rank 0 calls it;
 *   the caller broadcasts them, e.g. over torch.distributed).
 * fh_nccl_comm_create: ncclCommInitRank(nranks, id, rank) on the current
 *   device -> *comm (opaque; the caller destroys it after its trainers).
 * fh_trainer_dp_workspace_size / fh_trainer_set_comm: attach a communicator
 *   (comm NULL detaches) and caller-owned device workspace (shards of the
 *   reduce-scattered gradients and the small replicated tail + MLP buffer).
 *   From then on fh_train_step runs the whole data-parallel step: the encode
 *   backward's level groups (fh_train_bwd_ranges) are reduce-scattered
 *   (ncclReduceScatter, SUM) on an internal stream as soon as each group's
 *   gradients are final, overlapping the later groups; the < 4W + 4
 *   unaligned tail elements of every group and the MLP gradients are
 *   all-reduced; ONE Adam launch updates this rank's chunks and the tails;
 *   the fp16 shadow chunks are all-gathered (ncclAllGather, in place).  The
 *   caller's stream is ordered after all of it.  Same mathematics as
 *   fh_train_fwd_bwd + all-reduce + fh_train_apply.  Needs an FH_F16 table
 *   (the fp16 shadow is the replicated state: the fp32 masters and moments
 *   of a rank are current only inside its own chunks).
 * Errors: FH_E_STATE (NCCL not loadable, no fp16 shadow), FH_E_ARG,
 * FH_E_CUDA (NCCL failures, with NCCL's message). */
fh_status fh_nccl_unique_id(void *id128);
fh_status fh_nccl_comm_create(const void *id128, int nranks, int rank, void **comm);
fh_status fh_nccl_comm_destroy(void *comm);
size_t    fh_trainer_dp_workspace_size(fh_trainer tr, int nranks);
fh_status fh_trainer_set_comm(fh_trainer tr, void *comm, int nranks, int rank, void *workspace,
                              size_t workspace_bytes);

/* fh_train_fwd_bwd + fh_train_apply (single GPU); with a communicator
 * attached (fh_trainer_set_comm) the fused data-parallel step. */
fh_status fh_train_step(fh_trainer tr, const float *coords, const float *target, int64_t N_local,
                        int64_t N_global, float *loss_dev, fh_stream stream);

/* Synchronise `stream`; FH_E_DIVERGED if a non-finite loss was seen since
 * the last call (sticky flag, cleared by the read), FH_E_DOMAIN if the
 * encoder clamped coordinates, else FH_OK. */
fh_status fh_trainer_status(fh_trainer tr, fh_stream stream);
int64_t   fh_trainer_step_count(fh_trainer tr);
void      fh_trainer_destroy(fh_trainer tr);

/* ============================================================ inference
 * The renderer's model evaluation "V = model(S)" (Alg. 1) as ONE
 * fused kernel (NEXT-1): the encode forward of each 128-sample tile goes as
 * bf16 straight into the shared-memory X operand of the tcgen05 MLP forward
 * (small batches are cut into short tiles so they spread over the SMs), with
 * exactly the forward numerics of the train step (R13).
 * table: the encoder's table dtype (fp16 shadow or fp32, 32-byte aligned);
 * mlp_shadow bf16 (16-byte aligned) and mlp_master fp32 in the flat MLP
 * layout; y [N] f32 (device).  Workspace: none for the fused form
 * (fh_infer_workspace_size returns 0; workspace may be NULL); a LARGE batch
 * (>= 8 tiles per SM) over tables bigger than the forward's L2 budget is
 * faster in two launches -- fh_encode_fwd's L2-sized level groups into
 * max_batch * n_in bf16 of workspace, then the kernel's MLP-only mode --
 * and fh_infer_workspace_size(enc, mlp, max_batch) returns that size.
 * F-Hash encoders only.  Errors as fh_train_fwd_bwd (FH_E_ARG when a
 * two-launch batch gets too little workspace). */
size_t    fh_infer_workspace_size(fh_encoder enc, const fh_mlp_desc *mlp, int64_t max_batch);
fh_status fh_infer(fh_encoder enc, const fh_mlp_desc *mlp, const void *table, const void *mlp_shadow,
                   const float *mlp_master, const float *coords, int64_t N, float *y, void *workspace,
                   size_t workspace_bytes, fh_stream stream);

/* ARM marching pace, Alg. 1 line "N_s = max(min(N_r / N_a, 64), 1)"
 * (P:255): N_r read as the total number of rays (the symbol is undefined in
 * the paper; R19), integer division.  0 when no ray is alive. */
int64_t   fh_arm_pace(int64_t n_rays, int64_t n_alive);

/* ============================================================ encoding stats
 * fh_level_stats -- encoding_stats of one level (the
 * collision / bucket-waste contrast of Fig. 4): every lattice
 * vertex of the level (for an MHE encoder: of one key frame's R^3 grid) is
 * mapped to its bucket exactly as the encode maps corners, and *out (device,
 * uint64) receives the number of DISTINCT buckets hit.  With C vertices
 * (fh_level_info corners; R^3 for MHE) and T buckets (table_size; the MHE
 * T): collisions = C - distinct, utilisation = distinct / T.  F-Hash levels
 * (Eq. 9 / brick) give distinct = C = T.  Exhaustive -- a diagnostic, not on
 * the train path.  workspace (device, 16-byte aligned) of
 * fh_level_stats_workspace_size(enc, level) bytes (a T-bit bitmap).
 * Errors: FH_E_ARG, FH_E_CUDA. */
size_t    fh_level_stats_workspace_size(fh_encoder enc, int level);
fh_status fh_level_stats(fh_encoder enc, int level, void *workspace, size_t workspace_bytes, uint64_t *out,
                         fh_stream stream);

/* fh_encoder_scratch_size / fh_encoder_attach_scratch -- the caller-owned
 * shifted-pair scratch (see fh_encode_fwd), one per stream:
 * fh_encoder_scratch_size(enc) bytes (device, 256-byte aligned; covers every
 * pass of this encoder: the table copy up to the last level the forward may
 * shift, the fp32 gradient scratch of the shiftable backward levels or the
 * 64 replicated copies of a replicated level, and for F >= 4 the in-pass
 * replicated copies of the contended coarse levels -- up to 32 copies, at
 * most 2^20 entries, per level of at most 2^18 entries; a backward on a
 * stream without scratch runs without them, same result).  No initial contents are
 * needed: each range is written or zeroed right before use.  The library
 * never allocates, grows or frees it; ptr = NULL detaches (after
 * synchronising `stream`: attach is set-up, not stream-ordered).  Size 0 /
 * FH_E_ARG for MHE encoders; FH_E_ARG if too small or misaligned;
 * FH_E_STATE if all 8 stream slots are taken. */
size_t    fh_encoder_scratch_size(fh_encoder enc);
fh_status fh_encoder_attach_scratch(fh_encoder enc, fh_stream stream, void *ptr, size_t bytes);

/* fh_kernel_launches -- number of CUDA kernels this library has launched
 * so far (all threads, all encoders / trainers; the method's kernels, not
 * the fhash_bench.h / fhash_data.h harness kernels, not memset / memcpy).
 * Read before and after a region to count its launches. */
unsigned long long fh_kernel_launches(void);

/* Thread-local text of the last error on this thread ("" if none). */
const char *fh_last_error(void);

/* Library version string. */
const char *fh_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FHASH_H_ */
