/*
 * fhash_oracle.c -- CPU ORACLE for the F-Hash multi-resolution Tesseract
 * encode (arXiv 2507.03836).  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load this library.  It shares no code, header,
 * table or constant generator with the CUDA path in paper_2507_03836_b200/;
 * neither side includes or links the other.
 *
 * Plain, slow, obviously-correct: one sample at a time, one level at a time,
 * one corner at a time, accumulation in fp64.  Build with
 *     gcc -O2 -std=c11 -ffp-contract=off -fPIC -shared
 * (no fast-math, no FMA contraction: the one fp32 multiply that decides the
 * cell index must be a single IEEE round-to-nearest product, R2).
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n.
 * Readings R1..R18 are listed in DESIGN.md §3 (same numbering as SURVEY.md
 * §8(c) D1..D18).
 *
 * Pins (tests/test_oracle.py, -m "not gpu"): SPEC worked examples, Table-3
 * parameter counts, brute-force bijectivity / utilisation, partition of
 * unity, lattice exactness, multilinear reproduction, finite differences,
 * adjoint identity.  The capped-level hash (R5) is pinned only by its
 * integer definition plus brute-force collision statistics ("parity
 * unpinned by the paper").
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ a1 --
 * Fold schedule, Eqs. 4-8 + temporal analogue.
 *   Res^1 = S (Eq. 4); L_a = ceil(log_f S_a) (Eq. 5) computed as the least
 *   integer L >= 1 with f^L >= S_a (R8); L_s = max over axes (Eq. 6, R9,
 *   extended to t as S:279); Res^l = ceil(Res^{l-1}/f) if Res^{l-1} > f,
 *   else Tail = 2, for l = 2..L_s (Eqs. 7-8, R8).
 * out: [L][4] (x,y,z,t), level 1 (native, finest) first.  Returns L_s, or
 * -1 on bad arguments, or -2 if L_s > max_L.
 */
static int ceil_log(uint64_t S, uint64_t f)
{
    int L = 1;
    uint64_t p = f;
    while (p < S) { p *= f; L++; }
    return L;
}

int fho_fold_schedule(const uint32_t S_xyz[3], uint32_t n_t, uint32_t fold,
                      uint32_t *out, int max_L)
{
    if (fold < 2 || n_t < 2 || S_xyz[0] < 2 || S_xyz[1] < 2 || S_xyz[2] < 2) return -1;
    uint32_t S[4] = { S_xyz[0], S_xyz[1], S_xyz[2], n_t };
    int Ls = 0;
    for (int a = 0; a < 4; a++) {
        int La = ceil_log(S[a], fold);
        if (La > Ls) Ls = La;
    }
    if (Ls > max_L) return -2;
    for (int a = 0; a < 4; a++) {
        uint32_t r = S[a];
        out[0 * 4 + a] = r;
        for (int l = 1; l < Ls; l++) {
            if (r > fold) r = (r + fold - 1) / fold;  /* ceil(Res/f), Eq. 7 */
            else r = 2;                               /* Tail(l) = 2, Eq. 8 */
            out[l * 4 + a] = r;
        }
    }
    return Ls;
}

/* ------------------------------------------------------------------ a1 --
 * Level table.  Corner count C_l = Rx*Ry*Rz*Rt (64-bit) -- D2: the table is
 * "resolution-dependent ... scaling their sizes proportionally",
 * sized exactly to the vertex count (R1: Res = vertex count).  When a cap is
 * given and C_l > cap the level is hashed with T_l = cap (R5).  Offsets pack
 * the levels in the given order (R11).  Returns total entries, 0 on error.
 */
uint64_t fho_build_levels(const uint32_t *res, int L, uint64_t cap,
                          uint64_t *corners, uint64_t *tsize, int32_t *hashed,
                          uint64_t *offset)
{
    uint64_t off = 0;
    if (cap & (cap - 1)) return 0;  /* cap must be 0 or a power of two */
    for (int l = 0; l < L; l++) {
        uint64_t c = 1;
        for (int a = 0; a < 4; a++) {
            if (res[l * 4 + a] < 2) return 0;
            c *= res[l * 4 + a];
        }
        corners[l] = c;
        hashed[l] = (cap != 0 && c > cap);
        tsize[l] = hashed[l] ? cap : c;
        offset[l] = off;
        off += tsize[l];
    }
    return off;
}

/* ------------------------------------------------------------------ a4 --
 * F-Hash, Eq. 9:  t*Rx*Ry*Rz + z*Rx*Ry + y*Rx + x.
 */
uint64_t fho_fhash(const uint32_t r[4], uint64_t x, uint64_t y, uint64_t z, uint64_t t)
{
    uint64_t Rx = r[0], Ry = r[1], Rz = r[2];
    return t * Rx * Ry * Rz + z * Rx * Ry + y * Rx + x;
}

/* NEXT-2: a locality-preserving bijective linearization ("Other
 * linearizations like Morton and Z-order can also be used to construct F-Hash
 * with preserved locality"): tiled (one-level Z-order) order -- the
 * grid is cut into bricks of 2 x 2 x 2 x 2 vertices (clipped at the grid
 * edge), bricks are enumerated in row-major (x fastest) order and vertices
 * in row-major order inside a brick (reading R21):
 *   b_a = v_a / B_a, i_a = v_a % B_a, e_a = min(B_a, R_a - b_a B_a)
 *   idx = b_t B_t Rz Ry Rx + b_z B_z Ry Rx e_t + b_y B_y Rx e_z e_t
 *       + b_x B_x e_y e_z e_t + ((i_t e_z + i_z) e_y + i_y) e_x + i_x
 * Bijective onto [0, Rx Ry Rz Rt) (brute-force pinned in the tests). */
static const uint64_t kBrick[4] = { 2, 2, 2, 2 };

uint64_t fho_brick_index(const uint32_t r[4], uint64_t x, uint64_t y, uint64_t z, uint64_t t)
{
    uint64_t v[4] = { x, y, z, t }, b[4], i[4], e[4];
    for (int a = 0; a < 4; a++) {
        b[a] = v[a] / kBrick[a];
        i[a] = v[a] % kBrick[a];
        uint64_t rem = (uint64_t)r[a] - b[a] * kBrick[a];
        e[a] = rem < kBrick[a] ? rem : kBrick[a];
    }
    uint64_t Rx = r[0], Ry = r[1], Rz = r[2];
    return b[3] * kBrick[3] * Rz * Ry * Rx
         + b[2] * kBrick[2] * Ry * Rx * e[3]
         + b[1] * kBrick[1] * Rx * e[2] * e[3]
         + b[0] * kBrick[0] * e[1] * e[2] * e[3]
         + ((i[3] * e[2] + i[2]) * e[1] + i[1]) * e[0] + i[0];
}

/* Capped levels (R5; the paper never caps).  The primes of the MHE
 * spatial hash (Teschner et al., cited at P:174) on y, z and
 * t, with x entering additively (prime 1, added instead of xor-ed) so that
 * x-neighbours stay adjacent entries as in Eq. 9 (x fastest):
 *   (X + (Y*2654435761 xor Z*805459861 xor T*2246822519)) mod 2^32 mod T_l
 * uint32 wrap-around; T_l is a power of two.  The t-axis prime is our choice. */
uint64_t fho_spatial_hash(uint32_t X, uint32_t Y, uint32_t Z, uint32_t T, uint64_t tsize)
{
    uint32_t h = X + ((Y * 2654435761u) ^ (Z * 805459861u) ^ (T * 2246822519u));
    return (uint64_t)h % tsize;
}

/* ------------------------------------------------------------- a2, a3 --
 * Steps 1-2 on one axis, R2: coordinate p in [0,1] (clamped;
 * NaN -> 0; *bad set when clamping happened), s = fp32(p * fp32(R-1)) as ONE
 * rounded fp32 multiply, i = clamp(floor(s), 0, R-2), w = s - i (exact).
 */
static void locate_axis(float p, uint32_t R, uint32_t *i_out, float *w_out, int *bad)
{
    float pc;
    if (p >= 0.0f) {
        if (p <= 1.0f) pc = p;
        else { pc = 1.0f; *bad = 1; }
    } else { pc = 0.0f; *bad = 1; }  /* negative or NaN */
    volatile float Rm1 = (float)(R - 1);
    volatile float s = pc * Rm1;       /* single IEEE fp32 product */
    float fl = floorf(s);
    int64_t i = (int64_t)fl;
    if (i < 0) i = 0;
    if (i > (int64_t)R - 2) i = (int64_t)R - 2;
    *i_out = (uint32_t)i;
    *w_out = s - (float)i;
}

/* One (sample, level): the 16 corner indices (global, i.e. + level offset)
 * and fp64 weights.  Corner order c = bx + 2*by + 4*bz + 8*bt (R3).
 * Weight W_c = prod_a (b_a ? w_a : 1 - w_a), computed in fp64 from the fp32
 * fractions (R6: Eqs. 10-11 trilinear per time slice times the temporal
 * lerp of Eq. 12, expanded into the single 16-term sum). */
static int corners_one(const float *p /*x,y,z,t*/, const uint32_t r[4], int hashed,
                       uint64_t tsize, uint64_t offset, uint64_t idx[16], double W[16])
{
    uint32_t i[4];
    float w[4];
    int bad = 0;
    for (int a = 0; a < 4; a++) locate_axis(p[a], r[a], &i[a], &w[a], &bad);
    for (int c = 0; c < 16; c++) {
        uint32_t b[4] = { (uint32_t)(c & 1), (uint32_t)((c >> 1) & 1),
                          (uint32_t)((c >> 2) & 1), (uint32_t)((c >> 3) & 1) };
        uint32_t X = i[0] + b[0], Y = i[1] + b[1], Z = i[2] + b[2], T = i[3] + b[3];
        /* hashed: 0 = Eq. 9, 1 = capped hash (R5), 2 = brick order (NEXT-2, R21) */
        uint64_t local = hashed == 1 ? fho_spatial_hash(X, Y, Z, T, tsize)
                       : hashed == 2 ? fho_brick_index(r, X, Y, Z, T)
                                     : fho_fhash(r, X, Y, Z, T);
        idx[c] = offset + local;
        double Wc = 1.0;
        for (int a = 0; a < 4; a++) Wc *= b[a] ? (double)w[a] : 1.0 - (double)w[a];
        W[c] = Wc;
    }
    return bad;
}

/* Oracle-I: idx [N][L][16] (uint32 -- sums of T_l < 2^32 are required), W
 * [N][L][16] fp64 (may be NULL).  Returns number of samples with clamped
 * coordinates. */
int64_t fho_encode_indices(const uint32_t *res, const int32_t *hashed, const uint64_t *tsize,
                           const uint64_t *offset, int L, const float *coords, int64_t N,
                           uint32_t *idx, double *W)
{
    int64_t nbad = 0;
    for (int64_t n = 0; n < N; n++) {
        int bad = 0;
        for (int l = 0; l < L; l++) {
            uint64_t id[16];
            double w[16];
            bad |= corners_one(coords + 4 * n, res + 4 * l, hashed[l], tsize[l], offset[l], id, w);
            for (int c = 0; c < 16; c++) {
                idx[(n * L + l) * 16 + c] = (uint32_t)id[c];
                if (W) W[(n * L + l) * 16 + c] = w[c];
            }
        }
        nbad += bad;
    }
    return nbad;
}

/* Oracle-F, steps 1-4, Eqs. 10-12 + concatenation:
 *   out[n][l*F + f] = sum_{c=0}^{15} W_c * E[idx_c][f]     (fp64)
 * table: [sum T][F] fp64 (the caller converts the fp32/fp16 table exactly).
 * absout (may be NULL): sum_c W_c |E[idx_c][f]|, the tolerance scale. */
void fho_encode_fwd(const uint32_t *res, const int32_t *hashed, const uint64_t *tsize,
                    const uint64_t *offset, int L, int F, const float *coords, int64_t N,
                    const double *table, double *out, double *absout)
{
    for (int64_t n = 0; n < N; n++) {
        for (int l = 0; l < L; l++) {
            uint64_t id[16];
            double w[16];
            corners_one(coords + 4 * n, res + 4 * l, hashed[l], tsize[l], offset[l], id, w);
            for (int f = 0; f < F; f++) {
                double acc = 0.0, aacc = 0.0;
                for (int c = 0; c < 16; c++) {
                    double e = table[id[c] * (uint64_t)F + f];
                    acc += w[c] * e;
                    aacc += w[c] * fabs(e);
                }
                out[n * (int64_t)L * F + l * F + f] = acc;
                if (absout) absout[n * (int64_t)L * F + l * F + f] = aacc;
            }
        }
    }
}

/* Oracle-B (the adjoint of Oracle-F; "gradient
 * computation ... during backpropagation"):
 *   G[idx_c][f] += W_c * g[n][l*F + f]   accumulated in fp64, order n, l, c.
 *   A[idx_c][f] += |W_c * g[n][l*F + f]| (tolerance scale; may be NULL).
 * G and A are caller-zeroed [sum T][F]. */
void fho_encode_bwd(const uint32_t *res, const int32_t *hashed, const uint64_t *tsize,
                    const uint64_t *offset, int L, int F, const float *coords, int64_t N,
                    const double *dout, double *G, double *A)
{
    for (int64_t n = 0; n < N; n++) {
        for (int l = 0; l < L; l++) {
            uint64_t id[16];
            double w[16];
            corners_one(coords + 4 * n, res + 4 * l, hashed[l], tsize[l], offset[l], id, w);
            for (int c = 0; c < 16; c++) {
                for (int f = 0; f < F; f++) {
                    double g = dout[n * (int64_t)L * F + l * F + f];
                    G[id[c] * (uint64_t)F + f] += w[c] * g;
                    if (A) A[id[c] * (uint64_t)F + f] += fabs(w[c] * g);
                }
            }
        }
    }
}

/* ------------------------------------------------------------ NEXT-3 --
 * MHE baseline encoder (the comparison system of P:378 / Fig. 4, P:177-182;
 * SPEC baseline_encode S:321-329): one 3D multi-resolution hash encoder per
 * key frame, a FIXED table size T per level (bucket waste on small levels,
 * S:354), index = direct x + y R + z R^2 when R^3 <= T, else the spatial hash
 * (x*1 xor y*2654435761 xor z*805459861) mod T (uint32); trilinear blend of 8
 * corners.  Frame k of a sample: nearest key frame of its t (reading R20):
 * s = fp32(t * (n-1)), k = clamp(floor(s + 0.5), 0, n-1) with t clamped as
 * R2.  Level l of frame k occupies entries offset_l + k*T + [0, T).
 * Corner order c = bx + 2 by + 4 bz.  W_c in fp64 from the fp32 fractions. */
static int mhe_corners_one(const float *p, uint32_t R, uint32_t n_frames, uint64_t T, uint64_t offset,
                           uint64_t idx[8], double W[8])
{
    uint32_t i[3];
    float w[3];
    int bad = 0;
    for (int a = 0; a < 3; a++) locate_axis(p[a], R, &i[a], &w[a], &bad);
    uint32_t k_i;
    float k_w;
    /* frame: nearest vertex of an n_frames-vertex time axis */
    {
        float pc;
        if (p[3] >= 0.0f) { if (p[3] <= 1.0f) pc = p[3]; else { pc = 1.0f; bad = 1; } }
        else { pc = 0.0f; bad = 1; }
        volatile float nm1 = (float)(n_frames - 1);
        volatile float s = pc * nm1;
        float fl = floorf(s);
        int64_t k = (int64_t)fl + ((s - fl) >= 0.5f ? 1 : 0);
        if (k < 0) k = 0;
        if (k > (int64_t)n_frames - 1) k = (int64_t)n_frames - 1;
        k_i = (uint32_t)k;
        k_w = 0.0f;
        (void)k_w;
    }
    const uint64_t cube = (uint64_t)R * R * R;
    for (int c = 0; c < 8; c++) {
        uint32_t b[3] = { (uint32_t)(c & 1), (uint32_t)((c >> 1) & 1), (uint32_t)((c >> 2) & 1) };
        uint32_t X = i[0] + b[0], Y = i[1] + b[1], Z = i[2] + b[2];
        uint64_t local;
        if (cube <= T) local = (uint64_t)X + (uint64_t)Y * R + (uint64_t)Z * R * R;
        else local = (uint64_t)((X * 1u) ^ (Y * 2654435761u) ^ (Z * 805459861u)) % T;
        idx[c] = offset + (uint64_t)k_i * T + local;
        double Wc = 1.0;
        for (int a = 0; a < 3; a++) Wc *= b[a] ? (double)w[a] : 1.0 - (double)w[a];
        W[c] = Wc;
    }
    return bad;
}

/* res[L]: vertices per spatial axis; every level has T entries per frame. */
int64_t fho_mhe_indices(const uint32_t *res, int L, uint32_t n_frames, uint64_t T, const float *coords,
                        int64_t N, uint32_t *idx, double *W)
{
    int64_t nbad = 0;
    for (int64_t n = 0; n < N; n++) {
        int bad = 0;
        for (int l = 0; l < L; l++) {
            uint64_t id[8];
            double w[8];
            bad |= mhe_corners_one(coords + 4 * n, res[l], n_frames, T, (uint64_t)l * n_frames * T, id, w);
            for (int c = 0; c < 8; c++) {
                idx[(n * L + l) * 8 + c] = (uint32_t)id[c];
                if (W) W[(n * L + l) * 8 + c] = w[c];
            }
        }
        nbad += bad;
    }
    return nbad;
}

void fho_mhe_fwd(const uint32_t *res, int L, uint32_t n_frames, uint64_t T, int F, const float *coords,
                 int64_t N, const double *table, double *out, double *absout)
{
    for (int64_t n = 0; n < N; n++)
        for (int l = 0; l < L; l++) {
            uint64_t id[8];
            double w[8];
            mhe_corners_one(coords + 4 * n, res[l], n_frames, T, (uint64_t)l * n_frames * T, id, w);
            for (int f = 0; f < F; f++) {
                double acc = 0.0, aacc = 0.0;
                for (int c = 0; c < 8; c++) {
                    double e = table[id[c] * (uint64_t)F + f];
                    acc += w[c] * e;
                    aacc += w[c] * fabs(e);
                }
                out[n * (int64_t)L * F + l * F + f] = acc;
                if (absout) absout[n * (int64_t)L * F + l * F + f] = aacc;
            }
        }
}

void fho_mhe_bwd(const uint32_t *res, int L, uint32_t n_frames, uint64_t T, int F, const float *coords,
                 int64_t N, const double *dout, double *G, double *A)
{
    for (int64_t n = 0; n < N; n++)
        for (int l = 0; l < L; l++) {
            uint64_t id[8];
            double w[8];
            mhe_corners_one(coords + 4 * n, res[l], n_frames, T, (uint64_t)l * n_frames * T, id, w);
            for (int c = 0; c < 8; c++)
                for (int f = 0; f < F; f++) {
                    double g = dout[n * (int64_t)L * F + l * F + f];
                    G[id[c] * (uint64_t)F + f] += w[c] * g;
                    if (A) A[id[c] * (uint64_t)F + f] += fabs(w[c] * g);
                }
        }
}

/* MHE level statistics over one frame: distinct buckets hit by the R^3
 * vertices, collisions = R^3 - distinct, utilisation = distinct / T. */
int fho_mhe_level_stats(uint32_t R, uint64_t T, uint64_t max_vertices, uint64_t *distinct, uint64_t *collisions)
{
    uint64_t C = (uint64_t)R * R * R;
    if (C > max_vertices) return -1;
    uint8_t *hit = calloc(T, 1);
    if (!hit) return -2;
    uint64_t d = 0;
    for (uint32_t z = 0; z < R; z++)
        for (uint32_t y = 0; y < R; y++)
            for (uint32_t x = 0; x < R; x++) {
                uint64_t b = (C <= T) ? (uint64_t)x + (uint64_t)y * R + (uint64_t)z * R * R
                                      : (uint64_t)((x * 1u) ^ (y * 2654435761u) ^ (z * 805459861u)) % T;
                if (!hit[b]) { hit[b] = 1; d++; }
            }
    free(hit);
    *distinct = d;
    *collisions = C - d;
    return 0;
}

/* Oracle-S, encoding_stats: brute force over every lattice
 * vertex of level l: buckets hit, collisions = vertices - distinct buckets,
 * utilisation = distinct / T_l.  Returns -1 if the level has more than
 * max_vertices vertices (not enumerated). */
int fho_level_stats(const uint32_t r[4], int hashed, uint64_t tsize, uint64_t max_vertices,
                    uint64_t *distinct, uint64_t *collisions)
{
    uint64_t C = (uint64_t)r[0] * r[1] * r[2] * r[3];
    if (C > max_vertices) return -1;
    uint8_t *hit = calloc(tsize, 1);
    if (!hit) return -2;
    uint64_t d = 0, out_of_range = 0;
    for (uint32_t t = 0; t < r[3]; t++)
        for (uint32_t z = 0; z < r[2]; z++)
            for (uint32_t y = 0; y < r[1]; y++)
                for (uint32_t x = 0; x < r[0]; x++) {
                    uint64_t b = hashed == 1 ? fho_spatial_hash(x, y, z, t, tsize)
                               : hashed == 2 ? fho_brick_index(r, x, y, z, t) : fho_fhash(r, x, y, z, t);
                    if (b >= tsize) { out_of_range++; continue; }
                    if (!hit[b]) { hit[b] = 1; d++; }
                }
    free(hit);
    *distinct = d;
    *collisions = C - d;
    return out_of_range ? -3 : 0;
}
