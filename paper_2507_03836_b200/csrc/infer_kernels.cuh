// infer_kernels.cuh -- NEXT-1: the renderer's model evaluation V = model(S)
// (Alg. 1, "Inference F-Hash INR") as ONE kernel: the encode
// forward (steps 1-4 of §3.2.4, through the same device
// functions as fwd_kernel, encode_device.cuh) is written as bf16 straight
// into the shared-memory X operand of the tcgen05 MLP forward (MMA1 ->
// bias + ReLU -> MMA2 -> bias + ReLU -> 64 -> 1 output): no encoder-output
// round trip through global memory, one launch.
//
// Short tiles for small batches.  A 128-sample tile is 128 L corner-cell
// gathers, i.e. 8 x 128 L pair requests (16 K at L = 16), and one SM issues
// about one L2 request per cycle: a full tile gathered by one CTA costs
// >= 8 us (measured 22.7 us for one tile).  So a batch that does not fill
// the GPU is cut into tiles of R = 8 .. 128 samples (the smallest power of
// two that keeps one wave of CTAs), each CTA gathering and evaluating its
// own: the MMA still runs M = 128 rows, those past R are never read back.
// (Thread-block clusters sharing a tile's gathers through distributed
// shared memory were measured too -- never faster than short tiles, and
// slower at 4096 samples: 12.3 vs 10.7 us.)
//
// Roles per CTA: warps 0-3 (full tiles) or 0-7 (short tiles) run the MLP
// (TMEM lane = sample row t = 32 (warp % 4) + lane; with 8 warps each row's
// columns are split in two halves); the other warps gather, as G groups of 8 warps working on different
// tiles (more loads in flight per SM).  X buffers: NB = 4; mbarriers
//   full[b]   8 arrivals (the gather warps of the group that filled X[b]);
//   xfree[b]  1 arrival from the MLP thread once MMA1 has consumed X[b].
// The CTA's tile u (global tile blockIdx.x + gridDim.x u) uses X[u % NB].
//
// Numerics = fh_encode_fwd(FH_BF16) followed by the forward half of
// mlp_train_kernel: the same gather / lerp tree / RNE bf16 rounding of the
// encoding (R13), bf16 weights and activations, fp32 accumulation, the
// 64 -> 1 layer as 4 interleaved fp32 accumulators in column order.
#pragma once
#include "encode_device.cuh"
#include "mlp_kernels.cuh"

namespace fh {
namespace infer {

using mlp::H;
using mlp::TILE;

constexpr int kGatherWarps = 8;   // gather warps per group
// MLP warps: 8 in short-tile launches (two warps per TMEM lane quarter, each
// taking half the columns of every epilogue: the single-tile latency chain
// is then half as long), 4 in full-tile launches (register budget).
template <int G> struct MlpWarps { static constexpr int value = G == 1 ? 8 : 4; };
// Short-tile launches (small batches) use one gather group (384 threads: a
// smaller CTA launches faster); full tiles as many as the register file
// allows: 3 groups (896 threads, 72 registers) for F <= 2, 2 (640 threads,
// 96 registers) for wider entries.
template <int F> struct Groups { static constexpr int value = F <= 2 ? 3 : 2; };
template <int G> struct Threads { static constexpr int value = 32 * (MlpWarps<G>::value + G * kGatherWarps); };

template <int K0>
struct FusedLayout {
    static constexpr uint32_t SBO_X = (K0 / 8) * 128;
    static constexpr uint32_t SBO_H = (H / 8) * 128;
    static constexpr uint32_t BYTES_W1 = H * K0 * 2;
    static constexpr uint32_t BYTES_W2 = H * H * 2;
    static constexpr uint32_t BYTES_X = TILE * K0 * 2;
    static constexpr uint32_t BYTES_H = TILE * H * 2;
    static constexpr int NB = 4;   // X buffers per CTA
    static constexpr uint32_t SMEM = BYTES_W1 + BYTES_W2 + NB * BYTES_X + BYTES_H;
};

struct FusedArgs {
    const float4 *coords;          // [N][4]
    const void *table;             // [sum T][F] of the encoder's table dtype
    const __nv_bfloat16 *wsh;      // bf16 shadow of the flat MLP parameters
    const float *wmaster;          // fp32 master (biases, b3)
    float *y;                      // [N]
    int64_t N;
    int *flag;                     // encoder status word (out-of-domain coordinates)
    int rows;                      // samples per tile R (8 .. 128, a power of two)
    const __nv_bfloat16 *xin;      // NULL: gather; else the encoding [N][K0] bf16 already in global memory
                                   // (large batches over HBM-sized tables: fh_encode_fwd's L2-sized level
                                   // groups first, then this kernel as the MLP forward only)
};

// bf16 of the F blended features into the X tile at p.
template <int F>
__device__ __forceinline__ void st_x(uint8_t *p, const float (&v)[F]) {
    if constexpr (F == 1) {
        *reinterpret_cast<__nv_bfloat16 *>(p) = __float2bfloat16_rn(v[0]);
    } else if constexpr (F == 2) {
        *reinterpret_cast<uint32_t *>(p) = mlp::pack_bf16(v[0], v[1]);
    } else if constexpr (F == 4) {
        *reinterpret_cast<uint2 *>(p) = make_uint2(mlp::pack_bf16(v[0], v[1]), mlp::pack_bf16(v[2], v[3]));
    } else {
        *reinterpret_cast<uint4 *>(p) = make_uint4(mlp::pack_bf16(v[0], v[1]), mlp::pack_bf16(v[2], v[3]),
                                                   mlp::pack_bf16(v[4], v[5]), mlp::pack_bf16(v[6], v[7]));
    }
}

#ifdef FH_INFER_TRACE
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define TRACE(var) var = gtime()
#else
#define TRACE(var)
#endif

// Barrier over the MW warps of the MLP (named barrier 1).
template <int MW>
__device__ __forceinline__ void mlp_sync() { asm volatile("bar.sync 1, %0;" ::"n"(32 * MW) : "memory"); }

__device__ __forceinline__ void mbar_arrive(uint64_t *mbar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(mbar)) : "memory");
}

template <int F, typename T, int K0, int G>
__global__ void __launch_bounds__(Threads<G>::value, 1) infer_fused_kernel(const __grid_constant__ Params P, const FusedArgs a) {
    using Lo = FusedLayout<K0>;
    constexpr int NB = Lo::NB;
    constexpr int kMlpWarps = MlpWarps<G>::value;
    constexpr int HALVES = kMlpWarps / 4;    // threads per sample row
    constexpr int HC = H / HALVES;           // epilogue columns per thread
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *sW1 = smem;
    uint8_t *sW2 = sW1 + Lo::BYTES_W1;
    uint8_t *sX0 = sW2 + Lo::BYTES_W2;       // X[0 .. NB)
    uint8_t *sH = sX0 + NB * Lo::BYTES_X;
    __shared__ LevelSmem slv;
    __shared__ uint64_t full[NB], xfree[NB], mma_bar;
    __shared__ uint32_t tbase;
    __shared__ __align__(16) float b1[H], b2[H], w3[H];   // read as float4
    __shared__ float4 s_y[MlpWarps<G>::value / 4][TILE];   // per column half: the 4 output-layer accumulators

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
#ifdef FH_INFER_TRACE
    unsigned long long T0 = 0, T1 = 0, T2 = 0, T3 = 0, T4 = 0, T5 = 0, T6 = 0, T7 = 0;
#endif
    TRACE(T0);
    if (tid == 0) {
        for (int b = 0; b < NB; b++) {
            tc::mbar_init(&full[b], kGatherWarps);
            tc::mbar_init(&xfree[b], 1);
        }
        tc::mbar_init(&mma_bar, 1);
        tc::fence_mbar_init();
    }
    // (no 64-bit divisions on the start-up path: R is a power of two, and a
    // short-tile launch has at most one tile per CTA)
    const int R = a.rows;
    const int64_t n_tiles = (a.N + R - 1) >> (__ffs(R) - 1);
    const int64_t n_u = (int64_t)blockIdx.x >= n_tiles ? 0
                        : n_tiles <= (int64_t)gridDim.x ? 1
                        : (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int L = P.L;
    // Loads issued before the level-table barrier, so their latency overlaps
    // the CTA's start-up (the warps of a CTA start up to ~0.4 us apart):
    // MLP warps: the bf16 weights (core-matrix rows, stored to shared memory
    // after the barrier) and the fp32 biases; gather warps: the coordinates
    // of their first item.
    constexpr int NW1 = (H * K0 / 8 + 32 * kMlpWarps - 1) / (32 * kMlpWarps), NW2 = H * H / 8 / (32 * kMlpWarps);
    static_assert(NW2 * 32 * kMlpWarps == H * H / 8, "weight rows per thread");
    // (Short-tile launches only, G == 1: the full-tile variants run at the
    // register limit and many tiles per CTA, where start-up latency is noise.)
    constexpr bool kPre = G == 1;
    constexpr int CW = kPre ? 32 : 16;   // TMEM columns per load in the MLP epilogues (register budget)
    uint4 wr1[kPre ? NW1 : 1], wr2[kPre ? NW2 : 1];
    float pb1 = 0.f, pb2 = 0.f;
    __nv_bfloat16 pw3 = __float2bfloat16_rn(0.f);   // converted after the barrier (a use here would wait for the load)
    float4 c_first = make_float4(0.f, 0.f, 0.f, 0.f);
    if (!kPre) {
    } else if (warp < kMlpWarps) {
        const uint4 *w = reinterpret_cast<const uint4 *>(a.wsh);
#pragma unroll
        for (int k = 0; k < NW1; k++)
            if (tid + k * 32 * kMlpWarps < H * K0 / 8) wr1[k] = __ldg(w + (mlp::off_W1() / 8) + tid + k * 32 * kMlpWarps);
        const uint4 *w2 = reinterpret_cast<const uint4 *>(a.wsh + mlp::off_W2(K0));
#pragma unroll
        for (int k = 0; k < NW2; k++) wr2[k] = __ldg(w2 + tid + k * 32 * kMlpWarps);
        if (tid < H) {
            pb1 = __ldg(a.wmaster + mlp::off_b1(K0) + tid);
            pb2 = __ldg(a.wmaster + mlp::off_b2(K0) + tid);
            pw3 = a.wsh[mlp::off_w3(K0) + tid];
        }
    } else if (a.xin == nullptr) {
        const int gt = tid - 32 * kMlpWarps;   // one gather group (G == 1)
        const int64_t n = (int64_t)blockIdx.x * R + gt / L;
        if (gt < R * L && n < a.N) c_first = __ldg(a.coords + n);
    }
    load_levels(P, slv);   // ends with __syncthreads: barriers and level table ready
    TRACE(T1);

    if (warp >= kMlpWarps) {
        // ------------------------------------------------ gather warps
        const int gq = tid - 32 * kMlpWarps;
        const int grp = gq / (32 * kGatherWarps);     // this warp's gather group
        const int gt = gq % (32 * kGatherWarps);      // 0 .. 255 within the group
        const T *table = reinterpret_cast<const T *>(a.table);
        const int items = R * L;
        // tiles u = grp, grp + G, ...: tile u + NB (the next use of buffer
        // u % NB) may belong to another group, so the xfree wait orders them
        for (int64_t u = grp; u < n_u; u += G) {
            const int b = (int)(u % NB);
            const int64_t m = u / NB;                 // use index of the buffer
            if (m > 0) tc::mbar_wait(&xfree[b], (uint32_t)((m - 1) & 1));
            const int64_t tile = (int64_t)blockIdx.x + (int64_t)gridDim.x * u;
            uint8_t *sX = sX0 + b * Lo::BYTES_X;
            if (a.xin) {   // copy the tile's encoding rows (coalesced 16-byte chunks) into the X tile
                constexpr int CH = K0 / 8;
                const uint4 *src = reinterpret_cast<const uint4 *>(a.xin + tile * R * K0);
                for (int k = gt; k < R * CH; k += 32 * kGatherWarps) {
                    const int r = k / CH, q = k - r * CH;
                    const uint4 v = tile * R + r < a.N ? __ldg(src + k) : make_uint4(0u, 0u, 0u, 0u);
                    mlp::st16(sX, tc::core_off(r, 8 * q, Lo::SBO_X), v);
                }
            } else
#pragma unroll 1
            for (int i = gt; i < items; i += 32 * kGatherWarps) {
                const int s = i / L, l = i - s * L;
                const int64_t n = tile * R + s;
                float v[F];
                if (n < a.N) {
                    Cell c;
                    const float4 xyzt = (kPre && u == grp && i == gt) ? c_first : __ldg(a.coords + n);
#ifdef FH_INFER_TRACE
                    unsigned long long Ta = gtime();
#endif
                    if (cell_of(slv.get(l), xyzt, c) && l == 0) atomicOr(a.flag, 1);
#ifdef FH_INFER_TRACE
                    unsigned long long Tb = gtime();
#endif
                    float e[16][F];
                    gather16<T, F>(table, nullptr, c.idx, e);
                    blend16<F>(e, c.w, v);
#ifdef FH_INFER_TRACE
                    unsigned long long Tc = gtime();
                    if (blockIdx.x == 0 && (gt == 0 || gt == 100) && u == grp)
                        printf("TI %d %llu %llu %llu %llu %f\n", gt, T0, Ta, Tb, Tc, v[0]);
#endif
                } else {
#pragma unroll
                    for (int f = 0; f < F; f++) v[f] = 0.f;
                }
                st_x<F>(sX + tc::core_off(s, l * F, Lo::SBO_X), v);
            }
            // the stores (generic proxy) must be visible to the tensor core
            tc::fence_smem_to_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[b]);
#ifdef FH_INFER_TRACE
            if (blockIdx.x == 0 && lane == 0 && u == grp) {
                TRACE(T2);
                printf("TG %d %llu %llu %llu\n", warp, T0, T1, T2);
            }
#endif
        }
    } else {
        // ------------------------------------------------ MLP warps
        // TMEM and the weights are set up here, while the gather warps already gather
        if (warp == 0) tc::tmem_alloc(&tbase, 64);
        {   // weights -> shared memory (core-matrix layout, one 16-byte row segment per store)
            const uint4 *w = reinterpret_cast<const uint4 *>(a.wsh);
            const uint4 *w2 = reinterpret_cast<const uint4 *>(a.wsh + mlp::off_W2(K0));
#pragma unroll
            for (int k = 0; k < NW1; k++) {
                const int q = tid + k * 32 * kMlpWarps;
                const int r = q / (K0 / 8), c = (q % (K0 / 8)) * 8;
                if (q < H * K0 / 8)
                    mlp::st16(sW1, tc::core_off(r, c, Lo::SBO_X), kPre ? wr1[kPre ? k : 0] : __ldg(w + (mlp::off_W1() / 8) + q));
            }
#pragma unroll
            for (int k = 0; k < NW2; k++) {
                const int q = tid + k * 32 * kMlpWarps;
                const int r = q / (H / 8), c = (q % (H / 8)) * 8;
                mlp::st16(sW2, tc::core_off(r, c, Lo::SBO_H), kPre ? wr2[kPre ? k : 0] : __ldg(w2 + q));
            }
        }
        if (tid < H) {
            b1[tid] = kPre ? pb1 : a.wmaster[mlp::off_b1(K0) + tid];
            b2[tid] = kPre ? pb2 : a.wmaster[mlp::off_b2(K0) + tid];
            w3[tid] = __bfloat162float(kPre ? pw3 : a.wsh[mlp::off_w3(K0) + tid]);
        }
        tc::fence_smem_to_async();
        tc::fence_before_sync();
        mlp_sync<kMlpWarps>();                                       // named barrier 1 over the 128 MLP threads
        tc::fence_after_sync();
        TRACE(T2);
        const uint32_t tm = tbase;
        const int row = tid & 127;                        // TMEM lane = sample row
        const int hc0 = (warp >> 2) * HC;                 // this thread's first epilogue column
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t aH = tc::smem_u32(sH), aW1 = tc::smem_u32(sW1), aW2 = tc::smem_u32(sW2);
        constexpr uint32_t id_h = tc::idesc_bf16_f32(128, H, false, false);
        const float b3 = a.wmaster[mlp::off_b3(K0)];
        uint32_t phase = 0;
        for (int64_t u = 0; u < n_u; u++) {
            const int b = (int)(u % NB);
            tc::mbar_wait(&full[b], (uint32_t)((u / NB) & 1));
            tc::fence_after_sync();
            TRACE(T3);
            const uint32_t aX = tc::smem_u32(sX0 + b * Lo::BYTES_X);
            // ---- MMA1: Z1 = X . W1^T
            if (tid == 0) {
#pragma unroll
                for (int s = 0; s < K0 / 16; s++)
                    tc::mma_bf16(tm, tc::sdesc(aX + s * 256, 128, Lo::SBO_X), tc::sdesc(aW1 + s * 256, 128, Lo::SBO_X),
                                 id_h, s > 0);
                tc::commit(&mma_bar);
            }
            tc::mbar_wait(&mma_bar, phase); phase ^= 1;
            tc::fence_after_sync();
            TRACE(T4);
            // X[b] consumed: free it (only if a gather group will refill it)
            if (tid == 0 && u + NB < n_u) mbar_arrive(&xfree[b]);
            // ---- H1 = bf16(relu(Z1 + b1)) (packed pairs, as mlp_train_kernel)
#pragma unroll
            for (int c0 = hc0; c0 < hc0 + HC; c0 += CW) {
                float v[CW];
                mlp::tmem_ld_cols<CW>(tm + lane_off + c0, v);
#pragma unroll
                for (int j = 0; j < CW; j += 8) {
                    const int c = c0 + j;
                    const float4 ba = *reinterpret_cast<const float4 *>(b1 + c);
                    const float4 bb = *reinterpret_cast<const float4 *>(b1 + c + 4);
                    mlp::st16(sH, tc::core_off(row, c, Lo::SBO_H),
                              make_uint4(mlp::bias_relu_bf16x2(v[j], v[j + 1], ba.x, ba.y),
                                         mlp::bias_relu_bf16x2(v[j + 2], v[j + 3], ba.z, ba.w),
                                         mlp::bias_relu_bf16x2(v[j + 4], v[j + 5], bb.x, bb.y),
                                         mlp::bias_relu_bf16x2(v[j + 6], v[j + 7], bb.z, bb.w)));
                }
            }
            tc::fence_smem_to_async();
            tc::fence_before_sync();
            mlp_sync<kMlpWarps>();
            tc::fence_after_sync();
            TRACE(T5);
            // ---- MMA2: Z2 = H1 . W2^T
            if (tid == 0) {
#pragma unroll
                for (int s = 0; s < H / 16; s++)
                    tc::mma_bf16(tm, tc::sdesc(aH + s * 256, 128, Lo::SBO_H), tc::sdesc(aW2 + s * 256, 128, Lo::SBO_H),
                                 id_h, s > 0);
                tc::commit(&mma_bar);
            }
            tc::mbar_wait(&mma_bar, phase); phase ^= 1;
            tc::fence_after_sync();
            TRACE(T6);
            // ---- y = bf16(relu(Z2 + b2)) . w3 + b3 (4 accumulators in column order mod 4, as mlp_train_kernel)
            float2 ya01 = make_float2(0.f, 0.f), ya23 = make_float2(0.f, 0.f);
#pragma unroll
            for (int c0 = hc0; c0 < hc0 + HC; c0 += CW) {
                float v[CW];
                mlp::tmem_ld_cols<CW>(tm + lane_off + c0, v);
#pragma unroll
                for (int j = 0; j < CW; j += 4) {
                    const float4 b = *reinterpret_cast<const float4 *>(b2 + c0 + j);
                    const float4 w = *reinterpret_cast<const float4 *>(w3 + c0 + j);
                    ya01 = __ffma2_rn(mlp::unpack_bf16(mlp::bias_relu_bf16x2(v[j], v[j + 1], b.x, b.y)),
                                      make_float2(w.x, w.y), ya01);
                    ya23 = __ffma2_rn(mlp::unpack_bf16(mlp::bias_relu_bf16x2(v[j + 2], v[j + 3], b.z, b.w)),
                                      make_float2(w.z, w.w), ya23);
                }
            }
            const int64_t n = ((int64_t)blockIdx.x + (int64_t)gridDim.x * u) * R + row;
            if constexpr (HALVES == 2) {
                // the two column halves of a row meet in shared memory (the
                // two warps of a lane quarter, named barriers 2..5): each of the
                // 4 accumulators is the sum of the halves' partial sums
                s_y[warp >> 2][row] = make_float4(ya01.x, ya01.y, ya23.x, ya23.y);
                asm volatile("bar.sync %0, 64;" ::"r"(2 + (warp & 3)) : "memory");
                if (warp < 4) {
                    const float4 o = s_y[1][row];
                    ya01.x += o.x; ya01.y += o.y; ya23.x += o.z; ya23.y += o.w;
                }
            }
            if (warp < 4 && row < R && n < a.N) a.y[n] = ((ya01.x + ya01.y) + (ya23.x + ya23.y)) + b3;
#ifdef FH_INFER_TRACE
            TRACE(T7);
            if (tid == 0 && u == 0)
                printf("TR %d %llu %llu %llu %llu %llu %llu %llu %llu\n", blockIdx.x, T0, T1, T2, T3, T4, T5, T6, T7);
#endif
            tc::fence_before_sync();
            mlp_sync<kMlpWarps>();                            // TMEM and H reused by the next tile
            tc::fence_after_sync();
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tbase, 64);
}

}  // namespace infer
}  // namespace fh
