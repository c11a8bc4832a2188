// mlp_kernels.cuh -- the small MLP of the F-Hash INR on 5th-gen tensor
// cores (tcgen05 + TMEM), fused forward + MSE loss + backward, and the fused
// Adam optimiser.
//
// Paper: "a shallow network ... is used" on the concatenated encodings
// (P:233); "number of MLP layers = 2, number of neurons per layer = 64"
// (P:354); Adam, lr 0.01.  Readings R12 (Adam betas/eps,
// MSE over the global batch), R13 (bf16 operand rounding points), R15
// (ReLU hidden layers, identity output, biases) -- DESIGN.md §3.
//
// One persistent CTA per SM, 512 threads (two tile slots of 8 warps); each
// 128-sample tile is one
// M = 128 tcgen05 GEMM chain with the accumulators in TMEM:
//   MMA1  Z1  = X  . W1^T          (N = 64, K = K0)
//   MMA2  Z2  = H1 . W2^T          (N = 64, K = 64)
//   MMA3  dH1 = dZ2 . W2           (N = 64, K = 64)
//   MMA4  dX  = dZ1 . W1           (N = K0, K = 64)
//   MMA5  DW += [dZ2^T ; dZ1^T] . [H1 | X | 1]   (M = 128 hidden rows, K = 128 samples)
// MMA5 accumulates dW2 (top-left), dW1 (bottom, X columns) and, through the
// constant-one column, db2 / db1, in TMEM across all tiles of the CTA; the
// transposed operands are the SAME shared-memory tiles read through
// MN-major descriptors.  Two threads own sample row t of every tile (TMEM
// lane t), one per half of the columns, so every epilogue (bias, ReLU, bf16
// rounding, the 64 -> 1 output layer, the loss) runs in registers of those
// two threads; the output layer's two partial sums meet in shared memory.
#pragma once
#include <cuda.h>   // CUtensorMap
#include <cuda_bf16.h>
#include <stdint.h>

#include "tc_sm100.cuh"

namespace fh {
namespace mlp {

constexpr int H = 64;          // hidden width
constexpr int TILE = 128;      // samples per tile = TMEM lanes

// Flat fp32 parameter layout (master, grads, Adam moments; the bf16 shadow
// uses the same offsets): W1[H][K0], b1[H], W2[H][H], b2[H], w3[H], b3.
__host__ __device__ constexpr int off_W1() { return 0; }
__host__ __device__ constexpr int off_b1(int K0) { return H * K0; }
__host__ __device__ constexpr int off_W2(int K0) { return H * K0 + H; }
__host__ __device__ constexpr int off_b2(int K0) { return H * K0 + H + H * H; }
__host__ __device__ constexpr int off_w3(int K0) { return H * K0 + 2 * H + H * H; }
__host__ __device__ constexpr int off_b3(int K0) { return H * K0 + 3 * H + H * H; }
__host__ __device__ constexpr int param_count(int K0) { return H * K0 + 3 * H + H * H + 1; }

// Two independent tile "slots" per CTA (warps 0-7 and 8-15), each with its
// own shared-memory tiles, TMEM columns, mbarriers and MMA-issuing thread,
// so one slot's epilogue math overlaps the other slot's MMAs and loads.
// Within a slot the four per-tile accumulators Z1, Z2, dH1, dX share ONE
// 64-column TMEM region (each is consumed before the next MMA of the chain
// is issued); each slot accumulates its own DW block across all its tiles.
//
// Per slot: the [H1 | 1 0..0] tile; two 16 KB buffers that alternate
// between the tile's X operand (landed by TMA in the core-matrix layout, a
// tile ahead) and its h2 tile (the next tile's X lands in this tile's h2
// buffer once MMA6 has read it; this tile's X buffer takes the next tile's
// h2 once MMA5 has read it); the [dZ2 | dZ1] tile (also the dX staging);
// the [dy_hi dy_lo] tile.
template <int K0>
struct Layout {
    static constexpr int WH1 = H + 16;                    // columns of the [H1 | 1 0..0] tile
    static constexpr int WHX = WH1 + K0;                  // DW accumulator columns: [dW2 | db | dW1]
    static constexpr uint32_t SBO_H1 = (WH1 / 8) * 128;   // bytes per 8-sample row group: 1280
    static constexpr uint32_t SBO_X = (K0 / 8) * 128;
    static constexpr uint32_t SBO_DZ = (2 * H / 8) * 128; // [dZ2 | dZ1] tile: 2048
    static constexpr uint32_t SBO_W1 = (K0 / 8) * 128;
    static constexpr uint32_t SBO_W2 = (H / 8) * 128;
    static constexpr uint32_t BYTES_H1 = TILE * WH1 * 2;
    static constexpr uint32_t BYTES_X = TILE * K0 * 2;    // X tile (TMA transaction bytes)
    static constexpr uint32_t BYTES_XB = TILE * H * 2;    // one X / h2 buffer (h2: SBO 1024; K0 <= H)
    static constexpr uint32_t BYTES_DZ = TILE * 2 * H * 2;
    static constexpr uint32_t BYTES_DY = TILE * 16 * 2;   // [dy_hi, dy_lo, 0 x 14] per sample (SBO 256)
    static constexpr uint32_t BYTES_SLOT = BYTES_H1 + 2 * BYTES_XB + BYTES_DZ + BYTES_DY;
    static constexpr uint32_t BYTES_W1 = H * K0 * 2;
    static constexpr uint32_t BYTES_W2 = H * H * 2;
    static constexpr int SLOTS = 2;
    static constexpr uint32_t SMEM = SLOTS * BYTES_SLOT + BYTES_W1 + BYTES_W2;
    // TMEM columns (per slot, base = slot * 256)
    static constexpr uint32_t T_ACC = 0, T_DW = 64, T_D3 = 64 + WHX;  // T_D3: [dw3_hi, dw3_lo] accumulators
    // T_A: the A operand of MMA2 / MMA3 / MMA4 (H1, dZ2, dZ1 in turn: 128 x 64
    // bf16, two per column) written by the epilogues straight into TMEM, so
    // those MMAs read only B from shared memory (SS-mode MMAs with N = 64 are
    // bound by the shared-memory operand reads, A being two thirds of them)
    static constexpr uint32_t T_A = T_D3 + 16;
    static constexpr uint32_t TMEM_COLS = 512;
    static_assert(T_A + H / 2 <= 256, "slot TMEM region overflow");
    static_assert(K0 <= H && BYTES_X <= BYTES_XB, "X tile must fit an h2 buffer");
    static_assert(BYTES_H1 % 1024 == 0 && BYTES_XB % 1024 == 0 && BYTES_SLOT % 1024 == 0, "1 KB aligned tiles");
};

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&v);
}
__device__ __forceinline__ float bf16r(float a) { return __bfloat162float(__float2bfloat16_rn(a)); }
__device__ __forceinline__ float2 unpack_bf16(uint32_t u) {
    return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&u));
}

// Packed-pair epilogue arithmetic (sm_100 fp32x2 / bf16x2 instructions;
// element-wise identical to the scalar forms, half the instructions):
// bf16(relu(z + b)) of a pair (rounding is monotonic, so relu after the
// rounding gives the same value), and "p where h > 0, else +0" on bf16 pairs.
__device__ __forceinline__ uint32_t bf2_bits(__nv_bfloat162 h) { return *reinterpret_cast<uint32_t *>(&h); }
__device__ __forceinline__ __nv_bfloat162 bits_bf2(uint32_t u) { return *reinterpret_cast<__nv_bfloat162 *>(&u); }
__device__ __forceinline__ uint32_t bias_relu_bf16x2(float z0, float z1, float b0, float b1) {
    const float2 zb = __fadd2_rn(make_float2(z0, z1), make_float2(b0, b1));
    return bf2_bits(__hmax2(__float22bfloat162_rn(zb), __float2bfloat162_rn(0.f)));
}
__device__ __forceinline__ uint32_t where_pos(uint32_t p, uint32_t h) {
    return p & __hgt2_mask(bits_bf2(h), __float2bfloat162_rn(0.f));
}

struct TrainArgs {
    const __nv_bfloat16 *x;      // [N][K0] encoder output
    const float *target;         // [N]
    const __nv_bfloat16 *wsh;    // bf16 shadow of the flat parameters
    const float *wmaster;        // fp32 master (biases are read in fp32)
    float *dx;                   // [N][K0] dL/d(enc), fp32
    float *grad;                 // flat fp32 grads (+=, through partial + mlp_grad_reduce_kernel)
    float *partial;              // [2 gridDim.x][P] per-slot partial gradients (every element written)
    int P;                       // param_count(K0)
    float *loss;                 // += sum (y - t)^2 / N_global
    int *flag;                   // bit 1: non-finite loss
    int64_t N;
    float inv_n_global;
    int dx_lm_log2;              // 0: dx row-major [N][K0]; 2 / 3: level-major [L][N][F], F = 4 / 8
    int dx_direct;               // level-major only: dX stored from registers (no staging), MMA5 overlapping
};

// Write 8 bf16 (16 B) = one core-matrix row segment.
__device__ __forceinline__ void st16(uint8_t *base, uint32_t off, uint4 v) {
    *reinterpret_cast<uint4 *>(base + off) = v;
}

// Threads of the train kernel: two tile slots x 8 warps.  Warp ws (0..7) of
// a slot reads TMEM lane quarter ws & 3 (sample rows 32 (ws & 3) .. +31)
// and owns column half ws >> 2 of every epilogue, so each sample row's
// epilogue work is split over two threads.  (Round 1 / early round 2: 4
// warps per slot, one thread per row: the per-row epilogues were most of
// the per-tile chain -- 4.0 of 5.8 us at cfg4.)
constexpr int SLOT_THREADS = 256;
constexpr int TRAIN_THREADS = 2 * SLOT_THREADS;

// Barrier over the 256 threads of one slot (named barrier 1 + slot).
__device__ __forceinline__ void slot_sync(int slot) {
    asm volatile("bar.sync %0, 256;" ::"r"(1 + slot) : "memory");
}

// TMEM -> registers, N consecutive columns (N = 8, 16, 24 or 32), one wait.
template <int N>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, float (&v)[N]) {
    static_assert(N == 8 || N == 16 || N == 24 || N == 32, "column count");
    if constexpr (N == 32) {
        tc::tmem_ld32(taddr, v);
    } else if constexpr (N == 16) {
        tc::tmem_ld16(taddr, v);
    } else if constexpr (N == 8) {
        tc::tmem_ld8(taddr, v);
    } else {
        float a[16];
        tc::tmem_ld16(taddr, a);
        tc::tmem_ld8(taddr + 16, v + 16);
#pragma unroll
        for (int i = 0; i < 16; i++) v[i] = a[i];
    }
    tc::tmem_wait_ld();
}

// A thread's N bf16 of its row of an MMA A operand (N / 2 packed columns)
// into TMEM, then wait for the writes (the slot barrier follows).
template <int N>
__device__ __forceinline__ void store_a_tmem(uint32_t taddr, const uint32_t (&pk)[N / 2]) {
#pragma unroll
    for (int c = 0; c < N / 2; c += 8) {
        uint32_t r[8];
#pragma unroll
        for (int j = 0; j < 8; j++) r[j] = pk[c + j];
        tc::tmem_st8(taddr + c, r);
    }
    tc::tmem_wait_st();
}

// tm_x: 4-D tensor map of x ([N][K0] bf16) as (8 elements, row % 8, 16-byte
// chunk, row / 8): a box of 128 rows lands in the core-matrix layout
// (SWIZZLE_NONE, SBO = K0 * 16); rows past N read as zero.  tm_dx: 2-D map
// of dX ([N][K0] fp32), box 128 rows x 16 columns, 64-byte swizzle; rows
// past N are not written.  Both encoded per launch (train_api.cu).
template <int K0>
__global__ void __launch_bounds__(TRAIN_THREADS, 1) mlp_train_kernel(const TrainArgs a,
                                                                     const __grid_constant__ CUtensorMap tm_x,
                                                                     const __grid_constant__ CUtensorMap tm_dx) {
    using Lo = Layout<K0>;
    constexpr int HC = H / 2;            // hidden columns per thread
    constexpr int XC = K0 / 2;           // X / dX columns per thread
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *sW1 = smem;
    uint8_t *sW2 = sW1 + Lo::BYTES_W1;
    __shared__ uint64_t bar[2], xbar[2];
    __shared__ uint32_t tbase;
    __shared__ __align__(16) float b1[H];   // read as float4
    __shared__ __align__(16) float b2[H];
    __shared__ __align__(16) float w3[H];
    __shared__ float s_y[2][2][TILE];    // [slot][column half][row]: partial output-layer sums
    __shared__ float s_db3[16], s_loss[16];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int slot = warp >> 3;          // 0: warps 0-7, 1: warps 8-15
    const int ws = warp & 7;
    const int hf = ws >> 2;              // column half
    const int t = ((ws & 3) << 5) | lane;   // sample row within the slot's tile = TMEM lane
    const int ts = tid & (SLOT_THREADS - 1);
    uint8_t *sH1 = smem + Lo::BYTES_W1 + Lo::BYTES_W2 + slot * Lo::BYTES_SLOT;
    uint8_t *sXB = sH1 + Lo::BYTES_H1;   // the two X / h2 buffers
    uint8_t *sDZ = sXB + 2 * Lo::BYTES_XB;
    uint8_t *sDY = sDZ + Lo::BYTES_DZ;
    const int64_t n_tiles = (a.N + TILE - 1) / TILE;
    // the dX staging relies on the TMA swizzle's address pattern (512-byte atoms)
    if (tid == 0 && (tc::smem_u32(smem) & 1023u) != 0u) __trap();

    // ---- weights -> shared memory (bf16 shadow), once per CTA
    for (int i = tid; i < H * K0; i += blockDim.x) {
        const int r = i / K0, c = i % K0;
        *reinterpret_cast<__nv_bfloat16 *>(sW1 + tc::core_off(r, c, Lo::SBO_W1)) = a.wsh[off_W1() + i];
    }
    for (int i = tid; i < H * H; i += blockDim.x) {
        const int r = i / H, c = i % H;
        *reinterpret_cast<__nv_bfloat16 *>(sW2 + tc::core_off(r, c, Lo::SBO_W2)) = a.wsh[off_W2(K0) + i];
    }
    {   // constant columns [H, H + 16) of each slot's H1 tile: 1, 0, ..., 0
        const uint4 ones = make_uint4(pack_bf16(1.f, 0.f), 0u, 0u, 0u), zero = make_uint4(0u, 0u, 0u, 0u);
        st16(sH1, tc::core_off(t, H + 8 * hf, Lo::SBO_H1), hf ? zero : ones);
    }
    if (tid < H) {
        b1[tid] = a.wmaster[off_b1(K0) + tid];
        b2[tid] = a.wmaster[off_b2(K0) + tid];
        w3[tid] = __bfloat162float(a.wsh[off_w3(K0) + tid]);
    }
    const float b3 = a.wmaster[off_b3(K0)];

    if (warp == 0) tc::tmem_alloc(&tbase, Lo::TMEM_COLS);
    if (tid == 0) {
        for (int q = 0; q < 2; q++) { tc::mbar_init(&bar[q], 1); tc::mbar_init(&xbar[q], 1); }
        tc::fence_mbar_init();
    }
    tc::fence_smem_to_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    // X tiles arrive by TMA (tm_x), a tile ahead, into the buffer the
    // previous tile's h2 used (see Layout): the HBM latency of X overlaps the
    // previous tile's epilogues, and no thread touches X.
    uint64_t *xb = &xbar[slot];
    uint32_t xphase = 0;
    auto issue_x = [&](int64_t tl, uint32_t dst) {
        if (ts != 0 || tl >= n_tiles) return;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(xb)), "r"(Lo::BYTES_X)
                     : "memory");
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                     ::"r"(dst), "l"(reinterpret_cast<uint64_t>(&tm_x)), "r"(0), "r"(0), "r"(0), "r"((int)(tl * (TILE / 8))),
                     "r"(tc::smem_u32(xb)) : "memory");
    };
    issue_x(2 * (int64_t)blockIdx.x + slot, tc::smem_u32(sXB));
    const uint32_t tm = tbase + (uint32_t)slot * 256u;
    const uint32_t lane_off = (uint32_t)((ws & 3) * 32) << 16;
    uint64_t *mbar = &bar[slot];
    const bool issuer = (ts == 0);
    const bool direct = a.dx_direct != 0 && a.dx_lm_log2 != 0;
    const int hc0 = hf * HC;             // this thread's first hidden column

    const uint32_t aH1 = tc::smem_u32(sH1), aDZ = tc::smem_u32(sDZ), aDY = tc::smem_u32(sDY);
    const uint32_t aW1 = tc::smem_u32(sW1), aW2 = tc::smem_u32(sW2);
    constexpr uint32_t id_h = tc::idesc_bf16_f32(128, H, false, false);      // N = 64, K-major A,B
    constexpr uint32_t id_dh = tc::idesc_bf16_f32(128, H, false, true);      // B = W2 MN-major
    constexpr uint32_t id_dx = tc::idesc_bf16_f32(128, K0, false, true);     // B = W1 MN-major
    constexpr uint32_t id_dw = tc::idesc_bf16_f32(128, Lo::WH1, true, true); // both MN-major: [H1 | 1] block
    constexpr uint32_t id_dwx = tc::idesc_bf16_f32(128, K0, true, true);     // X block
    constexpr uint32_t id_d3 = tc::idesc_bf16_f32(64, 16, true, true);       // dw3: H2^T . [dy_hi dy_lo], M = 64

    uint32_t phase = 0;
    float db3_acc = 0.f, loss_acc = 0.f;
    bool bad = false;
    int my_tiles = 0;

    for (int64_t tile = 2 * (int64_t)blockIdx.x + slot; tile < n_tiles; tile += 2 * (int64_t)gridDim.x, my_tiles++) {
        const int64_t row = tile * TILE + t;
        const bool valid = row < a.N;
        // this tile's X buffer and h2 buffer (they swap every tile)
        const int xi = my_tiles & 1;
        uint8_t *sX = sXB + xi * Lo::BYTES_XB, *sH2 = sXB + (xi ^ 1) * Lo::BYTES_XB;
        const uint32_t aX = tc::smem_u32(sX), aH2 = tc::smem_u32(sH2);
        const float tgt = valid ? __ldg(a.target + row) : 0.f;
        if (a.N - tile * TILE < TILE) {
            // ragged last tile: the TMA zero-fills whole 8-row groups past N;
            // rows past N inside the last group are zeroed here
            tc::mbar_wait(xb, xphase);
            if (!valid) {
#pragma unroll
                for (int q = hf; q < K0 / 8; q += 2) st16(sX, tc::core_off(t, 8 * q, Lo::SBO_X), make_uint4(0u, 0u, 0u, 0u));
            }
            tc::fence_smem_to_async();
            tc::fence_before_sync();
            slot_sync(slot);
            tc::fence_after_sync();
        } else if (issuer) {
            tc::mbar_wait(xb, xphase);   // only the MMA issuer needs X
        }
        xphase ^= 1;
        // ---- MMA1: Z1 = X . W1^T
        if (issuer) {
#pragma unroll
            for (int s = 0; s < K0 / 16; s++)
                tc::mma_bf16(tm + Lo::T_ACC, tc::sdesc(aX + s * 256, 128, Lo::SBO_X),
                             tc::sdesc(aW1 + s * 256, 128, Lo::SBO_W1), id_h, s > 0);
            tc::commit(mbar);
        }
        tc::mbar_wait(mbar, phase); phase ^= 1;
        tc::fence_after_sync();
        // ---- epilogue 1: H1 = bf16(relu(Z1 + b1)) (its sign is the ReLU mask later)
        {
            float v[HC];
            tmem_ld_cols<HC>(tm + lane_off + Lo::T_ACC + hc0, v);
            uint32_t pk[HC / 2];
#pragma unroll
            for (int c = 0; c < HC; c += 8) {
                const float4 ba = *reinterpret_cast<const float4 *>(b1 + hc0 + c);
                const float4 bb = *reinterpret_cast<const float4 *>(b1 + hc0 + c + 4);
                pk[c / 2] = bias_relu_bf16x2(v[c], v[c + 1], ba.x, ba.y);
                pk[c / 2 + 1] = bias_relu_bf16x2(v[c + 2], v[c + 3], ba.z, ba.w);
                pk[c / 2 + 2] = bias_relu_bf16x2(v[c + 4], v[c + 5], bb.x, bb.y);
                pk[c / 2 + 3] = bias_relu_bf16x2(v[c + 6], v[c + 7], bb.z, bb.w);
                st16(sH1, tc::core_off(t, hc0 + c, Lo::SBO_H1), make_uint4(pk[c / 2], pk[c / 2 + 1], pk[c / 2 + 2], pk[c / 2 + 3]));
            }
            store_a_tmem<HC>(tm + lane_off + Lo::T_A + hc0 / 2, pk);
        }
        // the previous tile's dX stores have read the [dZ2 | dZ1] tile before
        // epilogue 2 rewrites it (this slot barrier orders the writes behind the wait)
        if (issuer) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        tc::fence_smem_to_async();
        tc::fence_before_sync();
        slot_sync(slot);
        tc::fence_after_sync();
        // ---- MMA2: Z2 = H1 . W2^T
        if (issuer) {
#pragma unroll
            for (int s = 0; s < H / 16; s++)
                tc::mma_bf16_ta(tm + Lo::T_ACC, tm + Lo::T_A + 8 * s, tc::sdesc(aW2 + s * 256, 128, Lo::SBO_W2), id_h,
                                s > 0);
            tc::commit(mbar);
        }
        tc::mbar_wait(mbar, phase); phase ^= 1;
        tc::fence_after_sync();
        // ---- epilogue 2: H2 = bf16(relu(Z2 + b2)); y = H2 . w3 + b3 (the two
        // halves' partial sums meet in shared memory); MSE; dZ2.  ReLU masks
        // are read as (h > 0): h = bf16(relu(z)) is > 0 iff z > 0.
        {
            float v[HC];
            tmem_ld_cols<HC>(tm + lane_off + Lo::T_ACC + hc0, v);
            float2 ya01 = make_float2(0.f, 0.f), ya23 = make_float2(0.f, 0.f);   // columns = 0, 1, 2, 3 mod 4
            uint32_t hp[HC / 2];
#pragma unroll
            for (int j = 0; j < HC; j += 4) {
                const float4 b = *reinterpret_cast<const float4 *>(b2 + hc0 + j);
                const float4 w = *reinterpret_cast<const float4 *>(w3 + hc0 + j);
                hp[j / 2] = bias_relu_bf16x2(v[j], v[j + 1], b.x, b.y);
                hp[j / 2 + 1] = bias_relu_bf16x2(v[j + 2], v[j + 3], b.z, b.w);
                ya01 = __ffma2_rn(unpack_bf16(hp[j / 2]), make_float2(w.x, w.y), ya01);
                ya23 = __ffma2_rn(unpack_bf16(hp[j / 2 + 1]), make_float2(w.z, w.w), ya23);
            }
#pragma unroll
            for (int c = 0; c < HC; c += 8)
                st16(sH2, tc::core_off(t, hc0 + c, 1024), make_uint4(hp[c / 2], hp[c / 2 + 1], hp[c / 2 + 2], hp[c / 2 + 3]));
            s_y[slot][hf][t] = (ya01.x + ya01.y) + (ya23.x + ya23.y);
            // only the two warps of this lane quarter exchange partial sums
            asm volatile("bar.sync %0, 64;" ::"r"(3 + 4 * slot + (ws & 3)) : "memory");
            const float y = (s_y[slot][0][t] + s_y[slot][1][t]) + b3;
            const float diff = valid ? (y - tgt) : 0.f;
            const float dy = 2.f * diff * a.inv_n_global;
            if (hf == 0) {
                if (!isfinite(diff)) bad = true;
                loss_acc = fmaf(diff, diff, loss_acc);
                db3_acc += dy;
                // dy as two bf16 (hi + lo: ~16 mantissa bits) for the dw3 GEMM below
                const float hi = bf16r(dy);
                st16(sDY, tc::core_off(t, 0, 256), make_uint4(pack_bf16(hi, dy - hi), 0u, 0u, 0u));
            } else {
                st16(sDY, tc::core_off(t, 8, 256), make_uint4(0u, 0u, 0u, 0u));
            }
#pragma unroll
            for (int c = 0; c < HC; c += 8) {
                const float4 wa = *reinterpret_cast<const float4 *>(w3 + hc0 + c);
                const float4 wb = *reinterpret_cast<const float4 *>(w3 + hc0 + c + 4);
                const float2 d2 = make_float2(dy, dy);
                const uint32_t p0 = bf2_bits(__float22bfloat162_rn(__fmul2_rn(d2, make_float2(wa.x, wa.y))));
                const uint32_t p1 = bf2_bits(__float22bfloat162_rn(__fmul2_rn(d2, make_float2(wa.z, wa.w))));
                const uint32_t p2 = bf2_bits(__float22bfloat162_rn(__fmul2_rn(d2, make_float2(wb.x, wb.y))));
                const uint32_t p3 = bf2_bits(__float22bfloat162_rn(__fmul2_rn(d2, make_float2(wb.z, wb.w))));
                hp[c / 2] = where_pos(p0, hp[c / 2]);          // h2 is no longer needed: hp takes dZ2
                hp[c / 2 + 1] = where_pos(p1, hp[c / 2 + 1]);
                hp[c / 2 + 2] = where_pos(p2, hp[c / 2 + 2]);
                hp[c / 2 + 3] = where_pos(p3, hp[c / 2 + 3]);
                st16(sDZ, tc::core_off(t, hc0 + c, Lo::SBO_DZ), make_uint4(hp[c / 2], hp[c / 2 + 1], hp[c / 2 + 2], hp[c / 2 + 3]));
            }
            store_a_tmem<HC>(tm + lane_off + Lo::T_A + hc0 / 2, hp);
        }
        tc::fence_smem_to_async();
        tc::fence_before_sync();
        slot_sync(slot);
        tc::fence_after_sync();
        // ---- MMA3: dH1 = dZ2 . W2 ; MMA6: [dw3_hi dw3_lo] += H2^T . [dy_hi dy_lo]
        // (MMA6: M = 64, hidden unit j in TMEM lane 32 (j / 16) + j % 16; was
        // M = 128 with A rows 64..127 read past the h2 tile and discarded)
        if (issuer) {
#pragma unroll
            for (int s = 0; s < H / 16; s++)
                tc::mma_bf16_ta(tm + Lo::T_ACC, tm + Lo::T_A + 8 * s, tc::sdesc(aW2 + s * 2 * Lo::SBO_W2, Lo::SBO_W2, 128),
                                id_dh, s > 0);
#pragma unroll
            for (int s = 0; s < TILE / 16; s++)
                tc::mma_bf16(tm + Lo::T_D3, tc::sdesc(aH2 + s * 2 * 1024, 1024, 128),
                             tc::sdesc(aDY + s * 2 * 256, 256, 128), id_d3, (my_tiles > 0 || s > 0) ? 1u : 0u);
            tc::commit(mbar);
        }
        tc::mbar_wait(mbar, phase); phase ^= 1;
        issue_x(tile + 2 * (int64_t)gridDim.x, aH2);   // the h2 buffer is free: the next tile's X
        tc::fence_after_sync();
        // ---- epilogue 3: dZ1 = bf16(dH1 * mask1), mask1 = (h1 > 0) from the H1 tile
        {
            float v[HC];
            uint32_t pk[HC / 2];
            tmem_ld_cols<HC>(tm + lane_off + Lo::T_ACC + hc0, v);
#pragma unroll
            for (int c = 0; c < HC; c += 8) {
                const uint4 ha = *reinterpret_cast<const uint4 *>(sH1 + tc::core_off(t, hc0 + c, Lo::SBO_H1));
                pk[c / 2] = where_pos(pack_bf16(v[c], v[c + 1]), ha.x);
                pk[c / 2 + 1] = where_pos(pack_bf16(v[c + 2], v[c + 3]), ha.y);
                pk[c / 2 + 2] = where_pos(pack_bf16(v[c + 4], v[c + 5]), ha.z);
                pk[c / 2 + 3] = where_pos(pack_bf16(v[c + 6], v[c + 7]), ha.w);
                st16(sDZ, tc::core_off(t, H + hc0 + c, Lo::SBO_DZ), make_uint4(pk[c / 2], pk[c / 2 + 1], pk[c / 2 + 2], pk[c / 2 + 3]));
            }
            store_a_tmem<HC>(tm + lane_off + Lo::T_A + hc0 / 2, pk);
        }
        tc::fence_smem_to_async();
        tc::fence_before_sync();
        slot_sync(slot);
        tc::fence_after_sync();
        // ---- MMA4: dX = dZ1 . W1 ; MMA5: DW += [dZ2^T; dZ1^T] . [H1 | 1 | X]
        // (two N blocks: the [H1 | 1] tile and the X buffer)
        if (issuer) {
#pragma unroll
            for (int s = 0; s < H / 16; s++)
                tc::mma_bf16_ta(tm + Lo::T_ACC, tm + Lo::T_A + 8 * s, tc::sdesc(aW1 + s * 2 * Lo::SBO_W1, Lo::SBO_W1, 128),
                                id_dx, s > 0);
            // direct dX (level-major): epilogue 4 needs only MMA4; MMA5 runs
            // under it, its completion covered by the next commit (the next
            // tile's MMA1, or the one after the loop)
            if (direct) tc::commit(mbar);
#pragma unroll
            for (int s = 0; s < TILE / 16; s++)
            {
                const uint64_t ad = tc::sdesc(aDZ + s * 2 * Lo::SBO_DZ, Lo::SBO_DZ, 128);
                const uint32_t acc = (my_tiles > 0 || s > 0) ? 1u : 0u;
                tc::mma_bf16(tm + Lo::T_DW, ad, tc::sdesc(aH1 + s * 2 * Lo::SBO_H1, Lo::SBO_H1, 128), id_dw, acc);
                tc::mma_bf16(tm + Lo::T_DW + Lo::WH1, ad, tc::sdesc(aX + s * 2 * Lo::SBO_X, Lo::SBO_X, 128), id_dwx, acc);
            }
            if (!direct) tc::commit(mbar);
        }
        tc::mbar_wait(mbar, phase); phase ^= 1;
        tc::fence_after_sync();
        // ---- epilogue 4: dX (fp32) -> shared staging -> TMA tensor stores.
        // The [dZ2 | dZ1] tile is free (MMA4/5 have completed); it takes the
        // 128 x K0 fp32 tile as K0 / 16 boxes of 128 rows x 16 columns in the
        // TMA's 64-byte swizzle (row t at 64 t, 16-byte chunk c at
        // c ^ ((t >> 1) & 3): conflict-free writes).  One thread issues the
        // stores; the copy engine writes dX while the slot goes on, and that
        // thread waits for the engine's reads before the tile is rewritten
        // (epilogue 2 of the next tile).  Earlier forms: 16-byte per-row
        // stores (half sectors, lg_throttle); a shared staging tile stored by
        // the threads with coalesced STGs (~1.2 us of the per-tile chain);
        // 32-byte st.global.v8 per row segment (slower).
        if (direct) {
            // level-major dX (F = 2^fl >= 4) straight from registers: a warp's
            // store of one level covers 32 consecutive rows = 32 x 4 F
            // contiguous bytes (whole lines); the [dZ2 | dZ1] tile stays
            // untouched for MMA5, which runs meanwhile
            float v[XC];
            tmem_ld_cols<XC>(tm + lane_off + Lo::T_ACC + hf * XC, v);
            const int fl = a.dx_lm_log2;
            if (valid) {
#pragma unroll
                for (int j = 0; j < XC; j += 4) {
                    const int col = hf * XC + j;
                    float *p = a.dx + ((((int64_t)(col >> fl) * a.N + row) << fl) + (col & ((1 << fl) - 1)));
                    __stcs(reinterpret_cast<float4 *>(p), make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]));
                }
            }
        } else {
            float v[XC];
            tmem_ld_cols<XC>(tm + lane_off + Lo::T_ACC + hf * XC, v);
            {   // rows past N (ragged last tile) are clipped by the TMA
                // level-major dX (F = 2^fl >= 4): a box is 16 / F levels of
                // 128 rows x F floats, row t of level-in-box lv at
                // lv * 512 F + t * 4 F bytes (F = 4: a warp's 32 rows are
                // 512 contiguous bytes, conflict-free)
                const int fl = a.dx_lm_log2;
#pragma unroll
                for (int j = 0; j < XC; j += 4) {
                    const int col = hf * XC + j, bx = col >> 4, c = (col >> 2) & 3, cc = col & 15;
                    const int off = fl ? bx * 8192 + ((cc >> fl) << (fl + 9)) + (t << (fl + 2)) + ((cc & ((1 << fl) - 1)) << 2)
                                       : bx * 8192 + t * 64 + 16 * (c ^ ((t >> 1) & 3));
                    *reinterpret_cast<float4 *>(sDZ + off) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                }
                tc::fence_smem_to_async();
                slot_sync(slot);
                if (issuer) {
                    if (fl) {
#pragma unroll
                        for (int bx = 0; bx < K0 / 16; bx++)
                            asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];"
                                         ::"l"(reinterpret_cast<uint64_t>(&tm_dx)), "r"(0), "r"((int)(tile * TILE)),
                                         "r"((16 * bx) >> fl), "r"(aDZ + 8192u * bx) : "memory");
                    } else {
#pragma unroll
                        for (int bx = 0; bx < K0 / 16; bx++)
                            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                                         ::"l"(reinterpret_cast<uint64_t>(&tm_dx)), "r"(16 * bx), "r"((int)(tile * TILE)),
                                         "r"(aDZ + 8192u * bx) : "memory");
                    }
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
            }
        }
        tc::fence_before_sync();
        slot_sync(slot);   // TMEM / smem reuse by this slot's next tile
        tc::fence_after_sync();
    }

    if (issuer) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");   // the last dX stores are done
    if (direct && my_tiles > 0) {   // the last tile's MMA5 (slot-uniform)
        if (issuer) tc::commit(mbar);
        tc::mbar_wait(mbar, phase); phase ^= 1;
        tc::fence_after_sync();
    }

    // ---- weight gradients out of TMEM: rows 0..63 -> dW2, db2; 64..127 -> dW1, db1,
    // written (not atomically added) into this slot's row of the partial
    // buffer; mlp_grad_reduce_kernel sums the rows.  (Per-slot atomics on
    // the same 6-8 k addresses from ~300 slots cost ~38 us per call at cfg3.)
    // The two column halves take alternate 16-column chunks.
    {
        const int r = t;  // TMEM lane = row of DW
        float *g = a.partial + (int64_t)(2 * blockIdx.x + slot) * a.P;
#pragma unroll 1
        for (int c = 16 * hf; c < Lo::WHX; c += 32) {
            float v[16];
            if (my_tiles > 0) {   // slot-uniform
                tc::tmem_ld16(tm + lane_off + Lo::T_DW + c, v);
                tc::tmem_wait_ld();
            } else {
#pragma unroll
                for (int j = 0; j < 16; j++) v[j] = 0.f;
            }
            // 16-column chunks lie entirely in one block: W2 (c < H), the bias chunk (c = H) or
            // W1 (c >= H + 16); the two weight blocks as float4 stores (rows padded to 4)
            float4 *dst = nullptr;
            if (r < H && c < H) dst = reinterpret_cast<float4 *>(g + off_W2(K0) + r * H + c);
            else if (r >= H && c >= Lo::WH1) dst = reinterpret_cast<float4 *>(g + off_W1() + (r - H) * K0 + (c - Lo::WH1));
            if (dst) {
#pragma unroll
                for (int j = 0; j < 16; j += 4) dst[j / 4] = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
            } else if (c == H) {
                if (r < H) g[off_b2(K0) + r] = v[0];
                else g[off_b1(K0) + (r - H)] = v[0];
            }
        }
        // dw3[j] = hi + lo columns of the D3 accumulator (M = 64 layout: j in
        // lane 32 (j / 16) + j % 16)
        if (hf == 0) {
            float d3[16] = {0.f};
            if (my_tiles > 0) {
                tc::tmem_ld16(tm + lane_off + Lo::T_D3, d3);
                tc::tmem_wait_ld();
            }
            if ((r & 31) < 16) g[off_w3(K0) + (r >> 5) * 16 + (r & 15)] = d3[0] + d3[1];
        }
    }
    // db3 and loss (column half 0 holds them): warp reduce, then one atomic per CTA
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        db3_acc += __shfl_xor_sync(0xffffffffu, db3_acc, o);
        loss_acc += __shfl_xor_sync(0xffffffffu, loss_acc, o);
    }
    if (lane == 0) { s_db3[warp] = db3_acc; s_loss[warp] = loss_acc; }
    if (bad) atomicOr(a.flag, 2);
    tc::fence_before_sync();
    __syncthreads();
    if (tid == 0) {
        float d = 0.f, l = 0.f;
        for (int w = 0; w < 16; w++) { d += s_db3[w]; l += s_loss[w]; }
        a.partial[(int64_t)(2 * blockIdx.x) * a.P + off_b3(K0)] = d;
        a.partial[(int64_t)(2 * blockIdx.x + 1) * a.P + off_b3(K0)] = 0.f;
        if (2 * (int64_t)blockIdx.x < n_tiles) atomicAdd(a.loss, l * a.inv_n_global);
    }
    if (warp == 0) tc::tmem_dealloc(tbase, Lo::TMEM_COLS);
}

// grad[p] += sum over the partial rows [0, rows) of partial[row][p]: block
// (x) = 256 parameters, block (y) = a chunk of 16 rows, one atomic per
// parameter per chunk.
__global__ void __launch_bounds__(256) mlp_grad_reduce_kernel(float *__restrict__ grad,
                                                              const float *__restrict__ partial, int rows, int P,
                                                              int n_params) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n_params) return;
    const int r0 = blockIdx.y * 16, r1 = min(rows, r0 + 16);
    float v = 0.f;
    for (int r = r0; r < r1; r++) v += partial[(int64_t)r * P + p];
    atomicAdd(grad + p, v);
}

// ------------------------------------------------------------------ Adam
// Bias-corrected Adam (R12), fp32 master/m/v, dense over every parameter:
//   m = b1 m + (1-b1) g;  v = b2 v + (1-b2) g^2
//   p -= lr * (m * c1) / (sqrt(v * c2) + eps),  c1 = 1/(1-b1^t), c2 = 1/(1-b2^t)
// then writes the low-precision shadow (fp16 table / bf16 MLP).  The grads are
// left as they are: every fh_train_fwd_bwd overwrites them.
struct AdamSeg {
    float *p, *g, *m, *v;
    void *shadow;        // __half* (kind 1), __nv_bfloat16* (kind 2), unused (kind 0)
    int64_t n;
    int kind;
    int vec;             // 1: p, g, m, v 16-byte and shadow 8-byte aligned -> float4 path
};

// Up to kMaxAdamSeg segments per launch (table ranges + the MLP); segment i
// owns blocks [block0[i], block0[i+1]).
constexpr int kMaxAdamSeg = 64;

struct AdamArgs {
    AdamSeg seg[kMaxAdamSeg];
    int64_t block0[kMaxAdamSeg + 1];
    int nseg;
    float lr, b1, b2, eps, c1, c2;
    float omb1, omb2;    // 1 - beta, rounded once from double (fp32 1.f - 0.999f is 5e-5 off)
};

__device__ __forceinline__ void adam_one(const AdamArgs &A, const AdamSeg &s, int64_t i) {
    const float g = s.g[i];
    const float m = fmaf(A.b1, s.m[i], A.omb1 * g);
    const float v = fmaf(A.b2, s.v[i], A.omb2 * g * g);
    const float p = s.p[i] - A.lr * (m * A.c1) / (sqrtf(v * A.c2) + A.eps);
    s.m[i] = m; s.v[i] = v; s.p[i] = p;
    if (s.kind == 1) reinterpret_cast<__half *>(s.shadow)[i] = __float2half_rn(p);
    else if (s.kind == 2) reinterpret_cast<__nv_bfloat16 *>(s.shadow)[i] = __float2bfloat16_rn(p);
    // kind 0: fp32 master only (FH_F32 tables are read directly), no shadow
}

__global__ void __launch_bounds__(256) adam_kernel(const __grid_constant__ AdamArgs A) {
    int si = 0;
    while (si + 1 < A.nseg && (int64_t)blockIdx.x >= A.block0[si + 1]) si++;
    const AdamSeg &s = A.seg[si];
    const int64_t b = (int64_t)blockIdx.x - A.block0[si];
    const int64_t nb = A.block0[si + 1] - A.block0[si];
    if (!s.vec) {   // unaligned segment (a tail range): scalar
        for (int64_t i = b * blockDim.x + threadIdx.x; i < s.n; i += nb * blockDim.x) adam_one(A, s, i);
        return;
    }
    // 4 elements per thread per iteration
    const int64_t n4 = s.n / 4;
    for (int64_t q = b * blockDim.x + threadIdx.x; q < n4; q += nb * blockDim.x) {
        float4 g = reinterpret_cast<const float4 *>(s.g)[q];
        float4 m = reinterpret_cast<const float4 *>(s.m)[q];
        float4 v = reinterpret_cast<const float4 *>(s.v)[q];
        float4 p = reinterpret_cast<const float4 *>(s.p)[q];
        float gg[4] = {g.x, g.y, g.z, g.w}, mm[4] = {m.x, m.y, m.z, m.w};
        float vv[4] = {v.x, v.y, v.z, v.w}, pp[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
        for (int k = 0; k < 4; k++) {
            mm[k] = fmaf(A.b1, mm[k], A.omb1 * gg[k]);
            vv[k] = fmaf(A.b2, vv[k], A.omb2 * gg[k] * gg[k]);
            pp[k] = pp[k] - A.lr * (mm[k] * A.c1) / (sqrtf(vv[k] * A.c2) + A.eps);
        }
        reinterpret_cast<float4 *>(s.m)[q] = make_float4(mm[0], mm[1], mm[2], mm[3]);
        reinterpret_cast<float4 *>(s.v)[q] = make_float4(vv[0], vv[1], vv[2], vv[3]);
        reinterpret_cast<float4 *>(s.p)[q] = make_float4(pp[0], pp[1], pp[2], pp[3]);
        if (s.kind == 1) {
            __half2 h0 = __floats2half2_rn(pp[0], pp[1]), h1 = __floats2half2_rn(pp[2], pp[3]);
            uint2 u;
            u.x = *reinterpret_cast<uint32_t *>(&h0);
            u.y = *reinterpret_cast<uint32_t *>(&h1);
            reinterpret_cast<uint2 *>(s.shadow)[q] = u;
        } else if (s.kind == 2) {
            __nv_bfloat162 h0 = __floats2bfloat162_rn(pp[0], pp[1]), h1 = __floats2bfloat162_rn(pp[2], pp[3]);
            uint2 u;
            u.x = *reinterpret_cast<uint32_t *>(&h0);
            u.y = *reinterpret_cast<uint32_t *>(&h1);
            reinterpret_cast<uint2 *>(s.shadow)[q] = u;
        }
    }
    // tail
    if (b == 0)
        for (int64_t i = n4 * 4 + threadIdx.x; i < s.n; i += blockDim.x) adam_one(A, s, i);
}

// ------------------------------------------------------------ fused DP step
// Reduce-scatter + Adam + all-gather in ONE kernel over peer memory
// (on NVLink peer pointers instead of an NVLS
// multicast object): segment i is a range of the flat table (or the MLP)
// that this rank updates; its gradient is the SUM over the W ranks' grad
// buffers read through peer pointers, Adam runs in registers on the local
// master / moments, and the fp16 shadow is stored into every rank's shadow
// buffer (broadcast segments: this rank's chunk) or only the local one
// (replicated segments every rank computes identically).  The caller orders
// it against the other ranks (all of them finished the gradients it reads;
// nobody reuses them before every rank is done).
constexpr int kMaxPeers = 8;

struct PeerArgs {
    const float *pg[kMaxPeers];    // each rank's flat table grad buffer
    __half *psh[kMaxPeers];        // each rank's fp16 table shadow
    const float *pmg[kMaxPeers];   // each rank's MLP grad buffer
    int W;
    int64_t off[kMaxAdamSeg];      // element offset of segment i in the peer buffers
    int src[kMaxAdamSeg];          // 0: table grads, 1: MLP grads
    int bcast[kMaxAdamSeg];        // 1: store the fp16 shadow into every rank's buffer
};

__global__ void __launch_bounds__(256) adam_peers_kernel(const __grid_constant__ AdamArgs A,
                                                         const __grid_constant__ PeerArgs P) {
    int si = 0;
    while (si + 1 < A.nseg && (int64_t)blockIdx.x >= A.block0[si + 1]) si++;
    const AdamSeg &s = A.seg[si];
    const int64_t b = (int64_t)blockIdx.x - A.block0[si];
    const int64_t nb = A.block0[si + 1] - A.block0[si];
    const float *const *G = P.src[si] ? P.pmg : P.pg;
    const int64_t off = P.off[si];
    auto update = [&](int64_t i, float g) {
        const float m = fmaf(A.b1, s.m[i], A.omb1 * g);
        const float v = fmaf(A.b2, s.v[i], A.omb2 * g * g);
        const float p = s.p[i] - A.lr * (m * A.c1) / (sqrtf(v * A.c2) + A.eps);
        s.m[i] = m; s.v[i] = v; s.p[i] = p;
        if (s.kind == 2) {
            reinterpret_cast<__nv_bfloat16 *>(s.shadow)[i] = __float2bfloat16_rn(p);
        } else if (s.kind == 1) {
            const __half h = __float2half_rn(p);
            if (P.bcast[si]) {
                for (int r = 0; r < P.W; r++) P.psh[r][off + i] = h;
            } else {
                reinterpret_cast<__half *>(s.shadow)[i] = h;
            }
        }
    };
    for (int64_t i = b * blockDim.x + threadIdx.x; i < s.n; i += nb * blockDim.x) {
        float g = 0.f;
        for (int r = 0; r < P.W; r++) g += G[r][off + i];   // ranks in order: same sum on every rank
        update(i, g);
    }
}

// ------------------------------------------------ fused DP step over NVLS
// The same reduce-scatter + Adam + all-gather through an NVLS multicast
// object (SURVEY.md §8(e) item 3 as written): the gradient of an element is
// ONE multimem.ld_reduce of its multicast address (the sum over every
// rank's buffer, formed by the NVSwitch), and the fp16 shadow of a
// broadcast range is ONE multimem.st to the multicast address (written into
// every rank's shadow).  Replicated ranges (every rank updates them) store
// the local shadow only.
struct McArgs {
    const float *g;                // multicast address of the flat table grad buffer
    __half *sh;                    // multicast address of the fp16 table shadow
    const float *mg;               // multicast address of the MLP grads
    int64_t off[kMaxAdamSeg];      // element offset of segment i in the multicast buffers
    int src[kMaxAdamSeg];          // 0: table grads, 1: MLP grads
    int bcast[kMaxAdamSeg];        // 1: multimem.st the fp16 shadow to every rank
};

__device__ __forceinline__ float4 mc_ld_reduce4(const float *p) {
    float4 v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}
__device__ __forceinline__ float mc_ld_reduce(const float *p) {
    float v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
    return v;
}
// (multimem.st has no 16-bit form: the fp16 shadow goes out as f16x2 pairs)
__device__ __forceinline__ void mc_st8(void *p, uint32_t a, uint32_t b) {   // 4 fp16 to every rank
    asm volatile("multimem.st.relaxed.sys.global.v2.f16x2 [%0], {%1, %2};" ::"l"(p), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void mc_st4(void *p, uint32_t a) {               // 2 fp16 to every rank
    asm volatile("multimem.st.relaxed.sys.global.f16x2 [%0], %1;" ::"l"(p), "r"(a) : "memory");
}

__global__ void __launch_bounds__(256) adam_multicast_kernel(const __grid_constant__ AdamArgs A,
                                                             const __grid_constant__ McArgs M) {
    int si = 0;
    while (si + 1 < A.nseg && (int64_t)blockIdx.x >= A.block0[si + 1]) si++;
    const AdamSeg &s = A.seg[si];
    const int64_t b = (int64_t)blockIdx.x - A.block0[si];
    const int64_t nb = A.block0[si + 1] - A.block0[si];
    const float *G = (M.src[si] ? M.mg : M.g) + M.off[si];
    const bool bc = M.bcast[si] != 0 && s.kind == 1;
    __half *msh = M.sh + M.off[si];
    auto one = [&](int64_t i, float g) -> float {   // the new master; stores the local shadow unless broadcast
        const float m = fmaf(A.b1, s.m[i], A.omb1 * g);
        const float v = fmaf(A.b2, s.v[i], A.omb2 * g * g);
        const float p = s.p[i] - A.lr * (m * A.c1) / (sqrtf(v * A.c2) + A.eps);
        s.m[i] = m; s.v[i] = v; s.p[i] = p;
        if (s.kind == 2) reinterpret_cast<__nv_bfloat16 *>(s.shadow)[i] = __float2bfloat16_rn(p);
        else if (s.kind == 1 && !bc) reinterpret_cast<__half *>(s.shadow)[i] = __float2half_rn(p);
        return p;
    };
    // 4 elements per thread when the segment and its multicast offset allow
    // 16-byte (grads) / 8-byte (shadow) accesses; else one at a time
    const bool vec = s.vec && (M.off[si] % 4) == 0;
    const int64_t n4 = vec ? s.n / 4 : 0;
    for (int64_t q = b * blockDim.x + threadIdx.x; q < n4; q += nb * blockDim.x) {
        const float4 g = mc_ld_reduce4(G + 4 * q);
        float4 m = reinterpret_cast<const float4 *>(s.m)[q];
        float4 v = reinterpret_cast<const float4 *>(s.v)[q];
        float4 p = reinterpret_cast<const float4 *>(s.p)[q];
        float gg[4] = {g.x, g.y, g.z, g.w}, mm[4] = {m.x, m.y, m.z, m.w};
        float vv[4] = {v.x, v.y, v.z, v.w}, pp[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
        for (int k = 0; k < 4; k++) {
            mm[k] = fmaf(A.b1, mm[k], A.omb1 * gg[k]);
            vv[k] = fmaf(A.b2, vv[k], A.omb2 * gg[k] * gg[k]);
            pp[k] = pp[k] - A.lr * (mm[k] * A.c1) / (sqrtf(vv[k] * A.c2) + A.eps);
        }
        reinterpret_cast<float4 *>(s.m)[q] = make_float4(mm[0], mm[1], mm[2], mm[3]);
        reinterpret_cast<float4 *>(s.v)[q] = make_float4(vv[0], vv[1], vv[2], vv[3]);
        reinterpret_cast<float4 *>(s.p)[q] = make_float4(pp[0], pp[1], pp[2], pp[3]);
        if (s.kind == 1) {
            __half2 h0 = __floats2half2_rn(pp[0], pp[1]), h1 = __floats2half2_rn(pp[2], pp[3]);
            const uint32_t u0 = *reinterpret_cast<uint32_t *>(&h0), u1 = *reinterpret_cast<uint32_t *>(&h1);
            if (bc) mc_st8(msh + 4 * q, u0, u1);
            else reinterpret_cast<uint2 *>(s.shadow)[q] = make_uint2(u0, u1);
        } else if (s.kind == 2) {
            __nv_bfloat162 h0 = __floats2bfloat162_rn(pp[0], pp[1]), h1 = __floats2bfloat162_rn(pp[2], pp[3]);
            uint2 u;
            u.x = *reinterpret_cast<uint32_t *>(&h0);
            u.y = *reinterpret_cast<uint32_t *>(&h1);
            reinterpret_cast<uint2 *>(s.shadow)[q] = u;
        }
    }
    if (bc) {   // broadcast scalar path: element pairs (even offsets and lengths, checked by the host)
        for (int64_t i = 4 * n4 + 2 * (b * blockDim.x + threadIdx.x); i < s.n; i += 2 * nb * blockDim.x) {
            const float p0 = one(i, mc_ld_reduce(G + i)), p1 = one(i + 1, mc_ld_reduce(G + i + 1));
            __half2 h = __floats2half2_rn(p0, p1);
            mc_st4(msh + i, *reinterpret_cast<uint32_t *>(&h));
        }
    } else {
        for (int64_t i = 4 * n4 + b * blockDim.x + threadIdx.x; i < s.n; i += nb * blockDim.x) one(i, mc_ld_reduce(G + i));
    }
}

}  // namespace mlp
}  // namespace fh
