// umma_probe.cu -- GPU test probe for the tcgen05 helpers in
// paper_2507_03836_b200/csrc/tc_sm100.cuh: one CTA computes
// D[128 x N] = A[128 x K] . B[N x K]^T with bf16 operands in shared memory
// (K-major or MN-major SWIZZLE_NONE layouts) and f32 accumulation in TMEM,
// and writes D to global memory.  Test infrastructure only.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../paper_2507_03836_b200/csrc/tc_sm100.cuh"

using namespace fh::tc;

// A: a_mn ? Am[K][128] : A[128][K];  B: b_mn ? Bm[K][N] : B[N][K]  (row-major bf16)
__global__ void __launch_bounds__(128) probe(const __nv_bfloat16 *A, const __nv_bfloat16 *B, float *D, int N, int K,
                                             int a_mn, int b_mn) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int M = 128;
    uint8_t *sA = smem;                 // 128*K*2 bytes
    uint8_t *sB = smem + M * K * 2;     // N*K*2 bytes
    const int t = threadIdx.x, warp = t >> 5;
    // ---- stage operands into core-matrix layouts
    // a_mn == 2: A[128][K] goes to TMEM (lane = row, two bf16 per column)
    for (int i = t; i < M * K && a_mn != 2; i += blockDim.x) {
        int m, k;
        uint32_t off;
        if (!a_mn) { m = i / K; k = i % K; off = core_off(m, k, (K / 8) * 128); }
        else { k = i / M; m = i % M; off = core_off(k, m, (M / 8) * 128); }
        *reinterpret_cast<__nv_bfloat16 *>(sA + off) = A[i];
    }
    for (int i = t; i < N * K; i += blockDim.x) {
        int n, k;
        uint32_t off;
        if (!b_mn) { n = i / K; k = i % K; off = core_off(n, k, (K / 8) * 128); }
        else { k = i / N; n = i % N; off = core_off(k, n, (N / 8) * 128); }
        *reinterpret_cast<__nv_bfloat16 *>(sB + off) = B[i];
    }
    if (warp == 0) tmem_alloc(&tbase, 256);
    if (t == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    fence_smem_to_async();
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t d = tbase;
    const uint32_t a_col = 160;        // A in TMEM (a_mn == 2): columns [160, 160 + K/2)
    if (a_mn == 2) {
        for (int c0 = 0; c0 < K / 2; c0 += 8) {
            uint32_t r[8];
            for (int j = 0; j < 8; j++) {
                const int k = 2 * (c0 + j);
                __nv_bfloat162 v;
                v.x = A[t * K + k];
                v.y = A[t * K + k + 1];
                r[j] = *reinterpret_cast<uint32_t *>(&v);
            }
            tmem_st8(d + ((uint32_t)(warp * 32) << 16) + a_col + c0, r);
        }
        tmem_wait_st();
        fence_before_sync();
        __syncthreads();
        fence_after_sync();
    }
    if (t == 0) {
        const uint32_t idesc = idesc_bf16_f32(M, N, a_mn == 1, b_mn);
        for (int s = 0; s < K / 16; s++) {
            uint64_t ad, bd;
            if (!a_mn) ad = sdesc(smem_u32(sA) + s * 256, 128, (K / 8) * 128);
            else ad = sdesc(smem_u32(sA) + s * 2 * (M / 8) * 128, (M / 8) * 128, 128);
            if (!b_mn) bd = sdesc(smem_u32(sB) + s * 256, 128, (K / 8) * 128);
            else bd = sdesc(smem_u32(sB) + s * 2 * (N / 8) * 128, (N / 8) * 128, 128);
            if (a_mn == 2) mma_bf16_ta(d, d + a_col + 8 * s, bd, idesc, s > 0);
            else mma_bf16(d, ad, bd, idesc, s > 0);
        }
        commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    fence_after_sync();
    for (int c = 0; c < N; c += 16) {
        float v[16];
        tmem_ld16(d + ((uint32_t)(warp * 32) << 16) + c, v);
        tmem_wait_ld();
        for (int j = 0; j < 16; j++) D[t * N + c + j] = v[j];
    }
    fence_before_sync();
    __syncthreads();
    if (warp == 0) tmem_dealloc(d, 256);
}

extern "C" int umma_probe(const void *A, const void *B, float *D, int N, int K, int a_mn, int b_mn) {
    const int smem = (128 * K + N * K) * 2;
    if (cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return -1;
    probe<<<1, 128, smem>>>((const __nv_bfloat16 *)A, (const __nv_bfloat16 *)B, D, N, K, a_mn, b_mn);
    if (cudaGetLastError() != cudaSuccess) return -2;
    return cudaDeviceSynchronize() == cudaSuccess ? 0 : -3;
}

// M = 64 variant (cta_group::1): A[64][K] (a_mn: stored [K][64]), B[N][K]
// (b_mn: [K][N]); D read back from all 128 TMEM lanes x N columns into
// Dall[128][N] (lanes the MMA does not write keep the 0 they were set to).
__global__ void __launch_bounds__(128) probe64(const __nv_bfloat16 *A, const __nv_bfloat16 *B, float *Dall, int N,
                                               int K, int a_mn, int b_mn, int lane0) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int M = 64;
    uint8_t *sA = smem;
    uint8_t *sB = smem + M * K * 2;
    const int t = threadIdx.x, warp = t >> 5;
    for (int i = t; i < M * K; i += blockDim.x) {
        int m, k;
        uint32_t off;
        if (!a_mn) { m = i / K; k = i % K; off = core_off(m, k, (K / 8) * 128); }
        else { k = i / M; m = i % M; off = core_off(k, m, (M / 8) * 128); }
        *reinterpret_cast<__nv_bfloat16 *>(sA + off) = A[i];
    }
    for (int i = t; i < N * K; i += blockDim.x) {
        int n, k;
        uint32_t off;
        if (!b_mn) { n = i / K; k = i % K; off = core_off(n, k, (K / 8) * 128); }
        else { k = i / N; n = i % N; off = core_off(k, n, (N / 8) * 128); }
        *reinterpret_cast<__nv_bfloat16 *>(sB + off) = B[i];
    }
    if (warp == 0) tmem_alloc(&tbase, 256);
    if (t == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    fence_smem_to_async();
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t d = tbase;
    {   // zero D (all lanes) first
        uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int c = 0; c < N; c += 8) tmem_st8(d + ((uint32_t)(warp * 32) << 16) + c, z);
        tmem_wait_st();
    }
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    if (t == 0) {
        const uint32_t idesc = idesc_bf16_f32(M, N, a_mn, b_mn);
        for (int s = 0; s < K / 16; s++) {
            uint64_t ad, bd;
            if (!a_mn) ad = sdesc(smem_u32(sA) + s * 256, 128, (K / 8) * 128);
            else ad = sdesc(smem_u32(sA) + s * 2 * (M / 8) * 128, (M / 8) * 128, 128);
            if (!b_mn) bd = sdesc(smem_u32(sB) + s * 256, 128, (K / 8) * 128);
            else bd = sdesc(smem_u32(sB) + s * 2 * (N / 8) * 128, (N / 8) * 128, 128);
            mma_bf16(d + ((uint32_t)lane0 << 16), ad, bd, idesc, 1);
        }
        commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    fence_after_sync();
    for (int c = 0; c < N; c += 16) {
        float v[16];
        tmem_ld16(d + ((uint32_t)(warp * 32) << 16) + c, v);
        tmem_wait_ld();
        for (int j = 0; j < 16; j++) Dall[t * N + c + j] = v[j];
    }
    fence_before_sync();
    __syncthreads();
    if (warp == 0) tmem_dealloc(d, 256);
}

// lane0: lane field of the D address (0, or 16 for the other half of the
// lanes when the M = 64 layout allows it)
extern "C" int umma_probe64(const void *A, const void *B, float *Dall, int N, int K, int a_mn, int b_mn, int lane0) {
    const int smem = (64 * K + N * K) * 2;
    if (cudaFuncSetAttribute(probe64, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return -1;
    probe64<<<1, 128, smem>>>((const __nv_bfloat16 *)A, (const __nv_bfloat16 *)B, Dall, N, K, a_mn, b_mn, lane0);
    if (cudaGetLastError() != cudaSuccess) return -2;
    return cudaDeviceSynchronize() == cudaSuccess ? 0 : -3;
}
