// infer_kernels.cuh -- NEXT-1: the renderer's model evaluation V = model(S)
// (Alg. 1, "Inference F-Hash INR") as ONE kernel: the encode
// forward (steps 1-4 of §3.2.4, through the same device
// functions as fwd_kernel, encode_device.cuh) is written as bf16 straight
// into the shared-memory X operand of the tcgen05 MLP forward (MMA1 ->
// bias + ReLU -> MMA2 -> bias + ReLU -> 64 -> 1 output): no encoder-output
// round trip through global memory, one launch.
//
// Why a cluster.  A 128-sample tile is 128 L corner-cell gathers, i.e.
// 8 x 128 L pair requests (16 K at L = 16): one SM issues about one L2
// request per cycle, so a tile gathered by one CTA costs >= 8 us however the
// loads are scheduled (measured: 22.7 us for a single tile).  Here a
// cluster of C = 8 CTAs (8 SMs) shares every tile: CTA r gathers the items
// i = r, r + C, ... of the tile and stores their bf16 features into the X
// tile of the tile's LEADER CTA through distributed shared memory; tiles
// rotate over the cluster's CTAs as leaders, so the MLP work is spread too.
//
// Large batches need no spreading: there the cluster size is 1 (every CTA
// gathers and evaluates its own tiles, CTA-scope fences only).
//
// Roles per CTA: warps 0-3 run the MLP of the tiles this CTA leads
// (thread t = TMEM lane = sample row t); the other warps gather, as 2-3
// groups of 8 warps working on different tiles (more loads in flight).  Per
// leader NB = 4 X buffers; mbarriers (no cluster-wide barrier in the loop):
//   full[b]     (in the leader)  C x 8 gather-warp arrivals: X[b] complete;
//   xfree[L][b] (in every CTA)   1 arrival from leader L's MLP thread once
//                                MMA1 has consumed L's X[b].
// Cluster-local tile u (global tile c + n_clusters u of cluster c) is led by
// rank u % C in buffer (u / C) % NB.
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

constexpr int kMaxCluster = 8;              // CTAs per cluster (portable maximum; 16 measured slower: fewer
                                            // resident clusters, longer waits for the slowest CTA)
constexpr int kMlpWarps = 4, kGatherWarps = 8;   // gather warps per group
// groups of gather warps work on different tiles concurrently (more loads in
// flight per SM); the register file bounds them: 3 groups (896 threads, 72
// registers) for F <= 2, 2 groups (640 threads, 96 registers) for wider entries
template <int F> struct Groups { static constexpr int value = F <= 2 ? 3 : 2; };
template <int F> struct Threads { static constexpr int value = 32 * (kMlpWarps + Groups<F>::value * kGatherWarps); };

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
};

// ---- cluster / DSMEM / mbarrier primitives (PTX ISA: mapa, st.shared::cluster,
// mbarrier.arrive.release.cluster, barrier.cluster)
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_id() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t n_clusters() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void wait_cluster(uint64_t *mbar, uint32_t parity) {
    const uint32_t a = tc::smem_u32(mbar);
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n\t}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}

// bf16 of the F blended features into X at a shared::cluster address.
template <int F>
__device__ __forceinline__ void st_x_remote(uint32_t addr, const float (&v)[F]) {
    if constexpr (F == 1) {
        const __nv_bfloat16 h = __float2bfloat16_rn(v[0]);
        asm volatile("st.shared::cluster.b16 [%0], %1;" ::"r"(addr), "h"(*reinterpret_cast<const unsigned short *>(&h))
                     : "memory");
    } else if constexpr (F == 2) {
        asm volatile("st.shared::cluster.b32 [%0], %1;" ::"r"(addr), "r"(mlp::pack_bf16(v[0], v[1])) : "memory");
    } else if constexpr (F == 4) {
        asm volatile("st.shared::cluster.v2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(mlp::pack_bf16(v[0], v[1])),
                     "r"(mlp::pack_bf16(v[2], v[3]))
                     : "memory");
    } else {
        asm volatile("st.shared::cluster.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(mlp::pack_bf16(v[0], v[1])),
                     "r"(mlp::pack_bf16(v[2], v[3])), "r"(mlp::pack_bf16(v[4], v[5])), "r"(mlp::pack_bf16(v[6], v[7]))
                     : "memory");
    }
}


template <int F, typename T, int K0>
__global__ void __launch_bounds__(Threads<F>::value, 1) infer_fused_kernel(const __grid_constant__ Params P, const FusedArgs a) {
    using Lo = FusedLayout<K0>;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *sW1 = smem;
    uint8_t *sW2 = sW1 + Lo::BYTES_W1;
    uint8_t *sX0 = sW2 + Lo::BYTES_W2;       // X[0 .. NB)
    uint8_t *sH = sX0 + Lo::NB * Lo::BYTES_X;
    constexpr int NB = Lo::NB;
    __shared__ LevelSmem slv;
    __shared__ uint64_t full[Lo::NB], xfree[kMaxCluster][Lo::NB], mma_bar;
    __shared__ uint32_t tbase;
    __shared__ float b1[H], b2[H], w3[H];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = cluster_rank(), cid = cluster_id(), ncl = n_clusters();
    const int C = (int)cluster_size();
    if (tid == 0) {
        for (int b = 0; b < NB; b++) {
            tc::mbar_init(&full[b], C * kGatherWarps);
            for (int l = 0; l < C; l++) tc::mbar_init(&xfree[l][b], 1);
        }
        tc::mbar_init(&mma_bar, 1);
        tc::fence_mbar_init();
    }
    tc::fence_smem_to_async();
    load_levels(P, slv);
    tc::fence_before_sync();
    cluster_sync_all();   // every CTA's barriers initialised before any remote arrive
    tc::fence_after_sync();

    constexpr int R = TILE;
    const int64_t n_tiles = (a.N + R - 1) / R;
    const int64_t n_u = (int64_t)cid < n_tiles ? (n_tiles - cid + ncl - 1) / ncl : 0;   // this cluster's tiles
    const int L = P.L;

    if (warp >= kMlpWarps) {
        // ------------------------------------------------ gather warps
        const int gq = tid - 32 * kMlpWarps;
        const int grp = gq / (32 * kGatherWarps);     // this warp's gather group
        const int gt = gq % (32 * kGatherWarps);      // 0 .. 255 within the group
        const T *table = reinterpret_cast<const T *>(a.table);
        const int items = R * L;
        const uint32_t x0 = tc::smem_u32(sX0);
        const uint32_t full0 = tc::smem_u32(&full[0]);
        // tiles u = grp, grp + G, ...: tiles u and u + NB C (the next use of a
        // leader's buffer) may belong to different groups, so the xfree wait
        // orders them
        for (int64_t u = grp; u < n_u; u += Groups<F>::value) {
            const uint32_t ld = (uint32_t)(u % C), b = (uint32_t)((u / C) % NB);
            const int64_t m = u / (NB * C);           // use index of (leader, buffer)
            if (m > 0) wait_cluster(&xfree[ld][b], (uint32_t)((m - 1) & 1));
            const int64_t tile = (int64_t)cid + (int64_t)ncl * u;
            const uint32_t xr = mapa(x0 + b * Lo::BYTES_X, ld);
#pragma unroll 1
            for (int i = (int)rank + C * gt; i < items; i += C * 32 * kGatherWarps) {
                const int s = i / L, l = i - s * L;
                const int64_t n = tile * R + s;
                float v[F];
                if (n < a.N) {
                    Cell c;
                    if (cell_of(slv.get(l), __ldg(a.coords + n), c) && l == 0) atomicOr(a.flag, 1);
                    float e[16][F];
                    gather16<T, F>(table, nullptr, c.idx, e);
                    blend16<F>(e, c.w, v);
                } else {
#pragma unroll
                    for (int f = 0; f < F; f++) v[f] = 0.f;
                }
                st_x_remote<F>(xr + tc::core_off(s, l * F, Lo::SBO_X), v);
            }
            // the stores (generic proxy) must be visible to the leader's tensor core
            if (C > 1) {   // stores into a peer's X: cluster-scope proxy fence + release
                asm volatile("fence.proxy.async;" ::: "memory");
                __syncwarp();
                if (lane == 0) arrive_remote(mapa(full0 + b * 8, ld));
            } else {       // own X: CTA scope is enough
                tc::fence_smem_to_async();
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(full0 + b * 8) : "memory");
            }
        }
    } else {
        // ------------------------------------------------ MLP warps (this CTA's tiles)
        // TMEM and the weights are set up here, while the gather warps already gather
        if (warp == 0) tc::tmem_alloc(&tbase, 64);
        // weights -> shared memory (core-matrix layout, one 16-byte row segment per store)
        {
            const uint4 *w = reinterpret_cast<const uint4 *>(a.wsh);
            for (int q = tid; q < H * K0 / 8; q += (32 * kMlpWarps)) {
                const int r = q / (K0 / 8), c = (q % (K0 / 8)) * 8;
                mlp::st16(sW1, tc::core_off(r, c, Lo::SBO_X), __ldg(w + (mlp::off_W1() / 8) + q));
            }
            const uint4 *w2 = reinterpret_cast<const uint4 *>(a.wsh + mlp::off_W2(K0));
            for (int q = tid; q < H * H / 8; q += (32 * kMlpWarps)) {
                const int r = q / (H / 8), c = (q % (H / 8)) * 8;
                mlp::st16(sW2, tc::core_off(r, c, Lo::SBO_H), __ldg(w2 + q));
            }
        }
        if (tid < H) {
            b1[tid] = a.wmaster[mlp::off_b1(K0) + tid];
            b2[tid] = a.wmaster[mlp::off_b2(K0) + tid];
            w3[tid] = __bfloat162float(a.wsh[mlp::off_w3(K0) + tid]);
        }
        tc::fence_smem_to_async();
        tc::fence_before_sync();
        mlp::slot_sync(0);                                // named barrier 1 over the 128 MLP threads
        tc::fence_after_sync();
        const uint32_t tm = tbase;
        const int row = tid;                              // TMEM lane = sample row
        const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
        const uint32_t aH = tc::smem_u32(sH), aW1 = tc::smem_u32(sW1), aW2 = tc::smem_u32(sW2);
        constexpr uint32_t id_h = tc::idesc_bf16_f32(128, H, false, false);
        const float b3 = a.wmaster[mlp::off_b3(K0)];
        const uint32_t xfree0 = tc::smem_u32(&xfree[rank][0]);
        uint32_t phase = 0;
        for (int64_t u = rank; u < n_u; u += C) {
            const uint32_t b = (uint32_t)((u / C) % NB);
            const int64_t m = u / (NB * C);
            wait_cluster(&full[b], (uint32_t)(m & 1));
            tc::fence_after_sync();
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
            // X[b] consumed: free it in every CTA of the cluster (lane j -> CTA j, in
            // parallel) -- only if the gather warps will refill it (tile u + NB C),
            // so every remote arrival targets a CTA that is still waiting for it
            if (tid < C && u + NB * C < n_u) {
                if (C > 1) arrive_remote(mapa(xfree0 + b * 8, (uint32_t)tid));
                else asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(xfree0 + b * 8) : "memory");
            }
            // ---- H1 = bf16(relu(Z1 + b1))
#pragma unroll
            for (int c = 0; c < H; c += 16) {
                float v[16];
                tc::tmem_ld16(tm + lane_off + c, v);
                tc::tmem_wait_ld();
                uint32_t p[8];
#pragma unroll
                for (int j = 0; j < 16; j += 2)
                    p[j / 2] = mlp::pack_bf16(fmaxf(v[j] + b1[c + j], 0.f), fmaxf(v[j + 1] + b1[c + j + 1], 0.f));
                mlp::st16(sH, tc::core_off(row, c, Lo::SBO_H), make_uint4(p[0], p[1], p[2], p[3]));
                mlp::st16(sH, tc::core_off(row, c + 8, Lo::SBO_H), make_uint4(p[4], p[5], p[6], p[7]));
            }
            tc::fence_smem_to_async();
            tc::fence_before_sync();
            mlp::slot_sync(0);                            // named barrier 1 over the 128 MLP threads
            tc::fence_after_sync();
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
            // ---- y = bf16(relu(Z2 + b2)) . w3 + b3
            float ya[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int c = 0; c < H; c += 16) {
                float v[16];
                tc::tmem_ld16(tm + lane_off + c, v);
                tc::tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 16; j++)
                    ya[j & 3] = fmaf(mlp::bf16r(fmaxf(v[j] + b2[c + j], 0.f)), w3[c + j], ya[j & 3]);
            }
            const int64_t n = ((int64_t)cid + (int64_t)ncl * u) * R + row;
            if (n < a.N) a.y[n] = ((ya[0] + ya[1]) + (ya[2] + ya[3])) + b3;
            tc::fence_before_sync();
            mlp::slot_sync(0);                            // TMEM and H reused by the next tile
            tc::fence_after_sync();
        }
    }
    // No closing cluster barrier: a CTA's X buffers and barriers are only
    // written by peers while it still waits for them (full[] before each of
    // its MLP tiles, xfree[] before each refill), so every CTA may exit as
    // soon as its own work is done.
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tbase, 64);
}

}  // namespace infer
}  // namespace fh
