// Probe: is a 32-byte fp32 reduction cheaper as ONE bulk async reduce
// (cp.reduce.async.bulk .add.f32 from shared memory) than as two red.v4?
// Random 32-byte-aligned chunks in a buffer of `mb` MiB; each thread does
// `per` chunks.  Prints G chunks/s for: 2 x red.global.add.v4.f32,
// 1 x red.v4 (16 B, half the payload: the op-rate reference), and the bulk form.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

__global__ void red2v4(float *buf, uint32_t nchunks, int per, uint32_t seed) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    for (int k = 0; k < per; k++) {
        const uint32_t c = hsh(t * 977u + k * 131071u + seed) % nchunks;
        float *p = buf + (size_t)c * 8;
        atomicAdd(reinterpret_cast<float4 *>(p), make_float4(1.f, 1.f, 1.f, 1.f));
        atomicAdd(reinterpret_cast<float4 *>(p + 4), make_float4(1.f, 1.f, 1.f, 1.f));
    }
}
__global__ void red1v4(float *buf, uint32_t nchunks, int per, uint32_t seed) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    for (int k = 0; k < per; k++) {
        const uint32_t c = hsh(t * 977u + k * 131071u + seed) % nchunks;
        atomicAdd(reinterpret_cast<float4 *>(buf + (size_t)c * 8), make_float4(1.f, 1.f, 1.f, 1.f));
    }
}
// each thread owns a 32-byte smem slot per in-flight op (DEPTH slots)
template <int DEPTH>
__global__ void bulkred(float *buf, uint32_t nchunks, int per, uint32_t seed) {
    __shared__ __align__(128) float slot[256][DEPTH][8];
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    for (int d = 0; d < DEPTH; d++)
        for (int j = 0; j < 8; j++) slot[threadIdx.x][d][j] = 1.f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int k = 0; k < per; k++) {
        const int d = k % DEPTH;
        if (k >= DEPTH) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(DEPTH - 1) : "memory");
        const uint32_t c = hsh(t * 977u + k * 131071u + seed) % nchunks;
        const uint32_t s = (uint32_t)__cvta_generic_to_shared(&slot[threadIdx.x][d][0]);
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 32;"
                     ::"l"(buf + (size_t)c * 8), "r"(s) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    for (int mb : {48, 64, 512}) {
        const uint32_t nchunks = (uint32_t)((size_t)mb * 1048576 / 32);
        float *buf;
        cudaMalloc(&buf, (size_t)mb * 1048576);
        cudaMemset(buf, 0, (size_t)mb * 1048576);
        const int blocks = 148 * 8, threads = 256, per = 64;
        const double n = (double)blocks * threads * per;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        auto run = [&](const char *name, auto launch) {
            launch(0u);
            cudaEventRecord(e0);
            for (int r = 0; r < 5; r++) launch(r + 1u);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("%4d MiB %-14s %8.2f G chunks/s  (%s)\n", mb, name, 5 * n / (ms * 1e-3) / 1e9,
                   cudaGetErrorString(cudaGetLastError()));
        };
        run("2x red.v4", [&](uint32_t s) { red2v4<<<blocks, threads>>>(buf, nchunks, per, s); });
        run("1x red.v4", [&](uint32_t s) { red1v4<<<blocks, threads>>>(buf, nchunks, per, s); });
        run("bulk32 d4", [&](uint32_t s) { bulkred<4><<<blocks, threads>>>(buf, nchunks, per, s); });
        run("bulk32 d2", [&](uint32_t s) { bulkred<2><<<blocks, threads>>>(buf, nchunks, per, s); });
        cudaFree(buf);
    }
    return 0;
}
