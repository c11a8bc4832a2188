// Probe: L2 reduction rate when every red.v4 is issued from an SM on the
// die that homes its address (4 KB-granular home map measured by atomic
// latency) vs from any SM.  Random 16-byte targets in a `mib` MiB buffer.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o die_red die_red.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}
__device__ __forceinline__ int smid() { int s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s)); return s; }
__device__ __forceinline__ uint32_t lat_atomic(unsigned *p, unsigned &acc) {
    long long t0 = clock64();
    unsigned v = atomicAdd(p, 1u);
    unsigned w;
    asm volatile("add.u32 %0, %1, 1;" : "=r"(w) : "r"(v));
    acc += w;
    long long t1 = clock64();
    asm volatile("" :: "r"(acc));
    return (uint32_t)(t1 - t0);
}
// every SM: latency to the first 64 chunks (for clustering SMs by die)
__global__ void sm_probe(unsigned *buf, uint32_t *lat, int *sm) {
    if (threadIdx.x) return;
    sm[blockIdx.x] = smid();
    unsigned acc = 0;
    for (int i = 0; i < 64; i++) {
        uint32_t b = 0xffffffffu;
        for (int r = 0; r < 3; r++) { uint32_t d = lat_atomic(buf + (size_t)i * 1024, acc); b = d < b ? d : b; }
        lat[blockIdx.x * 64 + i] = b;
    }
    if (acc == 0x12345678u) sm[0] = -1;
}
// chunks' home die, measured from die-0 SMs only
__global__ void chunk_probe(unsigned *buf, const int *die_of_sm, int nchunk, uint8_t *home, int *ctr) {
    if (die_of_sm[smid()] != 0 || threadIdx.x != 0) return;
    unsigned acc = 0;
    for (;;) {
        int c = atomicAdd(ctr, 1);
        if (c >= nchunk) break;
        uint32_t b = 0xffffffffu;
        for (int r = 0; r < 2; r++) { uint32_t d = lat_atomic(buf + (size_t)c * 1024, acc); b = d < b ? d : b; }
        home[c] = b < 450 ? 0 : 1;
    }
    if (acc == 0x12345678u) home[0] = 7;
}
__global__ void red_all(float *buf, uint32_t nslot, int per, uint32_t seed) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    for (int k = 0; k < per; k++) {
        const uint32_t c = hsh(t * 977u + k * 131071u + seed) % nslot;
        atomicAdd(reinterpret_cast<float4 *>(buf + (size_t)c * 4), make_float4(1.f, 1.f, 1.f, 1.f));
    }
}
// same candidate stream per thread pair-of-dies: each thread draws 2 per
// candidates and issues those homed on its own die (half in expectation)
__global__ void red_die(float *buf, uint32_t nslot, int per, uint32_t seed, const int *die_of_sm,
                        const uint8_t *home) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    const int d = die_of_sm[smid()];
    for (int k = 0; k < 2 * per; k++) {
        const uint32_t c = hsh(t * 977u + k * 131071u + seed) % nslot;
        if (__ldg(home + (c >> 8)) == d)
            atomicAdd(reinterpret_cast<float4 *>(buf + (size_t)c * 4), make_float4(1.f, 1.f, 1.f, 1.f));
    }
}

int main(int argc, char **argv) {
    const size_t mib = argc > 1 ? atoi(argv[1]) : 64;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    float *buf;
    const size_t bytes = mib << 20;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 0, bytes);
    uint32_t *lat; int *sm;
    cudaMalloc(&lat, nsm * 64 * 4); cudaMalloc(&sm, nsm * 4);
    sm_probe<<<nsm, 32>>>(reinterpret_cast<unsigned *>(buf), lat, sm);
    std::vector<uint32_t> hl(nsm * 64); std::vector<int> hs(nsm);
    cudaMemcpy(hl.data(), lat, hl.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(hs.data(), sm, nsm * 4, cudaMemcpyDeviceToHost);
    std::vector<int> die(nsm, 0);
    int n1 = 0;
    for (int b = 0; b < nsm; b++) {
        int agree = 0;
        for (int i = 0; i < 64; i++) agree += ((hl[b * 64 + i] < 450) == (hl[0 * 64 + i] < 450));
        die[hs[b]] = agree >= 32 ? 0 : 1;
        n1 += die[hs[b]];
    }
    printf("SMs on die 1: %d of %d; die by smid: ", n1, nsm);
    for (int s = 0; s < nsm; s++) printf("%d", die[s]);
    printf("\n");
    int *d_die; cudaMalloc(&d_die, nsm * 4); cudaMemcpy(d_die, die.data(), nsm * 4, cudaMemcpyHostToDevice);
    const int nchunk = (int)(bytes >> 12);
    uint8_t *home; int *ctr;
    cudaMalloc(&home, nchunk); cudaMalloc(&ctr, 4); cudaMemset(ctr, 0, 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    chunk_probe<<<nsm, 64>>>(reinterpret_cast<unsigned *>(buf), d_die, nchunk, home, ctr);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    std::vector<uint8_t> hh(nchunk); cudaMemcpy(hh.data(), home, nchunk, cudaMemcpyDeviceToHost);
    int h1 = 0; for (auto v : hh) h1 += v;
    printf("chunk map: %d chunks, %d on die 1, %.3f ms\n", nchunk, h1, ms);
    const uint32_t nslot = (uint32_t)(bytes / 16);
    const int threads = 256, blocks = nsm * 8, per = 64;
    const double ops = (double)threads * blocks * per;
    for (int rep = 0; rep < 3; rep++) {
        for (int mode = 0; mode < 2; mode++) {
            cudaEventRecord(e0);
            for (int it = 0; it < 10; it++) {
                if (mode == 0) red_all<<<blocks, threads>>>(buf, nslot, per, 1234u + it);
                else red_die<<<blocks, threads>>>(buf, nslot, per, 1234u + it, d_die, home);
            }
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            printf("%s: %.1f G red.v4/s (%.3f ms per 10 x %.0f M ops)\n", mode ? "die-local" : "any SM   ",
                   10 * ops / (ms * 1e-3) / 1e9, ms, ops / 1e6);
        }
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
