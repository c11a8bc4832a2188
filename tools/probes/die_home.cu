// Probe: which L2 half (die) is the home of each address?  One thread per
// CTA (one CTA per SM) times a returning atomicAdd to each probe address
// (min over reps); an SM on the address's home die sees the short latency,
// the others the fabric round trip.  Writes smid[grid] and lat[grid][n] to
// the output file for offline clustering.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o die_home die_home.cu
//   ./die_home out.bin [mib]
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__global__ void probe(unsigned *buf, const uint64_t *offs, int n, uint32_t *lat, int *smid, int reps) {
    if (threadIdx.x != 0) return;
    int sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    smid[blockIdx.x] = sm;
    unsigned acc = 0;
    for (int i = 0; i < n; i++) {
        unsigned *p = reinterpret_cast<unsigned *>(reinterpret_cast<char *>(buf) + offs[i]);
        uint32_t best = 0xffffffffu;
        for (int r = 0; r < reps; r++) {
            long long t0 = clock64();
            unsigned v = atomicAdd(p, 1u);
            unsigned w;
            asm volatile("add.u32 %0, %1, 1;" : "=r"(w) : "r"(v));
            acc += w;
            long long t1 = clock64();
            asm volatile("" :: "r"(acc));
            const uint32_t d = (uint32_t)(t1 - t0);
            best = d < best ? d : best;
        }
        lat[(size_t)blockIdx.x * n + i] = best;
    }
    if (acc == 0x12345678u) smid[0] = -1;
}

int main(int argc, char **argv) {
    const char *outp = argc > 1 ? argv[1] : "die_home.bin";
    const size_t mib = argc > 2 ? atoi(argv[2]) : 64;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    unsigned *buf;
    cudaMalloc(&buf, mib << 20);
    cudaMemset(buf, 0, mib << 20);
    std::vector<uint64_t> offs;
    for (int i = 0; i < 4096; i++) offs.push_back((uint64_t)i * 32);                 // 128 KB at 32 B
    for (int i = 0; i < 4096; i++) offs.push_back((uint64_t)i * ((mib << 20) / 4096)); // whole buffer
    const int n = (int)offs.size();
    uint64_t *d_offs;
    cudaMalloc(&d_offs, n * 8);
    cudaMemcpy(d_offs, offs.data(), n * 8, cudaMemcpyHostToDevice);
    const int grid = nsm;
    uint32_t *lat;
    int *smid;
    cudaMalloc(&lat, (size_t)grid * n * 4);
    cudaMalloc(&smid, grid * 4);
    probe<<<grid, 32>>>(buf, d_offs, n, lat, smid, 3);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<uint32_t> h((size_t)grid * n);
    std::vector<int> hs(grid);
    cudaMemcpy(h.data(), lat, h.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(hs.data(), smid, grid * 4, cudaMemcpyDeviceToHost);
    FILE *f = fopen(outp, "wb");
    int hdr[2] = {grid, n};
    fwrite(hdr, 4, 2, f);
    fwrite(hs.data(), 4, grid, f);
    fwrite(offs.data(), 8, n, f);
    fwrite(h.data(), 4, h.size(), f);
    fclose(f);
    printf("grid %d n %d buf %p\n", grid, n, (void *)buf);
    return 0;
}
