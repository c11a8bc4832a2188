// Launch-overhead probe for the fused inference kernel's shape: how long a
// near-empty kernel of 128 CTAs x 384 threads lasts (ncu gpu__time_duration
// and back-to-back event timing) with / without 60 KB of dynamic shared
// memory, TMEM alloc/dealloc and a 1 KB __grid_constant__ parameter block.
// nvcc -gencode arch=compute_100a,code=sm_100a -o launch_overhead launch_overhead.cu
#include <cstdio>
#include <cuda_runtime.h>
struct Big { unsigned v[320]; };
struct Big2 { unsigned v[514]; };
__global__ void k_plain(float *out) { if (threadIdx.x == 0 && blockIdx.x == 1000) out[0] = 1.f; }
__global__ void k_smem(float *out) {
    extern __shared__ float sm[];
    sm[threadIdx.x] = threadIdx.x;
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 1000) out[0] = sm[5];
}
__global__ void k_tmem(float *out, const __grid_constant__ Big b) {
    extern __shared__ float sm[];
    __shared__ unsigned tb;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"((unsigned)__cvta_generic_to_shared(&tb)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    sm[threadIdx.x] = b.v[threadIdx.x % 320];
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tb));
    if (threadIdx.x == 0 && blockIdx.x == 1000) out[0] = sm[5];
}
__global__ void k_tmem_only(float *out) {
    extern __shared__ float sm[];
    __shared__ unsigned tb;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"((unsigned)__cvta_generic_to_shared(&tb)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    sm[threadIdx.x] = threadIdx.x;
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tb));
    if (threadIdx.x == 0 && blockIdx.x == 1000) out[0] = sm[5];
}
__global__ void k_param_only(float *out, const __grid_constant__ Big b) {
    extern __shared__ float sm[];
    sm[threadIdx.x] = b.v[threadIdx.x % 320];
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 1000) out[0] = sm[5];
}
__global__ void k_param2k(float *out, const __grid_constant__ Big2 b) {
    extern __shared__ float sm[];
    sm[threadIdx.x] = b.v[threadIdx.x % 256];
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 1000) out[0] = sm[5];
}
__global__ void k_gload1k(float *out, const unsigned *g) {
    extern __shared__ float sm[];
    sm[threadIdx.x] = g[threadIdx.x % 256];
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 1000) out[0] = sm[5];
}
int main() {
    float *d; cudaMalloc(&d, 4);
    const int smem = 60 * 1024;
    cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_tmem, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_tmem_only, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_param_only, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_param2k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_gload1k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    Big2 b2{};
    unsigned *g; cudaMalloc(&g, 4096); cudaMemset(g, 0, 4096);
    Big b{};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int which = 0; which < 7; which++) {
        for (int rep = 0; rep < 2; rep++) {
            const int n = 2000;
            cudaEventRecord(e0);
            for (int i = 0; i < n; i++) {
                if (which == 0) k_plain<<<128, 384>>>(d);
                else if (which == 1) k_smem<<<128, 384, smem>>>(d);
                else if (which == 2) k_tmem<<<128, 384, smem>>>(d, b);
                else if (which == 3) k_tmem_only<<<128, 384, smem>>>(d);
                else if (which == 4) k_param_only<<<128, 384, smem>>>(d, b);
                else if (which == 5) k_param2k<<<128, 384, smem>>>(d, b2);
                else k_gload1k<<<128, 384, smem>>>(d, g);
            }
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (rep) printf("%s: %.2f us per launch back to back\n", which == 0 ? "plain" : which == 1 ? "smem60K" : which == 2 ? "smem60K+tmem+1KBparam" : which == 3 ? "smem60K+tmem" : which == 4 ? "smem60K+1KBparam" : which == 5 ? "smem60K+2KBparam" : "smem60K+global 1KB load", ms * 1e3 / n);
        }
    }
    return 0;
}
