// D2H of 4 GB: DMA copy (cudaMemcpyAsync from device to pinned host) vs SM
// stores straight into mapped pinned host memory (zero-copy), 16-B stores.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_store(uint4* __restrict__ dst, const uint4* __restrict__ src, size_t n16) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}
int main() {
    const size_t bytes = 4000000000ull;
    void *h, *d, *hd;
    cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
    cudaHostGetDevicePointer(&hd, h, 0);
    cudaMalloc(&d, bytes);
    cudaMemset(d, 1, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("DMA D2H: %.2f ms (%.1f GB/s)\n", ms, bytes / ms / 1e6);
    }
    for (int blocks : {148, 296, 592, 1184}) for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        k_store<<<blocks, 512>>>((uint4*)hd, (const uint4*)d, bytes / 16);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("SM stores (%d CTAs): %.2f ms (%.1f GB/s) %s\n", blocks, ms, bytes / ms / 1e6,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
