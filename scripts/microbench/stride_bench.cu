// Microbenchmark: K2's access pattern -- one lane per 2048-double block,
// 32-element chunks staged warp-cooperatively -- with blocks at a 16 KB
// stride (as the light / heavy lists are laid out) vs skewed by 256 B per
// block, to see whether the common 16 KB stride concentrates the concurrent
// requests on few HBM channels.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o stride_bench stride_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int BLK = 2048, C = 32;

__global__ void __launch_bounds__(64) k_chunks(const double* __restrict__ src, uint64_t nblocks,
                                               uint64_t stride, double* __restrict__ out) {
    __shared__ double tile[2][2][32][C + 1];
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const uint64_t b0 = (static_cast<uint64_t>(blockIdx.x) * 2 + wq) * 32;
    if (b0 >= nblocks) return;
    double acc = 0;
    for (int c = 0; c < BLK / C; ++c) {
        const int buf = c & 1;
#pragma unroll 4
        for (int r = 0; r < 32; ++r) {
            const double* p = src + (b0 + r) * stride + c * C + lane;
            const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(&tile[wq][buf][r][lane]));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(p));
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
        __syncwarp();
#pragma unroll 8
        for (int e = 0; e < C; ++e) acc += tile[wq][buf][lane][e];
        __syncwarp();
    }
    out[b0 + lane] = acc;
}

int main() {
    const uint64_t nblocks = 48830;
    double *src, *out;
    cudaMalloc(&src, (nblocks * (BLK + 64) + 64) * sizeof(double));
    cudaMalloc(&out, nblocks * sizeof(double));
    cudaMemset(src, 0, (nblocks * (BLK + 64) + 64) * sizeof(double));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (uint64_t skew : {0, 4, 16, 32, 64}) {
        float best = 1e9f;
        for (int r = 0; r < 4; ++r) {
            cudaEventRecord(a);
            k_chunks<<<(nblocks + 63) / 64, 64>>>(src, nblocks, BLK + skew, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r && ms < best) best = ms;
        }
        printf("block stride 2048+%-3llu doubles: %.3f ms  %.0f GB/s\n", (unsigned long long)skew, best,
               nblocks * BLK * 8.0 / best / 1e6);
    }
    return 0;
}
