// Microbenchmark: random 16-B row gathers from a table spread over the
// shared memory of a thread-block cluster (distributed shared memory), to
// see whether a cluster-resident table slice beats the ~240 G rows/s the L2
// random-access path delivers (l2_gather_bench.cu).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o dsmem_gather_bench dsmem_gather_bench.cu
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t hash32(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return static_cast<uint32_t>(z ^ (z >> 31));
}

template <int CL, int ROWS_PER_CTA>
__global__ void __launch_bounds__(512) k_dsmem(uint64_t iters, uint32_t* out) {
    extern __shared__ __align__(16) uint4 rows[];
    cg::cluster_group cluster = cg::this_cluster();
    for (int i = threadIdx.x; i < ROWS_PER_CTA; i += blockDim.x)
        rows[i] = make_uint4(i, blockIdx.x, 1, 2);
    cluster.sync();
    uint32_t acc = 0;
    const uint64_t base = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * iters;
    for (uint64_t it = 0; it < iters; it += 8) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t h = hash32(base + it + u);
            const uint32_t rank = h % CL;
            const uint32_t row = (h >> 8) % ROWS_PER_CTA;
            const uint4* remote = cluster.map_shared_rank(rows, rank);
            v[u] = remote[row];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].w;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    cluster.sync();
}

template <int CL>
void run(int sms) {
    constexpr int ROWS = 8192;  // 128 KB per CTA
    const size_t smem = ROWS * 16;
    auto k = k_dsmem<CL, ROWS>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (CL > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    const int ctas = (sms / CL) * CL;
    uint32_t* out;
    cudaMalloc(&out, ctas * 512 * 4);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const uint64_t iters = 4096;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9f;
    for (int r = 0; r < 4; ++r) {
        cudaEventRecord(a);
        cudaError_t e = cudaLaunchKernelEx(&cfg, k, iters, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        if (e != cudaSuccess) {
            printf("cluster %d: launch %s\n", CL, cudaGetErrorString(e));
            return;
        }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r && ms < best) best = ms;
    }
    const double rows = static_cast<double>(ctas) * 512 * iters;
    printf("cluster %2d (%3d CTAs, %d KB per CTA): %.3f ms  %.1f G rows/s  (%s)\n", CL, ctas,
           static_cast<int>(smem >> 10), best, rows / best / 1e6, cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main() {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<1>(sms);
    run<2>(sms);
    run<4>(sms);
    run<8>(sms);
    run<16>(sms);
    return 0;
}
