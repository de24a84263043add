// Microbenchmark: random 16-B gathers from a table of n buckets with the K5
// bucket-index formula, comparing load flavours (L1/L2 caching behaviour
// decides how many 32-B sectors each 16-B gather pulls from HBM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o gather_bench gather_bench.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
constexpr uint64_t G = 0x9e3779b97f4a7c15ull;

template <int V>
__device__ __forceinline__ uint4 ld(const uint4* p) {
    uint4 v;
    if (V == 0)
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    else if (V == 1)
        asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    else if (V == 2)
        asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    else if (V == 3)
        asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    else if (V == 4)
        asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    else
        asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

template <int V, int U>
__global__ void gather(const uint4* __restrict__ t, uint64_t n, uint64_t k, uint32_t* out,
                       uint64_t key) {
    const uint64_t span = (uint64_t)blockDim.x * U;
    for (uint64_t q0 = (uint64_t)blockIdx.x * span + threadIdx.x; q0 < k;
         q0 += (uint64_t)gridDim.x * span) {
        uint64_t idx[U];
#pragma unroll
        for (int u = 0; u < U; ++u) idx[u] = __umul64hi(mix(key + (2 * (q0 + u * blockDim.x) + 1) * G), n);
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ld<V>(t + idx[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t q = q0 + u * blockDim.x;
            if (q < k) out[q] = v[u].x ^ v[u].w;
        }
    }
}

int main() {
    const uint64_t k = 1ull << 30;
    uint32_t* out;
    cudaMalloc(&out, k * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char* name, auto launch) {
        float best = 1e30f;
        const int reps = getenv("ONCE") ? 1 : 4;
        for (int r = 0; r < reps; ++r) {
            cudaEventRecord(a);
            launch(r);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if ((r || reps == 1) && ms < best) best = ms;
        }
        printf("%-44s %8.3f ms -> %6.1f G/s\n", name, best, k / best / 1e6);
    };
    const unsigned grid = (unsigned)(k / 2048);
    for (uint64_t n : {1ull << 20, 100000000ull, 1000000000ull}) {
        uint4* t;
        if (cudaMalloc(&t, n * 16) != cudaSuccess) continue;
        cudaMemset(t, 3, n * 16);
        char buf[128];
#define V(X, NAME)                                                                         \
    snprintf(buf, sizeof buf, "n=%llu %s", (unsigned long long)n, NAME);                   \
    run(buf, [&](int r) { gather<X, 8><<<grid, 256>>>(t, n, k, out, 0x1234567ull * (r + 1)); });
        V(0, "ld.nc.L1::no_allocate")
        V(1, "ld.cg")
        V(2, "ld (default)")
        V(3, "ld.cs")
        V(4, "ld.nc")
        V(5, "ld.cv")
        cudaFree(t);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
