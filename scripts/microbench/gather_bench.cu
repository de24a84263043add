// Microbenchmark: random 16-B gathers from a table of n buckets (the K5 access
// pattern without the RNG cost), to find the B200's random-access ceiling and
// the effect of cudaLimitMaxL2FetchGranularity.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench gather_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

template <int U>
__global__ void gather(const uint4* __restrict__ t, uint64_t n, uint64_t k, uint32_t* out,
                       uint64_t salt) {
    const uint64_t span = (uint64_t)blockDim.x * U;
    for (uint64_t q0 = (uint64_t)blockIdx.x * span + threadIdx.x; q0 < k;
         q0 += (uint64_t)gridDim.x * span) {
        uint64_t idx[U];
#pragma unroll
        for (int u = 0; u < U; ++u) idx[u] = __umul64hi(mix(salt + q0 + u * blockDim.x), n);
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                         : "l"(t + idx[u]));
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t q = q0 + u * blockDim.x;
            if (q < k) out[q] = v[u].x ^ v[u].w;
        }
    }
}

// sequential copy for reference bandwidth
__global__ void copyk(const uint4* __restrict__ a, uint4* b, uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const uint64_t k = 1ull << 30;
    uint32_t* out;
    cudaMalloc(&out, k * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    uint64_t n = 100000000ull;
    uint4* t;
    cudaMalloc(&t, n * 16);
    cudaMemset(t, 3, n * 16);
    auto run = [&](const char* name, auto launch) {
        float best = 1e30f;
        for (int r = 0; r < 4; ++r) {
            cudaEventRecord(a);
            launch(r);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r && ms < best) best = ms;
        }
        printf("%-40s %.3f ms -> %.1f G/s\n", name, best, k / best / 1e6);
    };
    char buf[128];
    for (int bps : {1, 2, 3, 4, 8}) {
        for (int thr : {128, 256, 512}) {
            snprintf(buf, sizeof buf, "U8 blocks/SM=%d thr=%d", bps, thr);
            run(buf, [&](int r) { gather<8><<<sms * bps, thr>>>(t, n, k, out, r * 777); });
        }
    }
    run("U8 many-ctas 75776x256", [&](int r) { gather<8><<<75776, 256>>>(t, n, k, out, r * 777); });
    run("U8 exact grid k/2048 x256", [&](int r) { gather<8><<<(unsigned)(k / 2048), 256>>>(t, n, k, out, r * 777); });
    run("U4 exact grid k/1024 x256", [&](int r) { gather<4><<<(unsigned)(k / 1024), 256>>>(t, n, k, out, r * 777); });
    run("U16 exact grid x256", [&](int r) { gather<16><<<(unsigned)(k / 4096), 256>>>(t, n, k, out, r * 777); });
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
