// Microbenchmark: random 16-B gathers from an L2-resident 32 MB table with the
// indices streamed from HBM (the shape of k_region_gather), comparing the
// load paths: LDG through L1, LDG bypassing L1, and LDGSTS (cp.async) into
// shared memory.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o l2_gather_bench l2_gather_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return static_cast<uint32_t>(z ^ (z >> 31));
}

__global__ void k_idx(uint32_t* idx, uint64_t k, uint32_t n) {
    for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < k; i += gridDim.x * 256ull)
        idx[i] = __umulhi(hash32(i), n);
}

template <int V, int U>
__global__ void __launch_bounds__(256) k_ldg(const uint4* __restrict__ t, const uint32_t* __restrict__ idx,
                                             uint64_t k, uint32_t* __restrict__ out) {
    const uint64_t p0 = static_cast<uint64_t>(blockIdx.x) * (256 * U) + threadIdx.x;
    uint32_t r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = idx[p0 + u * 256];
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        if (V == 0)
            asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(t + r[u]));
        else if (V == 1)
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(t + r[u]));
        else
            asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(t + r[u]));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) out[p0 + u * 256] = v[u].x ^ v[u].w;
}

template <int U, bool CA = false>
__global__ void __launch_bounds__(256) k_ldgsts(const uint4* __restrict__ t, const uint32_t* __restrict__ idx,
                                                uint64_t k, uint32_t* __restrict__ out) {
    __shared__ uint4 buf[256 * U];
    const uint64_t p0 = static_cast<uint64_t>(blockIdx.x) * (256 * U) + threadIdx.x;
    uint32_t r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = idx[p0 + u * 256];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(&buf[u * 256 + threadIdx.x]));
        if (CA)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(s), "l"(t + r[u]));
        else
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(t + r[u]));
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const uint4 v = buf[u * 256 + threadIdx.x];
        out[p0 + u * 256] = v.x ^ v.w;
    }
}

// texture path: int4 texels through the TEX pipe (tex1Dfetch on a linear buffer)
template <int U>
__global__ void __launch_bounds__(256) k_tex(cudaTextureObject_t tex, const uint32_t* __restrict__ idx,
                                             uint64_t k, uint32_t* __restrict__ out) {
    const uint64_t p0 = static_cast<uint64_t>(blockIdx.x) * (256 * U) + threadIdx.x;
    uint32_t r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = idx[p0 + u * 256];
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = tex1Dfetch<int4>(tex, static_cast<int>(r[u]));
#pragma unroll
    for (int u = 0; u < U; ++u) out[p0 + u * 256] = static_cast<uint32_t>(v[u].x ^ v[u].w);
}

// half the rows through LDGSTS, half through the TEX pipe
template <int U>
__global__ void __launch_bounds__(256) k_mix_tex(cudaTextureObject_t tex, const uint4* __restrict__ t,
                                                 const uint32_t* __restrict__ idx, uint64_t k,
                                                 uint32_t* __restrict__ out) {
    __shared__ uint4 buf[256 * U];
    const uint64_t p0 = static_cast<uint64_t>(blockIdx.x) * (256 * U * 2) + threadIdx.x;
    uint32_t r[U], q[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        r[u] = idx[p0 + u * 256];
        q[u] = idx[p0 + (U + u) * 256];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(&buf[u * 256 + threadIdx.x]));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(t + r[u]));
    }
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = tex1Dfetch<int4>(tex, static_cast<int>(q[u]));
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const uint4 a = buf[u * 256 + threadIdx.x];
        out[p0 + u * 256] = a.x ^ a.w;
        out[p0 + (U + u) * 256] = static_cast<uint32_t>(v[u].x ^ v[u].w);
    }
}

int main() {
    const uint32_t n = 1u << 21;  // 32 MB table
    const uint64_t k = 1ull << 28;
    uint4* t;
    uint32_t *idx, *out;
    cudaMalloc(&t, (size_t)n * 16);
    cudaMalloc(&idx, k * 4);
    cudaMalloc(&out, k * 4);
    cudaMemset(t, 7, (size_t)n * 16);
    k_idx<<<148 * 16, 256>>>(idx, k, n);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto time = [&](const char* name, auto fn) {
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a);
            fn();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r && ms < best) best = ms;
        }
        printf("%-32s %8.3f ms  %7.1f G rows/s  (%s)\n", name, best, k / best / 1e6,
               cudaGetErrorString(cudaGetLastError()));
    };
    time("ldg.nc U8", [&] { k_ldg<0, 8><<<k / 2048, 256>>>(t, idx, k, out); });
    time("ldg.nc U16", [&] { k_ldg<0, 16><<<k / 4096, 256>>>(t, idx, k, out); });
    time("ldg.nc.L1::no_allocate U8", [&] { k_ldg<1, 8><<<k / 2048, 256>>>(t, idx, k, out); });
    time("ldg.cg U8", [&] { k_ldg<2, 8><<<k / 2048, 256>>>(t, idx, k, out); });
    time("ldgsts.cg U8", [&] { k_ldgsts<8><<<k / 2048, 256>>>(t, idx, k, out); });
    cudaResourceDesc rd{};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = t;
    rd.res.linear.desc = cudaCreateChannelDesc<int4>();
    rd.res.linear.sizeInBytes = (size_t)n * 16;
    cudaTextureDesc td{};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tex = 0;
    printf("tex create: %s\n", cudaGetErrorString(cudaCreateTextureObject(&tex, &rd, &td, nullptr)));
    time("tex1Dfetch int4 U8", [&] { k_tex<8><<<k / 2048, 256>>>(tex, idx, k, out); });
    time("tex1Dfetch int4 U16", [&] { k_tex<16><<<k / 4096, 256>>>(tex, idx, k, out); });
    time("mix ldgsts+tex U4+U4", [&] { k_mix_tex<4><<<k / 2048, 256>>>(tex, t, idx, k, out); });
    time("ldgsts.ca U8", [&] { k_ldgsts<8, true><<<k / 2048, 256>>>(t, idx, k, out); });
    time("ldgsts.cg U4", [&] { k_ldgsts<4><<<k / 1024, 256>>>(t, idx, k, out); });
    time("ldgsts.cg U12", [&] { k_ldgsts<12><<<k / 3072, 256>>>(t, idx, k, out); });
    return 0;
}
