// Microbenchmark: random 16-B row gathers from an L2-resident 32 MB table,
// LDG (one lane per row) vs TMA tile::gather4 (4 rows per instruction).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_gather_bench tma_gather_bench.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t hash32(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return static_cast<uint32_t>(z ^ (z >> 31));
}

__global__ void k_ldg(const uint4* __restrict__ t, uint32_t n, uint64_t k, uint32_t* out) {
    for (uint64_t q = blockIdx.x * 256ull * 8 + threadIdx.x; q < k; q += gridDim.x * 256ull * 8) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t r = __umulhi(hash32(q + u * 256), n);
            asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(t + r));
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) out[q + u * 256] = v[u].x ^ v[u].w;
    }
}

constexpr int BATCH = 1024;  // rows per CTA batch

__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n"
        ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(phase));
}

template <int ISSUERS>
__global__ void k_tma(const __grid_constant__ CUtensorMap tmap, uint32_t n, uint64_t k, uint32_t* out) {
    __shared__ __align__(128) uint4 buf[BATCH * 2];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    unsigned phase = 0;
    for (uint64_t b0 = blockIdx.x * (uint64_t)BATCH; b0 < k; b0 += gridDim.x * (uint64_t)BATCH) {
        if (threadIdx.x == 0) mbar_expect(&bar, BATCH * 16);
        __syncthreads();
        if (threadIdx.x < ISSUERS) {
            for (int g = threadIdx.x; g < BATCH / 4; g += ISSUERS) {
                int r[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) r[u] = (int)__umulhi(hash32(b0 + g * 4 + u), n);
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes "
                    "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                    ::"r"((unsigned)__cvta_generic_to_shared(&buf[g * 8])), "l"(&tmap), "r"(0), "r"(r[0]),
                      "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"((unsigned)__cvta_generic_to_shared(&bar))
                    : "memory");
            }
        }
        mbar_wait(&bar, phase);
        phase ^= 1;
        for (int i = threadIdx.x; i < BATCH; i += blockDim.x) out[b0 + i] = buf[(i / 4) * 8 + (i % 4)].x ^ buf[(i / 4) * 8 + (i % 4)].w;
        __syncthreads();
    }
}

// Mixed: warp 0 gathers the first TMA_ROWS of each batch with TMA gather4
// (lane 0 issues), the other warps gather the rest with LDGSTS -- do the two
// paths add up?
template <int TMA_ROWS>
__global__ void k_mixed(const __grid_constant__ CUtensorMap tmap, const uint4* __restrict__ t, uint32_t n,
                        uint64_t k, uint32_t* out) {
    __shared__ __align__(128) uint4 buf[BATCH * 2];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    unsigned phase = 0;
    for (uint64_t b0 = blockIdx.x * (uint64_t)BATCH; b0 < k; b0 += gridDim.x * (uint64_t)BATCH) {
        if (threadIdx.x == 0) mbar_expect(&bar, TMA_ROWS * 16);
        __syncthreads();
        if (threadIdx.x < 32) {
            for (int g = threadIdx.x; g < TMA_ROWS / 4; g += 32) {
                int r[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) r[u] = (int)__umulhi(hash32(b0 + g * 4 + u), n);
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes "
                    "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                    ::"r"((unsigned)__cvta_generic_to_shared(&buf[g * 8])), "l"(&tmap), "r"(0), "r"(r[0]),
                      "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"((unsigned)__cvta_generic_to_shared(&bar))
                    : "memory");
            }
        } else {
            for (int i = TMA_ROWS + threadIdx.x - 32; i < BATCH; i += blockDim.x - 32) {
                const uint32_t r = __umulhi(hash32(b0 + i), n);
                const unsigned s = (unsigned)__cvta_generic_to_shared(&buf[(i / 4) * 8 + (i % 4)]);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(t + r));
            }
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
        }
        mbar_wait(&bar, phase);
        phase ^= 1;
        __syncthreads();
        for (int i = threadIdx.x; i < BATCH; i += blockDim.x) out[b0 + i] = buf[(i / 4) * 8 + (i % 4)].x ^ buf[(i / 4) * 8 + (i % 4)].w;
        __syncthreads();
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const uint32_t n = 1u << 21;  // 32 MB table
    const uint64_t k = 1ull << 28;
    uint4* t;
    uint32_t* out;
    cudaMalloc(&t, (size_t)n * 16);
    cudaMalloc(&out, k * 4);
    cudaMemset(t, 7, (size_t)n * 16);
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult qr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &qr);
    CUtensorMap tm;
    cuuint64_t dims[2] = {4, n};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {4, 1};
    cuuint32_t estr[2] = {1, 1};
    CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, t, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode: %d\n", (int)cr);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto time = [&](const char* name, auto fn) {
        float best = 1e30f;
        for (int r = 0; r < 4; ++r) {
            cudaEventRecord(a);
            fn();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r && ms < best) best = ms;
        }
        printf("%-28s %8.3f ms  %7.1f G rows/s  (%s)\n", name, best, k / best / 1e6,
               cudaGetErrorString(cudaGetLastError()));
    };
    time("ldg", [&] { k_ldg<<<sms * 8, 256>>>(t, n, k, out); });
    uint32_t ref0;
    cudaMemcpy(&ref0, out + 12345, 4, cudaMemcpyDeviceToHost);
    time("tma gather4 x1 issuer", [&] { k_tma<1><<<sms * 6, 128>>>(tm, n, k, out); });
    time("tma gather4 x32 issuers", [&] { k_tma<32><<<sms * 6, 128>>>(tm, n, k, out); });
    time("tma gather4 x128 issuers", [&] { k_tma<128><<<sms * 6, 128>>>(tm, n, k, out); });
    time("ldgsts only (mixed<0>)", [&] { k_mixed<0><<<sms * 6, 256>>>(tm, t, n, k, out); });
    time("mixed 256 tma / 768 ldgsts", [&] { k_mixed<256><<<sms * 6, 256>>>(tm, t, n, k, out); });
    time("mixed 384 tma / 640 ldgsts", [&] { k_mixed<384><<<sms * 6, 256>>>(tm, t, n, k, out); });
    time("mixed 512 tma / 512 ldgsts", [&] { k_mixed<512><<<sms * 6, 256>>>(tm, t, n, k, out); });
    uint32_t v0;
    cudaMemcpy(&v0, out + 12345, 4, cudaMemcpyDeviceToHost);
    printf("check %u %u\n", ref0, v0);
    return 0;
}
