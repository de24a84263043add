// paper_1903_00227_b200/csrc/sample_kernels.cu -- K5, bulk alias sampling,
// plus the on-device uniform weight generator.
//
// K5 reproduces AliasTable::sample_many (alias.hpp:274-284) exactly: worker w
// of W owns the contiguous output slice worker_slice(k, W, w)
// (parallel.hpp:37-43) and draws it from RngStream(seed, 'alia').derive(w);
// query m of a slice consumes outputs 2m+1 (bucket via the 128-bit
// multiply-shift, rng.hpp:63-66) and 2m+2 (coin, rng.hpp:53-55) of that
// counter stream, then returns ia[x >= share] (alias.hpp:265-269).  Because
// the stream is counter-based every output position is computable on its own,
// so the GPU assigns positions to threads freely and still matches the
// reference bit for bit.
//
// Memory behaviour: one random 16-B bucket gather (one 32-B sector) plus one
// coalesced 4-B store per sample.  Each thread keeps kUnroll independent
// gathers in flight; outputs are written warp-contiguous.
#include "common.cuh"
#include "engine.h"

namespace wrsb {

constexpr int K5_THREADS = 256;
constexpr int K5_UNROLL = 8;

__device__ __forceinline__ uint4 ld_bucket(const Bucket* b, uint64_t i) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(b + i));
    return v;
}

struct SliceCursor {
    uint64_t per, rem, big;  // per = k/W, rem = k%W, big = rem*(per+1)
    __device__ __forceinline__ uint32_t worker_of(uint64_t q) const {
        return q < big ? static_cast<uint32_t>(q / (per + 1))
                       : static_cast<uint32_t>(rem + (q - big) / per);
    }
    __device__ __forceinline__ uint64_t lo_of(uint32_t w) const {
        return per * w + (w < rem ? w : rem);
    }
};

__global__ void __launch_bounds__(K5_THREADS)
k_sample(const Bucket* __restrict__ b, uint64_t n, double wn, uint64_t base_key, uint64_t k,
         uint32_t W, uint64_t q_begin, uint64_t q_end, uint32_t out_base,
         uint32_t* __restrict__ out) {
    const SliceCursor sl{k / W, k % W, (k % W) * (k / W + 1)};
    const uint64_t span = static_cast<uint64_t>(K5_THREADS) * K5_UNROLL;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * span;
    out -= q_begin;  // out[q] for q in [q_begin, q_end)
    for (uint64_t q0 = q_begin + static_cast<uint64_t>(blockIdx.x) * span + threadIdx.x;
         q0 < q_end; q0 += stride) {
        // worker of the first query; later ones advance past slice ends
        uint32_t w = sl.worker_of(q0);
        uint64_t lo = sl.lo_of(w);
        uint64_t hi = lo + sl.per + (w < sl.rem ? 1 : 0);
        uint64_t key = rng_derive(base_key, w);
        uint64_t bidx[K5_UNROLL];
        double x[K5_UNROLL];
#pragma unroll
        for (int u = 0; u < K5_UNROLL; ++u) {
            const uint64_t q = q0 + static_cast<uint64_t>(u) * K5_THREADS;
            if (q < q_end) {
                while (q >= hi) {
                    ++w;
                    lo = hi;
                    hi = lo + sl.per + (w < sl.rem ? 1 : 0);
                    key = rng_derive(base_key, w);
                }
                const uint64_t m = q - lo;
                const uint64_t r1 = mix64(key + (2 * m + 1) * kGolden);
                const uint64_t r2 = mix64(key + (2 * m + 2) * kGolden);
                bidx[u] = __umul64hi(r1, n);                              // bounded(n)
                x[u] = (static_cast<double>(r2 >> 11) * 0x1.0p-53) * wn;  // uniform01()*wn
            } else {
                bidx[u] = 0;
                x[u] = 0.0;
            }
        }
        uint4 bk[K5_UNROLL];
#pragma unroll
        for (int u = 0; u < K5_UNROLL; ++u) bk[u] = ld_bucket(b, bidx[u]);
#pragma unroll
        for (int u = 0; u < K5_UNROLL; ++u) {
            const uint64_t q = q0 + static_cast<uint64_t>(u) * K5_THREADS;
            if (q < q_end) {
                const double share = __hiloint2double(static_cast<int>(bk[u].y),
                                                      static_cast<int>(bk[u].x));
                out[q] = (x[u] >= share ? bk[u].w : bk[u].z) + out_base;
            }
        }
    }
}

__global__ void k_generate_uniform(double* __restrict__ w, uint64_t n, uint64_t offset,
                                   uint64_t key) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += stride) {
        // global item offset+i is output offset+i+1 of the stream
        const uint64_t r = mix64(key + (offset + i + 1) * kGolden);
        w[i] = 1.0 - static_cast<double>(r >> 11) * 0x1.0p-53;  // weight_file.hpp:36
    }
}

static int sm_count() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

cudaError_t launch_sample(const Bucket* d_b, uint64_t n, double wn, uint64_t seed,
                          uint64_t stream_id, uint64_t q_begin, uint64_t q_end, uint64_t k,
                          uint32_t workers, uint32_t base, uint32_t* d_out, cudaStream_t st) {
    if (q_end <= q_begin) return cudaSuccess;
    if (workers == 0) workers = 1;
    const uint64_t span = static_cast<uint64_t>(K5_THREADS) * K5_UNROLL;
    uint64_t blocks = (q_end - q_begin + span - 1) / span;
    const uint64_t cap = static_cast<uint64_t>(sm_count()) * 8 * 64;  // grid-stride beyond this
    if (blocks > cap) blocks = cap;
    k_sample<<<static_cast<unsigned>(blocks), K5_THREADS, 0, st>>>(
        d_b, n, wn, rng_key(seed, stream_id), k, workers, q_begin, q_end, base, d_out);
    return cudaGetLastError();
}

cudaError_t launch_generate_uniform(double* d_w, uint64_t n, uint64_t offset, uint64_t seed,
                                    cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    uint64_t blocks = (n + 255) / 256;
    const uint64_t cap = static_cast<uint64_t>(sm_count()) * 16;
    if (blocks > cap) blocks = cap;
    k_generate_uniform<<<static_cast<unsigned>(blocks), 256, 0, st>>>(
        d_w, n, offset, rng_key(seed, 0x67656e75u));
    return cudaGetLastError();
}

}  // namespace wrsb
