// paper_1903_00227_b200/csrc/verify_kernels.cu -- implied masses and the
// mass check on the device (verify.hpp:43-54, 92-98).
//
// implied_masses: m[item] gets each bucket's share, m[alias] its bucket_mean
// - share, Kahan-summed per item in bucket order.  Bit for bit here: the
// (alias, bucket) pairs are sorted by alias with a stable radix sort, so each
// item's alias contributions come in bucket order, and one thread per item
// merges its own bucket's share in at its position (own share before the
// alias contribution of the same bucket, as the reference's loop body).  The
// sort is CUB's (a library sort on the verification path, not the hot path).
#include <climits>
#include <cstring>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "engine.h"

namespace wrsb {

__global__ void k_alias_pairs(const Bucket* __restrict__ b, uint64_t n, uint32_t* __restrict__ keys,
                              uint32_t* __restrict__ vals, uint32_t* __restrict__ cnt) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += stride) {
        const uint32_t a = b[i].alias;
        keys[i] = a;
        vals[i] = static_cast<uint32_t>(i);
        atomicAdd(cnt + a, 1u);
    }
}

struct Kahan {  // kahan_sum, verify.hpp:26-38
    double s = 0.0, c = 0.0;
    __device__ __forceinline__ void add(double x) {
        const double y = x - c;
        const double t = s + y;
        c = (t - s) - y;
        s = t;
    }
};

// One thread per item; worst = max |m - w| / w as the bits of a non-negative
// double (their integer order is their numeric order).
__global__ void k_item_masses(const Bucket* __restrict__ b, uint64_t n, double wn,
                              const uint32_t* __restrict__ by_alias,
                              const uint32_t* __restrict__ off, const double* __restrict__ w,
                              double* __restrict__ m, unsigned long long* __restrict__ worst) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    double local = 0.0;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += stride) {
        Kahan k;
        uint32_t p = off[i];
        const uint32_t e = off[i + 1];
        // alias contributions of buckets before i, then bucket i's own share
        // (item == index in a PSA table), then the rest (incl. bucket i's
        // alias contribution when it aliases itself)
        while (p < e && by_alias[p] < i) k.add(wn - b[by_alias[p++]].share);
        k.add(b[i].share);
        while (p < e) k.add(wn - b[by_alias[p++]].share);
        if (m) m[i] = k.s;
        const double err = fabs(k.s - w[i]) / w[i];  // max_relative_mass_error, verify.hpp:92-98
        local = err > local ? err : local;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double y = __shfl_xor_sync(0xffffffffu, local, o);
        local = y > local ? y : local;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(worst, static_cast<unsigned long long>(__double_as_longlong(local)));
}

cudaError_t implied_masses_device(const Bucket* d_b, uint64_t n, double wn, const double* d_w,
                                  double* d_m, double* worst_host, cudaStream_t st) {
    if (n == 0) {
        *worst_host = 0.0;
        return cudaSuccess;
    }
    if (n > static_cast<uint64_t>(INT_MAX)) return cudaErrorInvalidValue;  // CUB int item counts
    uint32_t *keys = nullptr, *vals = nullptr, *keys2 = nullptr, *vals2 = nullptr;
    uint32_t *cnt = nullptr, *off = nullptr;
    unsigned long long* worst = nullptr;
    void* tmp = nullptr;
    size_t tmp_sort = 0, tmp_scan = 0;
    cudaError_t e = cudaSuccess;
    auto A = [&](auto*& p, size_t bytes) {
        if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&p), bytes);
    };
    int end_bit = 1;
    while (end_bit < 32 && (1ull << end_bit) < n) ++end_bit;
    A(keys, n * 4);
    A(vals, n * 4);
    A(keys2, n * 4);
    A(vals2, n * 4);
    A(cnt, (n + 1) * 4);
    A(off, (n + 1) * 4);
    A(worst, 8);
    if (e == cudaSuccess)
        e = cub::DeviceRadixSort::SortPairs(nullptr, tmp_sort, keys, keys2, vals, vals2,
                                            static_cast<int>(n), 0, end_bit, st);
    if (e == cudaSuccess)
        e = cub::DeviceScan::ExclusiveSum(nullptr, tmp_scan, cnt, off, static_cast<int>(n + 1), st);
    A(tmp, tmp_sort > tmp_scan ? tmp_sort : tmp_scan);
    if (e == cudaSuccess) e = cudaMemsetAsync(cnt, 0, (n + 1) * 4, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(worst, 0, 8, st);
    if (e == cudaSuccess) {
        const unsigned blocks = static_cast<unsigned>(umin64((n + 255) / 256, 148ull * 16));
        k_alias_pairs<<<blocks, 256, 0, st>>>(d_b, n, keys, vals, cnt);
        e = cudaGetLastError();
    }
    // stable: equal aliases keep bucket order
    if (e == cudaSuccess)
        e = cub::DeviceRadixSort::SortPairs(tmp, tmp_sort, keys, keys2, vals, vals2,
                                            static_cast<int>(n), 0, end_bit, st);
    if (e == cudaSuccess)
        e = cub::DeviceScan::ExclusiveSum(tmp, tmp_scan, cnt, off, static_cast<int>(n + 1), st);
    if (e == cudaSuccess) {
        const unsigned blocks = static_cast<unsigned>(umin64((n + 255) / 256, 148ull * 16));
        k_item_masses<<<blocks, 256, 0, st>>>(d_b, n, wn, vals2, off, d_w, d_m, worst);
        e = cudaGetLastError();
    }
    unsigned long long wbits = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&wbits, worst, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) std::memcpy(worst_host, &wbits, sizeof wbits);
    for (void* p : {static_cast<void*>(keys), static_cast<void*>(vals), static_cast<void*>(keys2),
                    static_cast<void*>(vals2), static_cast<void*>(cnt), static_cast<void*>(off),
                    static_cast<void*>(worst), tmp})
        if (p) cudaFree(p);
    return e;
}

unsigned long long check_failures_verify(unsigned* line) { return tu_check_failures(line); }

}  // namespace wrsb
