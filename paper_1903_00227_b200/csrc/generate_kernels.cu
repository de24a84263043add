// paper_1903_00227_b200/csrc/generate_kernels.cu -- the power-law generator's
// Fisher-Yates shuffle on the device (weight_file.hpp:42-54).
//
// The reference deals (i+1)^-s to positions with
//     for i = n .. 2:  j_i = rng.bounded(i);  swap(w[i-1], w[j_i])
// on RngStream(seed, 'genp').  The stream is counter-based, so every j_i is
// known up front (j_i uses output n-i+1), and the sequential swaps can be
// resolved in parallel with the identical result:
//   * position i-1 is final after step i and receives what position j_i held
//     just before step i;
//   * what position j held just before step i is the value moved into it by
//     the most recent earlier step targeting j -- the smallest i' > i with
//     j_i' = j -- i.e. what position i'-1 held just before step i' (call it
//     node i'), or the original w[j] if no earlier step targeted j;
//   * node i' in turn is node parent(i') with parent(i') = the smallest
//     i'' > i' with j_i'' = i'-1, or the original w[i'-1]: a forest whose
//     edges go to strictly earlier steps, resolved by pointer jumping.
// The (j_i, i) pairs are grouped by j with a stable radix sort (CUB), so each
// j's steps come in increasing i.  Scratch ~28 B per item.
#include <climits>
#include <cstring>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "engine.h"

namespace wrsb {

namespace {

__device__ __forceinline__ uint32_t mulhi_u32(uint64_t r, uint32_t n) {
    const uint64_t t = static_cast<uint64_t>(static_cast<uint32_t>(r)) * n;
    const uint64_t u = static_cast<uint64_t>(static_cast<uint32_t>(r >> 32)) * n + (t >> 32);
    return static_cast<uint32_t>(u >> 32);
}

__device__ __forceinline__ uint64_t tid_global() {
    return static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
}
__device__ __forceinline__ uint64_t stride_global() {
    return static_cast<uint64_t>(gridDim.x) * blockDim.x;
}

// step i (2 <= i <= n) sits at index s = i - 2: j_i = bounded(i) from output
// n - i + 1 of the stream (rng.hpp:63-66)
__global__ void k_fy_targets(uint64_t n, uint64_t key, uint32_t* __restrict__ keys,
                             uint32_t* __restrict__ vals, uint32_t* __restrict__ cnt) {
    for (uint64_t s = tid_global(); s + 2 <= n; s += stride_global()) {
        const uint64_t i = s + 2;
        const uint64_t r = mix64(key + (n - i + 1) * kGolden);
        const uint32_t j = mulhi_u32(r, static_cast<uint32_t>(i));
        keys[s] = j;
        vals[s] = static_cast<uint32_t>(i);
        atomicAdd(cnt + j, 1u);
    }
}

// next[i]: smallest i' > i with j_i' = j_i (0 if none); parent[i]: smallest
// i' > i with j_i' = i - 1 (0 if none); root[i] starts as parent or itself.
__global__ void k_fy_links(uint64_t n, const uint32_t* __restrict__ skeys,
                           const uint32_t* __restrict__ svals, const uint32_t* __restrict__ off,
                           uint32_t* __restrict__ next, uint32_t* __restrict__ root) {
    const uint64_t m = n - 1;  // steps
    for (uint64_t p = tid_global(); p < m; p += stride_global()) {
        const uint32_t j = skeys[p], i = svals[p];
        next[i] = (p + 1 < m && skeys[p + 1] == j) ? svals[p + 1] : 0u;
    }
    for (uint64_t i = tid_global() + 2; i <= n; i += stride_global()) {
        uint32_t lo = off[i - 1], hi = off[i];  // steps targeting position i - 1
        while (lo < hi) {  // first with step > i
            const uint32_t mid = lo + (hi - lo) / 2;
            if (svals[mid] > i) hi = mid;
            else lo = mid + 1;
        }
        root[i] = lo < off[i] ? svals[lo] : static_cast<uint32_t>(i);
    }
}

__global__ void k_fy_jump(uint64_t n, const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                          unsigned* __restrict__ changed) {
    bool any = false;
    for (uint64_t i = tid_global() + 2; i <= n; i += stride_global()) {
        const uint32_t r = in[i], rr = in[r];
        out[i] = rr;
        any |= rr != r;
    }
    if (__any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0) *changed = 1u;
}

__global__ void k_fy_out(uint64_t n, const double* __restrict__ w, const uint32_t* __restrict__ keys,
                         const uint32_t* __restrict__ svals, const uint32_t* __restrict__ off,
                         const uint32_t* __restrict__ next, const uint32_t* __restrict__ root,
                         double* __restrict__ out) {
    for (uint64_t i = tid_global() + 2; i <= n; i += stride_global()) {
        const uint32_t nx = next[i];
        out[i - 1] = nx ? w[root[nx] - 1] : w[keys[i - 2]];
    }
    if (tid_global() == 0) {  // position 0: after every step
        out[0] = off[1] > off[0] ? w[root[svals[off[0]]] - 1] : w[0];
    }
}

}  // namespace

cudaError_t fisher_yates_device(const double* d_in, double* d_out, uint64_t n, uint64_t key,
                                cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    if (n == 1) return cudaMemcpyAsync(d_out, d_in, sizeof(double), cudaMemcpyDeviceToDevice, st);
    if (n > static_cast<uint64_t>(INT_MAX)) return cudaErrorInvalidValue;  // CUB int item counts
    const uint64_t m = n - 1;
    uint32_t *keys = nullptr, *vals = nullptr, *skeys = nullptr, *svals = nullptr, *cnt = nullptr,
             *off = nullptr, *next = nullptr, *ra = nullptr, *rb = nullptr;
    unsigned* changed = nullptr;
    void* tmp = nullptr;
    size_t tmp_sort = 0, tmp_scan = 0;
    cudaError_t e = cudaSuccess;
    auto A = [&](auto*& p, size_t bytes) {
        if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&p), bytes);
    };
    int end_bit = 1;
    while (end_bit < 32 && (1ull << end_bit) < n) ++end_bit;
    A(keys, m * 4);
    A(vals, m * 4);
    A(skeys, m * 4);
    A(svals, m * 4);
    A(cnt, (n + 1) * 4);
    A(off, (n + 1) * 4);
    A(next, (n + 1) * 4);
    A(ra, (n + 1) * 4);
    A(rb, (n + 1) * 4);
    A(changed, 4);
    if (e == cudaSuccess)
        e = cub::DeviceRadixSort::SortPairs(nullptr, tmp_sort, keys, skeys, vals, svals,
                                            static_cast<int>(m), 0, end_bit, st);
    if (e == cudaSuccess)
        e = cub::DeviceScan::ExclusiveSum(nullptr, tmp_scan, cnt, off, static_cast<int>(n + 1), st);
    A(tmp, tmp_sort > tmp_scan ? tmp_sort : tmp_scan);
    const unsigned blocks = static_cast<unsigned>(umin64((n + 255) / 256, 148ull * 32));
    if (e == cudaSuccess) e = cudaMemsetAsync(cnt, 0, (n + 1) * 4, st);
    if (e == cudaSuccess) {
        k_fy_targets<<<blocks, 256, 0, st>>>(n, key, keys, vals, cnt);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess)  // stable: each j's steps stay in increasing i
        e = cub::DeviceRadixSort::SortPairs(tmp, tmp_sort, keys, skeys, vals, svals,
                                            static_cast<int>(m), 0, end_bit, st);
    if (e == cudaSuccess)
        e = cub::DeviceScan::ExclusiveSum(tmp, tmp_scan, cnt, off, static_cast<int>(n + 1), st);
    if (e == cudaSuccess) {
        k_fy_links<<<blocks, 256, 0, st>>>(n, skeys, svals, off, next, ra);
        e = cudaGetLastError();
    }
    // pointer jumping to the roots (parents are strictly later steps)
    for (int round = 0; e == cudaSuccess && round < 64; ++round) {
        unsigned h = 0;
        e = cudaMemsetAsync(changed, 0, 4, st);
        if (e == cudaSuccess) {
            k_fy_jump<<<blocks, 256, 0, st>>>(n, ra, rb, changed);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaMemcpyAsync(&h, changed, 4, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        std::swap(ra, rb);
        if (!h) break;
    }
    if (e == cudaSuccess) {
        k_fy_out<<<blocks, 256, 0, st>>>(n, d_in, keys, svals, off, next, ra, d_out);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    for (void* p : {static_cast<void*>(keys), static_cast<void*>(vals), static_cast<void*>(skeys),
                    static_cast<void*>(svals), static_cast<void*>(cnt), static_cast<void*>(off),
                    static_cast<void*>(next), static_cast<void*>(ra), static_cast<void*>(rb),
                    static_cast<void*>(changed), tmp})
        if (p) cudaFree(p);
    return e;
}

unsigned long long check_failures_generate(unsigned* line) { return tu_check_failures(line); }

}  // namespace wrsb
