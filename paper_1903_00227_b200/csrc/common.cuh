// paper_1903_00227_b200/csrc/common.cuh -- device-side building blocks shared
// by the PSA build (psa_kernels.cu) and the query kernel (sample_kernels.cu).
//
// Everything here reproduces a reference primitive bit for bit; the whole
// library is compiled with --fmad=false so no multiply-add is ever contracted
// (the reference's x86-64 build has no FMA).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace wrsb {

// 16-byte bucket with the byte layout of wrs::alias_bucket (alias.hpp:26-33):
// share at offset 0, item at 8, alias at 12.  Every bucket's item is its own
// index, so a query reads one aligned 16-B record = one 32-B sector.
struct alignas(16) Bucket {
    double share;
    uint32_t item;
    uint32_t alias;
};
static_assert(sizeof(Bucket) == 16, "bucket must stay 16 bytes");

// Device-resident scalars of one build (no host round trip between kernels).
struct DevScalars {
    double total;                  // pairwise W (weights.hpp:19-28)
    double wn;                     // W / n (alias.hpp:247-248)
    unsigned long long bad_index;  // first non-finite / non-positive weight, ~0 if none
    unsigned long long nl, nh;     // light / heavy counts (alias.hpp:41-46)
    unsigned int tile_counter;     // K1 dynamic tile ids
    unsigned int plan_error;       // psa_plan's logic_error (alias.hpp:230-231)
};

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;  // rng.hpp:23

// SplitMix64 finalizer, rng.hpp:16-20.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// RngStream(seed, stream).key (rng.hpp:36-37) and derive(salt).key (:40-45).
__host__ __device__ __forceinline__ uint64_t rng_key(uint64_t seed, uint64_t stream) {
    return mix64(mix64(seed + kGolden) ^ mix64(stream) ^ stream);
}
__host__ __device__ __forceinline__ uint64_t rng_derive(uint64_t key, uint64_t salt) {
    return mix64(key + mix64(salt + kGolden));
}

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// Philox4x32-10 (Salmon et al., SC'11 "Parallel random numbers: as easy as
// 1, 2, 3"): 10 rounds of two 32x32 multiplies on a 4-word counter with a
// 2-word key bumped by the Weyl constants.  Used by the optional Philox draw
// mode (north star), not by the reference-parity draws.
__host__ __device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
    constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#if defined(__CUDACC__)
#pragma unroll
#endif
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = static_cast<uint64_t>(M0) * c[0];
        const uint64_t p1 = static_cast<uint64_t>(M1) * c[2];
        const uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
        const uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
        const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0;
        c[1] = lo1;
        c[2] = n2;
        c[3] = lo0;
        k0 += W0;
        k1 += W1;
    }
}

#if defined(__CUDACC__)
// Neumaier compensated sum, parallel.hpp:70-81 (the isfinite guard keeps an
// infinite running value from poisoning the low word).  Written branch-free:
// the error term is always computed and the guarded update is a select, so
// the compiler can compute the error terms of a run of adds in parallel and
// leave only one dependent DADD per add on each of the hi and lo chains.  The
// values are identical to the guarded form.
struct CompSum {
    double hi, lo;
    __device__ __forceinline__ void add(double x) {
        const double t = hi + x;
        // (hi - t) + x if |hi| >= |x| else (x - t) + hi: select the operands,
        // then the same two roundings (2 DADD instead of 4 + a select)
        const bool big = fabs(hi) >= fabs(x);
        const double a = big ? hi : x, b = big ? x : hi;
        const double e = (a - t) + b;
        const double l2 = lo + e;
        lo = isfinite(t) ? l2 : lo;
        hi = t;
    }
    __device__ __forceinline__ double value() const { return hi + lo; }
};

// The same sum for chains whose terms and running values are all finite and
// >= 0 (prefix sums of validated weights whose total is far below DBL_MAX):
// then |hi| >= |x| is hi >= x, so the operands of the error term are
// max(hi, x) and min(hi, x), and isfinite(t) is always true, so the guarded
// update is the plain one.  Bit-identical to CompSum on such chains, with
// 4 DADD + one compare + selects per add and a one-DADD recurrence on lo.
struct CompSumPos {
    double hi, lo;
    __device__ __forceinline__ void add(double x) {
        const double t = hi + x;
        const bool big = hi >= x;
        const double a = big ? hi : x, b = big ? x : hi;
        lo = lo + ((a - t) + b);
        hi = t;
    }
    __device__ __forceinline__ double value() const { return hi + lo; }
};

// std::min / std::max argument order (the reference's share clamps).
__device__ __forceinline__ double std_min(double a, double b) { return b < a ? b : a; }
__device__ __forceinline__ double std_max(double a, double b) { return a < b ? b : a; }

// ---- async copies (sm_80+ LDGSTS; no register staging) --------------------
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// 16-byte streaming store of one bucket.
__device__ __forceinline__ void store_bucket(Bucket* b, uint64_t idx, double share,
                                             uint32_t item, uint32_t alias) {
    const unsigned long long s = static_cast<unsigned long long>(__double_as_longlong(share));
    uint4 v = make_uint4(static_cast<unsigned>(s), static_cast<unsigned>(s >> 32), item, alias);
    *reinterpret_cast<uint4*>(b + idx) = v;
}

#endif  // __CUDACC__

}  // namespace wrsb
