// paper_1903_00227_b200/csrc/common.cuh -- device-side building blocks shared
// by the PSA build (psa_kernels.cu) and the query kernel (sample_kernels.cu).
//
// Everything here reproduces a reference primitive bit for bit; the whole
// library is compiled with --fmad=false so no multiply-add is ever contracted
// (the reference's x86-64 build has no FMA).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
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
    unsigned int k2_ticket;        // fused K2b+K2c: CTA roles in start order
    unsigned int k2_work;          // fused K2b+K2c: next checkpoint warp unit
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

// ---- configs[3]'s lognormal weights (our own generator) ------
// The reference has no lognormal generator, so this one is defined here and
// restated in the oracle (oracle/wrs_oracle.c, wo_generate_lognormal): item
// i of generate_lognormal(n, sigma, seed) takes outputs 2i+1 and 2i+2 of
// RngStream(seed, 'logn'):
//     u1 = 1 - uniform01()  in (0, 1],  u2 = uniform01()  in [0, 1)
//     z  = sqrt(-2 log u1) cos(2 pi u2)          (Box-Muller, one variate)
//     w  = exp(sigma z)                          (lognormal(0, sigma))
// log, cos and exp are evaluated by the fixed sequences of IEEE additions,
// multiplications and divisions below (argument reduction + Horner series,
// no fused multiply-adds), so the CPU and the GPU produce the same bits.
constexpr uint64_t kLognStream = 0x6c6f676eu;  // "logn"
constexpr double kLn2Hi = 0x1.62e42fefa3800p-1, kLn2Lo = 0x1.ef35793c76730p-45;

// log x for x in (0, 1]: x = m 2^e, m in [sqrt(1/2), sqrt(2)); log m =
// 2 atanh(s), s = (m - 1) / (m + 1), |s| < 0.172: 13 odd terms.
__host__ __device__ inline double det_log(double x) {
    uint64_t b;
    memcpy(&b, &x, 8);
    int e = static_cast<int>((b >> 52) & 0x7ff) - 1023;
    b = (b & 0x000fffffffffffffull) | 0x3ff0000000000000ull;
    double m;
    memcpy(&m, &b, 8);
    if (m > 1.4142135623730951) {
        m = m * 0.5;
        e += 1;
    }
    const double s = (m - 1.0) / (m + 1.0);
    const double s2 = s * s;
    double p = 1.0 / 25.0;
    p = p * s2 + 1.0 / 23.0;
    p = p * s2 + 1.0 / 21.0;
    p = p * s2 + 1.0 / 19.0;
    p = p * s2 + 1.0 / 17.0;
    p = p * s2 + 1.0 / 15.0;
    p = p * s2 + 1.0 / 13.0;
    p = p * s2 + 1.0 / 11.0;
    p = p * s2 + 1.0 / 9.0;
    p = p * s2 + 1.0 / 7.0;
    p = p * s2 + 1.0 / 5.0;
    p = p * s2 + 1.0 / 3.0;
    p = p * s2 + 1.0;
    const double de = static_cast<double>(e);
    return de * kLn2Hi + (de * kLn2Lo + 2.0 * s * p);
}
// cos(2 pi u) for u in [0, 1): cos(2 pi u) = -cos(2 pi (u - 1/2)), folded to
// an angle in [0, pi/2]; even Taylor series, 13 terms.
__host__ __device__ inline double det_cos2pi(double u) {
    double a = u - 0.5;
    a = a < 0.0 ? -a : a;
    double sign = -1.0;
    if (a > 0.25) {
        a = 0.5 - a;
        sign = 1.0;
    }
    const double t = a * 6.283185307179586;
    const double t2 = t * t;
    double p = 1.0 / 620448401733239439360000.0;   // 1/24!
    p = p * -t2 + 1.0 / 1124000727777607680000.0;  // 1/22!
    p = p * -t2 + 1.0 / 2432902008176640000.0;     // 1/20!
    p = p * -t2 + 1.0 / 6402373705728000.0;        // 1/18!
    p = p * -t2 + 1.0 / 20922789888000.0;          // 1/16!
    p = p * -t2 + 1.0 / 87178291200.0;             // 1/14!
    p = p * -t2 + 1.0 / 479001600.0;               // 1/12!
    p = p * -t2 + 1.0 / 3628800.0;                 // 1/10!
    p = p * -t2 + 1.0 / 40320.0;                   // 1/8!
    p = p * -t2 + 1.0 / 720.0;                     // 1/6!
    p = p * -t2 + 1.0 / 24.0;                      // 1/4!
    p = p * -t2 + 1.0 / 2.0;                       // 1/2!
    p = p * -t2 + 1.0;
    return sign * p;
}
// exp x for |x| < 700: x = k ln2 + r, |r| <= ln2 / 2; Taylor series of e^r
// (18 terms) times 2^k.
__host__ __device__ inline double det_exp(double x) {
    const double kf = floor(x * 1.4426950408889634 + 0.5);
    const double r = (x - kf * kLn2Hi) - kf * kLn2Lo;
    double p = 1.0 / 355687428096000.0;  // 1/17!
    p = p * r + 1.0 / 20922789888000.0;  // 1/16!
    p = p * r + 1.0 / 1307674368000.0;   // 1/15!
    p = p * r + 1.0 / 87178291200.0;     // 1/14!
    p = p * r + 1.0 / 6227020800.0;      // 1/13!
    p = p * r + 1.0 / 479001600.0;       // 1/12!
    p = p * r + 1.0 / 39916800.0;        // 1/11!
    p = p * r + 1.0 / 3628800.0;         // 1/10!
    p = p * r + 1.0 / 362880.0;          // 1/9!
    p = p * r + 1.0 / 40320.0;           // 1/8!
    p = p * r + 1.0 / 5040.0;            // 1/7!
    p = p * r + 1.0 / 720.0;             // 1/6!
    p = p * r + 1.0 / 120.0;             // 1/5!
    p = p * r + 1.0 / 24.0;              // 1/4!
    p = p * r + 1.0 / 6.0;               // 1/3!
    p = p * r + 0.5;                     // 1/2!
    p = p * r + 1.0;
    p = p * r + 1.0;
    const uint64_t eb = static_cast<uint64_t>(static_cast<int64_t>(kf) + 1023) << 52;
    double scale;
    memcpy(&scale, &eb, 8);
    return p * scale;
}
// weight of item g (a global index) of generate_lognormal(., sigma, seed),
// key = rng_key(seed, kLognStream)
__host__ __device__ inline double lognormal_weight(uint64_t key, uint64_t g, double sigma) {
    const uint64_t r1 = mix64(key + (2 * g + 1) * kGolden);
    const uint64_t r2 = mix64(key + (2 * g + 2) * kGolden);
    const double u1 = 1.0 - static_cast<double>(r1 >> 11) * 0x1.0p-53;
    const double u2 = static_cast<double>(r2 >> 11) * 0x1.0p-53;
    const double z = sqrt(-2.0 * det_log(u1)) * det_cos2pi(u2);
    return det_exp(sigma * z);
}

#if defined(__CUDACC__)
// ---- checked builds (make checked -> libwrs_b200_checked.so) ---------------
// compute-sanitizer is not available on the GPU pool, so the library checks
// itself: in a checked build every WRS_CHECK'd index is tested on the device
// and a violation is counted (the first offending source line is kept) in a
// per-translation-unit counter that wrs_b200_check_failures() reads; scratch
// buffers are also filled with 0xFF bytes (NaN / huge indices) before use, so
// a read of anything not written first shows up in the parity checks.  In
// the normal build WRS_CHECK compiles to nothing.
#ifdef WRS_B200_CHECKED
static __device__ unsigned long long g_check_fail = 0;
static __device__ unsigned int g_check_line = 0;
__device__ __noinline__ static void check_fail(unsigned line) {
    atomicAdd(&g_check_fail, 1ull);
    atomicCAS(&g_check_line, 0u, line);
}
#define WRS_CHECK(c)                                 \
    do {                                             \
        if (!(c)) ::wrsb::check_fail(__LINE__);      \
    } while (0)
// this translation unit's count (and first line); host side
static inline unsigned long long tu_check_failures(unsigned* line) {
    unsigned long long c = 0;
    unsigned l = 0;
    cudaMemcpyFromSymbol(&c, g_check_fail, sizeof c);
    cudaMemcpyFromSymbol(&l, g_check_line, sizeof l);
    if (line && l && !*line) *line = l;
    return c;
}
#else
#define WRS_CHECK(c) \
    do {             \
    } while (0)
static inline unsigned long long tu_check_failures(unsigned*) { return 0; }
#endif

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
// mbarrier + bulk-copy (cp.async.bulk) helpers, CTA scope
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)),
                 "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n"
        ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
                   "r"((unsigned)__cvta_generic_to_shared(b)) : "memory");
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
