// paper_1903_00227_b200/csrc/sample_kernels.cu -- K5, bulk alias sampling,
// plus the on-device uniform weight generator.
//
// Semantics: AliasTable::sample_many (alias.hpp:274-284) bit for bit.  Worker
// w of W owns the contiguous output slice worker_slice(k, W, w)
// (parallel.hpp:37-43) and draws it from RngStream(seed, 'alia').derive(w);
// query m of a slice consumes outputs 2m+1 (bucket via the 128-bit
// multiply-shift, rng.hpp:63-66) and 2m+2 (coin, rng.hpp:53-55) of that
// counter stream and returns ia[x >= share] (alias.hpp:265-269).  The stream
// is counter-based, so every output position is computable on its own and the
// GPU is free to choose WHEN it computes each one.
//
// Two execution plans:
//   direct  (table L2-resident or few draws): one kernel, one 16-B gather per
//           draw straight from the table.
//   region  (table >> L2): measured on B200, every random 16-B gather from an
//           HBM-resident table moves a full 128-B line (ncu: 126 B/draw), so
//           the direct plan tops out near 6.5 TB/s / 132 B = 50 G draws/s.
//           The region plan reorders the WORK, not the results: draws are
//           bucketed by table region (2^21 buckets = 32 MB, L2-resident;
//           64 MB above 2^27 buckets, region_shift) with
//           a tile-local counting sort into per-region slabs (space claimed by
//           atomics), the gathers then sweep the table region by region so
//           every line is fetched from HBM about once, and a final pass puts
//           the answers back in output order.  Traffic per draw: 4 B record
//           (the draw's index) write + 4 B read + 2 B slot write + 2 B read +
//           4 B result write + 4 B read + 4 B output write, plus 16n B of
//           table per pass (passes of up to 3.5e9 draws).
//     RB  k_region_scatter   draw-index records, runs per (tile, region),
//                            each run one bulk copy to its slab
//     RC  k_region_gather    bucket + coin recomputed, bucket gather, region
//                            by region
//     RD  k_region_unpermute out[q] = result at the slot RB gave draw q; each
//                            of the tile's runs staged with one bulk copy
//   Aggregated draws reuse RB and count instead of writing (k_region_count,
//   k_count_fold, k_compact_*); k_two_level_sample routes two-level draws;
//   the Philox mode is a compile-time variant of every draw kernel.
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "engine.h"

namespace wrsb {

// ===========================================================================
// shared: where query q lives in the worker partition, and its two draws
// ===========================================================================
struct DrawGeom {
    uint64_t n;         // buckets
    double wn;          // bucket mean W/n
    uint64_t base_key;  // RngStream(seed, stream).key
    uint64_t k;         // total draws of the call (defines worker slices)
    uint32_t W;         // workers
    uint32_t philox;    // Philox draw mode (kPhiloxStream): W = 1, base_key = the raw seed
    uint64_t per, rem, big;  // k/W, k%W, rem*(per+1)
    double inv_p1, inv_p;    // 1/(per+1), 1/per for the division estimate
};

DrawGeom make_geom(uint64_t n, double wn, uint64_t seed, uint64_t stream_id, uint64_t k,
                   uint32_t W) {
    DrawGeom g{};
    g.n = n;
    g.wn = wn;
    g.philox = stream_id == kPhiloxStream;
    g.base_key = g.philox ? seed : rng_key(seed, stream_id);  // Philox keys on the raw seed
    g.k = k;
    if (g.philox) W = 1;  // one counter space: draw q uses counter q
    g.W = W ? W : 1;
    g.per = k / g.W;
    g.rem = k % g.W;
    g.big = g.rem * (g.per + 1);
    g.inv_p1 = 1.0 / static_cast<double>(g.per + 1);
    g.inv_p = g.per ? 1.0 / static_cast<double>(g.per) : 0.0;
    return g;
}

// floor(a / d) for a < 2^53 from a double estimate plus exact correction.
__device__ __forceinline__ uint64_t div_est(uint64_t a, uint64_t d, double inv) {
    uint64_t t = static_cast<uint64_t>(static_cast<double>(a) * inv);
    while (t * d > a) --t;
    while ((t + 1) * d <= a) ++t;
    return t;
}

// worker_slice inverse (parallel.hpp:37-43): q -> (worker, index in slice).
__device__ __forceinline__ void locate(const DrawGeom& g, uint64_t q, uint32_t& w, uint64_t& m) {
    if (g.W == 1) {
        w = 0;
        m = q;
    } else if (q < g.big) {
        const uint64_t t = div_est(q, g.per + 1, g.inv_p1);
        w = static_cast<uint32_t>(t);
        m = q - t * (g.per + 1);
    } else {
        const uint64_t r = q - g.big;
        const uint64_t t = div_est(r, g.per, g.inv_p);
        w = static_cast<uint32_t>(g.rem + t);
        m = r - t * g.per;
    }
}

// Per-thread cache of the last worker's derived key.
struct KeyCache {
    uint32_t w = 0xffffffffu;
    uint64_t key = 0;
    __device__ __forceinline__ uint64_t get(const DrawGeom& g, uint32_t wk) {
        if (wk != w) {
            w = wk;
            key = rng_derive(g.base_key, wk);  // RngStream(...).derive(worker), alias.hpp:280
        }
        return key;
    }
};

// Walks a thread's increasing query positions: the current worker slice
// [lo, hi) and its derived key.  W1 (a single worker, the common case)
// compiles the slice logic away.
template <bool W1>
struct DrawCursor {
    uint32_t w;
    uint64_t lo, hi, key;
    __device__ __forceinline__ void init(const DrawGeom& g, uint64_t q) {
        if (W1) {
            w = 0;
            lo = 0;
            hi = ~0ull;
        } else {
            uint64_t m;
            locate(g, q, w, m);
            lo = q - m;
            hi = lo + g.per + (w < g.rem ? 1 : 0);
        }
        key = rng_derive(g.base_key, w);  // RngStream(seed, 'alia').derive(w), alias.hpp:279-280
    }
    // counter of output 2m+1 of query q (m = q - lo); q must not decrease
    __device__ __forceinline__ uint64_t ctr1(const DrawGeom& g, uint64_t q) {
        if (!W1) {
            while (q >= hi) {
                ++w;
                lo = hi;
                hi = lo + g.per + (w < g.rem ? 1 : 0);
                key = rng_derive(g.base_key, w);
            }
        }
        return key + (2 * (q - lo) + 1) * kGolden;
    }
};

// bounded(n) of output 2m+1 (rng.hpp:63-66)
__device__ __forceinline__ uint64_t draw_bucket(const DrawGeom& g, uint64_t key, uint64_t m) {
    return __umul64hi(mix64(key + (2 * m + 1) * kGolden), g.n);
}
// (r * n) >> 64 for n < 2^32 (the table limit) in two 32x32->64 multiplies;
// equal to __umul64hi(r, n).
__device__ __forceinline__ uint32_t mulhi_n32(uint64_t r, uint32_t n) {
    const uint64_t t = static_cast<uint64_t>(static_cast<uint32_t>(r)) * n;
    const uint64_t u = static_cast<uint64_t>(static_cast<uint32_t>(r >> 32)) * n + (t >> 32);
    return static_cast<uint32_t>(u >> 32);
}
__device__ __forceinline__ uint64_t bucket_of_ctr(const DrawGeom& g, uint64_t c1) {
    return mulhi_n32(mix64(c1), static_cast<uint32_t>(g.n));
}
// uniform01() * bucket_mean of the output after c1 (rng.hpp:53-55)
__device__ __forceinline__ double coin_of_ctr(const DrawGeom& g, uint64_t c1) {
    const uint64_t r = mix64(c1 + kGolden);
    return (static_cast<double>(r >> 11) * 0x1.0p-53) * g.wn;
}
// uniform01() * bucket_mean of output 2m+2 (rng.hpp:53-55, alias.hpp:267)
__device__ __forceinline__ double draw_coin(const DrawGeom& g, uint64_t key, uint64_t m) {
    const uint64_t r = mix64(key + (2 * m + 2) * kGolden);
    return (static_cast<double>(r >> 11) * 0x1.0p-53) * g.wn;
}

// Philox draw mode: draw q = Philox4x32-10(counter (q_lo, q_hi, 0, 0), key
// (seed_lo, seed_hi)) -> words o0..o3; bucket = ((o1:o0) * n) >> 64, coin =
// ((o3:o2) >> 11) * 2^-53 * bucket_mean, answer ia[coin >= share].
__device__ __forceinline__ void philox_words(const DrawGeom& g, uint64_t q, uint32_t o[4]) {
    o[0] = static_cast<uint32_t>(q);
    o[1] = static_cast<uint32_t>(q >> 32);
    o[2] = 0;
    o[3] = 0;
    philox4x32_10(o, static_cast<uint32_t>(g.base_key), static_cast<uint32_t>(g.base_key >> 32));
}
__device__ __forceinline__ uint32_t philox_bucket(const DrawGeom& g, uint64_t q) {
    uint32_t o[4];
    philox_words(g, q, o);
    return mulhi_n32((static_cast<uint64_t>(o[1]) << 32) | o[0], static_cast<uint32_t>(g.n));
}
// bucket and coin of draw q from ONE Philox evaluation (the words feed both)
__device__ __forceinline__ void philox_draw(const DrawGeom& g, uint64_t q, uint32_t& bucket,
                                            double& coin) {
    uint32_t o[4];
    philox_words(g, q, o);
    bucket = mulhi_n32((static_cast<uint64_t>(o[1]) << 32) | o[0], static_cast<uint32_t>(g.n));
    const uint64_t r = (static_cast<uint64_t>(o[3]) << 32) | o[2];
    coin = (static_cast<double>(r >> 11) * 0x1.0p-53) * g.wn;
}
__device__ __forceinline__ double philox_coin(const DrawGeom& g, uint64_t q) {
    uint32_t o[4];
    philox_words(g, q, o);
    const uint64_t r = (static_cast<uint64_t>(o[3]) << 32) | o[2];
    return (static_cast<double>(r >> 11) * 0x1.0p-53) * g.wn;
}

__device__ __forceinline__ uint4 ld_bucket(const Bucket* b, uint64_t i) {
    uint4 v;
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(b + i));
    return v;
}
__device__ __forceinline__ uint32_t pick(const uint4& bk, double x) {
    const double share = __hiloint2double(static_cast<int>(bk.y), static_cast<int>(bk.x));
    return x >= share ? bk.w : bk.z;  // ia[x >= share] (alias.hpp:268)
}

// ===========================================================================
// direct plan
// ===========================================================================
constexpr int K5_THREADS = 256;
constexpr int K5_UNROLL = 8;

template <bool W1, bool PHX = false>
__global__ void __launch_bounds__(K5_THREADS)
k_sample(const Bucket* __restrict__ b, DrawGeom g, uint64_t q_begin, uint64_t q_end,
         uint32_t out_base, uint32_t* __restrict__ out) {
    const uint64_t span = static_cast<uint64_t>(K5_THREADS) * K5_UNROLL;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * span;
    out -= q_begin;  // out[q] for q in [q_begin, q_end)
    const uint64_t first = q_begin + static_cast<uint64_t>(blockIdx.x) * span + threadIdx.x;
    DrawCursor<W1> cur;
    cur.init(g, first < q_end ? first : q_begin);
    for (uint64_t q0 = first; q0 < q_end; q0 += stride) {
        uint64_t bidx[K5_UNROLL];
        double x[K5_UNROLL];
#pragma unroll
        for (int u = 0; u < K5_UNROLL; ++u) {
            const uint64_t q = q0 + static_cast<uint64_t>(u) * K5_THREADS;
            bidx[u] = 0;
            x[u] = 0.0;
            if (q < q_end) {
                if constexpr (PHX) {
                    uint32_t bb;
                    philox_draw(g, q, bb, x[u]);
                    bidx[u] = bb;
                    continue;
                }
                const uint64_t c1 = cur.ctr1(g, q);
                bidx[u] = bucket_of_ctr(g, c1);
                x[u] = coin_of_ctr(g, c1);
            }
        }
        uint4 bk[K5_UNROLL];
#pragma unroll
        for (int u = 0; u < K5_UNROLL; ++u) bk[u] = ld_bucket(b, bidx[u]);
#pragma unroll
        for (int u = 0; u < K5_UNROLL; ++u) {
            const uint64_t q = q0 + static_cast<uint64_t>(u) * K5_THREADS;
            WRS_CHECK(q >= q_end || bidx[u] < g.n);
            if (q < q_end) out[q] = pick(bk[u], x[u]) + out_base;
        }
    }
}

// ===========================================================================
// region plan
//   Tiles of TT * RS_ROWS consecutive draws (TT = 256, 512 or 1024 threads,
//   more for more regions, tile_threads_for); thread t computes draws t,
//   t + TT, ... of its tile.  Inside a tile
//   the draws are laid out by (region, warp, row, lane); each region's run of
//   the tile moves to and from global memory as one contiguous block through
//   shared memory.  Region r owns a fixed slab [r*cap, (r+1)*cap) of the
//   record array; tiles claim space in it with one atomicAdd per (tile,
//   region), so no counting pass is needed (the order of runs inside a slab
//   is arbitrary and does not affect any result).  A run that would overflow
//   its slab (cap has ~20 sigma of slack) goes to a shared overflow slab.
// ===========================================================================
constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_ROWS = 16;                        // rows of 32 draws per warp
constexpr int RS_TILE = RS_THREADS * RS_ROWS;      // 4096 draws per tile
constexpr int RS_MAX_REGIONS = 1024;

struct RegionGeom {
    DrawGeom g;
    uint64_t q0;       // first draw of this chunk
    uint64_t kc;       // draws in this chunk
    uint64_t ntiles;   // ceil(kc / tile)
    uint32_t nreg;     // regions
    int shift;         // region = bucket >> shift
    uint32_t cap;      // records per region slab
    uint32_t ov_cap;   // records in the overflow slab (after the nreg slabs)
};

// per (tile, region): slab position of the tile's run and the END of its
// padded slots in the tile's stage (the run starts where the previous ends)
struct RunInfo {
    uint32_t goff;
    uint32_t end;
};

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint2 ld_stream(const uint2* p, uint64_t pol) {
    uint2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
                 : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
                 : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_stream(uint32_t* p, uint32_t v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.u32 [%0], %1, %2;"
                 :: "l"(p), "r"(v), "l"(pol));
}
__device__ __forceinline__ uint4 ld_table(const Bucket* b, uint64_t i, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(b + i), "l"(pol));
    return v;
}

// RB: draws -> region slabs.  Each thread computes 16 draws' buckets and
// counts them per region (shared-memory atomics); a warp scan turns the counts
// into tile-local run starts while other warps claim the runs' slab space; each
// draw then takes a staging slot from its region's fill cursor, the (draw,
// bucket) records are staged in shared memory in region order, and each run is
// written to its slab as one contiguous block.  The tile slot of every draw
// is recorded (q order) for RD, so the (non-deterministic) order inside a run
// never needs to be reproduced.
// Runs are padded to whole groups of RUN_ALIGN records (slab and stage
// positions stay multiples of 4: 32-B aligned records, 16-B aligned results),
// so RB writes each run with one bulk copy and RD stages results with 16-B
// copies; a padding slot holds a record whose draw index is REC_PAD, which
// RC and the counting pass skip.
constexpr uint32_t RUN_ALIGN = 4;
constexpr uint32_t REC_PAD = 0xffffffffu;  // (draw indices within a chunk are < 2^32 - 1)
__host__ __device__ inline uint32_t stage_slots(uint32_t nreg, uint32_t tile) {
    return tile + (RUN_ALIGN - 1) * nreg;
}
__host__ __device__ inline size_t scatter_smem_bytes(uint32_t nreg, uint32_t tile, size_t rec_bytes) {
    const size_t head = (4 * static_cast<size_t>(nreg) + 2) * 4;
    return ((head + 15) & ~size_t(15)) + stage_slots(nreg, tile) * rec_bytes;
}

// ORDER = false (aggregated draws): the answers are only counted, never put
// back in draw order, so the tile slots and the run table are not written.
// FULL: every tile of the launch holds TT * RS_ROWS draws, so no per-draw
// bounds test is compiled (the one partial tile of a chunk, if any, is a
// separate one-CTA launch with tile0 = its index).
// Phases: (1) buckets + per-region counts (shared atomics, no return value,
// so only the 16 buckets stay in registers); (2) warp 0 scans the counts while
// the other warps claim slab space for the tile's runs (global atomics), so the
// two latencies overlap; (3) each draw takes its staging slot with a second
// shared atomic on its region's fill cursor; (4) the staged records go out
// run by run as contiguous blocks.
#ifndef RC_ROWS
#define RC_ROWS 12  // records per gather / count thread (8.02 vs 8.06 ms at 8, 1e9 draws, n = 1e8)
#endif
constexpr int RC_SPAN = RC_ROWS * 256;  // slab positions per gather / count CTA
#ifndef RC_COIN_EARLY
#define RC_COIN_EARLY 1  // gather: coins computed while the bucket rows are in flight
#endif
#ifndef RC_MIN_CTAS
#define RC_MIN_CTAS 4  // gather / count CTAs per SM (48 KB of bucket rows each)
#endif
#ifndef RD_MIN_CTAS
#define RD_MIN_CTAS 8  // unpermute (256-thread) CTAs per SM (32 regs)
#endif
#ifndef RS_MIN_CTAS
#define RS_MIN_CTAS 6  // 256-thread CTAs per SM the register budget must allow (40 regs; 8.05 vs 8.16 ms at 5)
#endif
#ifndef RS32_SM_THREADS
#define RS32_SM_THREADS 1024  // 32-row scatter threads per SM the registers must allow (64 each)
#endif
// ROWS: draws per thread (tile = TT * ROWS); 32 rows keep 256-thread CTAs
// for 8192-draw tiles (4 CTAs per SM: 64 registers for the 32 buckets).
template <bool W1, bool ORDER = true, bool PHX = false, int TT = RS_THREADS, bool FULL = false,
          int ROWS = RS_ROWS>
__global__ void __launch_bounds__(TT, (ROWS == RS_ROWS ? RS_MIN_CTAS * 256 : ROWS == 32 ? RS32_SM_THREADS : 512) / TT)
k_region_scatter(RegionGeom rg, uint32_t tile0, uint32_t* __restrict__ cursor,
                 unsigned* __restrict__ overflow, void* __restrict__ rec_out,
                 uint16_t* __restrict__ slot_of, RunInfo* __restrict__ runs) {
    // 4-B records, the draw's index in the chunk (the gather / counting pass
    // recomputes its bucket and coin from the counter-based stream)
    using Rec = uint32_t;
    Rec* const rec = static_cast<Rec*>(rec_out);
    extern __shared__ __align__(16) unsigned char rs_smem[];
    const uint32_t nreg = rg.nreg;
    uint32_t* cnt = reinterpret_cast<uint32_t*>(rs_smem);  // [nreg] draws per region
    uint32_t* start = cnt + nreg;                          // [nreg + 1] run starts in the stage
    uint32_t* fill = start + nreg + 1;                     // [nreg] fill cursors
    uint32_t* goff = fill + nreg;                          // [nreg] the runs' slab positions
    Rec* stage = reinterpret_cast<Rec*>(rs_smem + (((4 * nreg + 2) * 4 + 15) & ~15u));  // padded runs
    const uint64_t tile = static_cast<uint64_t>(tile0) + blockIdx.x;
    const uint64_t tbase = tile * (TT * ROWS);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t i = threadIdx.x; i < nreg; i += TT) cnt[i] = 0;
    __syncthreads();

    uint32_t bk[ROWS];
    const uint32_t kc_left =
        FULL ? (TT * ROWS) : static_cast<uint32_t>(umin64(rg.kc - tbase, (TT * ROWS)));
    const uint32_t n32 = static_cast<uint32_t>(rg.g.n);
    if (W1) {
        // single worker: counter of draw q is key + (2q + 1) G, and the rows of
        // a thread are TT draws apart
        uint64_t c1 = rng_derive(rg.g.base_key, 0) +
                      (2 * (rg.q0 + tbase + threadIdx.x) + 1) * kGolden;
        const uint64_t step = 2ull * TT * kGolden;
        if constexpr (PHX) {
#pragma unroll
            for (int r = 0; r < ROWS; ++r)
                bk[r] = philox_bucket(rg.g, rg.q0 + tbase + r * TT + threadIdx.x);
        } else {
#pragma unroll
            for (int r = 0; r < ROWS; ++r) {
                bk[r] = mulhi_n32(mix64(c1), n32);
                c1 += step;
            }
        }
    } else {
        DrawCursor<W1> cur;
        cur.init(rg.g, rg.q0 + tbase + threadIdx.x);
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
            const uint32_t e = r * TT + threadIdx.x;
            bk[r] = e < kc_left
                        ? static_cast<uint32_t>(bucket_of_ctr(rg.g, cur.ctr1(rg.g, rg.q0 + tbase + e)))
                        : 0u;
        }
    }
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
        const uint32_t e = r * TT + threadIdx.x;
        if (e < kc_left) atomicAdd(&cnt[bk[r] >> rg.shift], 1u);
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the region counts, 32 at a time
        uint32_t carry = 0;
        for (uint32_t r0 = 0; r0 < nreg; r0 += 32) {
            const uint32_t reg = r0 + lane;
            const uint32_t c = reg < nreg ? (cnt[reg] + RUN_ALIGN - 1) & ~(RUN_ALIGN - 1) : 0;
            uint32_t x = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (reg < nreg) {
                start[reg] = carry + x - c;
                fill[reg] = carry + x - c;
            }
            carry += __shfl_sync(0xffffffffu, x, 31);
        }
        if (lane == 0) start[nreg] = carry;
    } else {  // claim slab space for each non-empty run of this tile
        for (uint32_t reg = threadIdx.x - 32; reg < nreg; reg += TT - 32) {
            const uint32_t c = (cnt[reg] + RUN_ALIGN - 1) & ~(RUN_ALIGN - 1);  // padded run
            uint32_t g = 0;
            if (c) {
                const uint32_t base = atomicAdd(&cursor[reg], c);
                if (base + c <= rg.cap) {
                    g = reg * rg.cap + base;
                } else {
                    // the slab keeps only the runs claimed below this one:
                    // positions from here on are never written
                    atomicMin(&cursor[nreg + 1 + reg], base);
                    const uint32_t ob = atomicAdd(&cursor[nreg], c);
                    if (ob + c > rg.ov_cap) atomicOr(overflow, 1u);
                    g = nreg * rg.cap + (ob + c <= rg.ov_cap ? ob : 0);
                }
            }
            goff[reg] = g;
        }
    }
    __syncthreads();
    // run table and padding records (slots [start + cnt, next start), disjoint
    // from the slots the draws take below)
    for (uint32_t reg = threadIdx.x; reg < nreg; reg += TT) {
        if (ORDER) runs[tile * nreg + reg] = RunInfo{goff[reg], start[reg + 1]};
        for (uint32_t i = start[reg] + cnt[reg]; i < start[reg + 1]; ++i) stage[i] = REC_PAD;
    }
    const uint32_t t32 = static_cast<uint32_t>(tbase);
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
        const uint32_t e = r * TT + threadIdx.x;
        if (e < kc_left) {
            const uint32_t slot = atomicAdd(&fill[bk[r] >> rg.shift], 1u);
            stage[slot] = t32 + e;
            if constexpr (ORDER) slot_of[tbase + e] = static_cast<uint16_t>(slot);
        }
    }
    // (no early exit on overflow: an overflowed run is written to the start
    // of the overflow slab, which stays in bounds, and RD recomputes the whole
    // chunk directly whenever the flag is set)
    // staged tile -> slabs: one bulk copy per run (32-B aligned on both
    // sides, whole 32-B groups), issued by the run's thread once every
    // thread's generic-proxy stage writes are ordered before the async proxy
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const uint64_t pol = policy_evict_first();
    bool issued = false;
    // run reg is issued by lane reg / WARPS of warp reg % WARPS: the per-lane
    // issue loop the bulk copy compiles to is spread over every warp
    constexpr uint32_t WARPS = TT / 32;
    for (uint32_t reg = warp + WARPS * lane; reg < nreg; reg += TT) {
        const uint32_t len = start[reg + 1] - start[reg];
        if (len) {
            WRS_CHECK(goff[reg] % RUN_ALIGN == 0 &&
                      goff[reg] + len <= static_cast<uint64_t>(rg.nreg) * rg.cap + rg.ov_cap);
            const unsigned src = static_cast<unsigned>(__cvta_generic_to_shared(stage + start[reg]));
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
                         :: "l"(rec + goff[reg]), "r"(src),
                            "r"(len * static_cast<uint32_t>(sizeof(Rec))), "l"(pol) : "memory");
            issued = true;
        }
    }
    if (issued) {  // the stage must stay intact until the copies have read it
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
}

// End of the written records of slab `slab` (nreg = the overflow slab):
// cursor[0, nreg) are the region fill cursors, cursor[nreg] the overflow
// slab's, cursor[nreg + 1 + r] the base of region r's first run that did not
// fit (~0 if none; every run claimed below it was written).
// p0: a position inside the slab (the overflow slab may be longer than cap).
__device__ __forceinline__ uint64_t slab_valid_end(const RegionGeom& rg, const uint32_t* cursor,
                                                   uint64_t p0) {
    const uint32_t slab = static_cast<uint32_t>(umin64(p0 / rg.cap, rg.nreg));
    const uint64_t slab0 = static_cast<uint64_t>(slab) * rg.cap;
    if (slab < rg.nreg)
        return slab0 + umin64(umin64(cursor[slab], rg.cap), cursor[rg.nreg + 1 + slab]);
    return slab0 + umin64(cursor[rg.nreg], rg.ov_cap);
}

// RC: slab by slab, the coin flip of every record against its bucket.  One
// contiguous run of RC_SPAN slab positions per CTA, so the resident CTAs of the
// GPU sweep the table region by region; table loads are marked evict-last,
// record / result streams evict-first.
template <bool W1, bool PHX = false>
__global__ void __launch_bounds__(256, RC_MIN_CTAS)
k_region_gather(RegionGeom rg, const Bucket* __restrict__ b, const uint32_t* __restrict__ cursor,
                const unsigned* __restrict__ overflow, const uint32_t* __restrict__ rec,
                uint32_t* __restrict__ res) {
    if (*overflow) return;  // the overflow slab overflowed: RD recomputes the chunk directly
    const uint64_t p0 = static_cast<uint64_t>(blockIdx.x) * RC_SPAN;
    const uint64_t valid_end = slab_valid_end(rg, cursor, p0);
    if (p0 >= valid_end) return;
    const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
    KeyCache kc;
    const uint64_t key0 = rng_derive(rg.g.base_key, 0);  // W1: the single worker's key
    const uint32_t n32 = static_cast<uint32_t>(rg.g.n);
    // the records are draw indices: each draw's counter, bucket and coin are
    // recomputed here from the counter-based stream (the gather has issue
    // slots to spare; the scatter writes and this kernel reads 4 B per
    // record instead of 8)
    auto ctr1 = [&](uint32_t e) -> uint64_t {
        const uint64_t q = rg.q0 + e;
        if (W1) return key0 + (2 * q + 1) * kGolden;
        uint32_t w;
        uint64_t m;
        locate(rg.g, q, w, m);
        return kc.get(rg.g, w) + (2 * m + 1) * kGolden;
    };
    uint32_t r[RC_ROWS];
    double xph[RC_ROWS];  // Philox mode: the coins, from the same evaluation as the buckets
#pragma unroll
    for (int u = 0; u < RC_ROWS; ++u) {
        const uint64_t p = p0 + u * 256 + threadIdx.x;
        r[u] = p < valid_end ? ld_stream(rec + p, pf) : REC_PAD;
    }
    // bucket gathers as LDGSTS into shared memory: measured 232 G random
    // L2-resident 16-B rows/s vs 200 G for LDG (scripts/microbench/
    // l2_gather_bench.cu); each thread reads back only its own rows.
    // Padding records (REC_PAD) are skipped.
    __shared__ uint4 bk_s[RC_ROWS * 256];
#pragma unroll
    for (int u = 0; u < RC_ROWS; ++u) {
        const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(&bk_s[u * 256 + threadIdx.x]));
        if (r[u] != REC_PAD) {
            uint32_t bi;
            uint64_t c1 = 0;
            if constexpr (PHX) {
                philox_draw(rg.g, rg.q0 + r[u], bi, xph[u]);
            } else {
                c1 = ctr1(r[u]);
                bi = mulhi_n32(mix64(c1), n32);
            }
            WRS_CHECK(bi < rg.g.n);
            asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n"
                         ::"r"(s), "l"(b + bi), "l"(pl) : "memory");
#if RC_COIN_EARLY
            // the coin while the row is in flight (not after the wait)
            if constexpr (!PHX) xph[u] = coin_of_ctr(rg.g, c1);
#endif
        }
    }
    cp_async_commit();
    cp_async_wait<0>();
#pragma unroll
    for (int u = 0; u < RC_ROWS; ++u) {
        const uint64_t p = p0 + u * 256 + threadIdx.x;
        const uint4 bk = bk_s[u * 256 + threadIdx.x];
        if (r[u] != REC_PAD) {  // (positions past valid_end read as padding)
            double x;
            if constexpr (PHX || RC_COIN_EARLY)
                x = xph[u];
            else
                x = coin_of_ctr(rg.g, ctr1(r[u]));
            st_stream(res + p, pick(bk, x), pf);
        }
    }
}

// RD: results back to draw order.  Each region run of the tile is read as one
// contiguous block into shared memory at its tile-local start; every draw
// then picks its answer at the slot RB recorded for it.  If a slab ever
// overflowed (not expected: ~20 sigma of slack), the tile recomputes its
// draws directly instead, so the output is correct in every case.
template <bool W1, bool PHX = false, int TT = RS_THREADS, bool BULK = true>
__global__ void __launch_bounds__(TT, RD_MIN_CTAS * 256 / TT)
k_region_unpermute(RegionGeom rg, const Bucket* __restrict__ b,
                   const unsigned* __restrict__ overflow, const RunInfo* __restrict__ runs,
                   const uint16_t* __restrict__ slot_of, const uint32_t* __restrict__ res,
                   uint32_t out_base, uint32_t* __restrict__ out) {
    extern __shared__ __align__(16) uint32_t stage[];  // stage_slots() results (padded runs)
    const uint64_t tile = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t tbase = tile * (TT * RS_ROWS);
    const uint32_t tcount = static_cast<uint32_t>(umin64((TT * RS_ROWS), rg.kc - tbase));
    if (*overflow) {
        DrawCursor<W1> cur;
        cur.init(rg.g, rg.q0 + tbase + threadIdx.x);
        for (uint32_t e = threadIdx.x; e < tcount; e += TT) {
            const uint64_t q = rg.q0 + tbase + e;
            if constexpr (PHX) {
                uint32_t bb;
                double xx;
                philox_draw(rg.g, q, bb, xx);
                out[tbase + e] = pick(ld_bucket(b, bb), xx) + out_base;
                continue;
            }
            const uint64_t c1 = cur.ctr1(rg.g, q);
            out[tbase + e] = pick(ld_bucket(b, bucket_of_ctr(rg.g, c1)), coin_of_ctr(rg.g, c1)) +
                             out_base;
        }
        return;
    }
    const RunInfo* tr = runs + tile * rg.nreg;
    // full tiles with a 16-B aligned output: each thread owns 4 consecutive
    // draws per pass (one 8-B slot vector, one 16-B output store); the slot
    // vectors are loaded first so they are in flight during the staging
    constexpr int VP = (TT * RS_ROWS) / (TT * 4);  // passes of 4 draws
    const bool vec = tcount == (TT * RS_ROWS) && (reinterpret_cast<uintptr_t>(out + tbase) & 15) == 0;
    uint2 sv[VP];
    if (vec) {
#pragma unroll
        for (int i = 0; i < VP; ++i)
            sv[i] = *reinterpret_cast<const uint2*>(slot_of + tbase + (i * TT + threadIdx.x) * 4);
    }
    constexpr uint32_t WARPS = TT / 32;
    if constexpr (BULK) {
        // this tile's runs -> shared memory, one cp.async.bulk per run (runs
        // are padded to 4 results: 16-B aligned and sized on both sides),
        // completion counted on one mbarrier expecting the tile's padded
        // total.  Run reg is issued by lane reg / WARPS of warp reg % WARPS,
        // so the per-lane issue loop the bulk copy compiles to stays short in
        // every warp.  (~11 instructions per run instead of ~50 for a warp-
        // wide LDGSTS loop: the difference at 256 regions per tile, n = 2^30.)
        __shared__ uint64_t mbar;
        if (threadIdx.x == 0) mbar_init(&mbar, 1);
        __syncthreads();
        if (threadIdx.x == 0) mbar_expect(&mbar, tr[rg.nreg - 1].end * 4u);
        for (uint32_t reg = warp + WARPS * lane; reg < rg.nreg; reg += 32 * WARPS) {
            const uint32_t loc = reg ? tr[reg - 1].end : 0u;
            const RunInfo ri = tr[reg];
            const uint32_t len = ri.end - loc;
            WRS_CHECK(ri.goff % RUN_ALIGN == 0 && loc % RUN_ALIGN == 0 && len % RUN_ALIGN == 0 &&
                      ri.end <= stage_slots(rg.nreg, TT * RS_ROWS));
            if (len) bulk_g2s(&stage[loc], res + ri.goff, len * 4u, &mbar);
        }
        mbar_wait(&mbar, 0);
    }
    // this tile's runs -> shared memory with 16-B LDGSTS (runs are padded to
    // 4 results, 16-B aligned in the slab and the stage): no register
    // staging, so every element of the tile is in flight at once.  Warp w
    // owns runs w, w + WARPS, ...; their descriptors are loaded by one lane
    // each, all at once, and handed round by shuffles.
    const uint32_t ldgsts_regions = BULK ? 0u : rg.nreg;  // (the bulk form staged above)
    for (uint32_t r0 = warp; r0 < ldgsts_regions; r0 += 32 * WARPS) {
        const uint32_t reg = r0 + lane * WARPS;
        uint32_t goff = 0, loc = 0, end = 0;
        if (reg < rg.nreg) {
            const RunInfo ri = tr[reg];
            goff = ri.goff;
            end = ri.end;
            loc = reg ? tr[reg - 1].end : 0u;
        }
        const uint32_t nrun = min(32u, (rg.nreg - r0 + WARPS - 1) / WARPS);
        for (uint32_t j = 0; j < nrun; ++j) {
            const uint32_t g = __shfl_sync(0xffffffffu, goff, j);
            const uint32_t l = __shfl_sync(0xffffffffu, loc, j);
            const uint32_t len = __shfl_sync(0xffffffffu, end, j) - l;
            WRS_CHECK(g % RUN_ALIGN == 0 && l % RUN_ALIGN == 0 && len % RUN_ALIGN == 0 &&
                      l + len <= stage_slots(rg.nreg, TT * RS_ROWS));
            for (uint32_t t = 4 * lane; t < len; t += 128) cp_async16(&stage[l + t], res + g + t);
        }
    }
    if constexpr (!BULK) {
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
    }
    if (vec) {
#pragma unroll
        for (int i = 0; i < VP; ++i) {
            const uint32_t e0 = (i * TT + threadIdx.x) * 4;
            uint4 o;
            o.x = stage[sv[i].x & 0xffffu] + out_base;
            o.y = stage[sv[i].x >> 16] + out_base;
            o.z = stage[sv[i].y & 0xffffu] + out_base;
            o.w = stage[sv[i].y >> 16] + out_base;
            *reinterpret_cast<uint4*>(out + tbase + e0) = o;
        }
    } else {
        for (uint32_t e = threadIdx.x; e < tcount; e += TT) {
            WRS_CHECK(slot_of[tbase + e] < stage_slots(rg.nreg, TT * RS_ROWS));
            out[tbase + e] = stage[slot_of[tbase + e]] + out_base;
        }
    }
}

// ===========================================================================
// aggregated draws: (item, count) pairs of sample_many(seed, k, workers)
//   The draws are the same as above; only their answers are counted.  Each
//   bucket b gets two 32-bit counters: draws answered by b itself
//   (x < share) and draws answered by its alias.  With
//   the region plan the counters of a region are L2-resident while the
//   gather sweeps it.  A fold then adds the own count to count[b] and pushes
//   the alias count to count[alias[b]] (aliases are near b: PSA jobs pair index-
//   ordered lights and heavies), and a compaction writes the nonzero counts in
//   item order.  Chunks of <= 2^31 draws keep each counter below 2^32.
// ===========================================================================
// hits[0, n): draws answered by bucket b itself; hits[n, 2n): by its alias
__device__ __forceinline__ void count_hit(uint32_t* hits, uint64_t n, uint32_t b, bool alias) {
    WRS_CHECK(b < n);
    atomicAdd(hits + (alias ? n + b : b), 1u);
}

template <bool W1, bool PHX = false>
__global__ void __launch_bounds__(256, RC_MIN_CTAS)
k_region_count(RegionGeom rg, const Bucket* __restrict__ b, const uint32_t* __restrict__ cursor,
               const unsigned* __restrict__ overflow, const uint32_t* __restrict__ rec,
               uint32_t* __restrict__ hits) {
    if (*overflow) return;  // k_count_direct<.., true> recounts the chunk
    const uint64_t p0 = static_cast<uint64_t>(blockIdx.x) * RC_SPAN;
    const uint64_t valid_end = slab_valid_end(rg, cursor, p0);
    if (p0 >= valid_end) return;
    const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
    KeyCache kc;
    const uint64_t key0 = rng_derive(rg.g.base_key, 0);
    const uint32_t n32 = static_cast<uint32_t>(rg.g.n);
    // records are draw indices, as for the plain gather: bucket and coin are
    // recomputed here (one counter per draw, kept for the coin)
    uint32_t r[RC_ROWS], bi[RC_ROWS];
    double x[RC_ROWS];
#pragma unroll
    for (int u = 0; u < RC_ROWS; ++u) {
        const uint64_t p = p0 + u * 256 + threadIdx.x;
        r[u] = p < valid_end ? ld_stream(rec + p, pf) : REC_PAD;
    }
    __shared__ uint4 bk_s[RC_ROWS * 256];
#pragma unroll
    for (int u = 0; u < RC_ROWS; ++u) {
        const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(&bk_s[u * 256 + threadIdx.x]));
        bi[u] = 0;
        x[u] = 0.0;
        if (r[u] != REC_PAD) {  // (padding records: no draw)
            const uint64_t q = rg.q0 + r[u];
            if constexpr (PHX) {
                philox_draw(rg.g, q, bi[u], x[u]);
            } else {
                uint64_t c1;
                if (W1) {
                    c1 = key0 + (2 * q + 1) * kGolden;
                } else {
                    uint32_t w;
                    uint64_t m;
                    locate(rg.g, q, w, m);
                    c1 = kc.get(rg.g, w) + (2 * m + 1) * kGolden;
                }
                bi[u] = mulhi_n32(mix64(c1), n32);
                x[u] = coin_of_ctr(rg.g, c1);
            }
            WRS_CHECK(bi[u] < rg.g.n);
            asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n"
                         ::"r"(s), "l"(b + bi[u]), "l"(pl) : "memory");
        }
    }
    cp_async_commit();
    cp_async_wait<0>();
#pragma unroll
    for (int u = 0; u < RC_ROWS; ++u) {
        const uint4 bk = bk_s[u * 256 + threadIdx.x];
        if (r[u] != REC_PAD) {
            const double share = __hiloint2double(static_cast<int>(bk.y), static_cast<int>(bk.x));
            count_hit(hits, rg.g.n, bi[u], x[u] >= share);  // ia[x >= share]
        }
    }
}

// Direct counting of draws [q_begin, q_end): the whole call when the table
// is L2-resident, or (IF_OVERFLOW) the region chunk whose slabs overflowed.
template <bool W1, bool IF_OVERFLOW, bool PHX = false>
__global__ void __launch_bounds__(K5_THREADS)
k_count_direct(const Bucket* __restrict__ b, DrawGeom g, uint64_t q_begin, uint64_t q_end,
               const unsigned* __restrict__ overflow, uint32_t* __restrict__ hits) {
    if (IF_OVERFLOW && !*overflow) return;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * K5_THREADS;
    const uint64_t first = q_begin + static_cast<uint64_t>(blockIdx.x) * K5_THREADS + threadIdx.x;
    DrawCursor<W1> cur;
    cur.init(g, first < q_end ? first : q_begin);
    for (uint64_t q = first; q < q_end; q += stride) {
        uint32_t bi;
        double x;
        if constexpr (PHX) {
            philox_draw(g, q, bi, x);
        } else {
            const uint64_t c1 = cur.ctr1(g, q);
            bi = static_cast<uint32_t>(bucket_of_ctr(g, c1));
            x = coin_of_ctr(g, c1);
        }
        const uint4 bk = ld_bucket(b, bi);
        const double share = __hiloint2double(static_cast<int>(bk.y), static_cast<int>(bk.x));
        count_hit(hits, g.n, bi, x >= share);
    }
}

// Fold: count[b] += own[b], count[alias[b]] += alias hits[b], counters reset.
// Lanes pushing to the same alias (runs of lights share their heavy) combine
// first, so most alias pushes are one atomic per run.
__global__ void __launch_bounds__(256)
k_count_fold(const Bucket* __restrict__ b, uint64_t n, uint32_t* __restrict__ hits,
             unsigned long long* __restrict__ count) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * 256;
    for (uint64_t i0 = static_cast<uint64_t>(blockIdx.x) * 256; i0 < n; i0 += stride) {
        const uint64_t i = i0 + threadIdx.x;
        uint32_t self = 0, al = 0, alias = 0xffffffffu;
        if (i < n) {
            self = hits[i];
            al = hits[n + i];
            if (self) hits[i] = 0;
            if (al) {
                hits[n + i] = 0;
                alias = b[i].alias;
            }
        }
        if (self) atomicAdd(count + i, static_cast<unsigned long long>(self));
        const uint32_t key = al ? alias : 0xffffffffu;
        const unsigned peers = __match_any_sync(0xffffffffu, key);
        const uint32_t sum = __reduce_add_sync(peers, al);
        if (key != 0xffffffffu && (threadIdx.x & 31) == __ffs(peers) - 1)
            atomicAdd(count + key, static_cast<unsigned long long>(sum));
    }
}

// Compaction of the nonzero counts in item order: per-tile counts, one-CTA
// scan, then each tile writes its (item, count) pairs at its offset.
constexpr int CC_THREADS = 256;
constexpr int CC_TILE = CC_THREADS * 16;

__global__ void __launch_bounds__(CC_THREADS)
k_compact_count(const unsigned long long* __restrict__ count, uint64_t n, uint32_t* __restrict__ tile_cnt) {
    const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * CC_TILE;
    uint32_t c = 0;
#pragma unroll 4
    for (int r = 0; r < 16; ++r) {
        const uint64_t i = t0 + r * CC_THREADS + threadIdx.x;
        c += (i < n && count[i] != 0) ? 1u : 0u;
    }
    __shared__ uint32_t red[CC_THREADS / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < CC_THREADS / 32; ++w) t += red[w];
        tile_cnt[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(1024)
k_compact_scan(const uint32_t* __restrict__ tile_cnt, uint64_t ntiles, uint64_t* __restrict__ tile_off,
               unsigned long long* __restrict__ n_unique) {
    __shared__ uint64_t wsum[32];
    __shared__ uint64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint64_t base = 0; base < ntiles; base += 1024) {
        const uint64_t t = base + threadIdx.x;
        const uint64_t c = t < ntiles ? tile_cnt[t] : 0;
        uint64_t x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint64_t v = wsum[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t y = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += y;
            }
            wsum[lane] = v;
        }
        __syncthreads();
        const uint64_t before = carry + (warp ? wsum[warp - 1] : 0) + x - c;
        if (t < ntiles) tile_off[t] = before;
        __syncthreads();
        if (threadIdx.x == 1023) carry = before + c;
        __syncthreads();
    }
    if (threadIdx.x == 0) *n_unique = carry;
}

__global__ void __launch_bounds__(CC_THREADS)
k_compact_write(const unsigned long long* __restrict__ count, uint64_t n,
                const uint64_t* __restrict__ tile_off, uint32_t* __restrict__ items,
                uint64_t* __restrict__ counts) {
    __shared__ uint32_t wcnt[CC_THREADS / 32];
    __shared__ uint64_t base;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * CC_TILE;
    if (threadIdx.x == 0) base = tile_off[blockIdx.x];
    __syncthreads();
    uint64_t run = base;
    // rows of CC_THREADS consecutive items, in order
    for (int r = 0; r < 16; ++r) {
        const uint64_t i = t0 + r * CC_THREADS + threadIdx.x;
        const unsigned long long c = i < n ? count[i] : 0ull;
        const unsigned m = __ballot_sync(0xffffffffu, c != 0);
        if (lane == 0) wcnt[warp] = __popc(m);
        __syncthreads();
        uint32_t before = 0, total = 0;
#pragma unroll
        for (int w = 0; w < CC_THREADS / 32; ++w) {
            const uint32_t v = wcnt[w];
            before += w < warp ? v : 0;
            total += v;
        }
        if (c) {
            const uint64_t o = run + before + __popc(m & lanemask_lt());
            items[o] = static_cast<uint32_t>(i);
            counts[o] = c;
        }
        run += total;
        __syncthreads();
    }
}

// ===========================================================================
// routed two-level draws (two_level.hpp:66-81)
//   Query m of worker w's slice consumes outputs 4m+1..4m+4 of
//   RngStream(seed, '2lvl').derive(w): bucket and coin in the top table pick
//   group g, bucket and coin in g's table the local item; the answer is
//   bases[g] + item.  Group tables may live on peer GPUs (NVLink loads).
// ===========================================================================
template <bool W1>
__global__ void __launch_bounds__(256)
k_two_level_sample(const __grid_constant__ TwoLevelDev tl, DrawGeom g, uint64_t q_begin,
                   uint64_t q_end, uint32_t* __restrict__ out) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * 256;
    const uint64_t first = q_begin + static_cast<uint64_t>(blockIdx.x) * 256 + threadIdx.x;
    if (first >= q_end) return;
    uint32_t w;
    uint64_t m;
    locate(g, first, w, m);
    uint64_t lo = first - m;
    uint64_t hi = W1 ? ~0ull : lo + g.per + (w < g.rem ? 1 : 0);
    uint64_t key = rng_derive(g.base_key, w);
    const uint32_t top_n = static_cast<uint32_t>(tl.groups);
    for (uint64_t q = first; q < q_end; q += stride) {
        if (!W1) {
            while (q >= hi) {
                ++w;
                lo = hi;
                hi = lo + g.per + (w < g.rem ? 1 : 0);
                key = rng_derive(g.base_key, w);
            }
        }
        const uint64_t c = key + (4 * (q - lo) + 1) * kGolden;  // output 4m+1
        // top table: AliasTable::sample (alias.hpp:265-269)
        const uint4 tb = ld_bucket(tl.top, mulhi_n32(mix64(c), top_n));
        const double tx = (static_cast<double>(mix64(c + kGolden) >> 11) * 0x1.0p-53) * tl.top_mean;
        const uint32_t grp = pick(tb, tx);
        WRS_CHECK(grp < tl.groups);
        // the group's own table
        const uint4 lb = ld_bucket(tl.tables[grp],
                                   mulhi_n32(mix64(c + 2 * kGolden), static_cast<uint32_t>(tl.sizes[grp])));
        const double lx =
            (static_cast<double>(mix64(c + 3 * kGolden) >> 11) * 0x1.0p-53) * tl.means[grp];
        out[q - q_begin] = static_cast<uint32_t>(tl.bases[grp]) + pick(lb, lx);
    }
}

// ===========================================================================
// host side
// ===========================================================================
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

__global__ void k_generate_lognormal(double* __restrict__ w, uint64_t n, uint64_t offset,
                                     uint64_t key, double sigma) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += stride)
        w[i] = lognormal_weight(key, offset + i, sigma);  // common.cuh
}

static int sm_count() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

// Region = 2^shift buckets: 32 MB regions up to 2^27 buckets, 64 MB above.
// Measured (1e9 draws, scripts/draw_probe.py): 32 MB wins at n <= 2^26 (8.86
// vs 9.19 ms at 2^26: the 64-MB region crowds the L2 during the gather), the
// two tie at 2^27, 64 MB wins above (9.72 vs 10.19 ms at 2e8, 13.30 vs 15.22
// at 2^30: half the regions, so longer runs per tile and half the per-tile
// scan / claim / run-table work).  WRS_B200_REGION_SHIFT overrides.
static int region_shift(uint64_t n) {
    if (const char* env = getenv("WRS_B200_REGION_SHIFT")) {
        const int v = atoi(env);
        if (v >= 16 && v <= 24) return v;
    }
    return n > (1ull << 27) ? 22 : 21;
}

bool use_region_plan(uint64_t n, uint64_t k) {
    const int sh = region_shift(n);
    const uint64_t nreg = (n + (1ull << sh) - 1) >> sh;
    if (const char* env = getenv("WRS_B200_PLAN")) {  // experiments: force a plan
        if (env[0] == 'd') return false;
        if (env[0] == 'r') return nreg <= RS_MAX_REGIONS;
    }
    // table beyond ~116 MB (measured crossover on B200 with the round-2 region
    // plan: direct / region 7.50 / 7.73 ms per 1e9 draws at 112 MB, 8.39 / 7.59
    // at 128 MB, 9.28 / 7.55 at 144 MB) and enough draws per bucket to reuse
    // the lines
    return n * sizeof(Bucket) > (116ull << 20) && k * 8 >= n && nreg <= RS_MAX_REGIONS;
}

struct RegionPlan {
    RegionGeom rg;
    uint64_t rec_slots;  // nreg * cap + ov_cap
    int tt;              // threads of a scatter / unpermute CTA (tile = tt * RS_ROWS draws)
    uint32_t tile;
};

// Tile size by region count: a tile's runs (one per region) should average
// tens of draws, or the slab writes and the unpermute's run reads fragment
// (measured at n = 2^30, 512 regions: 8 draws per run with 4096-draw tiles).
static int tile_threads_for(uint32_t nreg, bool counts) {
    if (const char* env = getenv("WRS_B200_TILE_THREADS")) {  // tests: force a tile size
        const int t = atoi(env);
        if (t == 256 || t == 512 || t == 1024) return t;
    }
    // (aggregated draws, 4-B records and the 32-row scatter: 1e9 draws at
    // n = 1e8 with 4096 / 8192 / 16384-draw tiles 10.77 / 10.70 / 10.88 ms)
    (void)counts;
    // 8192-draw tiles up to 320 regions, 16384 above (bulk-copied unpermute
    // runs, 32-row scatter; 1e9 draws with 4096 / 8192 / 16384-draw tiles:
    // n = 2e7 7.40 / 7.38 / 7.64 ms, 1e8 7.92 / 7.75 / 7.89, 2^28 8.52 / 8.25 /
    // 8.36, 2^30 11.34 / 10.25 / 10.45; scripts/tt_rows_sweep.sh)
    return nreg <= 320 ? 512 : 1024;
}

static RegionPlan plan_regions(const DrawGeom& g, uint64_t chunk, bool counts = false) {
    RegionPlan p{};
    p.rg.g = g;
    p.rg.shift = region_shift(g.n);
    p.rg.nreg = static_cast<uint32_t>((g.n + (1ull << p.rg.shift) - 1) >> p.rg.shift);
    // expected draws per full region + ~20 sigma + two tiles of slack
    const double mu = static_cast<double>(chunk) *
                      (static_cast<double>(1ull << p.rg.shift) / static_cast<double>(g.n));
    p.tt = tile_threads_for(p.rg.nreg, counts);
    p.tile = static_cast<uint32_t>(p.tt * RS_ROWS);
    // + the runs' padding: up to RUN_ALIGN - 1 slots per (tile, region)
    const double pad = static_cast<double>(RUN_ALIGN - 1) * static_cast<double>((chunk + p.tile - 1) / p.tile);
    const double cap = mu + 20.0 * std::sqrt(mu) + 2.0 * p.tile + pad;
    // slabs are whole multiples of the gather CTA's RC_SPAN positions
    auto round2k = [](uint64_t x) { return static_cast<uint32_t>((x + RC_SPAN - 1) / RC_SPAN * RC_SPAN); };
    const double most = static_cast<double>(chunk) + pad;  // every draw of the chunk in one region
    p.rg.cap = round2k(static_cast<uint64_t>(cap < most ? cap : most) + p.tile);
    p.rg.ov_cap = round2k(chunk / 64 + 8 * p.tile);
    // tests: shrink the slabs to force the redirect / overflow paths
    if (const char* e = getenv("WRS_B200_TEST_SLAB_CAP")) p.rg.cap = round2k(strtoull(e, nullptr, 10));
    if (const char* e = getenv("WRS_B200_TEST_OV_CAP")) p.rg.ov_cap = round2k(strtoull(e, nullptr, 10));
    p.rec_slots = static_cast<uint64_t>(p.rg.nreg) * p.rg.cap + p.rg.ov_cap;
    return p;
}

static uint64_t region_chunk_max() {
    uint64_t chunk_max = 1ull << 30;  // draws per region pass
    if (const char* env = getenv("WRS_B200_DRAW_CHUNK")) {
        const unsigned long long v = strtoull(env, nullptr, 10);
        if (v >= RS_TILE) chunk_max = v < 3500000000ull ? v : 3500000000ull;
    }
    return chunk_max;
}

struct RegionBuffers {
    uint32_t* rec;  // draw-index records
    uint32_t* res;
    uint16_t* slot_of;
    RunInfo* runs;
    uint32_t* cursor;
    unsigned* overflow;
};

// fill cursors and the overflow flag to 0, the failed-run bases to ~0
static cudaError_t reset_cursors(const RegionGeom& rg, const RegionBuffers& B, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(B.cursor, 0, (rg.nreg + 1) * 4, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(B.cursor + rg.nreg + 1, 0xff, rg.nreg * 4, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(B.overflow, 0, 4, st);
    return e;
}

static uint64_t region_bytes(const RegionPlan& p, uint64_t chunk, RegionBuffers* b, void* base) {
    const uint64_t ntiles = (chunk + p.tile - 1) / p.tile;
    uint64_t off = 0;
    auto take = [&](uint64_t bytes) {
        const uint64_t o = off;
        off += (bytes + 255) & ~uint64_t(255);
        return static_cast<char*>(base) + o;
    };
    char* rec = take(p.rec_slots * sizeof(uint32_t));
    char* res = take(p.rec_slots * sizeof(uint32_t));
    char* slot = take(chunk * sizeof(uint16_t));
    char* runs = take(ntiles * p.rg.nreg * sizeof(RunInfo));
    char* cur = take((2 * p.rg.nreg + 1) * 4 + 4);
    if (b) {
        b->rec = reinterpret_cast<uint32_t*>(rec);
        b->res = reinterpret_cast<uint32_t*>(res);
        b->slot_of = reinterpret_cast<uint16_t*>(slot);
        b->runs = reinterpret_cast<RunInfo*>(runs);
        b->cursor = reinterpret_cast<uint32_t*>(cur);
        b->overflow = reinterpret_cast<unsigned*>(cur) + 2 * p.rg.nreg + 1;
    }
    return off;
}

cudaError_t SampleWorkspace::reserve(uint64_t need) {
    if (need <= bytes) return cudaSuccess;
    release();
    cudaError_t e = dev_malloc(&base, need);
    if (e == cudaSuccess) bytes = need;
    return e;
}

void SampleWorkspace::release() {
    if (base) dev_free(base);
    base = nullptr;
    bytes = 0;
}

// RB over a chunk: the full tiles in one launch, the partial last tile (if
// any) in a one-CTA launch of the bounds-checked variant.
template <bool W1, bool ORDER, bool PHX, int TT, int ROWS = RS_ROWS>
static void launch_scatter(const RegionGeom& rg, const RegionBuffers& B, int smem, cudaStream_t s) {
    const uint64_t full = rg.kc / (static_cast<uint64_t>(TT) * ROWS);
    if (full) {
        cudaFuncSetAttribute(k_region_scatter<W1, ORDER, PHX, TT, true, ROWS>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_region_scatter<W1, ORDER, PHX, TT, true, ROWS>,
                             cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
        k_region_scatter<W1, ORDER, PHX, TT, true, ROWS><<<static_cast<unsigned>(full), TT, smem, s>>>(
            rg, 0u, B.cursor, B.overflow, B.rec, B.slot_of, B.runs);
    }
    if (rg.ntiles > full) {
        cudaFuncSetAttribute(k_region_scatter<W1, ORDER, PHX, TT, false, ROWS>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        k_region_scatter<W1, ORDER, PHX, TT, false, ROWS><<<1, TT, smem, s>>>(
            rg, static_cast<uint32_t>(full), B.cursor, B.overflow, B.rec, B.slot_of, B.runs);
    }
}
// The scatter of a TT * 16-draw tile as TT / 2 threads x 32 rows (default)
// or TT / 4 x 64 / TT x 16 (WRS_B200_SCATTER_ROWS=64 / 16, A/B): fewer,
// longer-lived threads per tile (1e9 draws, n = 1e8: scatter 1.88 -> 1.65 ms
// at 8192-draw tiles).
static int scatter_rows() {
    const char* e = getenv("WRS_B200_SCATTER_ROWS");
    const int r = e ? atoi(e) : 32;
    return r == 16 || r == 64 ? r : 32;
}
template <bool W1, bool ORDER, bool PHX, int TT>
static void launch_scatter_tt(const RegionGeom& rg, const RegionBuffers& B, int smem, cudaStream_t s) {
    const int rows = scatter_rows();
    if (rows == 32) return launch_scatter<W1, ORDER, PHX, TT / 2, 32>(rg, B, smem, s);
    if (rows == 64) return launch_scatter<W1, ORDER, PHX, TT / 4, 64>(rg, B, smem, s);
    launch_scatter<W1, ORDER, PHX, TT>(rg, B, smem, s);
}

// RD staging: one bulk copy per run (default) or warp-wide 16-B LDGSTS
// loops (WRS_B200_RD_BULK=0, the earlier form, kept for A/B and tests).
static bool rd_bulk() {
    const char* e = getenv("WRS_B200_RD_BULK");
    return !(e && e[0] == '0');
}
template <bool W1, bool PHX, int TT, bool BULK>
static void launch_unpermute(const RegionGeom& rg, const Bucket* d_b, const RegionBuffers& B,
                             uint32_t base, uint32_t* o, unsigned tiles, int smem, cudaStream_t st) {
    cudaFuncSetAttribute(k_region_unpermute<W1, PHX, TT, BULK>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_region_unpermute<W1, PHX, TT, BULK><<<tiles, TT, smem, st>>>(
        rg, d_b, B.overflow, B.runs, B.slot_of, B.res, base, o);
}

// One chunk of the region plan with TT-thread tiles: RB (on the side stream
// when asked), then RC and RD on st.
template <int TT>
static cudaError_t region_pass(const RegionPlan& plan, const RegionGeom& rg, const DrawGeom& g,
                               const Bucket* d_b, const RegionBuffers& B, uint32_t base,
                               uint32_t* o, cudaStream_t st, bool on_side, cudaStream_t side,
                               cudaEvent_t side_ev) {
    const int sm_scatter = static_cast<int>(scatter_smem_bytes(rg.nreg, plan.tile, sizeof(uint32_t)));
    const int sm_unperm = static_cast<int>(stage_slots(rg.nreg, plan.tile) * sizeof(uint32_t));
    const bool w1 = g.W == 1;
    cudaStream_t ss = on_side ? side : st;
    poison(B.rec, plan.rec_slots * sizeof(uint32_t), ss);  // checked builds only (4-B records)
    poison(B.res, plan.rec_slots * sizeof(uint32_t), ss);
    cudaError_t e = reset_cursors(rg, B, ss);
    if (e != cudaSuccess) return e;
    const unsigned tiles = static_cast<unsigned>(rg.ntiles);
    const uint64_t gblocks = (plan.rec_slots + RC_SPAN - 1) / RC_SPAN;
    if (g.philox)
        launch_scatter_tt<true, true, true, TT>(rg, B, sm_scatter, ss);
    else if (w1)
        launch_scatter_tt<true, true, false, TT>(rg, B, sm_scatter, ss);
    else
        launch_scatter_tt<false, true, false, TT>(rg, B, sm_scatter, ss);
    if (on_side) {
        if ((e = cudaEventRecord(side_ev, side)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(st, side_ev, 0)) != cudaSuccess) return e;
    }
    const unsigned gb = static_cast<unsigned>(gblocks);
    const uint32_t* rec = B.rec;
    if (g.philox)
        k_region_gather<true, true><<<gb, 256, 0, st>>>(rg, d_b, B.cursor, B.overflow, rec, B.res);
    else if (w1)
        k_region_gather<true><<<gb, 256, 0, st>>>(rg, d_b, B.cursor, B.overflow, rec, B.res);
    else
        k_region_gather<false><<<gb, 256, 0, st>>>(rg, d_b, B.cursor, B.overflow, rec, B.res);
    const bool bulk = rd_bulk();
    if (g.philox)
        bulk ? launch_unpermute<true, true, TT, true>(rg, d_b, B, base, o, tiles, sm_unperm, st)
             : launch_unpermute<true, true, TT, false>(rg, d_b, B, base, o, tiles, sm_unperm, st);
    else if (w1)
        bulk ? launch_unpermute<true, false, TT, true>(rg, d_b, B, base, o, tiles, sm_unperm, st)
             : launch_unpermute<true, false, TT, false>(rg, d_b, B, base, o, tiles, sm_unperm, st);
    else
        bulk ? launch_unpermute<false, false, TT, true>(rg, d_b, B, base, o, tiles, sm_unperm, st)
             : launch_unpermute<false, false, TT, false>(rg, d_b, B, base, o, tiles, sm_unperm, st);
    return cudaGetLastError();
}

// Draws per region pass for a plain draw of cnt draws: every pass sweeps the
// whole table once more (16 GB at n = 1e9), so big draws take as few,
// equal passes of up to kPassMax draws as keep the slab positions 32-bit and
// the scratch (~10 B per draw) well inside free device memory; 2^30-draw
// passes otherwise (or what WRS_B200_DRAW_CHUNK says).  1e10 draws: 3 passes
// instead of 5 of 2^31.
static uint64_t draw_chunk_for(const DrawGeom& g, uint64_t cnt, const SampleWorkspace* ws) {
    if (getenv("WRS_B200_DRAW_CHUNK")) return region_chunk_max();
    constexpr uint64_t kBase = 1ull << 30, kPassMax = 3500000000ull;
    if (cnt <= kBase) return kBase;
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
        cudaGetLastError();
        return kBase;
    }
    for (uint64_t passes = (cnt + kPassMax - 1) / kPassMax;; ++passes) {
        const uint64_t c = (cnt + passes - 1) / passes;
        if (c <= kBase) return kBase;
        const RegionPlan p = plan_regions(g, c);
        if (p.rec_slots < (1ull << 32) - RC_SPAN &&
            region_bytes(p, c, nullptr, nullptr) < 0.6 * (free_b + ws->bytes))
            return c;
    }
}

cudaError_t launch_sample(const Bucket* d_b, uint64_t n, double wn, uint64_t seed,
                          uint64_t stream_id, uint64_t q_begin, uint64_t q_end, uint64_t k,
                          uint32_t workers, uint32_t base, uint32_t* d_out, cudaStream_t st,
                          SampleWorkspace* ws, cudaStream_t side, cudaEvent_t side_ev) {
    if (q_end <= q_begin) return cudaSuccess;
    const DrawGeom g = make_geom(n, wn, seed, stream_id, k, workers);
    const uint64_t cnt = q_end - q_begin;
    if (!ws || !use_region_plan(n, cnt)) {
        const uint64_t span = static_cast<uint64_t>(K5_THREADS) * K5_UNROLL;
        uint64_t blocks = (cnt + span - 1) / span;
        const uint64_t cap = static_cast<uint64_t>(sm_count()) * 8 * 64;
        if (blocks > cap) blocks = cap;
        if (g.philox)
            k_sample<true, true><<<static_cast<unsigned>(blocks), K5_THREADS, 0, st>>>(
                d_b, g, q_begin, q_end, base, d_out);
        else if (g.W == 1)
            k_sample<true><<<static_cast<unsigned>(blocks), K5_THREADS, 0, st>>>(d_b, g, q_begin,
                                                                              q_end, base, d_out);
        else
            k_sample<false><<<static_cast<unsigned>(blocks), K5_THREADS, 0, st>>>(d_b, g, q_begin,
                                                                               q_end, base, d_out);
        return cudaGetLastError();
    }
    const uint64_t chunk_max = draw_chunk_for(g, cnt, ws);
    const uint64_t chunk = cnt < chunk_max ? cnt : chunk_max;
    RegionPlan plan = plan_regions(g, chunk);
    cudaError_t e = ws->reserve(region_bytes(plan, chunk, nullptr, nullptr));
    if (e != cudaSuccess) return e;
    RegionBuffers B;
    region_bytes(plan, chunk, &B, ws->base);
    ws->overflow = B.overflow;
    for (uint64_t c0 = q_begin; c0 < q_end; c0 += chunk) {
        RegionGeom rg = plan.rg;
        rg.q0 = c0;
        rg.kc = (q_end - c0) < chunk ? (q_end - c0) : chunk;
        rg.ntiles = (rg.kc + plan.tile - 1) / plan.tile;
        // first chunk's scatter on the side stream (if any): it does not read
        // the table; later chunks reuse the scratch behind RD on st
        const bool on_side = side && side_ev && c0 == q_begin;
        uint32_t* o = d_out + (c0 - q_begin);
        switch (plan.tt) {
            case 256: e = region_pass<256>(plan, rg, g, d_b, B, base, o, st, on_side, side, side_ev); break;
            case 512: e = region_pass<512>(plan, rg, g, d_b, B, base, o, st, on_side, side, side_ev); break;
            default: e = region_pass<1024>(plan, rg, g, d_b, B, base, o, st, on_side, side, side_ev); break;
        }
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// RB for aggregated draws (no slots / run table) at the plan's tile size.
template <bool W1>
static cudaError_t count_scatter(int tt, const RegionGeom& rg, const RegionBuffers& B,
                                 int sm_scatter, cudaStream_t st) {
    // (32 rows per scatter thread, as for plain draws: 10.89 -> 10.77 ms per
    // 1e9 aggregated draws at n = 1e8 with 4-B records)
    switch (tt) {
        case 256: launch_scatter_tt<W1, false, false, 256>(rg, B, sm_scatter, st); break;
        case 512: launch_scatter_tt<W1, false, false, 512>(rg, B, sm_scatter, st); break;
        default: launch_scatter_tt<W1, false, false, 1024>(rg, B, sm_scatter, st); break;
    }
    return cudaGetLastError();
}

cudaError_t CountWorkspace::reserve(uint64_t need) {
    if (need <= n && hits) return cudaSuccess;
    release();
    const uint64_t nt = (need + CC_TILE - 1) / CC_TILE + 1;
    cudaError_t e = dev_malloc(reinterpret_cast<void**>(&hits), 2 * need * sizeof(uint32_t));
    if (e == cudaSuccess) e = dev_malloc(reinterpret_cast<void**>(&count), need * sizeof(unsigned long long));
    if (e == cudaSuccess) e = dev_malloc(reinterpret_cast<void**>(&tile_cnt), nt * sizeof(uint32_t));
    if (e == cudaSuccess) e = dev_malloc(reinterpret_cast<void**>(&tile_off), nt * sizeof(uint64_t));
    if (e != cudaSuccess) {
        release();
        return e;
    }
    n = need;
    return cudaSuccess;
}

void CountWorkspace::release() {
    for (void* p : {static_cast<void*>(hits), static_cast<void*>(count),
                    static_cast<void*>(tile_cnt), static_cast<void*>(tile_off)})
        if (p) dev_free(p);
    hits = nullptr;
    count = nullptr;
    tile_cnt = nullptr;
    tile_off = nullptr;
    n = 0;
}

cudaError_t launch_count(const Bucket* d_b, uint64_t n, double wn, uint64_t seed,
                         uint64_t stream_id, uint64_t k, uint32_t workers, cudaStream_t st,
                         SampleWorkspace* ws, CountWorkspace* cw, uint32_t* d_items,
                         uint64_t* d_counts, unsigned long long* d_n_unique) {
    cudaError_t e = cw->reserve(n);
    if (e != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(cw->hits, 0, 2 * n * sizeof(uint32_t), st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(cw->count, 0, n * sizeof(unsigned long long), st)) != cudaSuccess) return e;
    const DrawGeom g = make_geom(n, wn, seed, stream_id, k, workers);
    const bool w1 = g.W == 1;
    const bool region = ws && use_region_plan(n, k);
    constexpr uint64_t kHalf = 1ull << 31;  // per-fold draws: each counter stays < 2^32
    uint64_t chunk = region ? region_chunk_max() : kHalf;
    if (chunk > kHalf) chunk = kHalf;
    if (chunk > k) chunk = k ? k : 1;
    RegionPlan plan{};
    RegionBuffers B{};
    int sm_scatter = 0;
    if (region) {
        plan = plan_regions(g, chunk, true);
        if ((e = ws->reserve(region_bytes(plan, chunk, nullptr, nullptr))) != cudaSuccess) return e;
        region_bytes(plan, chunk, &B, ws->base);
        ws->overflow = B.overflow;
        sm_scatter = static_cast<int>(scatter_smem_bytes(plan.rg.nreg, plan.tile, sizeof(uint32_t)));
    }
    const unsigned fold_blocks = static_cast<unsigned>(
        umin64((n + 255) / 256, static_cast<uint64_t>(sm_count()) * 8));
    for (uint64_t c0 = 0; c0 < k; c0 += chunk) {
        const uint64_t c1 = k - c0 < chunk ? k : c0 + chunk;
        if (region) {
            RegionGeom rg = plan.rg;
            rg.q0 = c0;
            rg.kc = c1 - c0;
            rg.ntiles = (rg.kc + plan.tile - 1) / plan.tile;
            if ((e = reset_cursors(rg, B, st)) != cudaSuccess) return e;
            const unsigned gblocks = static_cast<unsigned>((plan.rec_slots + RC_SPAN - 1) / RC_SPAN);
            const uint64_t span = static_cast<uint64_t>(K5_THREADS);
            const unsigned dblocks = static_cast<unsigned>(
                umin64((rg.kc + span - 1) / span, static_cast<uint64_t>(sm_count()) * 8));
            if (w1) {
                if ((e = count_scatter<true>(plan.tt, rg, B, sm_scatter, st)) != cudaSuccess) return e;
                k_region_count<true><<<gblocks, 256, 0, st>>>(
                    rg, d_b, B.cursor, B.overflow, B.rec, cw->hits);
                k_count_direct<true, true><<<dblocks, K5_THREADS, 0, st>>>(d_b, g, c0, c1, B.overflow,
                                                                           cw->hits);
            } else {
                if ((e = count_scatter<false>(plan.tt, rg, B, sm_scatter, st)) != cudaSuccess) return e;
                k_region_count<false><<<gblocks, 256, 0, st>>>(
                    rg, d_b, B.cursor, B.overflow, B.rec, cw->hits);
                k_count_direct<false, true><<<dblocks, K5_THREADS, 0, st>>>(d_b, g, c0, c1,
                                                                            B.overflow, cw->hits);
            }
        } else {
            const uint64_t span = static_cast<uint64_t>(K5_THREADS);
            const unsigned dblocks = static_cast<unsigned>(
                umin64((c1 - c0 + span - 1) / span, static_cast<uint64_t>(sm_count()) * 8));
            if (w1)
                k_count_direct<true, false><<<dblocks, K5_THREADS, 0, st>>>(d_b, g, c0, c1, nullptr,
                                                                            cw->hits);
            else
                k_count_direct<false, false><<<dblocks, K5_THREADS, 0, st>>>(d_b, g, c0, c1, nullptr,
                                                                             cw->hits);
        }
        k_count_fold<<<fold_blocks, 256, 0, st>>>(d_b, n, cw->hits, cw->count);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    const uint64_t ntiles = (n + CC_TILE - 1) / CC_TILE;
    k_compact_count<<<static_cast<unsigned>(ntiles), CC_THREADS, 0, st>>>(cw->count, n, cw->tile_cnt);
    k_compact_scan<<<1, 1024, 0, st>>>(cw->tile_cnt, ntiles, cw->tile_off, d_n_unique);
    k_compact_write<<<static_cast<unsigned>(ntiles), CC_THREADS, 0, st>>>(cw->count, n, cw->tile_off,
                                                                         d_items, d_counts);
    return cudaGetLastError();
}

cudaError_t launch_two_level(const TwoLevelDev& tl, uint64_t seed, uint64_t q_begin,
                             uint64_t q_end, uint64_t k, uint32_t workers, uint32_t* d_out,
                             cudaStream_t st) {
    if (q_end <= q_begin) return cudaSuccess;
    const DrawGeom g = make_geom(tl.groups, tl.top_mean, seed, kTwoLevelStream, k, workers);
    uint64_t blocks = (q_end - q_begin + 255) / 256;
    const uint64_t cap = static_cast<uint64_t>(sm_count()) * 16;
    if (blocks > cap) blocks = cap;
    if (g.W == 1)
        k_two_level_sample<true><<<static_cast<unsigned>(blocks), 256, 0, st>>>(tl, g, q_begin,
                                                                                q_end, d_out);
    else
        k_two_level_sample<false><<<static_cast<unsigned>(blocks), 256, 0, st>>>(tl, g, q_begin,
                                                                                 q_end, d_out);
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

cudaError_t launch_generate_lognormal(double* d_w, uint64_t n, uint64_t offset, uint64_t seed,
                                      double sigma, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    uint64_t blocks = (n + 255) / 256;
    const uint64_t cap = static_cast<uint64_t>(sm_count()) * 16;
    if (blocks > cap) blocks = cap;
    k_generate_lognormal<<<static_cast<unsigned>(blocks), 256, 0, st>>>(
        d_w, n, offset, rng_key(seed, kLognStream), sigma);
    return cudaGetLastError();
}

unsigned long long check_failures_sample(unsigned* line) { return tu_check_failures(line); }

}  // namespace wrsb
