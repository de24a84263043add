// paper_1903_00227_b200/csrc/psa_kernels.cu -- the PSA alias-table build on
// sm_100a.  Five stages, each bit-exact with the reference CPU code it
// replaces (line citations are to /root/reference/proj):
//
//   K0  k_total        WeightTable ctor: validation + pairwise_sum tree
//                      (weights.hpp:19-46), one CTA per subtree, top of the
//                      tree combined by arrival counters.
//   K1  k_partition    partition_items' stable light/heavy split
//                      (alias.hpp:48-80): one pass, decoupled look-back,
//                      emits heavy ids and the gathered light / heavy weights
//                      (light ids stay implicit: K4b recovers them).
//   K2a k_scan_blocks  prefix_sums pass 1 (parallel.hpp:110-115): Neumaier
//                      total of every 2048-element block, thread per block,
//                      warp-transposed through shared memory (smaller tables:
//                      k_scan_blocks_direct, register-direct loads, or
//                      k_scan_blocks_split, each chain split over warps).
//   K2b k_scan_carry_split  pass 2 (:116-121): serial Neumaier chain of the
//                      block totals, light and heavy lists in parallel, the
//                      chain's hi / error / lo parts on separate warps
//                      (k_scan_carry: the guarded form, W >= 1e300).
//   K2c k_scan_blocks  pass 3 (:122-129): block chains seeded with the carry,
//                      writing the exclusive prefix arrays (alias.hpp:82-95);
//                      same three forms as K2a.
//   K3  k_split        psa_split binary searches (alias.hpp:122-149), the
//                      same probe sequence, one thread per split.
//   K4a k_pack         psa_pack (alias.hpp:160-209), one lane per job, run in
//                      S-step phases over per-lane windows staged by warp-wide
//                      coalesced async copies; list-order outputs flushed per
//                      phase.
//   K4b k_assemble     the table in index order (full-line 16-B buckets) from
//                      the weights and K4a's list-order outputs.
//
// No stage needs a host round trip: counts live in DevScalars and every grid
// is sized from upper bounds.
#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <cstdio>
#include <math_constants.h>

#include "common.cuh"
#include "engine.h"

namespace wrsb {

// ===========================================================================
// K0: validation + pairwise total
// ===========================================================================
constexpr int K0_NODE = 4096;   // max items of one CTA's subtree
constexpr int K0_THREADS = 128; // >= leaves per subtree (4096 / 32)

__device__ __forceinline__ int pad32(int e) { return e + (e >> 5); }

// (start, size) of node t at `depth` of the floor-halving tree over [0, n)
// (weights.hpp:26-27: left half = n/2).  Caller guarantees every node above
// `depth` is internal.
__host__ __device__ __forceinline__ void tree_node(uint64_t n, int depth, uint64_t t,
                                                   uint64_t& start, uint64_t& size) {
    start = 0;
    size = n;
    for (int l = 0; l < depth; ++l) {
        const uint64_t half = size / 2;
        if ((t >> (depth - 1 - l)) & 1) {
            start += half;
            size -= half;
        } else {
            size = half;
        }
    }
}

__global__ void __launch_bounds__(K0_THREADS)
k_total(const double* __restrict__ w, uint64_t n, int D, double* node_val,
        unsigned* node_cnt, DevScalars* sc) {
    __shared__ double buf[K0_NODE + K0_NODE / 32];
    __shared__ double val[K0_THREADS];
    const int tid = threadIdx.x;
    const uint64_t t = blockIdx.x;
    uint64_t s0, m64;
    tree_node(n, D, t, s0, m64);
    const int m = static_cast<int>(m64);

    // coalesced load + validation (weights.hpp:36-41)
    unsigned long long bad = ~0ull;
    for (int base = 0; base < m; base += K0_THREADS * 8) {
        double xs[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = base + u * K0_THREADS + tid;
            xs[u] = e < m ? __ldg(w + s0 + e) : 1.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = base + u * K0_THREADS + tid;
            if (e < m) {
                const double x = xs[u];
                if (!isfinite(x) || !(x > 0.0)) bad = min(bad, static_cast<unsigned long long>(s0 + e));
                buf[pad32(e)] = x;
            }
        }
    }
    if (bad != ~0ull) atomicMin(&sc->bad_index, bad);

    // subtree depth: smallest d with ceil(m / 2^d) <= 32
    int ds = 0;
    while (((m64 + (1ull << ds) - 1) >> ds) > 32) ++ds;
    __syncthreads();

    // leaves: sequential sums of <= 32 items (weights.hpp:20-24)
    if (tid < (1 << ds)) {
        uint64_t s = 0, sz = m64;
        bool rep = true;
        for (int l = 0; l < ds; ++l) {
            if (sz <= 32) {
                rep = (tid & ((1 << (ds - l)) - 1)) == 0;
                break;
            }
            const uint64_t half = sz / 2;
            if ((tid >> (ds - 1 - l)) & 1) {
                s += half;
                sz -= half;
            } else {
                sz = half;
            }
        }
        if (rep) {
            double acc = 0.0;
            for (int i = 0; i < static_cast<int>(sz); ++i) acc += buf[pad32(static_cast<int>(s) + i)];
            val[tid] = acc;
        }
    }
    // internal nodes inside the subtree: left + right (weights.hpp:27)
    for (int l = ds - 1; l >= 0; --l) {
        __syncthreads();
        if (tid < (1 << l)) {
            uint64_t sz = m64;
            bool exists = true;
            for (int i = 0; i < l; ++i) {
                if (sz <= 32) {
                    exists = false;
                    break;
                }
                sz = ((tid >> (l - 1 - i)) & 1) ? sz - sz / 2 : sz / 2;
            }
            if (exists && sz > 32) {
                const int slot = tid << (ds - l);
                val[slot] = val[slot] + val[slot + (1 << (ds - l - 1))];
            }
        }
    }
    __syncthreads();
    if (tid != 0) return;

    // climb the tree above the cut: the second child to arrive adds.
    double v = val[0];
    uint64_t u = t;
    int l = D;
    node_val[((1ull << l) - 1) + u] = v;
    while (l > 0) {
        __threadfence();
        const unsigned old = atomicAdd(&node_cnt[((1ull << (l - 1)) - 1) + (u >> 1)], 1u);
        if (old == 0) return;
        __threadfence();
        const uint64_t left = u & ~1ull;
        const double vl = __ldcg(&node_val[((1ull << l) - 1) + left]);
        const double vr = __ldcg(&node_val[((1ull << l) - 1) + left + 1]);
        v = vl + vr;
        --l;
        u >>= 1;
        node_val[((1ull << l) - 1) + u] = v;
    }
    sc->total = v;
    sc->wn = v / static_cast<double>(n);  // alias.hpp:50
}

// ===========================================================================
// Tile classification shared by K1 (partition) and K4b (assemble): a tile of
// K1_TILE items, row r covering items [r*256, r*256+256); per (row, warp)
// ballots of light / heavy flags and exclusive light / heavy offsets in index
// order.
// ===========================================================================
#ifndef K1_THREADS_DEF
#define K1_THREADS_DEF 256
#endif
constexpr int K1_THREADS = K1_THREADS_DEF;
constexpr int K1_WARPS = K1_THREADS / 32;
#ifndef K1_ROWS_DEF
#define K1_ROWS_DEF 16
#endif
constexpr int K1_ROWS = K1_ROWS_DEF;
constexpr int K1_TILE = K1_THREADS * K1_ROWS;  // 4096
constexpr int K1_SLOTS = K1_ROWS * (K1_THREADS / 32);  // (row, warp) cells
constexpr int K1_CPL = K1_SLOTS / 32;                  // cells per lane in the tile scan
constexpr unsigned long long FLAG_A = 1ull << 62, FLAG_P = 2ull << 62,
                             VAL_MASK = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long* p) {
    return *reinterpret_cast<const volatile unsigned long long*>(p);
}
__device__ __forceinline__ void st_volatile(unsigned long long* p, unsigned long long v) {
    *reinterpret_cast<volatile unsigned long long*>(p) = v;
}

struct TileCells {
    uint32_t lm[K1_SLOTS], hm[K1_SLOTS];      // ballots per (row, warp)
    uint32_t exL[K1_SLOTS], exH[K1_SLOTS];    // exclusive offsets per cell
    uint32_t totL, totH;
};

// Loads the tile's weights into xs (when KEEP), fills cells (ballots, offsets,
// totals).  Ends with __syncthreads().
// classify_cells: the same from weights already in registers (xs[r] = item
// base + r * K1_THREADS + tid).
__device__ __forceinline__ void classify_cells(const double* xs, uint64_t n, uint64_t base,
                                               double wn, TileCells& C);
template <bool KEEP>
__device__ __forceinline__ void classify_tile(const double* __restrict__ w, uint64_t n,
                                              uint64_t base, double wn, double* xs,
                                              TileCells& C) {
    const int tid = threadIdx.x;
    double x[K1_ROWS];
#pragma unroll
    for (int r = 0; r < K1_ROWS; ++r) {
        const uint64_t gi = base + r * K1_THREADS + tid;
        x[r] = gi < n ? __ldg(w + gi) : 0.0;
        if (KEEP) xs[r] = x[r];
    }
    classify_cells(x, n, base, wn, C);
}

__device__ __forceinline__ void classify_cells(const double* xs, uint64_t n, uint64_t base,
                                               double wn, TileCells& C) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int r = 0; r < K1_ROWS; ++r) {
        const uint64_t gi = base + r * K1_THREADS + tid;
        const double x = xs[r];
        const bool valid = gi < n;
        const bool light = valid && x <= wn;  // ties are light (alias.hpp:60)
        const unsigned lm = __ballot_sync(0xffffffffu, light);
        const unsigned hm = __ballot_sync(0xffffffffu, valid && !light);
        if (lane == 0) {
            C.lm[r * K1_WARPS + warp] = lm;
            C.hm[r * K1_WARPS + warp] = hm;
        }
    }
    __syncthreads();
    if (warp == 0) {
        uint32_t a[K1_CPL], b[K1_CPL], sa = 0, sb = 0;
#pragma unroll
        for (int q = 0; q < K1_CPL; ++q) {
            a[q] = __popc(C.lm[lane * K1_CPL + q]);
            b[q] = __popc(C.hm[lane * K1_CPL + q]);
            sa += a[q];
            sb += b[q];
        }
        uint32_t ia = sa, ib = sb;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t ya = __shfl_up_sync(0xffffffffu, ia, o);
            const uint32_t yb = __shfl_up_sync(0xffffffffu, ib, o);
            if (lane >= o) {
                ia += ya;
                ib += yb;
            }
        }
        uint32_t ea = ia - sa, eb = ib - sb;
#pragma unroll
        for (int q = 0; q < K1_CPL; ++q) {
            C.exL[lane * K1_CPL + q] = ea;
            C.exH[lane * K1_CPL + q] = eb;
            ea += a[q];
            eb += b[q];
        }
        if (lane == 31) {
            C.totL = ia;
            C.totH = ib;
        }
    }
    __syncthreads();
}

#ifndef K1_LOOKBACK_WIN
#define K1_LOOKBACK_WIN 1  // look-back windows of 32 tiles per round (measured: 2, 4, 8 are slower)
#endif
// Decoupled look-back (warp 0 of the tile's CTA): publishes the tile's light
// count, sums predecessors' counts back to the first inclusive prefix, then
// publishes its own inclusive prefix; s_excl = lights before the tile.
__device__ __forceinline__ void k1_lookback(uint64_t tile, uint64_t ntiles, uint64_t n,
                                            uint32_t totL, unsigned long long* status,
                                            DevScalars* sc, unsigned long long& s_excl) {
    const int lane = threadIdx.x & 31;
    unsigned long long excl = 0;
    if (tile == 0) {
        if (lane == 0) st_volatile(&status[0], FLAG_P | totL);
    } else {
        if (lane == 0) st_volatile(&status[tile], FLAG_A | totL);
        // 128 predecessors per round (4 per lane): with hundreds of tiles
        // in flight the inclusive prefixes lag far behind, and a round is
        // one memory latency
        constexpr int LB = K1_LOOKBACK_WIN;
        long long p = static_cast<long long>(tile) - 1;
        while (true) {
            unsigned long long v[LB];
#pragma unroll
            for (int u = 0; u < LB; ++u) {
                const long long idx = p - (u * 32 + lane);
                v[u] = FLAG_P;
                if (idx >= 0) v[u] = ld_volatile(&status[idx]);
            }
#pragma unroll
            for (int u = 0; u < LB; ++u) {
                const long long idx = p - (u * 32 + lane);
                while ((v[u] >> 62) == 0) v[u] = ld_volatile(&status[idx]);
            }
            bool done = false;
#pragma unroll
            for (int u = 0; u < LB; ++u) {
                if (!done) {
                    const unsigned pm = __ballot_sync(0xffffffffu, (v[u] >> 62) == 2);
                    unsigned long long c = v[u] & VAL_MASK;
                    if (pm) {
                        const int first = __ffs(pm) - 1;
                        if (lane > first) c = 0;
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
                    excl += c;
                    done = pm != 0;
                }
            }
            if (done) break;
            p -= 32 * LB;
        }
        if (lane == 0) st_volatile(&status[tile], FLAG_P | (excl + totL));
    }
    if (lane == 0) {
        s_excl = excl;
        if (tile + 1 == ntiles) {
            sc->nl = excl + totL;
            sc->nh = n - (excl + totL);
        }
    }
}

// ===========================================================================
// K1: stable light/heavy partition with decoupled look-back
//   in : w (8 B/item)
//   out: light weights lw (list order), heavy ids + weights hidx/hw.
//   The light ids are never materialised: K4b recovers them from the tile
//   prefix counts this kernel leaves in `status`.
// ===========================================================================
#ifndef K1_MIN_CTAS
#define K1_MIN_CTAS 5  // 48 registers, 42 KB of shared memory: 5 CTAs per SM
#endif
__global__ void __launch_bounds__(K1_THREADS, K1_MIN_CTAS)
k_partition(const double* __restrict__ w, uint64_t n, uint64_t ntiles, DevScalars* sc,
            unsigned long long* status, double* __restrict__ lw, uint32_t* __restrict__ hidx,
            double* __restrict__ hw) {
    extern __shared__ __align__(16) unsigned char k1_smem[];
    double* sw = reinterpret_cast<double*>(k1_smem);              // K1_TILE
    uint16_t* sidx = reinterpret_cast<uint16_t*>(sw + K1_TILE);   // K1_TILE tile-local ids
    __shared__ TileCells C;
    __shared__ unsigned s_tile;
    __shared__ unsigned long long s_excl;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(&sc->tile_counter, 1u);
    __syncthreads();
    const uint64_t tile = s_tile;
    const uint64_t base = tile * K1_TILE;
    double xs[K1_ROWS];
    classify_tile<true>(w, n, base, __ldcg(&sc->wn), xs, C);

    if (warp == 0) {
        const uint32_t totL = C.totL;
        // decoupled look-back for the number of lights before this tile
        unsigned long long excl = 0;
        if (tile == 0) {
            if (lane == 0) st_volatile(&status[0], FLAG_P | totL);
        } else {
            if (lane == 0) st_volatile(&status[tile], FLAG_A | totL);
            long long p = static_cast<long long>(tile) - 1;
            while (true) {
                const long long idx = p - lane;
                unsigned long long v = FLAG_P;
                if (idx >= 0) {
                    do {
                        v = ld_volatile(&status[idx]);
                    } while ((v >> 62) == 0);
                }
                const unsigned pm = __ballot_sync(0xffffffffu, (v >> 62) == 2);
                unsigned long long c = v & VAL_MASK;
                if (pm) {
                    const int first = __ffs(pm) - 1;
                    if (lane > first) c = 0;
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
                excl += c;
                if (pm) break;
                p -= 32;
            }
            if (lane == 0) st_volatile(&status[tile], FLAG_P | (excl + totL));
        }
        if (lane == 0) {
            s_excl = excl;
            if (tile + 1 == ntiles) {
                sc->nl = excl + totL;
                sc->nh = n - (excl + totL);
            }
        }
    }
    // the tile-local compaction does not need the look-back's result: the
    // other warps do it while warp 0 waits on its predecessors
    const uint32_t totL = C.totL, totH = C.totH;
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int r = 0; r < K1_ROWS; ++r) {
        const int cell = r * K1_WARPS + warp;
        const unsigned lm = C.lm[cell], hm = C.hm[cell];
        if ((lm >> lane) & 1) {
            sw[C.exL[cell] + __popc(lm & lt)] = xs[r];
        } else if ((hm >> lane) & 1) {
            const uint32_t p = totL + C.exH[cell] + __popc(hm & lt);
            sidx[p] = static_cast<uint16_t>(r * K1_THREADS + threadIdx.x);
            sw[p] = xs[r];
        }
    }
    __syncthreads();
    const uint64_t L0 = s_excl, H0 = base - s_excl;
    WRS_CHECK(L0 + totL <= n && H0 + totH <= n);
    for (uint32_t p = tid; p < totL; p += K1_THREADS) lw[L0 + p] = sw[p];
    for (uint32_t p = tid; p < totH; p += K1_THREADS) {
        hidx[H0 + p] = static_cast<uint32_t>(base + sidx[totL + p]);
        hw[H0 + p] = sw[totL + p];
    }
}

// K1, unstaged form (the default): the same tile classification and
// look-back, but every thread keeps its 16 weights in registers and, once the
// tile's list offsets are known, writes its lights / heavies straight to their
// list positions (a warp row's lights, and its heavies, are consecutive
// there).  No 40-KB staging buffer and one barrier less per tile; measured at
// n = 1e8: 0.50 vs 0.53 ms for the staged form.
#ifndef K1D_MINB
#define K1D_MINB 5
#endif
__global__ void __launch_bounds__(K1_THREADS, K1D_MINB)
k_partition_direct(const double* __restrict__ w, uint64_t n, uint64_t ntiles, DevScalars* sc,
                   unsigned long long* status, double* __restrict__ lw, uint32_t* __restrict__ hidx,
                   double* __restrict__ hw) {
    __shared__ TileCells C;
    __shared__ unsigned s_tile;
    __shared__ unsigned long long s_excl;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(&sc->tile_counter, 1u);
    __syncthreads();
    const uint64_t tile = s_tile;
    const uint64_t base = tile * K1_TILE;
    double xs[K1_ROWS];
    classify_tile<true>(w, n, base, __ldcg(&sc->wn), xs, C);
    if (warp == 0) k1_lookback(tile, ntiles, n, C.totL, status, sc, s_excl);
    __syncthreads();
    const uint64_t L0 = s_excl, H0 = base - s_excl;
    const unsigned lt = lanemask_lt();
    WRS_CHECK(tile < ntiles && L0 + C.totL <= n && H0 + C.totH <= n);
#pragma unroll
    for (int r = 0; r < K1_ROWS; ++r) {
        const int cell = r * K1_WARPS + warp;
        const unsigned lm = C.lm[cell], hm = C.hm[cell];
        if ((lm >> lane) & 1) {
            lw[L0 + C.exL[cell] + __popc(lm & lt)] = xs[r];
        } else if ((hm >> lane) & 1) {
            const uint64_t p = H0 + C.exH[cell] + __popc(hm & lt);
            hidx[p] = static_cast<uint32_t>(base + r * K1_THREADS + tid);
            hw[p] = xs[r];
        }
    }
}


// ===========================================================================
// K2a / K2c: per-2048-block Neumaier chains, one lane per block
// ===========================================================================
constexpr int SCAN_BLOCK = 2048;  // kScanBlock, parallel.hpp:60
#ifndef K2_WARPS_DEF
#define K2_WARPS_DEF 2
#endif
constexpr int K2_WARPS = K2_WARPS_DEF;
constexpr int K2_C = 32;          // chunk of each block staged per step
#ifndef K2_ROW_UNROLL
#define K2_ROW_UNROLL 4
#endif
constexpr int K2_ROW_U = K2_ROW_UNROLL;  // rows per unrolled step of the staging loops

struct K2Lane {
    const double* src;
    double* dst;
    int len;
};

// PASS3 = false: pass 1 (block totals).  PASS3 = true: pass 3 (prefixes).
// CS = CompSumPos when the weights' total is far below DBL_MAX (every chain
// value is then finite and >= 0), else the guarded CompSum.
template <bool PASS3, class CS>
__global__ void __launch_bounds__(K2_WARPS * 32)
k_scan_blocks(const double* __restrict__ lw, const double* __restrict__ hw,
              double* __restrict__ lpre, double* __restrict__ hpre, const DevScalars* sc,
              double* __restrict__ totals, const double* __restrict__ carries) {
    __shared__ double tile[K2_WARPS][2][32][K2_C + 1];
    __shared__ K2Lane lanes[K2_WARPS][32];
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const uint64_t nl = sc->nl, nh = sc->nh;
    const uint64_t nbl = (nl + SCAN_BLOCK - 1) / SCAN_BLOCK;
    const uint64_t nbh = (nh + SCAN_BLOCK - 1) / SCAN_BLOCK;
    const uint64_t b = (static_cast<uint64_t>(blockIdx.x) * K2_WARPS + wq) * 32 + lane;

    K2Lane me{nullptr, nullptr, 0};
    if (b < nbl) {
        me.src = lw + b * SCAN_BLOCK;
        me.dst = lpre + 1 + b * SCAN_BLOCK;
        me.len = static_cast<int>(umin64(SCAN_BLOCK, nl - b * SCAN_BLOCK));
    } else if (b - nbl < nbh) {
        const uint64_t hb = b - nbl;
        me.src = hw + hb * SCAN_BLOCK;
        me.dst = hpre + 1 + hb * SCAN_BLOCK;
        me.len = static_cast<int>(umin64(SCAN_BLOCK, nh - hb * SCAN_BLOCK));
    }
    lanes[wq][lane] = me;
    int maxlen = me.len;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
    if (maxlen == 0) return;
    __syncwarp();

    const int nchunks = (maxlen + K2_C - 1) / K2_C;
    auto load_chunk = [&](int c, int buf) {
#pragma unroll K2_ROW_U
        for (int r = 0; r < 32; ++r) {
            const K2Lane L = lanes[wq][r];
            const int e = c * K2_C + lane;
            if (e < L.len) cp_async8(&tile[wq][buf][r][lane], L.src + e);
        }
        cp_async_commit();
    };

    CS cs{0.0, 0.0};
    if (PASS3 && me.len > 0) cs.add(carries[b]);  // run.add(carry[b]), parallel.hpp:124
    load_chunk(0, 0);
    for (int c = 0; c < nchunks; ++c) {
        const int buf = c & 1;
        if (c + 1 < nchunks) {
            load_chunk(c + 1, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncwarp();
        const int cnt = min(K2_C, me.len - c * K2_C);
        double* row = tile[wq][buf][lane];
        if (cnt == K2_C) {
            // full chunk: the running (hi, lo) pairs are kept and the outputs
            // hi + lo formed after each group of 8 adds, so the output DADDs
            // do not sit between the adds of the in-order chain
#pragma unroll
            for (int e0 = 0; e0 < K2_C; e0 += 8) {
                double hs[8], ls[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    cs.add(row[e0 + u]);
                    hs[u] = cs.hi;
                    ls[u] = cs.lo;
                }
                if (PASS3) {
#pragma unroll
                    for (int u = 0; u < 8; ++u) row[e0 + u] = hs[u] + ls[u];  // run.value(), :127
                }
            }
        } else {
            for (int e = 0; e < cnt; ++e) {
                cs.add(row[e]);
                if (PASS3) row[e] = cs.value();  // out[i] = run.value(), :127
            }
        }
        __syncwarp();
        if (PASS3) {
#pragma unroll K2_ROW_U
            for (int r = 0; r < 32; ++r) {
                const K2Lane L = lanes[wq][r];
                const int e = c * K2_C + lane;
                if (e < L.len) L.dst[e] = tile[wq][buf][r][lane];
            }
            __syncwarp();
        }
    }
    if (!PASS3 && me.len > 0) totals[b] = cs.value();  // carry[b] = local.value(), :114
}

// K2c, checkpoint form (large tables, W < 1e300): the same block chains as
// k_scan_blocks<true>, but instead of every prefix value it keeps the chain's
// state (hi, lo) BEFORE every 16th element of each block -- 1 B per item
// instead of 8.  K3 only needs prefix values at its probe points, and any
// prefix value is the state at the checkpoint at or before it plus at most
// 16 more compensated adds (k_split_ckpt).  Checkpoint index = position / 16
// (blocks are multiples of 16); the state at a block start is run.add(carry)
// = (carry, 0) exactly (parallel.hpp:124).
constexpr int CK_STRIDE = 16;
typedef double K2Tile[2][32][K2_C + 1];  // one warp's double-buffered block chunks

// acquire load of a progress counter published by another CTA
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Fused K2b+K2c publication flags: per list, one word per chunk of K2F_S
// carries, each on its own 128-B line so the waiting warps poll many lines
// rather than one.  nb_flags = chunk slots per list.
#ifndef K2F_S_DEF
#define K2F_S_DEF 512
#endif
constexpr int K2F_S = K2F_S_DEF;  // totals per chain chunk (publication granularity)
__host__ __device__ inline uint64_t k2_flag_slots(uint64_t n) {
    return ((n + SCAN_BLOCK - 1) / SCAN_BLOCK + 2 + K2F_S - 1) / K2F_S + 1;
}
// (flag lines, then the same number of count lines: K2a units completed per
// chunk of K2F_S blocks, for the launch that also runs K2a)
__host__ __device__ inline uint64_t k2_flag_words(uint64_t n) { return 4 * 32 * k2_flag_slots(n); }
__device__ __forceinline__ const unsigned* k2_flag(const unsigned* f, bool heavy, uint64_t slots,
                                                   uint64_t chunk) {
    return f + 32 * ((heavy ? slots : 0) + chunk);
}
__device__ __forceinline__ unsigned* k2_tdone(unsigned* f, bool heavy, uint64_t slots, uint64_t chunk) {
    return f + 32 * (2 * slots + (heavy ? slots : 0) + chunk);
}

// One warp's 32 block chains of K2c (warp unit `wu` of the launch).  done
// (fused K2b+K2c only): per list, how many carries the chain has published;
// the lane waits for its block's before reading it (the chunk loads are
// already in flight).
__device__ __forceinline__ void ckpt_warp(uint64_t wu, K2Tile& tile, K2Lane* lanes,
                                          const double* __restrict__ lw, const double* __restrict__ hw,
                                          double2* __restrict__ lck, double2* __restrict__ hck,
                                          const DevScalars* sc, const double* carries,
                                          const unsigned* done, uint64_t nb_flags) {
    const int lane = threadIdx.x & 31;
    const uint64_t nl = sc->nl, nh = sc->nh;
    const uint64_t nbl = (nl + SCAN_BLOCK - 1) / SCAN_BLOCK;
    const uint64_t nbh = (nh + SCAN_BLOCK - 1) / SCAN_BLOCK;
    const uint64_t b = wu * 32 + lane;

    K2Lane me{nullptr, nullptr, 0};
    double2* ck = nullptr;
    if (b < nbl) {
        me.src = lw + b * SCAN_BLOCK;
        ck = lck + b * (SCAN_BLOCK / CK_STRIDE);
        me.len = static_cast<int>(umin64(SCAN_BLOCK, nl - b * SCAN_BLOCK));
    } else if (b - nbl < nbh) {
        const uint64_t hb = b - nbl;
        me.src = hw + hb * SCAN_BLOCK;
        ck = hck + hb * (SCAN_BLOCK / CK_STRIDE);
        me.len = static_cast<int>(umin64(SCAN_BLOCK, nh - hb * SCAN_BLOCK));
    }
    lanes[lane] = me;
    int maxlen = me.len;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
    if (maxlen == 0) return;
    __syncwarp();

    const int nchunks = (maxlen + K2_C - 1) / K2_C;
    auto load_chunk = [&](int c, int buf) {
#pragma unroll K2_ROW_U
        for (int r = 0; r < 32; ++r) {
            const K2Lane L = lanes[r];
            const int e = c * K2_C + lane;
            if (e < L.len) cp_async8(&tile[buf][r][lane], L.src + e);
        }
        cp_async_commit();
    };

    load_chunk(0, 0);  // first chunk in flight while the carry arrives
    CompSumPos cs{0.0, 0.0};
    if (me.len > 0) {
        double carry;
        if (done) {  // published by the chain CTA of this launch: acquire, then an L2 load
            const bool heavy = b >= nbl;
            const unsigned* f = k2_flag(done, heavy, nb_flags, (heavy ? b - nbl : b) / K2F_S);
            // relaxed polls (an acquire per poll invalidates the SM's L1 each
            // time), one acquire fence once the flag is seen
            while (*reinterpret_cast<const volatile unsigned*>(f) == 0) __nanosleep(128);
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            carry = __ldcg(carries + b);
        } else {
            carry = __ldg(carries + b);
        }
        cs.add(carry);  // run.add(carry[b]) = (carry, 0), parallel.hpp:124
    }
    for (int c = 0; c < nchunks; ++c) {
        const int buf = c & 1;
        if (c + 1 < nchunks) {
            load_chunk(c + 1, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncwarp();
        const int cnt = min(K2_C, me.len - c * K2_C);
        const double* row = tile[buf][lane];
        if (cnt > 0) {
            // the two checkpoints of this 32-element chunk: one full 32-B sector
            double2 k0, k1;
            k0 = make_double2(cs.hi, cs.lo);
            if (cnt == K2_C) {
#pragma unroll
                for (int e = 0; e < CK_STRIDE; ++e) cs.add(row[e]);
                k1 = make_double2(cs.hi, cs.lo);
#pragma unroll
                for (int e = CK_STRIDE; e < K2_C; ++e) cs.add(row[e]);
            } else {
                k1 = k0;
                for (int e = 0; e < cnt; ++e) {
                    if (e == CK_STRIDE) k1 = make_double2(cs.hi, cs.lo);
                    cs.add(row[e]);
                }
            }
            double2* d = ck + 2 * c;
            WRS_CHECK(static_cast<uint64_t>(c) * K2_C < static_cast<uint64_t>(me.len));
            __stcs(d, k0);
            __stcs(d + 1, k1);
        }
        __syncwarp();
    }
}

__global__ void __launch_bounds__(K2_WARPS * 32)
k_scan_blocks_ckpt(const double* __restrict__ lw, const double* __restrict__ hw,
                   double2* __restrict__ lck, double2* __restrict__ hck, const DevScalars* sc,
                   const double* __restrict__ carries) {
    __shared__ K2Tile tile[K2_WARPS];
    __shared__ K2Lane lanes[K2_WARPS][32];
    const int wq = threadIdx.x >> 5;
    ckpt_warp(static_cast<uint64_t>(blockIdx.x) * K2_WARPS + wq, tile[wq], lanes[wq], lw, hw, lck,
              hck, sc, carries, nullptr, 0);
}

// K2a with TMA bulk copies (experiment, WRS_B200_K2_BULK=1): each warp's
// lane 0 moves the warp's 32 block-chunk rows (256 B each, contiguous in
// global memory) with cp.async.bulk into 16-B-aligned shared rows, completion
// counted on a per-warp, per-buffer mbarrier; the lanes then read their rows
// as 16-B pairs (conflict-free at a 34-double row stride).
template <class CS>
__global__ void __launch_bounds__(K2_WARPS * 32)
k_scan_totals_bulk(const double* __restrict__ lw, const double* __restrict__ hw, const DevScalars* sc,
                   double* __restrict__ totals) {
    __shared__ __align__(16) double tile[K2_WARPS][2][32][K2_C + 2];
    __shared__ K2Lane lanes[K2_WARPS][32];
    __shared__ __align__(8) uint64_t mbar[K2_WARPS][2];
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const uint64_t nl = sc->nl, nh = sc->nh;
    const uint64_t nbl = (nl + SCAN_BLOCK - 1) / SCAN_BLOCK;
    const uint64_t nbh = (nh + SCAN_BLOCK - 1) / SCAN_BLOCK;
    const uint64_t b = (static_cast<uint64_t>(blockIdx.x) * K2_WARPS + wq) * 32 + lane;
    K2Lane me{nullptr, nullptr, 0};
    if (b < nbl) {
        me.src = lw + b * SCAN_BLOCK;
        me.len = static_cast<int>(umin64(SCAN_BLOCK, nl - b * SCAN_BLOCK));
    } else if (b - nbl < nbh) {
        const uint64_t hb = b - nbl;
        me.src = hw + hb * SCAN_BLOCK;
        me.len = static_cast<int>(umin64(SCAN_BLOCK, nh - hb * SCAN_BLOCK));
    }
    lanes[wq][lane] = me;
    int maxlen = me.len;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
    if (maxlen == 0) return;
    if (lane == 0) {
        mbar_init(&mbar[wq][0], 1);
        mbar_init(&mbar[wq][1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int nchunks = (maxlen + K2_C - 1) / K2_C;
    auto load_chunk = [&](int c, int buf) {
        if (lane == 0) {
            unsigned total = 0;
            for (int r = 0; r < 32; ++r) {
                const int len = lanes[wq][r].len - c * K2_C;
                if (len > 0) total += ((min(len, K2_C) * 8 + 15) & ~15);
            }
            mbar_expect(&mbar[wq][buf], total);
            for (int r = 0; r < 32; ++r) {
                const K2Lane L = lanes[wq][r];
                const int len = L.len - c * K2_C;
                if (len > 0)
                    bulk_g2s(&tile[wq][buf][r][0], L.src + c * K2_C,
                             (min(len, K2_C) * 8 + 15) & ~15, &mbar[wq][buf]);
            }
        }
    };
    CS cs{0.0, 0.0};
    unsigned phase[2] = {0, 0};
    load_chunk(0, 0);
    for (int c = 0; c < nchunks; ++c) {
        const int buf = c & 1;
        if (c + 1 < nchunks) load_chunk(c + 1, buf ^ 1);
        mbar_wait(&mbar[wq][buf], phase[buf]);
        phase[buf] ^= 1;
        const int cnt = min(K2_C, me.len - c * K2_C);
        const double2* row = reinterpret_cast<const double2*>(tile[wq][buf][lane]);
        if (cnt == K2_C) {
#pragma unroll
            for (int e = 0; e < K2_C / 2; ++e) {
                const double2 v = row[e];
                cs.add(v.x);
                cs.add(v.y);
            }
        } else {
            const double* r1 = tile[wq][buf][lane];
            for (int e = 0; e < cnt; ++e) cs.add(r1[e]);
        }
        __syncwarp();
    }
    if (me.len > 0) totals[b] = cs.value();  // carry[b] = local.value(), parallel.hpp:114
}

// Small tables (a few block chains per SM, so the chains' latency is the
// kernel's time): one lane per block as above, but the block is read straight
// into registers with 16-B loads, the next 32 elements in flight while the
// current 32 are summed, and (pass 3) written back with 16-B stores (the
// prefix arrays start one element in, so each 32 goes out as 1 + 15 pairs +
// 1).  No staging loop.  Measured per-pass time of a lone 2048-step chain:
// 0.12 / 0.21 ms (k_scan_blocks, pass 1 / 3) -> 0.05 / 0.06 ms.
#ifndef K2S_U_DEF
#define K2S_U_DEF 32
#endif
constexpr int K2S_U = K2S_U_DEF;  // elements per chunk (the next chunk is in flight)

// N adds of a CompSumPos chain over x[], software-pipelined by hand: pairs
// of adds pass through three stages in consecutive steps -- the hi chain
// (t = hi + x), the error terms e = (max - t) + min, the lo chain (lo += e)
// with the run's value t + lo after each add -- and step v runs hi(v),
// e(v-1), lo(v-2) interleaved, so the in-order warp finds independent work
// between the dependent DADDs.  Exactly CompSumPos::add's additions, in order.
template <int N, bool OUT>
__device__ __forceinline__ void chain_pos_pipelined(const double (&x)[N], double (&o)[N],
                                                    CompSumPos& cs) {
    constexpr int B = 2, NB = N / B;
    static_assert(N % B == 0, "pairs");
    double H[3][B], T[3][B], E[3][B];
    double hi = cs.hi, lo = cs.lo;
#pragma unroll
    for (int v = 0; v < NB + 2; ++v) {
        const int sh = v % 3, se = (v + 2) % 3, sl = (v + 1) % 3;  // sets of v, v-1, v-2
#pragma unroll
        for (int u = 0; u < B; ++u) {
            if (v < NB) {
                H[sh][u] = hi;
                T[sh][u] = hi + x[v * B + u];
                hi = T[sh][u];
            }
            if (v >= 1 && v - 1 < NB) {
                const double xv = x[(v - 1) * B + u];
                const bool big = H[se][u] >= xv;
                const double a = big ? H[se][u] : xv, b = big ? xv : H[se][u];
                E[se][u] = (a - T[se][u]) + b;
            }
            if (v >= 2) {
                lo = lo + E[sl][u];
                if (OUT) o[(v - 2) * B + u] = T[sl][u] + lo;
            }
        }
    }
    cs.hi = hi;
    cs.lo = lo;
}
template <int N, bool OUT>
__device__ __forceinline__ void chain_pos_pipelined(const double (&x)[N], double (&o)[N],
                                                    CompSum& cs) {
#pragma unroll
    for (int u = 0; u < N; ++u) {
        cs.add(x[u]);
        if (OUT) o[u] = cs.value();
    }
}
template <bool PASS3, class CS>
__global__ void __launch_bounds__(64)
k_scan_blocks_direct(const double* __restrict__ lw, const double* __restrict__ hw,
                     double* __restrict__ lpre, double* __restrict__ hpre, const DevScalars* sc,
                     double* __restrict__ totals, const double* __restrict__ carries, int lpw) {
    const uint64_t nl = sc->nl, nh = sc->nh;
    const uint64_t nbl = (nl + SCAN_BLOCK - 1) / SCAN_BLOCK;
    const uint64_t nbh = (nh + SCAN_BLOCK - 1) / SCAN_BLOCK;
    // lpw chains per warp: fewer lanes per warp spread the chains over more
    // schedulers (each SMSP's FP64 pipe serves 16 lanes per cycle)
    const int lane = threadIdx.x & 31;
    if (lane >= lpw) return;
    const uint64_t b = (static_cast<uint64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5)) * lpw + lane;
    const double* src;
    double* dst;
    int len;
    if (b < nbl) {
        src = lw + b * SCAN_BLOCK;
        dst = lpre + 1 + b * SCAN_BLOCK;
        len = static_cast<int>(umin64(SCAN_BLOCK, nl - b * SCAN_BLOCK));
    } else if (b - nbl < nbh) {
        const uint64_t hb = b - nbl;
        src = hw + hb * SCAN_BLOCK;
        dst = hpre + 1 + hb * SCAN_BLOCK;
        len = static_cast<int>(umin64(SCAN_BLOCK, nh - hb * SCAN_BLOCK));
    } else {
        return;
    }
    CS cs{0.0, 0.0};
    if (PASS3) cs.add(carries[b]);  // run.add(carry[b]), parallel.hpp:124
    const int full = len / K2S_U;
    double2 nx[K2S_U / 2];
    if (full > 0) {
#pragma unroll
        for (int u = 0; u < K2S_U / 2; ++u) nx[u] = __ldcs(reinterpret_cast<const double2*>(src) + u);
    }
    for (int c = 0; c < full; ++c) {
        double x[K2S_U];
#pragma unroll
        for (int u = 0; u < K2S_U / 2; ++u) {
            x[2 * u] = nx[u].x;
            x[2 * u + 1] = nx[u].y;
        }
        if (c + 1 < full) {
#pragma unroll
            for (int u = 0; u < K2S_U / 2; ++u)
                nx[u] = __ldcs(reinterpret_cast<const double2*>(src + (c + 1) * K2S_U) + u);
        }
        double o[K2S_U];
        chain_pos_pipelined<K2S_U, PASS3>(x, o, cs);  // out[i] = run.value(), parallel.hpp:127
        if (PASS3) {
            double* d = dst + c * K2S_U;  // 8 mod 16: one scalar, pairs, one scalar
            d[0] = o[0];
#pragma unroll
            for (int u = 0; u < K2S_U / 2 - 1; ++u)
                __stcs(reinterpret_cast<double2*>(d + 1) + u, make_double2(o[2 * u + 1], o[2 * u + 2]));
            d[K2S_U - 1] = o[K2S_U - 1];
        }
    }
    for (int e = full * K2S_U; e < len; ++e) {
        cs.add(src[e]);
        if (PASS3) dst[e] = cs.value();
    }
    if (!PASS3 && len > 0) totals[b] = cs.value();  // carry[b] = local.value(), parallel.hpp:114
}

// ===========================================================================
// K2b: serial carry chain over the block totals (parallel.hpp:116-121)
//   CompSumPos (W < 1e300): k_scan_carry_split, the chain's parts on separate
//   warps.  Guarded CompSum: k_scan_carry, one lane per list runs the chain
//   while the rest of the warp streams the totals into shared memory.
// ===========================================================================
constexpr int K2B_CHUNK = 1024;

// K2a / K2c for a few blocks (CompSumPos): one CTA per 2048-block whose warps
// run the parts of the block's chain concurrently, chunk-pipelined like
// k_scan_carry_split -- warp 0 loads chunk c+1 and runs the hi chain of
// chunk c (T[k] = hi = hi + x[k]), warp 1 the error terms of chunk c-1 (all
// lanes), warp 2 the lo chain of chunk c-2 (L[k] = lo after the add), warp 3
// the run's values T[k] + L[k] of chunk c-3 (pass 3, coalesced stores).
// Pass 3 starts from run.add(carry[b]), which leaves (hi, lo) = (carry, 0)
// exactly.  Bit-identical to the single-lane chain; worth it when the chains
// are few enough that their latency is the kernel's time.
constexpr int K2P_C = 256;  // elements per chunk
template <bool PASS3>
__global__ void __launch_bounds__(128)
k_scan_blocks_split(const double* __restrict__ lw, const double* __restrict__ hw,
                    double* __restrict__ lpre, double* __restrict__ hpre, const DevScalars* sc,
                    double* __restrict__ totals, const double* __restrict__ carries) {
    __shared__ __align__(16) double X[3][K2P_C];
    __shared__ __align__(16) double T[4][K2P_C];
    __shared__ __align__(16) double E[2][K2P_C];
    __shared__ __align__(16) double Lo[2][K2P_C];
    __shared__ double hin[4];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t nl = sc->nl, nh = sc->nh;
    const uint64_t nbl = (nl + SCAN_BLOCK - 1) / SCAN_BLOCK;
    const uint64_t nbh = (nh + SCAN_BLOCK - 1) / SCAN_BLOCK;
    const uint64_t b = blockIdx.x;
    const double* src;
    double* dst;
    int len;
    if (b < nbl) {
        src = lw + b * SCAN_BLOCK;
        dst = lpre + 1 + b * SCAN_BLOCK;
        len = static_cast<int>(umin64(SCAN_BLOCK, nl - b * SCAN_BLOCK));
    } else if (b - nbl < nbh) {
        const uint64_t hb = b - nbl;
        src = hw + hb * SCAN_BLOCK;
        dst = hpre + 1 + hb * SCAN_BLOCK;
        len = static_cast<int>(umin64(SCAN_BLOCK, nh - hb * SCAN_BLOCK));
    } else {
        return;
    }
    const int nch = (len + K2P_C - 1) / K2P_C;
    auto cnt_of = [&](int c) { return min(K2P_C, len - c * K2P_C); };
    auto load = [&](int c) {
        if (c < nch) {
            const int cnt = cnt_of(c);
            for (int i = lane; i < cnt; i += 32) cp_async8(&X[c % 3][i], src + c * K2P_C + i);
        }
        cp_async_commit();
    };
    auto h_at = [&](int c, int k) { return k ? T[c % 4][k - 1] : hin[c % 4]; };
    double hi = PASS3 ? carries[b] : 0.0, lo = 0.0;  // run.add(carry[b]) = {carry, 0}
    if (warp == 0) {
        load(0);
        cp_async_wait<0>();
    }
    __syncthreads();
    for (int it = 0; it < nch + 3; ++it) {
        if (warp == 0) {
            load(it + 1);
            const int c = it;
            if (c < nch && lane == 0) {
                const int cnt = cnt_of(c);
                hin[c % 4] = hi;
                int k = 0;
                for (; k + 16 <= cnt; k += 16) {
                    double x[16];
#pragma unroll
                    for (int u = 0; u < 16; ++u) x[u] = X[c % 3][k + u];
#pragma unroll
                    for (int u = 0; u < 16; ++u) {
                        hi = hi + x[u];
                        x[u] = hi;
                    }
#pragma unroll
                    for (int u = 0; u < 16; ++u) T[c % 4][k + u] = x[u];
                }
                for (; k < cnt; ++k) {
                    hi = hi + X[c % 3][k];
                    T[c % 4][k] = hi;
                }
            }
            cp_async_wait<0>();
        } else if (warp == 1) {
            const int c = it - 1;
            if (c >= 0 && c < nch) {
                const int cnt = cnt_of(c);
                for (int k = lane; k < cnt; k += 32) {
                    const double h = h_at(c, k), x = X[c % 3][k];
                    const bool big = h >= x;  // CompSumPos::add
                    const double a = big ? h : x, bb = big ? x : h;
                    E[c % 2][k] = (a - T[c % 4][k]) + bb;
                }
            }
        } else if (warp == 2) {
            const int c = it - 2;
            if (c >= 0 && c < nch && lane == 0) {
                const int cnt = cnt_of(c);
                int k = 0;
                for (; k + 16 <= cnt; k += 16) {
                    double e[16];
#pragma unroll
                    for (int u = 0; u < 16; ++u) e[u] = E[c % 2][k + u];
#pragma unroll
                    for (int u = 0; u < 16; ++u) {
                        lo = lo + e[u];
                        e[u] = lo;
                    }
#pragma unroll
                    for (int u = 0; u < 16; ++u) Lo[c % 2][k + u] = e[u];
                }
                for (; k < cnt; ++k) {
                    lo = lo + E[c % 2][k];
                    Lo[c % 2][k] = lo;
                }
            }
        } else if (PASS3) {
            const int c = it - 3;
            if (c >= 0 && c < nch) {
                const int cnt = cnt_of(c);
                for (int k = lane; k < cnt; k += 32)
                    dst[c * K2P_C + k] = T[c % 4][k] + Lo[c % 2][k];  // run.value(), parallel.hpp:127
            }
        }
        __syncthreads();
    }
    if (!PASS3 && warp == 2 && lane == 0 && len > 0) {
        const int c = nch - 1;  // the last total's hi is in T, its lo in this lane
        totals[b] = T[c % 4][cnt_of(c) - 1] + lo;  // carry[b] = local.value(), parallel.hpp:114
    }
}

// K2b for CompSumPos, split over warps: one CTA per list, whose warps run the
// parts of the compensated chain concurrently on different schedulers, chunk
// by chunk (a CTA barrier between steps):
//   warp 0  streams chunk c+1 of the totals into shared memory;
//   warp 1  the hi chain of chunk c:        T[k] = hi = hi + x[k];
//   warp 2  the error terms of chunk c-1:   e[k] = (max(H, x) - T) + min(H, x),
//           H[k] = T[k-1] (the hi before the add), all lanes;
//   warp 3  the lo chain of chunk c-2:      L[k] = lo, lo = lo + e[k];
//   warp 4  the carries of chunk c-3:       carry[k] = H[k] + L[k], all lanes,
//           coalesced stores.
// The two sequential chains are one dependent DADD per total each, so a step
// costs about one FP64 latency per total instead of a whole compensated add
// issued by one warp (chain_bench: 8.3 vs 22 cycles).  The same additions as
// CompSumPos::add, in the same order: carries are bit-identical.
constexpr int K2W_S = 1024;               // totals per chunk
// x ring RX, T ring 4, e ring 2, L ring 2, hin ring 4
__host__ __device__ constexpr int k2w_smem(int S, int RX) { return (RX + 8) * S * 8 + 4 * 8; }
constexpr int K2W_SMEM = k2w_smem(K2W_S, 3);
// The chain of one list (heavy: the heavy list) over chunks of S totals, the
// totals prefetched D chunks ahead into a ring of RX >= D + 2 buffers (chunk c
// is read in steps c and c + 1).  done (fused K2b+K2c only): the flag line
// of chunk c is released one step after its carries were stored, so the
// fence finds the stores complete instead of stalling the chain.
template <int K2W_S, int D = 1, int RX = 3>
__device__ __forceinline__ void carry_chain(bool heavy, double* k2w, const DevScalars* sc,
                                            const double* __restrict__ totals, double* carries,
                                            double* lpre, double* hpre, unsigned* done,
                                            uint64_t nb_flags, bool wait_totals = false) {
    static_assert(RX >= D + 2, "x ring too short for the prefetch depth");
    double* X = k2w;             // [RX][S] totals
    double* T = X + RX * K2W_S;  // [4][S] hi after each add
    double* E = T + 4 * K2W_S;   // [2][S] error terms
    double* L = E + 2 * K2W_S;   // [2][S] lo before each add
    double* hin = L + 2 * K2W_S;  // [4] hi entering each chunk
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t nl = sc->nl, nh = sc->nh;
    const uint64_t nbl = (nl + SCAN_BLOCK - 1) / SCAN_BLOCK;
    const uint64_t nbh = (nh + SCAN_BLOCK - 1) / SCAN_BLOCK;
    const uint64_t nb = heavy ? nbh : nbl;
    const uint64_t off = heavy ? nbl : 0;
    if (threadIdx.x == 0) (heavy ? hpre : lpre)[0] = 0.0;  // prefix[0] = 0, alias.hpp:89
    if (nb == 0) return;
    const double* src = totals + off;
    double* dst = carries + off;
    const int nch = static_cast<int>((nb + K2W_S - 1) / K2W_S);
    auto cnt_of = [&](int c) {
        return static_cast<int>(umin64(K2W_S, nb - static_cast<uint64_t>(c) * K2W_S));
    };
    auto load = [&](int c) {
        if (c < nch) {
            const int cnt = cnt_of(c);
            if (wait_totals) {  // the chunk's K2a units (same launch) have stored its totals
                if (lane == 0) {
                    const unsigned* t = k2_tdone(done, heavy, nb_flags, c);
                    while (*reinterpret_cast<const volatile unsigned*>(t) < static_cast<unsigned>(cnt))
                        __nanosleep(128);
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                }
                __syncwarp();
            }
            double* xb = X + (c % RX) * K2W_S;
            if (wait_totals) {
                // totals written during this launch: L2 loads (a cp.async may
                // allocate the line in L1, and a line straddling the previous
                // chunk -- the heavy list starts at block nbl -- could then be
                // served stale)
                for (int i = lane; i < cnt; i += 32)
                    xb[i] = __ldcg(src + static_cast<uint64_t>(c) * K2W_S + i);
            } else {
                for (int i = lane; i < cnt; i += 32)
                    cp_async8(xb + i, src + static_cast<uint64_t>(c) * K2W_S + i);
            }
        }
        cp_async_commit();
    };
    // H[k] of chunk c: the hi entering total k
    auto h_at = [&](int c, int k) {
        return k ? T[(c % 4) * K2W_S + k - 1] : hin[c % 4];
    };
    double hi = 0.0, lo = 0.0;  // warp 1 / warp 3, lane 0
    if (warp == 0) {
#pragma unroll
        for (int d = 0; d < D; ++d) load(d);
        cp_async_wait<D - 1>();  // chunk 0 landed
    }
    __syncthreads();
    const int steps = nch + 3 + (done ? 1 : 0);  // + the last chunk's publication
    for (int it = 0; it < steps; ++it) {
        if (warp == 0) {
            load(it + D);  // read by warp 1 D steps from now
        } else if (warp == 1) {
            const int c = it;
            if (c < nch && lane == 0) {
                const int cnt = cnt_of(c);
                const double* __restrict__ xb = X + (c % RX) * K2W_S;
                double* __restrict__ tb = T + (c % 4) * K2W_S;
                hin[c % 4] = hi;
                int k = 0;
                // 16 at a time, the next 16 loaded while these add (the rings
                // never alias): the chain runs at the DADD latency
                double x[16];
                if (cnt >= 16) {
#pragma unroll
                    for (int u = 0; u < 16; ++u) x[u] = xb[u];
                }
                for (; k + 16 <= cnt; k += 16) {
                    // (past the chunk's end these read the next ring buffer or
                    // T, inside the allocation; the values go unused)
                    double y[16];
#pragma unroll
                    for (int u = 0; u < 16; ++u) y[u] = xb[k + 16 + u];
#pragma unroll
                    for (int u = 0; u < 16; ++u) {
                        hi = hi + x[u];
                        x[u] = hi;
                    }
#pragma unroll
                    for (int u = 0; u < 16; ++u) tb[k + u] = x[u];
#pragma unroll
                    for (int u = 0; u < 16; ++u) x[u] = y[u];
                }
                for (; k < cnt; ++k) {
                    hi = hi + xb[k];
                    tb[k] = hi;
                }
            }
        } else if (warp == 2) {
            const int c = it - 1;
            if (c >= 0 && c < nch) {
                const int cnt = cnt_of(c);
                const double* xb = X + (c % RX) * K2W_S;
                const double* tb = T + (c % 4) * K2W_S;
                double* eb = E + (c % 2) * K2W_S;
                for (int k = lane; k < cnt; k += 32) {
                    const double h = h_at(c, k), x = xb[k];
                    const bool big = h >= x;  // CompSumPos::add
                    const double a = big ? h : x, b = big ? x : h;
                    eb[k] = (a - tb[k]) + b;
                }
            }
        } else if (warp == 3) {
            const int c = it - 2;
            if (c >= 0 && c < nch && lane == 0) {
                const int cnt = cnt_of(c);
                const double* __restrict__ eb = E + (c % 2) * K2W_S;
                double* __restrict__ lb = L + (c % 2) * K2W_S;
                int k = 0;
                double e[16];  // as the hi chain: next 16 in flight
                if (cnt >= 16) {
#pragma unroll
                    for (int u = 0; u < 16; ++u) e[u] = eb[u];
                }
                for (; k + 16 <= cnt; k += 16) {
                    double f[16];  // (past the end: E's next buffer or L, unused)
#pragma unroll
                    for (int u = 0; u < 16; ++u) f[u] = eb[k + 16 + u];
#pragma unroll
                    for (int u = 0; u < 16; ++u) {
                        const double l = lo;
                        lo = lo + e[u];
                        e[u] = l;
                    }
#pragma unroll
                    for (int u = 0; u < 16; ++u) lb[k + u] = e[u];
#pragma unroll
                    for (int u = 0; u < 16; ++u) e[u] = f[u];
                }
                for (; k < cnt; ++k) {
                    lb[k] = lo;
                    lo = lo + eb[k];
                }
            }
        } else if (warp == 4) {  // (warps beyond 4, if any, only keep the barriers)
            const int c = it - 3;
            if (done && c >= 1 && c - 1 < nch) {  // chunk c-1, stored a step ago -> its flag
                __threadfence();
                __syncwarp();
                if (lane == 0)
                    asm volatile("st.release.gpu.global.u32 [%0], %1;"
                                 ::"l"(k2_flag(done, heavy, nb_flags, c - 1)), "r"(1u) : "memory");
            }
            if (c >= 0 && c < nch) {
                const int cnt = cnt_of(c);
                const double* lb = L + (c % 2) * K2W_S;
                double* out = dst + static_cast<uint64_t>(c) * K2W_S;
                for (int k = lane; k < cnt; k += 32)
                    out[k] = h_at(c, k) + lb[k];  // carry[b] = acc.value(), parallel.hpp:116-121
            }
        }
        if (warp == 0) cp_async_wait<D - 1>();  // chunk it + 1 landed
        __syncthreads();
    }
}

__global__ void __launch_bounds__(160)
k_scan_carry_split(const DevScalars* sc, const double* __restrict__ totals, double* carries,
                   double* lpre, double* hpre) {
    extern __shared__ __align__(16) double k2w[];
    carry_chain<K2W_S>(blockIdx.x == 1, k2w, sc, totals, carries, lpre, hpre, nullptr, 0);
}

// ---------------------------------------------------------------------------
// K2a / K2c, bulk-copy form (large tables, CompSumPos; the default): a warp
// owns 32 consecutive blocks, one lane each, as before, but each lane's next
// 128 elements (1 KB, contiguous in its block) arrive by one cp.async.bulk
// that the lane issues itself, counted on a per-warp mbarrier, two chunks in
// flight.  The smem-staged form moves 256 B per row per step with one chunk
// in flight, so a warp's 32 blocks take ~0.22 ms however few warps compete
// (measured inside the fused kernel) -- a whole-list wave; here a warp
// streams 32 KB per step and finishes its 32 blocks in tens of microseconds,
// so three warps per SM saturate HBM and the units are short.  Rows are 130
// doubles apart: 16-B aligned for the bulk copy, and lanes r and r + 8 k read
// different 16-B bank groups, so the LDS.128 reads take the minimum 4
// wavefronts.  Same additions in the same order: bit-identical outputs.
#ifndef KB_C_DEF
#define KB_C_DEF 96
#endif
#ifndef KB_NB_DEF
#define KB_NB_DEF 2
#endif
#ifndef KB_WARPS_DEF
#define KB_WARPS_DEF 4
#endif
constexpr int KB_C = KB_C_DEF;          // elements per row chunk
constexpr int KB_RS = KB_C + 2;         // row stride (doubles)
constexpr int KB_NB = KB_NB_DEF;        // chunk buffers per warp
constexpr int KB_WARPS = KB_WARPS_DEF;  // bulk-form warps per CTA (200 KB of rows)
static_assert(KB_C % 32 == 0, "whole 32-element checkpoint pairs per chunk");
struct __align__(128) KBWarp {
    double tile[KB_NB][32][KB_RS];
    uint64_t bar[KB_NB];
};
__device__ __forceinline__ bool mbar_try(uint64_t* b, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok) : "r"((unsigned)__cvta_generic_to_shared(b)), "r"(parity) : "memory");
    return ok != 0;
}
// mbarriers of a warp's buffers (count 1: lane 0's arrive.expect_tx)
__device__ __forceinline__ void kb_init(KBWarp& W) {
    if ((threadIdx.x & 31) == 0) {
        for (int i = 0; i < KB_NB; ++i) mbar_init(&W.bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
}

// One 32-block unit.  CK = false: block totals (pass 1, parallel.hpp:104-114);
// CK = true: checkpoints from run.add(carry[b]) (pass 3 state, :122-127).
// par: the buffers' mbarrier phase bits, carried across units.  flags
// (fused launch only): wait for the chain's flag of the block's carry chunk.
template <bool CK>
__device__ __forceinline__ void kb_unit(uint64_t wu, KBWarp& W, unsigned& par,
                                        const double* __restrict__ lw, const double* __restrict__ hw,
                                        const DevScalars* sc, double* __restrict__ totals,
                                        double2* __restrict__ lck, double2* __restrict__ hck,
                                        const double* carries, const unsigned* flags,
                                        uint64_t nb_flags, double* __restrict__ bmax = nullptr,
                                        unsigned* tdone = nullptr) {
    const int lane = threadIdx.x & 31;
    const uint64_t nl = sc->nl, nh = sc->nh;
    const uint64_t nbl = (nl + SCAN_BLOCK - 1) / SCAN_BLOCK;
    const uint64_t nbh = (nh + SCAN_BLOCK - 1) / SCAN_BLOCK;
    // units alternate between the lists (light 0, heavy 0, light 1, ...):
    // the two chains publish block j's carries at about the same time, so
    // units taken in order follow both chains
    const uint64_t nlu = (nbl + 31) / 32, nhu = (nbh + 31) / 32;
    const uint64_t m = nlu < nhu ? nlu : nhu;
    bool heavy;
    uint64_t idx;
    if (wu < 2 * m) {
        heavy = wu & 1;
        idx = wu >> 1;
    } else {
        heavy = nhu > nlu;
        idx = wu - m;
    }
    const uint64_t j = idx * 32 + lane;  // block within its list
    const double* src = nullptr;
    double2* ck = nullptr;
    int len = 0;
    if (!heavy && j < nbl) {
        src = lw + j * SCAN_BLOCK;
        ck = lck + j * (SCAN_BLOCK / CK_STRIDE);
        len = static_cast<int>(umin64(SCAN_BLOCK, nl - j * SCAN_BLOCK));
    } else if (heavy && j < nbh) {
        src = hw + j * SCAN_BLOCK;
        ck = hck + j * (SCAN_BLOCK / CK_STRIDE);
        len = static_cast<int>(umin64(SCAN_BLOCK, nh - j * SCAN_BLOCK));
    }
    const uint64_t b = heavy ? nbl + j : j;  // index into totals / carries
    int maxlen = len;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
    if (maxlen == 0) return;
    const int nch = (maxlen + KB_C - 1) / KB_C;
    auto issue = [&](int c) {
        const int buf = c % KB_NB;
        const int cnt = max(0, min(KB_C, len - c * KB_C));
        const unsigned bytes = static_cast<unsigned>(cnt & ~1) * 8u;  // whole 16-B pairs
        unsigned tot = bytes;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        // the buffer's last readers are done (__syncwarp in the caller); order
        // their generic-proxy reads before the async-proxy writes
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (lane == 0) mbar_expect(&W.bar[buf], tot);
        if (bytes) bulk_g2s(&W.tile[buf][lane][0], src + c * KB_C, bytes, &W.bar[buf]);
        if (cnt & 1) W.tile[buf][lane][cnt - 1] = __ldg(src + c * KB_C + cnt - 1);  // odd tail
    };
#pragma unroll
    for (int c = 0; c < KB_NB; ++c)
        if (c < nch) issue(c);
    CompSumPos cs{0.0, 0.0};
    // (K2a, heavy blocks) an upper bound of the block's weights for K3's
    // coarse brackets: the largest high word (positive doubles order like
    // their bit patterns), one integer max per element
    const bool want_max = !CK && heavy && bmax;
    int mxh = 0;
    if (CK && len > 0) {
        double carry;
        if (flags) {  // the chain CTA of this launch publishes the carries
            const unsigned* f = k2_flag(flags, heavy, nb_flags, j / K2F_S);
            // relaxed polls (an acquire per poll invalidates the SM's L1), one
            // acquire fence once the flag is seen
            while (*reinterpret_cast<const volatile unsigned*>(f) == 0) __nanosleep(128);
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            carry = __ldcg(carries + b);
        } else {
            carry = __ldg(carries + b);
        }
        cs.add(carry);  // run.add(carry[b]) = (carry, 0), parallel.hpp:124
    }
    for (int c = 0; c < nch; ++c) {
        const int buf = c % KB_NB;
        while (!mbar_try(&W.bar[buf], (par >> buf) & 1u)) {
        }
        par ^= 1u << buf;
        const int cnt = min(KB_C, len - c * KB_C);
        if (cnt == KB_C) {
            const double2* row = reinterpret_cast<const double2*>(&W.tile[buf][lane][0]);
#pragma unroll 1
            for (int q = 0; q < KB_C / 32; ++q) {
                double2 k0, k1;
                k0 = make_double2(cs.hi, cs.lo);
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const double2 v = row[q * 16 + e];
                    cs.add(v.x);
                    cs.add(v.y);
                    if (want_max) mxh = max(mxh, max(__double2hiint(v.x), __double2hiint(v.y)));
                }
                k1 = make_double2(cs.hi, cs.lo);
#pragma unroll
                for (int e = 8; e < 16; ++e) {
                    const double2 v = row[q * 16 + e];
                    cs.add(v.x);
                    cs.add(v.y);
                    if (want_max) mxh = max(mxh, max(__double2hiint(v.x), __double2hiint(v.y)));
                }
                if (CK) {
                    double2* d = ck + (c * KB_C + q * 32) / CK_STRIDE;
                    __stcs(d, k0);
                    __stcs(d + 1, k1);
                }
            }
        } else if (cnt > 0) {
            const double* row = &W.tile[buf][lane][0];
            for (int q = 0; q * 32 < cnt; ++q) {  // 32-element sub-chunks, as k_scan_blocks_ckpt
                const int n32 = min(32, cnt - q * 32);
                double2 k0 = make_double2(cs.hi, cs.lo), k1 = k0;
                for (int e = 0; e < n32; ++e) {
                    if (e == CK_STRIDE) k1 = make_double2(cs.hi, cs.lo);
                    cs.add(row[q * 32 + e]);
                    if (want_max) mxh = max(mxh, __double2hiint(row[q * 32 + e]));
                }
                if (CK) {
                    double2* d = ck + (c * KB_C + q * 32) / CK_STRIDE;
                    __stcs(d, k0);
                    __stcs(d + 1, k1);
                }
            }
        }
        __syncwarp();
        if (c + KB_NB < nch) issue(c + KB_NB);
    }
    if (!CK && len > 0) {
        totals[b] = cs.value();  // carry[b] = local.value(), parallel.hpp:114
        if (want_max) bmax[b] = __hiloint2double(mxh, -1);  // >= every weight of the block
    }
    if (!CK && tdone) {  // one launch with the chain: count this unit's totals in
        __threadfence();
        const unsigned done = __popc(__ballot_sync(0xffffffffu, len > 0));
        if (lane == 0 && done)
            atomicAdd(k2_tdone(tdone, heavy, nb_flags, (idx * 32) / K2F_S), done);
    }
}

// K2a, bulk form: warp units in a grid stride.
__global__ void __launch_bounds__(KB_WARPS * 32, 1)
k_totals_kb(const double* __restrict__ lw, const double* __restrict__ hw, const DevScalars* sc,
            double* __restrict__ totals, uint32_t wunits, double* __restrict__ bmax) {
    extern __shared__ __align__(128) unsigned char kbs[];
    KBWarp& W = reinterpret_cast<KBWarp*>(kbs)[threadIdx.x >> 5];
    kb_init(W);
    unsigned par = 0;
    for (uint32_t wu = blockIdx.x * KB_WARPS + (threadIdx.x >> 5); wu < wunits;
         wu += gridDim.x * KB_WARPS)
        kb_unit<false>(wu, W, par, lw, hw, sc, totals, nullptr, nullptr, nullptr, nullptr, 0, bmax);
}

// K2c, bulk form, after a separate K2b (WRS_B200_K2_FUSE=0).
__global__ void __launch_bounds__(KB_WARPS * 32, 1)
k_ckpt_kb(const double* __restrict__ lw, const double* __restrict__ hw, double2* __restrict__ lck,
          double2* __restrict__ hck, const DevScalars* sc, const double* __restrict__ carries,
          uint32_t wunits) {
    extern __shared__ __align__(128) unsigned char kbs[];
    KBWarp& W = reinterpret_cast<KBWarp*>(kbs)[threadIdx.x >> 5];
    kb_init(W);
    unsigned par = 0;
    for (uint32_t wu = blockIdx.x * KB_WARPS + (threadIdx.x >> 5); wu < wunits;
         wu += gridDim.x * KB_WARPS)
        kb_unit<true>(wu, W, par, lw, hw, sc, nullptr, lck, hck, carries, nullptr, 0);
}
constexpr int KB_SMEM = KB_WARPS * static_cast<int>(sizeof(KBWarp));

// K2b and K2c fused (the checkpoint form): the chain is one dependent FP64
// add per block total -- ~0.16 ms at n = 1e8 on two CTAs while the other SMs
// idle -- so the checkpoint units run concurrently and start each block as
// soon as the chain has published its carry chunk.  CTAs take roles from a
// ticket in the order they start: tickets 0 and 1 run the light / heavy
// chains, every other CTA's warps take 32-block units in order from a
// counter.  A CTA waits only on chain CTAs that already hold their tickets,
// so they are resident and the waits end.
constexpr int K2F_D = 4, K2F_RX = 6;  // chain prefetch depth / x ring (loaded L2 latency)
// one CTA per SM (the bulk rows fill shared memory), so the chain CTAs have
// their SMs to themselves
constexpr int K2F_SMEM = KB_SMEM > k2w_smem(K2F_S, K2F_RX) ? KB_SMEM : k2w_smem(K2F_S, K2F_RX);
constexpr int K2F_THREADS = 32 * (KB_WARPS > 5 ? KB_WARPS : 5);  // chain: 5 warps
__global__ void __launch_bounds__(K2F_THREADS, 1)
k_carry_ckpt(DevScalars* sc, double* totals, double* carries, double* lpre,
             double* hpre, const double* __restrict__ lw, const double* __restrict__ hw,
             double2* __restrict__ lck, double2* __restrict__ hck, unsigned* flags,
             uint64_t nb_flags, uint32_t wunits, uint32_t units_a, double* bmax) {
    extern __shared__ __align__(128) double k2f[];
    __shared__ unsigned role;
    if (threadIdx.x == 0) role = atomicAdd(&sc->k2_ticket, 1u);
    __syncthreads();
    const unsigned t = role;
    if (t < 2) {
        carry_chain<K2F_S, K2F_D, K2F_RX>(t == 1, k2f, sc, totals, carries, lpre, hpre, flags,
                                          nb_flags, units_a > 0);
        return;
    }
    const int wq = threadIdx.x >> 5;
    if (wq >= KB_WARPS) return;
    KBWarp& W = reinterpret_cast<KBWarp*>(k2f)[wq];
    kb_init(W);
    unsigned par = 0;
    const int lane = threadIdx.x & 31;
    // units in order: with units_a > 0 (K2a in this launch too) the K2a units
    // come first -- none of them waits on anything, so the chains they feed
    // always progress -- then the checkpoint units, earliest carries first
    for (;;) {
        unsigned wu = 0;
        if (lane == 0) wu = atomicAdd(&sc->k2_work, 1u);
        wu = __shfl_sync(0xffffffffu, wu, 0);
        if (wu >= units_a + wunits) break;
        if (wu < units_a)
            kb_unit<false>(wu, W, par, lw, hw, sc, totals, nullptr, nullptr, nullptr, nullptr,
                           nb_flags, bmax, flags);
        else
            kb_unit<true>(wu - units_a, W, par, lw, hw, sc, nullptr, lck, hck, carries, flags,
                          nb_flags);
    }
}


template <class CS>
__global__ void __launch_bounds__(32)
k_scan_carry(const DevScalars* sc, const double* __restrict__ totals, double* carries,
             double* lpre, double* hpre) {
    __shared__ __align__(16) double buf[2][K2B_CHUNK];
    const int lane = threadIdx.x;
    const uint64_t nl = sc->nl, nh = sc->nh;
    const uint64_t nbl = (nl + SCAN_BLOCK - 1) / SCAN_BLOCK;
    const uint64_t nbh = (nh + SCAN_BLOCK - 1) / SCAN_BLOCK;
    const bool heavy = blockIdx.x == 1;
    const uint64_t nb = heavy ? nbh : nbl;
    const uint64_t off = heavy ? nbl : 0;
    if (lane == 0) (heavy ? hpre : lpre)[0] = 0.0;  // prefix[0] = 0, alias.hpp:89
    if (nb == 0) return;
    const double* src = totals + off;
    double* dst = carries + off;
    const uint64_t nchunks = (nb + K2B_CHUNK - 1) / K2B_CHUNK;
    auto load = [&](uint64_t c, int bsel) {
        for (int i = lane; i < K2B_CHUNK; i += 32) {
            const uint64_t g = c * K2B_CHUNK + i;
            if (g < nb) cp_async8(&buf[bsel][i], src + g);
        }
        cp_async_commit();
    };
    CS acc{0.0, 0.0};
    load(0, 0);
    for (uint64_t c = 0; c < nchunks; ++c) {
        const int bsel = static_cast<int>(c & 1);
        if (c + 1 < nchunks) {
            load(c + 1, bsel ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncwarp();
        if (lane == 0) {
            const int cnt = static_cast<int>(umin64(K2B_CHUNK, nb - c * K2B_CHUNK));
            double* out = dst + c * K2B_CHUNK;
            const double* in = buf[bsel];
            int i = 0;
            for (; i + 16 <= cnt; i += 16) {
                double t[16], hs[16], ls[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) t[u] = in[i + u];
                // carry[b] = acc.value(), then acc.add(total): keep the (hi, lo)
                // pairs and form the values after the adds (off the chain)
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    hs[u] = acc.hi;
                    ls[u] = acc.lo;
                    acc.add(t[u]);
                }
#pragma unroll
                for (int u = 0; u < 16; ++u) out[i + u] = hs[u] + ls[u];
            }
            for (; i < cnt; ++i) {
                const double t = in[i];
                out[i] = acc.value();
                acc.add(t);
            }
        }
        __syncwarp();
    }
}

// ===========================================================================
// K3: split points (psa_split, alias.hpp:122-149) -- one thread per split
// ===========================================================================
// K3 over checkpointed prefixes (k_scan_blocks_ckpt): the same probe
// sequence as k_split, each probe decided from a bracket first.  The prefix
// value at x lies between the values of the checkpoints around it (prefix
// values of non-negative terms only grow, up to rounding: each is within a
// few ulps of the exact prefix sum), widened by 1e-13 relative; rounding is
// monotone, so f(mid) = (L + H) + w lies between the same expressions of the
// bracket ends.  Only when the target falls inside does the probe recompute
// the exact L and H: the checkpoint state plus <= 16 compensated adds, the
// additions k_scan_blocks<true> makes.  Results are identical to k_split's.
struct CkList {
    const double* w;    // the list's gathered weights
    const double2* ck;  // states before every 16th element
    uint64_t len;
};
__device__ __forceinline__ double ck_value(const CkList& L, uint64_t m) {
    WRS_CHECK(m * CK_STRIDE < L.len);
    const double2 s = __ldg(L.ck + m);
    return s.x + s.y;
}
// exact prefix value at x (alias.hpp:82-95: prefix[x] = out[x-1], prefix[0] = 0)
__device__ __forceinline__ double ck_exact(const CkList& L, uint64_t x) {
    if (x == 0) return 0.0;
    const uint64_t e = x - 1;
    WRS_CHECK(e < L.len);
    const uint64_t base = e & ~static_cast<uint64_t>(CK_STRIDE - 1);
    const int cnt = static_cast<int>(e - base) + 1;
    // all (<= 16) terms in flight at once, then the chain
    double v[CK_STRIDE];
#pragma unroll
    for (int u = 0; u < CK_STRIDE; ++u) v[u] = u < cnt ? __ldg(L.w + base + u) : 0.0;
    const double2 s = __ldg(L.ck + (e / CK_STRIDE));
    CompSumPos cs{s.x, s.y};
#pragma unroll
    for (int u = 0; u < CK_STRIDE; ++u)
        if (u < cnt) cs.add(v[u]);
    return cs.value();
}
__device__ __forceinline__ void ck_bracket(const CkList& L, uint64_t x, double& lo, double& hi) {
    if (x == 0) {
        lo = hi = 0.0;
        return;
    }
    const uint64_t m = (x - 1) / CK_STRIDE;
    lo = ck_value(L, m) * (1.0 - 1e-13);
    hi = (m + 1) * CK_STRIDE < L.len ? ck_value(L, m + 1) * (1.0 + 1e-13) : CUDART_INF;
}

// Where the prefix values K3 probes come from: the full prefix arrays
// (k_scan_blocks<true>) or the checkpoints (k_scan_blocks_ckpt).
struct SplitSrc {
    const double* lpre;
    const double* hpre;
    CkList L, H;
    const double* hw;
    bool ckpt;
    // coarse brackets (checkpoint form with the bulk-copy K2a): the carries
    // (prefix at every block start; light blocks, then heavy from nbl) and
    // the heavy blocks' largest weights decide most probes from L2-resident
    // data before any checkpoint or weight is read
    const double* carries;
    const double* bmax;
    bool coarse;
};

// prefix of a list at x from its block carries: between the carry of x's
// block and the next (widened like ck_bracket; +inf past the last block)
__device__ __forceinline__ void coarse_bracket(const double* car, uint64_t nb, uint64_t x,
                                               double& lo, double& hi) {
    if (x == 0) {
        lo = hi = 0.0;
        return;
    }
    const uint64_t blk = (x - 1) / SCAN_BLOCK;
    lo = __ldg(car + blk) * (1.0 - 1e-13);
    hi = blk + 1 < nb ? __ldg(car + blk + 1) * (1.0 + 1e-13) : CUDART_INF;
}

struct Boundary {
    uint32_t i, j;
    double spill;
};

// Boundary b of psa_plan (alias.hpp:214-238): b = 0 -> (0, 0, w(heavy[0]));
// b = P -> (nl, nh, 0); else psa_split (alias.hpp:122-149) after the first
// n' = ceil(n b / P) buckets, with the reference's probe sequence.  With
// checkpoints every probe is decided from a bracket first: the prefix value
// at x lies between the values of the checkpoints around it (prefix values of
// non-negative terms only grow, up to rounding: each is within a few ulps of
// the exact prefix sum), widened by 1e-13 relative; rounding is monotone, so
// f(mid) = (L + H) + w lies between the same expressions of the bracket ends.
// Only when the target falls inside does the probe recompute the exact L
// and H (the checkpoint state plus <= 16 compensated adds, the additions
// k_scan_blocks<true> makes).  Results are identical either way.
__device__ __forceinline__ Boundary psa_boundary(uint64_t b, uint64_t n, uint64_t P, uint64_t nl,
                                                 uint64_t nh, double wn, const SplitSrc& S) {
    if (b == 0) return Boundary{0u, 0u, __ldg(S.hw)};  // carry of job 0 = w(heavy[0]), alias.hpp:219
    if (b >= P) return Boundary{static_cast<uint32_t>(nl), static_cast<uint32_t>(nh), 0.0};
    const uint64_t m = n * b;
    const uint64_t np = m / P + (m % P != 0);  // alias.hpp:227
    const double target = static_cast<double>(np) * wn;
    uint64_t lo = np > nl ? np - nl : 0;
    uint64_t hi = np < nh ? np : nh;
    while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        bool above;  // f(mid) > target
        if (mid >= nh) {
            above = true;  // f = inf
        } else {
            int coarse = 2;  // 1: above, 0: not, 2: undecided
            if (S.coarse) {
                // f(mid) = (L(np - mid) + H(mid)) + w with w in (wn, block max]
                // (heavies are > wn); floating-point + is monotone, so the
                // bracket ends bound f
                const uint64_t nbl = (nl + SCAN_BLOCK - 1) / SCAN_BLOCK;
                const uint64_t nbh = (nh + SCAN_BLOCK - 1) / SCAN_BLOCK;
                double l0, l1, h0, h1;
                coarse_bracket(S.carries, nbl, np - mid, l0, l1);
                coarse_bracket(S.carries + nbl, nbh, mid, h0, h1);
                if ((l0 + h0) + wn > target)
                    coarse = 1;
                else if ((l1 + h1) + __ldg(S.bmax + nbl + mid / SCAN_BLOCK) <= target)
                    coarse = 0;
            }
            const double w = coarse == 2 ? __ldg(S.hw + mid) : 0.0;
            if (coarse != 2) {
                above = coarse == 1;
            } else if (!S.ckpt) {
                above = (__ldg(S.lpre + (np - mid)) + __ldg(S.hpre + mid)) + w > target;
            } else {
                double l0, l1, h0, h1;
                ck_bracket(S.L, np - mid, l0, l1);
                ck_bracket(S.H, mid, h0, h1);
                if ((l0 + h0) + w > target)
                    above = true;
                else if ((l1 + h1) + w <= target)
                    above = false;
                else
                    above = (ck_exact(S.L, np - mid) + ck_exact(S.H, mid)) + w > target;
            }
        }
        if (above)
            hi = mid;
        else
            lo = mid + 1;
    }
    double spill = 0.0;
    if (lo < nh) {
        const double sig = S.ckpt ? ck_exact(S.L, np - lo) + ck_exact(S.H, lo)
                                  : __ldg(S.lpre + (np - lo)) + __ldg(S.hpre + lo);
        spill = std_max(0.0, (__ldg(S.hw + lo) + sig) - target);
    }
    return Boundary{static_cast<uint32_t>(np - lo), static_cast<uint32_t>(lo), spill};
}

// K3: one thread per boundary.
__global__ void __launch_bounds__(256)
k_split(uint64_t n, uint64_t P, const DevScalars* sc, SplitSrc S, uint32_t* split_l,
        uint32_t* split_h, double* split_s) {
    const uint64_t b = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t nl = sc->nl, nh = sc->nh;
    if (nh == 0 || b > P) return;  // uniform fill, K4
    S.L.len = nl;
    S.H.len = nh;
    const Boundary r = psa_boundary(b, n, P, nl, nh, sc->wn, S);
    split_l[b] = r.i;
    split_h[b] = r.j;
    split_s[b] = r.spill;
}

// ===========================================================================
// K4a: pack (psa_pack, alias.hpp:160-209) -- one lane per job
//   Each lane runs its job's sequential compensated sweep (the remainder
//   chain is not associative, so a job IS a sequential chain; parallelism is
//   the job count).  The lane's light and heavy weights stream through two
//   per-lane rings of K4_R doubles in shared memory, refilled one phase
//   ahead by warp-wide coalesced async copies (one half-warp per lane's row),
//   so the copies of phase p+1 are in flight while phase p sweeps.  Outputs
//   are written back in place (a light slot's low word takes its alias rank,
//   a heavy slot its share) and flushed per phase in list order:
//     lrank[p]  = the heavy RANK j the light at list position p was paired
//                 with (its alias is heavy[min(j, nh-1)], alias.hpp:186-197),
//     hshare[j] = the share of the heavy at list position j.
//   The heavy ids are never read here: K4b maps ranks to ids, and a heavy's
//   alias is always heavy[min(j+1, nh-1)] (alias.hpp:175-183, 200-206), so it
//   needs no output at all.
// ===========================================================================
constexpr int K4_S = 14;          // steps per phase (items consumed per list <= S)
constexpr int K4_R = 32;          // ring slots per list (power of two, >= 2S + 4)
constexpr int K4_RS = K4_R + 2;   // row stride in doubles (16-B aligned rows for the pair copies)
#ifndef K4_WARPS_DEF
#define K4_WARPS_DEF 12           // 17.6 KB of rings per warp: 12 warps fill 211 KB
#endif
constexpr int K4_WARPS = K4_WARPS_DEF;
static_assert(2 * K4_S + 4 <= K4_R, "a refill must not reach the slots of unflushed outputs");

enum : int { ST_MAIN = 0, ST_TAILA = 1, ST_TAILB = 2, ST_DONE = 3 };

struct __align__(16) K4Rings {
    double l[32][K4_RS];  // light weights in, alias ranks (low word) out
    double h[32][K4_RS];  // heavy weights in, shares out
    uint4 pos[32];        // per lane: flush-light, flush-heavy, refill-light, refill-heavy starts
    uint32_t cnt[32];     // per lane: the four counts, one byte each
};
static_assert(K4_WARPS * sizeof(K4Rings) <= 232448, "K4a rings exceed 227 KB of shared memory");

__device__ __forceinline__ uint32_t& low_word(double& d) { return reinterpret_cast<uint32_t*>(&d)[0]; }

// 16-B cp.async, ordered (compiler) after the preceding shared-memory reads of
// this thread; the hardware issues it after them.
__device__ __forceinline__ void cp_async16_ordered(void* smem, const void* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}

// The warp's per-phase data movement over its 32 rings.  Iteration t serves
// rows 4t .. 4t+3, one quarter-warp each; lane q of a quarter handles the
// aligned position pair (2q, 2q+1) past the even position at or below the
// range start (plus 16 per extra pass), for all four ranges of its row:
//   flush : lights [fi, fi + fl) -> lrank (ranks, low words of the light
//           slots), heavies [fj, fj + fh) -> hshare (shares);
//   refill: lights [lf, lf + rl) and heavies [hf, hf + rh), global -> ring,
//           asynchronously, as 16-B pairs (an edge pair also rewrites the
//           neighbouring slot: with its own input if that position is still
//           ahead, or with the pair's other input into the slot of a position
//           32 back, whose output this same pass has already read).
// A refill may target a slot a flush of the same row reads in the same
// iteration: the flush's loads feed its stores, which issue before the copy.
#ifndef K4R_UNROLL
#define K4R_UNROLL 4
#endif
constexpr int K4R_U = K4R_UNROLL;  // row iterations unrolled
template <int PASSES>
__device__ __forceinline__ void k4_rows(K4Rings& R, const double* __restrict__ lw,
                                        const double* __restrict__ hw, uint32_t* __restrict__ lrank,
                                        double* __restrict__ hshare, uint64_t nl, uint64_t nh) {
    const int lane = threadIdx.x & 31;
    const uint32_t q2 = 2u * (lane & 7);
    const int quarter = lane >> 3;
#pragma unroll K4R_U
    for (int t = 0; t < 8; ++t) {
        const int r = 4 * t + quarter;
        const uint4 d = R.pos[r];
        const uint32_t c = R.cnt[r];
        const uint32_t fle = d.x + (c & 0xffu), fhe = d.y + ((c >> 8) & 0xffu);
        const uint32_t rle = d.z + ((c >> 16) & 0xffu), rhe = d.w + (c >> 24);
        // flushes stay inside the lists; refills may read one pair element
        // past a list end (the buffers' slack)
        WRS_CHECK(fle <= nl && fhe <= nh && rle <= nl + 2 && rhe <= nh + 2);
        (void)nl, (void)nh;
        double* const Lr = R.l[r];
        double* const Hr = R.h[r];
#pragma unroll
        for (int ps = 0; ps < PASSES; ++ps) {
            const uint32_t off = q2 + 16u * ps;
            // flush, branch-free: the pair is read whole (one 16-B load), then
            // one of three predicated stores (both elements / first / second)
            {
                const uint32_t b = (d.x & ~1u) + off;
                const bool v0 = b >= d.x && b < fle, v1 = b + 1 < fle;
                const double2 pr = *reinterpret_cast<const double2*>(&Lr[b & (K4_R - 1)]);
                const uint32_t r0 = static_cast<uint32_t>(__double_as_longlong(pr.x));
                const uint32_t r1 = static_cast<uint32_t>(__double_as_longlong(pr.y));
                if (v0 && v1) *reinterpret_cast<uint2*>(lrank + b) = make_uint2(r0, r1);
                if (v0 && !v1) lrank[b] = r0;
                if (!v0 && v1) lrank[b + 1] = r1;
            }
            {
                const uint32_t b = (d.y & ~1u) + off;
                const bool v0 = b >= d.y && b < fhe, v1 = b + 1 < fhe;
                const double2 pr = *reinterpret_cast<const double2*>(&Hr[b & (K4_R - 1)]);
                if (v0 && v1) *reinterpret_cast<double2*>(hshare + b) = pr;
                if (v0 && !v1) hshare[b] = pr.x;
                if (!v0 && v1) hshare[b + 1] = pr.y;
            }
            // refill (pairs; the inputs have >= 64 B of slack past their ends)
            {
                const uint32_t b = (d.z & ~1u) + off;
                if (b < rle && d.z < rle)
                    cp_async16_ordered(&Lr[b & (K4_R - 1)], lw + b);
            }
            {
                const uint32_t b = (d.w & ~1u) + off;
                if (b < rhe && d.w < rhe)
                    cp_async16_ordered(&Hr[b & (K4_R - 1)], hw + b);
            }
        }
    }
}

// FIN: the weights' total is far below DBL_MAX, so the remainder and every
// term stay finite and the comp_sum finite-check never fires (the fast
// phases skip it).
template <bool FIN>
__global__ void __launch_bounds__(K4_WARPS * 32)
k_pack(uint64_t P, DevScalars* sc, const double* __restrict__ lw, const double* __restrict__ hw,
       const uint32_t* __restrict__ split_l, const uint32_t* __restrict__ split_h,
       const double* __restrict__ split_s, uint32_t* __restrict__ lrank,
       double* __restrict__ hshare) {
    extern __shared__ __align__(16) unsigned char k4_smem[];
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    K4Rings& R = reinterpret_cast<K4Rings*>(k4_smem)[wq];
    const uint64_t nh64 = sc->nh;
    if (nh64 == 0) return;  // all items tie with the mean: K4b fills (alias.hpp:288-297)
    const uint32_t hlast = static_cast<uint32_t>(nh64 - 1);  // last heavy position
    const double wn = sc->wn;
    double* const Lr = R.l[lane];
    double* const Hr = R.h[lane];
    auto lslot = [&](uint32_t p) -> double& { return Lr[p & (K4_R - 1)]; };
    auto hslot = [&](uint32_t p) -> double& { return Hr[p & (K4_R - 1)]; };

    const uint64_t k = (static_cast<uint64_t>(blockIdx.x) * (blockDim.x >> 5) + wq) * 32 + lane;
    uint32_t i = 0, lhi = 0, j = 0, hhi = 0;
    int mode = ST_DONE;
    double rhi = 0.0, rlo = 0.0;  // the remainder, comp_sum (parallel.hpp:70-81)
    if (k < P) {
        i = split_l[k];
        lhi = split_l[k + 1];
        j = split_h[k];
        hhi = split_h[k + 1];
        if (lhi < i || hhi < j) {
            atomicOr(&sc->plan_error, 1u);  // alias.hpp:230-231
            lhi = i;
            hhi = j;
        } else {
            mode = ST_MAIN;
            rhi = j < nh64 ? split_s[k] : CUDART_INF;  // alias.hpp:168
        }
    }
    // heavy weights the job reads: positions j+1 .. min(hhi, nh-1)
    const uint32_t hlim = umin64(hhi, hlast);
    const uint32_t hend = mode == ST_DONE ? 0u : hlim + 1;  // exclusive
    uint32_t lfill = i, hfill = j + 1;  // next positions to fetch
    uint32_t fi = i, fj = j;            // first positions not yet flushed

    // post this lane's flush [fi, i), [fj, j) and refill [lfill, i + 2S), [hfill, j + 1 + 2S)
    // (refill ends are rounded up to even positions, so every refill after the
    // prologue starts on a pair boundary and never rewrites a slot behind it;
    // the one extra input read past a range end is never used)
    auto post = [&]() {
        const uint32_t lto = lhi - i > 2 * K4_S ? i + 2 * K4_S : lhi;
        const uint32_t hto = (hend > j + 1 && hend - (j + 1) > 2 * K4_S) ? j + 1 + 2 * K4_S : hend;
        const uint32_t rl = lto > lfill ? ((lto - lfill + (lfill & 1u) + 1u) & ~1u) - (lfill & 1u) : 0u;
        const uint32_t rh = hto > hfill ? ((hto - hfill + (hfill & 1u) + 1u) & ~1u) - (hfill & 1u) : 0u;
        R.pos[lane] = make_uint4(fi, fj, lfill, hfill);
        R.cnt[lane] = (i - fi) | ((j - fj) << 8) | (rl << 16) | (rh << 24);
        lfill += rl;
        hfill += rh;
        fi = i;
        fj = j;
        __syncwarp();
    };
    post();
    k4_rows<2>(R, lw, hw, lrank, hshare, sc->nl, nh64);  // prologue: two phases' worth of inputs
    cp_async_commit();
    cp_async_commit();  // (empty: phase 0 waits for the prologue alone)

    while (__any_sync(0xffffffffu, mode != ST_DONE)) {
        // this phase's inputs (posted two phases ago) have landed; the copies
        // posted at the end of the last phase stay in flight
        cp_async_wait<1>();
        __syncwarp();
        // Fast phase: every lane in the main loop with >= S lights and >= S
        // next heavies left, so no tail loop or last-heavy reset can start:
        // the step is the main loop's body alone (alias.hpp:175-189).
        const bool fast = __all_sync(0xffffffffu, mode == ST_MAIN && lhi - i >= K4_S &&
                                                      hlim >= j + K4_S);
        if (fast) {
#pragma unroll
            for (int s = 0; s < K4_S; ++s) {
                const double v = rhi + rlo;  // rem.value()
                const bool gt = v > wn;
                // the next light w[i] or the next heavy w[j+1], read once the
                // direction is known
                const double x = (gt ? lslot(i) : hslot(j + 1)) - wn;
                // rem.add(x): the guarded Neumaier add, branch-free
                const double t = rhi + x;
                const bool big = fabs(rhi) >= fabs(x);
                const double a = big ? rhi : x, b = big ? x : rhi;
                const double l2 = rlo + ((a - t) + b);
                rlo = (FIN || isfinite(t)) ? l2 : rlo;
                rhi = t;
                if (gt) {  // light bucket {w, {idx, heavy_at(j)}}: rank j
                    low_word(lslot(i)) = j;
                } else {   // heavy bucket {max(0, min(rem, wn)), ...}; rem <= wn here,
                           // so the share is rem if rem > 0 else +0.0.  With FIN, v is
                           // finite, so clearing every bit when the sign is set does
                           // it in integer ops (the compiler's fmax-style sequence
                           // for `v > 0 ? v : 0` was ~10 instructions per step)
                    const long long vb = __double_as_longlong(v);
                    hslot(j) = __longlong_as_double(FIN ? vb & ~(vb >> 63) : (v > 0.0 ? vb : 0ll));
                }
                i += gt;
                j += !gt;
            }
        } else {
#pragma unroll 2
            for (int s = 0; s < K4_S; ++s) {
                const double v = rhi + rlo;
                const bool gt = v > wn;
                const bool lightsLeft = i < lhi, heaviesLeft = j < hhi;
                int st = mode;
                if (st == ST_MAIN && gt && !lightsLeft) st = ST_TAILA;   // alias.hpp:172
                if (st == ST_MAIN && !gt && !heaviesLeft) st = ST_TAILB; // alias.hpp:191
                const bool isMain = st == ST_MAIN;
                const bool lightOp = (isMain && gt) || (st == ST_TAILB && lightsLeft);
                const bool heavyOp = (isMain && !gt) || (st == ST_TAILA && heaviesLeft);
                if (!lightOp && !heavyOp) st = ST_DONE;  // tail loops exhausted: return
                mode = st;
                // remainder: rem.add(w - wn), or the reset at the last heavy
                const bool hasNext = j < hlast;
                const double x = (lightOp ? lslot(i) : hslot(j + 1)) - wn;
                const bool doAdd = (lightOp && isMain) || (heavyOp && hasNext);
                const bool doReset = heavyOp && !hasNext;
                const double t = rhi + x;
                const bool big = fabs(rhi) >= fabs(x);
                const double a = big ? rhi : x, b = big ? x : rhi;
                const double l2 = rlo + ((a - t) + b);
                const double nlo = isfinite(t) ? l2 : rlo;
                const double resetHi = isMain ? CUDART_INF : wn;  // rem = {inf} / rem = {wn}
                // light bucket {w, {idx, heavy_at(j)}} (alias.hpp:186-189, 194-197)
                if (lightOp) low_word(lslot(i)) = j;
                // heavy bucket {clamp(rem), {idx, heavy_at(j+1)}} (alias.hpp:175-183, 200-206)
                if (heavyOp) hslot(j) = isMain ? std_max(0.0, std_min(v, wn)) : std_min(v, wn);
                rhi = doAdd ? t : (doReset ? resetHi : rhi);
                rlo = doAdd ? nlo : (doReset ? 0.0 : rlo);
                i += lightOp;
                j += heavyOp;
            }
        }
        __syncwarp();
        // this phase's outputs out, the phase after next's inputs in
        post();
        k4_rows<1>(R, lw, hw, lrank, hshare, sc->nl, nh64);
        cp_async_commit();
    }
    cp_async_wait<0>();
}

// ===========================================================================
// K4b: assemble the 16-B buckets in index order (one CTA per K1 tile)
//   light item i : {w_i, i, heavy[min(lrank[rank of i], nh-1)]}  (alias.hpp:186-197)
//   heavy item i : {hshare[rank], i, heavy[min(rank+1, nh-1)]}    (alias.hpp:175-206)
//   no heavy at all: {w_i, i, i}                                  (alias.hpp:288-297)
//   Ranks come from the same tile classification as K1 plus K1's inclusive
//   tile prefix; every warp stores 32 consecutive buckets = 512 contiguous B.
// ===========================================================================
#ifndef K4B_SMEM_KB
#define K4B_SMEM_KB 36
#endif
constexpr uint32_t K4B_SMEM = K4B_SMEM_KB * 1024;  // 5 CTAs per SM (the register budget)
#ifndef K4B_KEEP
#define K4B_KEEP 1  // the lights' weights from classify's registers (0.58 vs 0.60 ms)
#endif
#ifndef K4B_PAD_DEF
#define K4B_PAD_DEF 64
#endif
constexpr uint32_t K4B_PAD = K4B_PAD_DEF;  // heavy ids staged either side of the tile's own
#ifndef K4B_MINB
#define K4B_MINB 5
#endif
__global__ void __launch_bounds__(K1_THREADS, K4B_MINB)
k_assemble(const double* __restrict__ w, uint64_t n, const DevScalars* sc,
           const unsigned long long* __restrict__ status, const uint32_t* __restrict__ lrank,
           const double* __restrict__ hshare, const uint32_t* __restrict__ hidx,
           Bucket* __restrict__ out) {
    // The tile's lights are the contiguous light-list run [L0, L0 + totL) and
    // its heavies the run [H0, H0 + totH): their lrank / hshare runs are
    // staged into shared memory with coalesced async copies.  The aliases are
    // heavy ids by rank: a heavy's is rank H0 + q + 1; a light's is the rank
    // the pack paired it with, which lies within a few dozen of the tile's own
    // heavy ranks (jobs balance light and heavy weight at every split).  So
    // the ids of ranks [H0 - PAD, H0 + totH + PAD) are staged too -- the
    // tile's own heavies write theirs (no load), the two PAD-wide edges are
    // copied from `heavy` -- and only a rank outside that window (rare, or a
    // tile whose runs do not fit the budget) reads `heavy` from global memory.
    extern __shared__ __align__(16) unsigned char k4b_smem[];
    __shared__ TileCells C;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t tile = blockIdx.x;
    const uint64_t base = tile * K1_TILE;
    const uint64_t nh = sc->nh;
#if K4B_KEEP
    double xs[K1_ROWS];  // the tile's weights stay in registers (no re-read for the lights)
    classify_tile<true>(w, n, base, sc->wn, xs, C);
#else
    classify_tile<false>(w, n, base, sc->wn, nullptr, C);
#endif
    const unsigned lt = lanemask_lt();
    if (nh == 0) {  // fill_uniform_if_no_heavy (alias.hpp:288-297)
#pragma unroll 4
        for (int r = 0; r < K1_ROWS; ++r) {
            const uint64_t gi = base + r * K1_THREADS + threadIdx.x;
            if (gi < n) store_bucket(out, gi, __ldg(w + gi), static_cast<uint32_t>(gi),
                                     static_cast<uint32_t>(gi));
        }
        return;
    }
    const uint32_t totL = C.totL, totH = C.totH;
    const uint64_t L0 = (status[tile] & VAL_MASK) - totL;
    const uint64_t H0 = base - L0;
    const uint64_t wlo = H0 > K4B_PAD ? H0 - K4B_PAD : 0;
    const uint64_t whi = umin64(H0 + totH + K4B_PAD, nh);
    const uint32_t b_la = (4u * totL + 15u) & ~15u;
    const uint32_t b_hs = 8u * totH;
    const bool ids = b_la + b_hs + 4u * static_cast<uint32_t>(whi - wlo) <= K4B_SMEM;
    uint32_t* d_la = reinterpret_cast<uint32_t*>(k4b_smem);
    double* d_hs = reinterpret_cast<double*>(k4b_smem + b_la);
    uint32_t* d_id = reinterpret_cast<uint32_t*>(k4b_smem + b_la + b_hs);  // ranks [wlo, whi)
    for (uint32_t q = threadIdx.x; q < totL; q += K1_THREADS) cp_async4(&d_la[q], lrank + L0 + q);
    for (uint32_t q = threadIdx.x; q < totH; q += K1_THREADS) cp_async8(&d_hs[q], hshare + H0 + q);
    if (ids) {
        const uint32_t e0 = static_cast<uint32_t>(H0 - wlo), e1 = static_cast<uint32_t>(H0 + totH - wlo);
        const uint32_t e2 = static_cast<uint32_t>(whi - wlo);
        for (uint32_t q = threadIdx.x; q < e0; q += K1_THREADS) cp_async4(&d_id[q], hidx + wlo + q);
        for (uint32_t q = e1 + threadIdx.x; q < e2; q += K1_THREADS) cp_async4(&d_id[q], hidx + wlo + q);
        // the tile's own heavies: rank H0 + q is item gi
#pragma unroll 4
        for (int r = 0; r < K1_ROWS; ++r) {
            const int cell = r * K1_WARPS + warp;
            const unsigned hm = C.hm[cell];
            if ((hm >> lane) & 1)
                d_id[e0 + C.exH[cell] + __popc(hm & lt)] =
                    static_cast<uint32_t>(base + r * K1_THREADS + threadIdx.x);
        }
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    const uint32_t hmax = static_cast<uint32_t>(nh - 1);
    const uint32_t wlo32 = static_cast<uint32_t>(wlo), wn32 = static_cast<uint32_t>(whi - wlo);
#if K4B_KEEP
#pragma unroll
#else
#pragma unroll 4
#endif
    for (int r = 0; r < K1_ROWS; ++r) {
        const uint64_t gi = base + r * K1_THREADS + threadIdx.x;
        if (gi >= n) continue;
        const int cell = r * K1_WARPS + warp;
        const unsigned lm = C.lm[cell];
        double share;
        uint32_t rank;
        if ((lm >> lane) & 1) {
#if K4B_KEEP
            share = xs[r];
#else
            share = __ldg(w + gi);
#endif
            rank = min(d_la[C.exL[cell] + __popc(lm & lt)], hmax);  // heavy_at(j)
        } else {
            const uint32_t q = C.exH[cell] + __popc(C.hm[cell] & lt);
            share = d_hs[q];
            rank = min(static_cast<uint32_t>(H0) + q + 1, hmax);  // heavy_at(j + 1)
        }
        const uint32_t o = rank - wlo32;
        WRS_CHECK(rank < nh);
        const uint32_t id = (ids && o < wn32) ? d_id[o] : __ldg(hidx + rank);
        store_bucket(out, gi, share, static_cast<uint32_t>(gi), id);
    }
}

// ===========================================================================
// host side
// ===========================================================================
static int k0_depth(uint64_t n) {
    int D = 0;
    while (((n + (1ull << D) - 1) >> D) > static_cast<uint64_t>(K0_NODE)) ++D;
    return D;
}

template <typename T>
static cudaError_t ws_alloc(Workspace& ws, T*& ptr, uint64_t count) {
    const uint64_t by = count * sizeof(T) + 64;
    cudaError_t e = dev_malloc(reinterpret_cast<void**>(&ptr), by);
    if (e == cudaSuccess) ws.bytes += by;
    return e;
}

cudaError_t workspace_alloc(Workspace& ws, uint64_t n, uint64_t P, bool separate_outputs) {
    workspace_free(ws);
    ws.n = n;
    ws.P = P;
    ws.k0_depth = k0_depth(n);
    const uint64_t nodes = (2ull << ws.k0_depth) - 1;
    const uint64_t cnts = (1ull << ws.k0_depth);
    const uint64_t ntiles = (n + K1_TILE - 1) / K1_TILE;
    const uint64_t nblocks = (n + SCAN_BLOCK - 1) / SCAN_BLOCK + 2;
    cudaError_t e = cudaSuccess;
    auto A = [&](auto*& p, uint64_t c) {
        if (e == cudaSuccess) e = ws_alloc(ws, p, c);
    };
    A(ws.node_val, nodes);
    A(ws.node_cnt, cnts);
    A(ws.tile_status, ntiles);
    A(ws.hidx, n);
    A(ws.lw, n);
    A(ws.hw, n);
    A(ws.lpre, n + 1);
    A(ws.hpre, n + 1);
    A(ws.totals, nblocks);
    A(ws.carries, nblocks);
    A(ws.bmax, nblocks);
    A(ws.lck, n / CK_STRIDE + 2);
    A(ws.hck, n / CK_STRIDE + 2);
    A(ws.split_l, P + 1);
    A(ws.split_h, P + 1);
    A(ws.split_s, P + 1);
    A(ws.sc, 1);
    A(ws.k2_flags, k2_flag_words(n));
    if (separate_outputs) {
        A(ws.lrank_own, n);
        A(ws.hshare_own, n);
        ws.lrank = ws.lrank_own;
        ws.hshare = ws.hshare_own;
    } else {
        // K4a runs after K3, the last reader of the prefix arrays: reuse them.
        ws.lrank = reinterpret_cast<uint32_t*>(ws.lpre);
        ws.hshare = ws.hpre;
    }
    if (e != cudaSuccess) workspace_free(ws);
    return e;
}

cudaError_t workspace_alloc_total(Workspace& ws, uint64_t n) {
    workspace_free(ws);
    ws.n = n;
    ws.k0_depth = k0_depth(n);
    cudaError_t e = ws_alloc(ws, ws.node_val, (2ull << ws.k0_depth) - 1);
    if (e == cudaSuccess) e = ws_alloc(ws, ws.node_cnt, 1ull << ws.k0_depth);
    if (e == cudaSuccess) e = ws_alloc(ws, ws.sc, 1);
    if (e != cudaSuccess) workspace_free(ws);
    return e;
}

void workspace_free(Workspace& ws) {
    void* ptrs[] = {ws.node_val, ws.node_cnt, ws.tile_status, ws.hidx,       ws.lw,
                    ws.hw,       ws.lpre,     ws.hpre,        ws.totals,
                    ws.carries,  ws.split_l,  ws.split_h,     ws.split_s,    ws.sc,
                    ws.lrank_own, ws.hshare_own, ws.lck,       ws.hck,    ws.k2_flags,
                    ws.bmax};
    for (void* p : ptrs)
        if (p) dev_free(p);
    ws = Workspace{};
}

// DevScalars of a build, written by a one-thread kernel: total and wn travel
// as launch parameters (captured at launch), so no host staging buffer can be
// reused while a copy from it is still pending, however many builds are in
// flight.
__global__ void k_reset_scalars(DevScalars* sc, double total, double wn) {
    DevScalars v{};
    v.bad_index = ~0ull;
    v.total = total;
    v.wn = wn;
    *sc = v;
}

static cudaError_t reset_scalars(Workspace& ws, cudaStream_t st, double total, double wn) {
    k_reset_scalars<<<1, 1, 0, st>>>(ws.sc, total, wn);
    return cudaGetLastError();
}

cudaError_t launch_total(const double* d_w, uint64_t n, Workspace& ws, cudaStream_t st) {
    cudaError_t e = reset_scalars(ws, st, 0.0, 0.0);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(ws.node_cnt, 0, sizeof(unsigned) << ws.k0_depth, st);
    if (e != cudaSuccess) return e;
    k_total<<<static_cast<unsigned>(1ull << ws.k0_depth), K0_THREADS, 0, st>>>(
        d_w, n, ws.k0_depth, ws.node_val, ws.node_cnt, ws.sc);
    return cudaGetLastError();
}

// Block count up to which K2a/K2c split each chain over warps
// (k_scan_blocks_split; WRS_B200_K2_SPLIT_MAX: experiments).
static uint64_t k2_split_max_blocks() {
    const char* e = std::getenv("WRS_B200_K2_SPLIT_MAX");
    return e ? std::strtoull(e, nullptr, 10) : 1536;  // measured: better up to 2^21 items, worse at 2^22
}

// Chains per warp of k_scan_blocks_direct (WRS_B200_K2_LPW: experiments).
static int k2_direct_lpw(uint64_t nblocks) {
    if (const char* e = std::getenv("WRS_B200_K2_LPW")) {
        const int v = std::atoi(e);
        if (v >= 1 && v <= 32) return v;
    }
    // measured (scripts/stage_probe.py): one chain per warp up to ~1e3
    // chains, then about 1024-1280 warps (lpw 2 at 2^22 items, 8 at 2^24)
    int lpw = 1;
    while (lpw < 32 && static_cast<uint64_t>(lpw) * 1280 < nblocks) lpw <<= 1;
    return lpw;
}

// Item count up to which K2a/K2c use k_scan_blocks_direct (WRS_B200_K2_DIRECT_MAX
// overrides; results are identical either way).  Builds with the direct form /
// the bulk-copy fused form: n = 4.2e6 0.25 / 0.29 ms, 1e7 0.39 / 0.39, 2^24
// 0.55 / 0.52, 2^25 0.95 / 0.85.
static uint64_t k2_direct_max() {
    const char* e = std::getenv("WRS_B200_K2_DIRECT_MAX");  // read per build (tests flip it)
    return e ? std::strtoull(e, nullptr, 10) : 12000000ull;
}

// K1 form: unstaged unless WRS_B200_K1=staged (tests run both)
static bool k1_staged() {
    const char* e = std::getenv("WRS_B200_K1");
    return e && e[0] == 's';
}

// Checkpointed prefixes for the staged K2 form (WRS_B200_K2_CKPT=0: full
// prefix arrays, as the small-table forms always write).
static bool k2_ckpt_enabled() {
    const char* e = std::getenv("WRS_B200_K2_CKPT");
    return !(e && e[0] == '0');
}

static int sm_count_psa() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

// K3's coarse brackets from block carries + block maxima (WRS_B200_K3_COARSE=0: off).
static bool k3_coarse_enabled() {
    const char* e = std::getenv("WRS_B200_K3_COARSE");
    return !(e && e[0] == '0');
}

// Bulk-copy K2a / K2c (WRS_B200_K2_KB=0: the smem-staged kernels).
static bool k2_kb_enabled() {
    const char* e = std::getenv("WRS_B200_K2_KB");
    return !(e && e[0] == '0');
}

// K2a, K2b and the checkpoint pass in one launch (default);
// WRS_B200_K2_FUSE=1: K2a separate; =0: three kernels.
static bool k2_fuse_enabled() {
    const char* e = std::getenv("WRS_B200_K2_FUSE");
    return !(e && e[0] == '0');
}
static bool k2_fuse_all_enabled() {
    const char* e = std::getenv("WRS_B200_K2_FUSE");
    return !(e && (e[0] == '0' || e[0] == '1'));
}

cudaError_t launch_psa_build(const double* d_w, uint64_t n, double total, uint64_t P,
                             Bucket* d_b, Workspace& ws, cudaStream_t st, cudaEvent_t* ev) {
    const int k1_smem = K1_TILE * 10;
    // warps per K4a CTA: 11 fill an SM's shared memory; with fewer jobs than
    // 11 warps on every SM, smaller CTAs spread the sequential chains over
    // more SMs (a lone chain is issue-latency bound, so it runs faster with a
    // scheduler to itself)
    const uint64_t k4_warps_total = (P + 31) / 32;
    const int k4_warps = static_cast<int>(std::min<uint64_t>(
        K4_WARPS, std::max<uint64_t>(1, (k4_warps_total + 147) / 148)));
    const int k4_smem = k4_warps * static_cast<int>(sizeof(K4Rings));
    // per-device attribute; cheap enough to set on every build
    cudaFuncSetAttribute(k_partition, cudaFuncAttributeMaxDynamicSharedMemorySize, k1_smem);
    cudaFuncSetAttribute(k_pack<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, k4_smem);
    cudaFuncSetAttribute(k_pack<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, k4_smem);
    cudaFuncSetAttribute(k_scan_carry_split, cudaFuncAttributeMaxDynamicSharedMemorySize, K2W_SMEM);
    cudaFuncSetAttribute(k_carry_ckpt, cudaFuncAttributeMaxDynamicSharedMemorySize, K2F_SMEM);
    cudaFuncSetAttribute(k_totals_kb, cudaFuncAttributeMaxDynamicSharedMemorySize, KB_SMEM);
    cudaFuncSetAttribute(k_ckpt_kb, cudaFuncAttributeMaxDynamicSharedMemorySize, KB_SMEM);
    cudaFuncSetAttribute(k_assemble, cudaFuncAttributeMaxDynamicSharedMemorySize, K4B_SMEM);
    const uint64_t ntiles = (n + K1_TILE - 1) / K1_TILE;
    const uint64_t nblocks = (n + SCAN_BLOCK - 1) / SCAN_BLOCK + 1;  // light + heavy blocks
    const unsigned k2_grid = static_cast<unsigned>((nblocks + K2_WARPS * 32 - 1) / (K2_WARPS * 32));
    const unsigned k4_grid = static_cast<unsigned>((P + k4_warps * 32 - 1) / (k4_warps * 32));
    cudaError_t e;
#define REC(i)                                          \
    do {                                                \
        if (ev) cudaEventRecord(ev[i], st);             \
    } while (0)
    // bucket_mean_ = W / n (alias.hpp:247-248) with the weights' pairwise W
    e = reset_scalars(ws, st, total, total / static_cast<double>(n));
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(ws.tile_status, 0, ntiles * sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    // checked builds: every scratch array starts as 0xFF garbage
    poison(ws.lw, ws.n * 8, st);
    poison(ws.hw, ws.n * 8, st);
    poison(ws.hidx, ws.n * 4, st);
    poison(ws.lpre, (ws.n + 1) * 8, st);
    poison(ws.hpre, (ws.n + 1) * 8, st);
    poison(ws.lck, (ws.n / CK_STRIDE + 2) * 16, st);
    poison(ws.hck, (ws.n / CK_STRIDE + 2) * 16, st);
    poison(ws.totals, (ws.n / SCAN_BLOCK + 3) * 8, st);
    poison(ws.carries, (ws.n / SCAN_BLOCK + 3) * 8, st);
    poison(ws.split_l, (P + 1) * 4, st);
    poison(ws.split_h, (P + 1) * 4, st);
    poison(ws.split_s, (P + 1) * 8, st);
    poison(d_b, n * sizeof(Bucket), st);
    REC(0);
    if (k1_staged())
        k_partition<<<static_cast<unsigned>(ntiles), K1_THREADS, k1_smem, st>>>(
            d_w, n, ntiles, ws.sc, ws.tile_status, ws.lw, ws.hidx, ws.hw);
    else
        k_partition_direct<<<static_cast<unsigned>(ntiles), K1_THREADS, 0, st>>>(
            d_w, n, ntiles, ws.sc, ws.tile_status, ws.lw, ws.hidx, ws.hw);
    REC(1);
    // every prefix-chain value is finite and >= 0 when W is far below DBL_MAX
    const bool pos = total < 1e300;
    // few chains per SM: their latency sets the time, so the leaner direct form
    const bool direct = n <= k2_direct_max();
    // a few blocks (n up to ~3e6 items): each chain split over four warps
    const bool split = pos && nblocks <= k2_split_max_blocks();
    const int lpw = k2_direct_lpw(nblocks);
    const unsigned k2d_grid = static_cast<unsigned>((nblocks + 2 * lpw - 1) / (2 * lpw));
#define K2_LAUNCH(PASS3)                                                                          \
    do {                                                                                          \
        if (split)                                                                                \
            k_scan_blocks_split<PASS3><<<static_cast<unsigned>(nblocks), 128, 0, st>>>(           \
                ws.lw, ws.hw, ws.lpre, ws.hpre, ws.sc, ws.totals, ws.carries);                    \
        else if (direct && pos)                                                                   \
            k_scan_blocks_direct<PASS3, CompSumPos><<<k2d_grid, 64, 0, st>>>(                     \
                ws.lw, ws.hw, ws.lpre, ws.hpre, ws.sc, ws.totals, ws.carries, lpw);               \
        else if (direct)                                                                          \
            k_scan_blocks_direct<PASS3, CompSum><<<k2d_grid, 64, 0, st>>>(                        \
                ws.lw, ws.hw, ws.lpre, ws.hpre, ws.sc, ws.totals, ws.carries, lpw);               \
        else if (pos)                                                                             \
            k_scan_blocks<PASS3, CompSumPos><<<k2_grid, K2_WARPS * 32, 0, st>>>(                  \
                ws.lw, ws.hw, ws.lpre, ws.hpre, ws.sc, ws.totals, ws.carries);                    \
        else                                                                                      \
            k_scan_blocks<PASS3, CompSum><<<k2_grid, K2_WARPS * 32, 0, st>>>(                     \
                ws.lw, ws.hw, ws.lpre, ws.hpre, ws.sc, ws.totals, ws.carries);                    \
    } while (0)
    // large tables: the bulk-copy forms of K2a / K2c (WRS_B200_K2_KB=0: the
    // smem-staged forms)
    const bool kb = pos && !split && !direct && k2_kb_enabled();
    // ... and K2a in the same launch as the chain and the checkpoints (see
    // k_carry_ckpt; WRS_B200_K2_FUSE=1 launches K2a on its own)
    const bool bulk_exp = pos && !split && !direct && std::getenv("WRS_B200_K2_BULK");
    const bool fuse_all = kb && k2_ckpt_enabled() && k2_fuse_all_enabled() && !bulk_exp;
    // K2a's bulk form also bounds every heavy block's weights (K3's coarse brackets)
    const bool have_bmax = kb && !bulk_exp;
    const int sms = sm_count_psa();
    // per-list units: nlu + nhu <= (blocks + 31) / 32 + 1 (empty ones return at once)
    const uint32_t kb_units = static_cast<uint32_t>((nblocks + 31) / 32 + 1);
    const unsigned kb_grid = static_cast<unsigned>(
        std::min<uint64_t>((kb_units + KB_WARPS - 1) / KB_WARPS, sms));
    if (bulk_exp)
        k_scan_totals_bulk<CompSumPos><<<k2_grid, K2_WARPS * 32, 0, st>>>(ws.lw, ws.hw, ws.sc,
                                                                          ws.totals);
    else if (kb && !fuse_all)
        k_totals_kb<<<kb_grid, KB_WARPS * 32, KB_SMEM, st>>>(ws.lw, ws.hw, ws.sc, ws.totals, kb_units,
                                                             ws.bmax);
    else if (!fuse_all)
        K2_LAUNCH(false);
    REC(2);
    // large tables: checkpoints instead of full prefix arrays (1 B per item
    // written instead of 8; K3 recomputes what it probes)
    ws.ckpt = pos && !split && !direct && k2_ckpt_enabled();
    // ... and the carry chain fused with them (WRS_B200_K2_FUSE=0: separate)
    const bool fuse = ws.ckpt && kb && k2_fuse_enabled();
    if (fuse) {
        // one CTA per SM: two chains, the rest checkpoint units
        const unsigned grid = static_cast<unsigned>(
            std::min<uint64_t>(2 + (kb_units + KB_WARPS - 1) / KB_WARPS, sms));
        e = cudaMemsetAsync(ws.k2_flags, 0, k2_flag_words(ws.n) * 4, st);
        if (e != cudaSuccess) return e;
        k_carry_ckpt<<<grid, K2F_THREADS, K2F_SMEM, st>>>(ws.sc, ws.totals, ws.carries, ws.lpre, ws.hpre,
                                                  ws.lw, ws.hw, ws.lck, ws.hck, ws.k2_flags,
                                                  k2_flag_slots(ws.n), kb_units,
                                                  fuse_all ? kb_units : 0u, ws.bmax);
    } else if (pos) {
        k_scan_carry_split<<<2, 160, K2W_SMEM, st>>>(ws.sc, ws.totals, ws.carries, ws.lpre, ws.hpre);
    } else {
        k_scan_carry<CompSum><<<2, 32, 0, st>>>(ws.sc, ws.totals, ws.carries, ws.lpre, ws.hpre);
    }
    REC(3);  // (fused: K2c ran inside the launch above, so its stage time is ~0)
    if (!fuse && ws.ckpt && kb)
        k_ckpt_kb<<<kb_grid, KB_WARPS * 32, KB_SMEM, st>>>(ws.lw, ws.hw, ws.lck, ws.hck, ws.sc,
                                                          ws.carries, kb_units);
    else if (!fuse && ws.ckpt)
        k_scan_blocks_ckpt<<<k2_grid, K2_WARPS * 32, 0, st>>>(ws.lw, ws.hw, ws.lck, ws.hck, ws.sc,
                                                              ws.carries);
    else if (!fuse)
        K2_LAUNCH(true);
#undef K2_LAUNCH
    REC(4);
    {
        SplitSrc src{ws.lpre, ws.hpre, CkList{ws.lw, ws.lck, 0}, CkList{ws.hw, ws.hck, 0}, ws.hw,
                     ws.ckpt, ws.carries, ws.bmax, ws.ckpt && have_bmax && k3_coarse_enabled()};
        const unsigned grid = static_cast<unsigned>((P + 1 + 255) / 256);
        k_split<<<grid, 256, 0, st>>>(n, P, ws.sc, src, ws.split_l, ws.split_h, ws.split_s);
    }
    REC(5);
    if (pos)  // W < 1e300: the remainder stays finite
        k_pack<true><<<k4_grid, k4_warps * 32, k4_smem, st>>>(
            P, ws.sc, ws.lw, ws.hw, ws.split_l, ws.split_h, ws.split_s, ws.lrank, ws.hshare);
    else
        k_pack<false><<<k4_grid, k4_warps * 32, k4_smem, st>>>(
            P, ws.sc, ws.lw, ws.hw, ws.split_l, ws.split_h, ws.split_s, ws.lrank, ws.hshare);
    REC(6);
    k_assemble<<<static_cast<unsigned>(ntiles), K1_THREADS, K4B_SMEM, st>>>(
        d_w, n, ws.sc, ws.tile_status, ws.lrank, ws.hshare, ws.hidx, d_b);
    REC(7);
#undef REC
    return cudaGetLastError();
}

unsigned long long check_failures_psa(unsigned* line) { return tu_check_failures(line); }

void poison(void* p, size_t bytes, cudaStream_t st) {
#ifdef WRS_B200_CHECKED
    if (p && bytes) cudaMemsetAsync(p, 0xff, bytes, st);
#else
    (void)p, (void)bytes, (void)st;
#endif
}

}  // namespace wrsb
