// paper_1903_00227_b200/csrc/engine.h -- host-side interface between the C ABI
// (capi.cpp) and the kernels (psa_kernels.cu, sample_kernels.cu).  Internal:
// not installed, not part of the ABI.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "common.cuh"

namespace wrsb {

// Checked builds: device-side index violations counted per translation unit
// (common.cuh WRS_CHECK); *line gets the first offending source line.
unsigned long long check_failures_psa(unsigned* line);
unsigned long long check_failures_sample(unsigned* line);
unsigned long long check_failures_verify(unsigned* line);
unsigned long long check_failures_generate(unsigned* line);
// Checked builds fill scratch with 0xFF bytes (no-op otherwise).
void poison(void* p, size_t bytes, cudaStream_t st);

// Caching device allocator for the library's large buffers (alloc.cpp).
cudaError_t dev_malloc(void** p, size_t bytes);
void dev_free(void* p);
// While an armed SyncedFrees is in scope on this thread, dev_free skips its
// device-wide synchronise: the caller has already synchronised every stream
// that used the buffers it frees (so a free on one host thread no longer
// waits for another thread's copies and kernels on other streams).
struct SyncedFrees {
    bool armed = false;
    void arm();
    ~SyncedFrees();
};
// Returns every cached block to the driver; the bytes released.
size_t release_cache();

// PSA job count used by algo "psa": one job = one thread's sequential pack
// chain, so P sets the build's parallelism and the job length its latency.
// Jobs of J = n / 49152 items rounded down to a power of two, clamped to
// [32, 1024]: large tables (n >= ~5e7) get 1024-item jobs (~1e5 chains for
// 148 SMs), smaller ones shorter chains so there are still ~5e4 of them.  A
// function of n only, so tables are reproducible on
// any GPU and launch shape.
// Wave fit: K4a keeps kK4Lanes jobs resident on a B200 (148 SMs x 12 warps x
// 32 lanes); when the jobs of that length would leave a last K4a wave less
// than half full, the jobs are stretched to fill the whole waves before it
// (measured builds: n = 1.25e8 2.79 -> 2.61 ms (J 1024 -> 1100), 2^24 0.59 ->
// 0.55, 1e7 0.43 -> 0.40; n = 1e8, whose last wave is 72 % full, keeps
// J = 1024).
constexpr uint64_t kJobBucketsMax = 1024, kJobBucketsMin = 32, kJobTarget = 49152;
constexpr uint64_t kK4Lanes = 148ull * 12 * 32;
inline uint64_t default_job_items(uint64_t n) {
    if (const char* e = std::getenv("WRS_B200_JOB_ITEMS")) {  // experiments only
        const uint64_t v = std::strtoull(e, nullptr, 10);
        if (v >= 1) return v;
    }
    uint64_t j = kJobBucketsMin;
    while (j < kJobBucketsMax && 2 * j <= n / kJobTarget) j *= 2;
    const uint64_t p = (n + j - 1) / j;
    const uint64_t waves = p / kK4Lanes, last = p % kK4Lanes;
    // (jobs shorter than the 1024 cap: any partial last wave; measured at
    // n = 1.2e7, 1.65 waves of J = 128: build 0.470 -> 0.437 ms with J = 212)
    if (waves >= 1 && last != 0 && (j < kJobBucketsMax || last < kK4Lanes / 2))
        j = (n + waves * kK4Lanes - 1) / (waves * kK4Lanes);
    return j;
}
inline uint64_t default_jobs(uint64_t n) {
    const uint64_t j = default_job_items(n);
    const uint64_t p = (n + j - 1) / j;
    return p ? p : 1;
}

// Scratch of one build, sized for n items and P jobs.  Light and heavy lists
// each get n slots (their split is only known on the device).
struct Workspace {
    uint64_t n = 0, P = 0;
    int k0_depth = 0;
    double* node_val = nullptr;      // K0 pairwise tree nodes above the CTA cut
    unsigned* node_cnt = nullptr;    // K0 arrival counters
    unsigned long long* tile_status = nullptr;  // K1 decoupled look-back
    unsigned* k2_flags = nullptr;  // fused K2b+K2c: per list, one 128-B line per published chunk
    uint32_t* hidx = nullptr;        // heavy item ids, ascending (light ids stay implicit)
    double* lw = nullptr;            // gathered light weights
    double* hw = nullptr;            // gathered heavy weights
    double* lpre = nullptr;          // exclusive light prefix, nl + 1 entries
    double* hpre = nullptr;          // exclusive heavy prefix, nh + 1 entries
    double2* lck = nullptr;          // (or) chain states before every 16th light ...
    double2* hck = nullptr;          // ... and heavy: the checkpointed prefixes
    bool ckpt = false;               // the last build kept checkpoints, not prefixes
    uint32_t* lrank = nullptr;       // K4a: alias heavy RANK of every light, list order
    double* hshare = nullptr;        // K4a: share of every heavy, list order
    uint32_t* lrank_own = nullptr;   // separate storage (else lrank aliases lpre)
    double* hshare_own = nullptr;    // separate storage (else hshare aliases hpre)
    double* totals = nullptr;        // K2a block totals (light blocks, then heavy)
    double* carries = nullptr;       // K2b exclusive carries
    double* bmax = nullptr;          // K2a (bulk form) per-block max weight, for K3's coarse brackets
    bool coarse = false;             // bmax is valid for this build
    uint32_t* split_l = nullptr;     // K3 boundaries, P + 1
    uint32_t* split_h = nullptr;
    double* split_s = nullptr;       // spill entering each job
    DevScalars* sc = nullptr;
    uint64_t bytes = 0;
};

// separate_outputs keeps K4a's outputs out of the prefix arrays' storage, so
// every intermediate stays inspectable (WRS_B200_KEEP_WORKSPACE).
cudaError_t workspace_alloc(Workspace& ws, uint64_t n, uint64_t P, bool separate_outputs);
// Only what K0 needs (weights handles: validation + total).
cudaError_t workspace_alloc_total(Workspace& ws, uint64_t n);
void workspace_free(Workspace& ws);

// K0: validation + bit-exact pairwise total of d_w into ws.sc (total, wn,
// bad_index).  Asynchronous.
cudaError_t launch_total(const double* d_w, uint64_t n, Workspace& ws, cudaStream_t st);

// K1..K4b: the PSA build of AliasTable(wt, psa, P) into d_b, given the
// weights' pairwise total (computed once by K0 when the weights handle was
// made, as WeightTable does).  `ev` (8 events or null) brackets the seven
// stages for timing.  Asynchronous; plan errors are latched in ws.sc.
cudaError_t launch_psa_build(const double* d_w, uint64_t n, double total, uint64_t P,
                             Bucket* d_b, Workspace& ws, cudaStream_t st, cudaEvent_t* ev);

// Scratch of the region-ordered draw plan (sample_kernels.cu); grows on demand.
struct SampleWorkspace {
    void* base = nullptr;
    uint64_t bytes = 0;
    unsigned* overflow = nullptr;  // device flag: a region slab overflowed (never expected)
    cudaError_t reserve(uint64_t bytes);
    void release();
};

// K5: AliasTable::sample_many(seed, k, workers) (alias.hpp:274-284), output
// positions [q_begin, q_end) of the k into d_out[0 .. q_end - q_begin).
// `stream_id` is the reference's sample stream 0x616c6961 ("alia").  `base` is
// added to every output (global ids of a shard).  With a workspace, large
// tables use the region-ordered plan; without, the direct gather kernel.
// `side` (optional; the C ABI passes it with WRS_B200_SIDE_SCATTER=1): a
// stream on which the region plan's first scatter runs.
// The scatter reads nothing but (n, seed, k), so it need not wait for the
// table: it only waits for what `side` already carries (the previous user of
// the scratch), and st waits for it (side_ev) before the first gather.  A
// draw issued right behind a rebuild thus scatters while the build runs.
constexpr uint64_t kSampleStream = 0x616c6961u;
// stream_id selecting the Philox draw mode (north star: counter-based Philox
// uniforms): draw q from Philox4x32-10(counter q, key seed), workers ignored.
constexpr uint64_t kPhiloxStream = ~0ull;
cudaError_t launch_sample(const Bucket* d_b, uint64_t n, double wn, uint64_t seed,
                          uint64_t stream_id, uint64_t q_begin, uint64_t q_end, uint64_t k,
                          uint32_t workers, uint32_t base, uint32_t* d_out, cudaStream_t st,
                          SampleWorkspace* ws, cudaStream_t side = nullptr,
                          cudaEvent_t side_ev = nullptr);
bool use_region_plan(uint64_t n, uint64_t k);

// Aggregated draws: the (item, count) pairs of sample_many(seed, k, workers)
// (the same draws as launch_sample), items ascending, into d_items /
// d_counts (min(k, n) entries) and *d_n_unique (device).  Per-bucket hit
// counters + fold + compaction; scratch grows on demand.
struct CountWorkspace {
    uint32_t* hits = nullptr;             // 2n: own answers per bucket, then alias answers
    unsigned long long* count = nullptr;  // per item
    uint32_t* tile_cnt = nullptr;
    uint64_t* tile_off = nullptr;
    uint64_t n = 0;
    cudaError_t reserve(uint64_t n);
    void release();
};
cudaError_t launch_count(const Bucket* d_b, uint64_t n, double wn, uint64_t seed,
                         uint64_t stream_id, uint64_t k, uint32_t workers, cudaStream_t st,
                         SampleWorkspace* ws, CountWorkspace* cw, uint32_t* d_items,
                         uint64_t* d_counts, unsigned long long* d_n_unique);

// Routed two-level draws (two_level.hpp:66-81): outputs [q_begin, q_end) of
// TwoLevelTable::sample_many(seed, k, workers) given the group tables (each
// on this GPU or a peer's, e.g. opened from an IPC handle), their sizes,
// bucket means and first global ids, and the top table over the group totals.
constexpr int kTwoLevelMaxGroups = 256;
struct TwoLevelDev {
    const Bucket* tables[kTwoLevelMaxGroups];
    uint64_t sizes[kTwoLevelMaxGroups];
    double means[kTwoLevelMaxGroups];
    uint64_t bases[kTwoLevelMaxGroups];
    const Bucket* top;
    uint64_t groups;
    double top_mean;
};
constexpr uint64_t kTwoLevelStream = 0x326c766cu;  // "2lvl", two_level.hpp:75
cudaError_t launch_two_level(const TwoLevelDev& tl, uint64_t seed, uint64_t q_begin,
                             uint64_t q_end, uint64_t k, uint32_t workers, uint32_t* d_out,
                             cudaStream_t st);

// implied_masses + max_relative_mass_error (verify.hpp:43-54, 92-98) on the
// device, bit-exact: per-item masses into d_m (may be null), the worst
// relative error into *worst (host).  Synchronous on st.  n < 2^31.
cudaError_t implied_masses_device(const Bucket* d_b, uint64_t n, double wn, const double* d_w,
                                  double* d_m, double* worst, cudaStream_t st);

// The power-law generator's Fisher-Yates deal (weight_file.hpp:47-52) on the
// device, identical to the sequential swaps: d_out = shuffle of d_in with
// RngStream key `key`.  Synchronous on st.  n < 2^31.
cudaError_t fisher_yates_device(const double* d_in, double* d_out, uint64_t n, uint64_t key,
                                cudaStream_t st);

// generate_uniform on the device (weight_file.hpp:32-38): counter-based, so
// every element is independent and bit-exact; items [offset, offset + n) of
// the global vector (a shard's slice).
cudaError_t launch_generate_uniform(double* d_w, uint64_t n, uint64_t offset, uint64_t seed,
                                    cudaStream_t st);
// configs[3]'s lognormal(0, sigma) weights (common.cuh: lognormal_weight),
// items [offset, offset + n) of the global vector.
cudaError_t launch_generate_lognormal(double* d_w, uint64_t n, uint64_t offset, uint64_t seed,
                                      double sigma, cudaStream_t st);

}  // namespace wrsb
