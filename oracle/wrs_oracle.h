/*
 * oracle/wrs_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's PSA alias-table build and bulk
 * alias sampling (arXiv 1903.00227 reference, /root/reference/proj).  It is
 * the checker the GPU path is compared against; nothing in the product
 * (paper_1903_00227_b200/) links or calls it.  Only tests/, the smoke() entry
 * and bench.py's cpu_baseline leg may load it.
 *
 * Parity is pinned two ways:
 *   - against the reference itself, compiled from its own headers into
 *     oracle/_ref/libwrs_ref.so by oracle/Makefile (ref_shim.cpp);
 *   - against golden vectors in tests/golden/ produced by that build.
 *
 * Every function cites the reference file:line it restates.
 */
#ifndef WRS_ORACLE_H
#define WRS_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 16-byte bucket, byte layout of wrs::alias_bucket (alias.hpp:26-33). */
typedef struct wo_bucket {
    double share;
    uint32_t item;
    uint32_t alias;
} wo_bucket;

/* Counter RNG state (rng.hpp:32-82). */
typedef struct wo_rng {
    uint64_t key;
    uint64_t ctr;
} wo_rng;

uint64_t wo_mix64(uint64_t z);
wo_rng wo_rng_make(uint64_t seed, uint64_t stream);
wo_rng wo_rng_derive(const wo_rng* r, uint64_t salt);
uint64_t wo_rng_next(wo_rng* r);
double wo_rng_uniform01(wo_rng* r);
uint64_t wo_rng_bounded(wo_rng* r, uint64_t n);
void wo_rng_outputs(uint64_t seed, uint64_t stream, int64_t salt, uint64_t count, uint64_t* out);

/* Weight generators (weight_file.hpp:32-54). Return 0 on success. */
void wo_generate_uniform(uint64_t n, uint64_t seed, double* out);
int wo_generate_powerlaw(uint64_t n, double s, uint64_t seed, double* out);
/* configs[3]'s lognormal(0, sigma) weights: the library's own generator
 * (common.cuh lognormal_weight), restated. */
void wo_generate_lognormal(uint64_t n, double sigma, uint64_t seed, double* out);

/* WeightTable (weights.hpp:19-46): returns 0 if valid, else 1 and *bad =
 * first offending index.  *total = pairwise_sum. */
double wo_pairwise_sum(const double* v, uint64_t n);
int wo_weights_check(const double* w, uint64_t n, uint64_t* bad, double* total,
                     double* wmin, double* wmax);

/* prefix_sums (parallel.hpp:104-130), inclusive, out[0..n). */
void wo_prefix_sums(const double* in, double* out, uint64_t n);
/* The pass-1 block totals and pass-2 carries, exposed for per-pass parity. */
void wo_scan_block_totals(const double* in, uint64_t n, double* totals);
void wo_scan_carries(double* totals_to_carries, uint64_t nblocks);

/* partition_items (alias.hpp:48-97). Arrays malloc'ed; free with
 * wo_partition_free. */
typedef struct wo_partition {
    uint64_t nl, nh;
    uint32_t* light;
    uint32_t* heavy;
    double* light_prefix; /* nl + 1 */
    double* heavy_prefix; /* nh + 1 */
    double wn;
} wo_partition;
int wo_partition_items(const double* w, uint64_t n, double total, wo_partition* p);
void wo_partition_free(wo_partition* p);

typedef struct wo_split {
    uint64_t light_count, heavy_count;
    double spill;
} wo_split;
/* psa_split (alias.hpp:122-149). */
wo_split wo_psa_split(const wo_partition* p, const double* w, uint64_t n_prime);

typedef struct wo_job {
    uint64_t light_lo, light_hi, heavy_lo, heavy_hi;
    double spill;
} wo_job;
/* psa_plan (alias.hpp:214-238): jobs[0..P). Returns 0, or 1 when the
 * boundaries decrease (the reference throws std::logic_error). */
int wo_psa_plan(const wo_partition* p, const double* w, uint64_t n, uint64_t P,
                wo_job* jobs);
/* psa_pack (alias.hpp:160-209). */
void wo_psa_pack(const wo_partition* p, const double* w, const wo_job* job,
                 wo_bucket* buckets);

/* AliasTable(wt, Build::psa, P) (alias.hpp:246-257, 288-297, 411-419).
 * Returns 0 on success, 1 invalid weights, 2 n too large, 3 plan error.
 * *bucket_mean = W/n. */
int wo_psa_build(const double* w, uint64_t n, uint64_t P, wo_bucket* buckets,
                 double* bucket_mean);

/* AliasTable::sample_many (alias.hpp:265-284, parallel.hpp:37-43). */
void wo_sample_many(const wo_bucket* b, uint64_t n, double bucket_mean, uint64_t seed,
                    uint64_t k, uint32_t workers, uint32_t* out);
/* Same, but only worker slice [q_lo, q_hi) of the global output. */
void wo_sample_range(const wo_bucket* b, uint64_t n, double bucket_mean,
                     uint64_t seed, uint64_t k, uint32_t workers, uint64_t q_lo,
                     uint64_t q_hi, uint32_t* out);

/* TwoLevelTable::sample_many (two_level.hpp:66-81), positions [q_lo, q_hi)
 * of the k outputs: the top table (groups buckets, mean top_mean) picks group
 * g, table g (sizes[g] buckets, mean means[g]) the local item, output
 * bases[g] + item; query m of worker w's slice consumes outputs 4m+1..4m+4
 * of RngStream(seed, 0x326c766c).derive(w). */
void wo_two_level_sample_range(const wo_bucket* const* tables, const uint64_t* sizes,
                               const double* means, const uint64_t* bases, uint64_t groups,
                               const wo_bucket* top, double top_mean, uint64_t seed,
                               uint64_t k, uint32_t workers, uint64_t q_lo, uint64_t q_hi,
                               uint32_t* out);

/* Philox4x32-10 (Salmon et al. SC'11, Random123): c[4] in place, key (k0, k1). */
void wo_philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1);
/* Philox draw mode replay (include/wrs_b200.h): draws [q_lo, q_hi) of the
 * table with uniforms from Philox4x32-10(counter q, key seed) through the
 * reference's ia[x >= share] rule (alias.hpp:265-269). */
void wo_sample_philox_range(const wo_bucket* b, uint64_t n, double bucket_mean, uint64_t seed,
                            uint64_t q_lo, uint64_t q_hi, uint32_t* out);

/* implied_masses + max_relative_mass_error (verify.hpp:43-54, 92-98). */
void wo_implied_masses(const wo_bucket* b, uint64_t n, double bucket_mean, double* m);
double wo_max_relative_mass_error(const double* m, const double* w, uint64_t n);

#ifdef __cplusplus
}
#endif
#endif
