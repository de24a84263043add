/*
 * oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
 *
 * extern "C" face over the UNMODIFIED reference headers
 * (/root/reference/proj/include, included read-only by oracle/Makefile) so the
 * tests, the golden-vector script and bench.py's CPU baseline can run the
 * reference's own code: AliasTable(wt, Build::psa, workers),
 * AliasTable::sample_many, the detail:: PSA pieces at an arbitrary job count,
 * implied_masses, the generators, binomial_split and TwoLevelTable.  No
 * reference source is copied; this file only calls it.  Output goes to
 * oracle/_ref/libwrs_ref.so (git-ignored).
 */
#include <wrs/alias.hpp>
#include <wrs/binomial.hpp>
#include <wrs/parallel.hpp>
#include <wrs/rng.hpp>
#include <wrs/two_level.hpp>
#include <wrs/verify.hpp>
#include <wrs/weight_file.hpp>
#include <wrs/weights.hpp>

#include <atomic>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <thread>
#include <vector>

namespace {

wrs::WeightTable table_of(const double* w, uint64_t n) {
    return wrs::WeightTable(std::vector<double>(w, w + n));
}

void copy_buckets(std::span<const wrs::alias_bucket> b, void* out) {
    std::memcpy(out, b.data(), b.size() * sizeof(wrs::alias_bucket));
}

} // namespace

extern "C" {

int ref_weights_check(const double* w, uint64_t n, double* total, double* wmin,
                      double* wmax) {
    try {
        auto wt = table_of(w, n);
        *total = wt.total();
        *wmin = wt.min_weight();
        *wmax = wt.max_weight();
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    }
}

double ref_pairwise_sum(const double* v, uint64_t n) { return wrs::pairwise_sum(v, n); }

void ref_prefix_sums(const double* in, double* out, uint64_t n, unsigned workers) {
    wrs::prefix_sums(in, out, n, workers);
}

void ref_generate_uniform(uint64_t n, uint64_t seed, double* out) {
    const auto w = wrs::generate_uniform(n, seed);
    std::memcpy(out, w.data(), n * sizeof(double));
}

int ref_generate_powerlaw(uint64_t n, double s, uint64_t seed, double* out) {
    try {
        const auto w = wrs::generate_powerlaw(n, s, seed);
        std::memcpy(out, w.data(), n * sizeof(double));
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

uint64_t ref_rng_outputs(uint64_t seed, uint64_t stream, int64_t derive_salt,
                         uint64_t count, uint64_t* out) {
    wrs::RngStream r(seed, stream);
    if (derive_salt >= 0)
        r = r.derive(static_cast<uint64_t>(derive_salt));
    for (uint64_t i = 0; i < count; ++i)
        out[i] = r.next();
    return count;
}

/* AliasTable(wt, Build::psa, workers): the reference's own threaded build
 * (one OS thread per job). Returns 0 on success. */
int ref_psa_build(const double* w, uint64_t n, unsigned workers, void* buckets,
                  double* bucket_mean) {
    try {
        auto wt = table_of(w, n);
        wrs::AliasTable t(wt, wrs::AliasTable::Build::psa, workers);
        copy_buckets(t.buckets(), buckets);
        *bucket_mean = t.bucket_mean();
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

/* The same build at an arbitrary job count P without P OS threads:
 * detail::partition_items + detail::psa_plan(P) + detail::psa_pack per job,
 * jobs spread over `threads` workers (alias.hpp:411-419).  Bytewise equal to
 * AliasTable(wt, psa, P) (survey probe; re-checked in tests). */
int ref_psa_build_jobs(const double* w, uint64_t n, uint64_t P, unsigned threads,
                       void* out, double* bucket_mean) {
    try {
        auto wt = table_of(w, n);
        const double wn = wt.total() / static_cast<double>(n);
        *bucket_mean = wn;
        auto* b = static_cast<wrs::alias_bucket*>(out);
        bool heavy = false;
        for (uint64_t i = 0; i < n && !heavy; ++i)
            heavy = wt[i] > wn;
        if (!heavy) { // fill_uniform_if_no_heavy, alias.hpp:288-297
            for (uint64_t i = 0; i < n; ++i)
                b[i] = {wt[i], {static_cast<uint32_t>(i), static_cast<uint32_t>(i)}};
            return 0;
        }
        const auto part = wrs::detail::partition_items(wt, threads ? threads : 1);
        const auto jobs = wrs::detail::psa_plan(part, wt, static_cast<unsigned>(P));
        std::atomic<uint64_t> next{0};
        wrs::run_workers(threads ? threads : 1, [&](unsigned) {
            for (uint64_t k = next.fetch_add(1024); k < jobs.size(); k = next.fetch_add(1024))
                for (uint64_t e = k; e < std::min<uint64_t>(k + 1024, jobs.size()); ++e)
                    wrs::detail::psa_pack(part, wt, jobs[e], b);
        });
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

/* detail::partition_items (alias.hpp:48-97): counts, lists and prefix arrays.
 * Call with null arrays first to get the counts. */
int ref_partition(const double* w, uint64_t n, uint64_t* nl, uint64_t* nh,
                  uint32_t* light, uint32_t* heavy, double* light_prefix,
                  double* heavy_prefix, double* bucket_mean) {
    try {
        auto wt = table_of(w, n);
        const auto part = wrs::detail::partition_items(wt, 4);
        *nl = part.light.size();
        *nh = part.heavy.size();
        *bucket_mean = part.bucket_mean;
        if (light) {
            std::memcpy(light, part.light.data(), part.light.size() * 4);
            std::memcpy(heavy, part.heavy.data(), part.heavy.size() * 4);
            std::memcpy(light_prefix, part.light_prefix.data(), part.light_prefix.size() * 8);
            std::memcpy(heavy_prefix, part.heavy_prefix.data(), part.heavy_prefix.size() * 8);
        }
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

/* detail::psa_plan (alias.hpp:214-238) -> P rows of
 * (light_lo, light_hi, heavy_lo, heavy_hi) and spill. Returns 2 on
 * logic_error. */
int ref_psa_plan(const double* w, uint64_t n, uint64_t P, uint64_t* bounds, double* spill) {
    try {
        auto wt = table_of(w, n);
        const auto part = wrs::detail::partition_items(wt, 1);
        const auto jobs = wrs::detail::psa_plan(part, wt, static_cast<unsigned>(P));
        for (uint64_t k = 0; k < jobs.size(); ++k) {
            bounds[4 * k + 0] = jobs[k].light_lo;
            bounds[4 * k + 1] = jobs[k].light_hi;
            bounds[4 * k + 2] = jobs[k].heavy_lo;
            bounds[4 * k + 3] = jobs[k].heavy_hi;
            spill[k] = jobs[k].spill;
        }
        return 0;
    } catch (const std::logic_error&) {
        return 2;
    } catch (const std::exception&) {
        return 1;
    }
}

/* AliasTable(wt, Build::vose / Build::sweep) -- the reference's other
 * builders (alias.hpp:299-409), extra oracles for the masses.
 * method: 0 = vose, 1 = sweep.  Returns 0 on success. */
int ref_build_method(const double* w, uint64_t n, int method, void* buckets, double* bucket_mean) {
    try {
        auto wt = table_of(w, n);
        wrs::AliasTable t(wt, method == 0 ? wrs::AliasTable::Build::vose : wrs::AliasTable::Build::sweep);
        copy_buckets(t.buckets(), buckets);
        *bucket_mean = t.bucket_mean();
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

/* A reference table kept alive for sampling / verification. */
void* ref_table_new(const double* w, uint64_t n, unsigned workers) {
    try {
        auto wt = table_of(w, n);
        return new wrs::AliasTable(wt, wrs::AliasTable::Build::psa, workers);
    } catch (const std::exception&) {
        return nullptr;
    }
}

void ref_table_free(void* h) { delete static_cast<wrs::AliasTable*>(h); }

void ref_table_buckets(void* h, void* out, double* bucket_mean) {
    auto* t = static_cast<wrs::AliasTable*>(h);
    copy_buckets(t->buckets(), out);
    *bucket_mean = t->bucket_mean();
}

/* AliasTable::sample_many (alias.hpp:274-284) into a caller buffer. */
void ref_table_sample_many(void* h, uint64_t seed, uint64_t k, unsigned workers,
                           uint32_t* out) {
    auto* t = static_cast<wrs::AliasTable*>(h);
    std::vector<uint32_t> buf;
    buf.reserve(k);
    t->sample_many(seed, k, workers, buf);
    std::memcpy(out, buf.data(), k * sizeof(uint32_t));
}

/* The CPU baseline's pieces (BASELINE.md "CPU baseline plan"): the
 * WeightTable is made outside the timed region, AliasTable(wt, psa, T) is
 * timed alone (bucket allocation and first touch included, alias.hpp:251). */
void* ref_wt_new(const double* w, uint64_t n) {
    try {
        return new wrs::WeightTable(table_of(w, n));
    } catch (const std::exception&) {
        return nullptr;
    }
}
void ref_wt_free(void* wt) { delete static_cast<wrs::WeightTable*>(wt); }
void* ref_table_from_wt(const void* wt, unsigned workers) {
    try {
        return new wrs::AliasTable(*static_cast<const wrs::WeightTable*>(wt),
                                   wrs::AliasTable::Build::psa, workers);
    } catch (const std::exception&) {
        return nullptr;
    }
}

/* Time-honest variant for the CPU baseline: the caller's vector is reused
 * across calls, as the reference's own benchmark does (alias.hpp:271-273). */
void* ref_outbuf_new(uint64_t k) {
    auto* v = new std::vector<uint32_t>();
    v->resize(k);
    return v;
}
void ref_outbuf_free(void* v) { delete static_cast<std::vector<uint32_t>*>(v); }
const uint32_t* ref_outbuf_data(void* v) { return static_cast<std::vector<uint32_t>*>(v)->data(); }
void ref_table_sample_into(void* h, uint64_t seed, uint64_t k, unsigned workers, void* v) {
    static_cast<wrs::AliasTable*>(h)->sample_many(seed, k, workers,
                                                  *static_cast<std::vector<uint32_t>*>(v));
}

/* implied_masses over a caller-supplied bucket array (verify.hpp:43-54). */
void ref_implied_masses(const void* buckets, uint64_t n, double bucket_mean, double* out) {
    std::span<const wrs::alias_bucket> b(static_cast<const wrs::alias_bucket*>(buckets), n);
    const auto m = wrs::implied_masses(b, bucket_mean);
    std::memcpy(out, m.data(), n * sizeof(double));
}

/* binomial_split (binomial.hpp:161-170) on RngStream(seed, stream).derive(salt). */
uint64_t ref_binomial_split(uint64_t seed, uint64_t stream, int64_t salt, uint64_t k,
                            double wl, double wr) {
    wrs::RngStream r(seed, stream);
    if (salt >= 0)
        r = r.derive(static_cast<uint64_t>(salt));
    return wrs::binomial_split(r, k, wl, wr);
}

/* TwoLevelTable group layout and totals (two_level.hpp:30-58): the group
 * boundaries come from the reference object; the totals are not exposed, so
 * they are recomputed exactly as :49-51 does (a WeightTable per group). */
uint64_t ref_two_level_group_totals(const double* w, uint64_t n, uint64_t groups,
                                    double* totals) {
    auto wt = table_of(w, n);
    wrs::TwoLevelTable t(wt, wrs::AliasTable::Build::sweep, 1, groups);
    for (size_t g = 0; g < t.groups(); ++g) {
        const size_t lo = t.group_begin(g);
        const size_t hi = g + 1 < t.groups() ? t.group_begin(g + 1) : n;
        totals[g] = wrs::WeightTable(std::vector<double>(w + lo, w + hi)).total();
    }
    return t.groups();
}

/* TwoLevelTable(wt, psa, 1, groups) itself (two_level.hpp:26-58): its local
 * and top tables and sample_many (:71-81), for the routed-draw pins. */
void* ref_two_level_new(const double* w, uint64_t n, uint64_t groups) {
    try {
        auto wt = table_of(w, n);
        return new wrs::TwoLevelTable(wt, wrs::AliasTable::Build::psa, 1, groups);
    } catch (...) {
        return nullptr;
    }
}
void ref_two_level_free(void* h) { delete static_cast<wrs::TwoLevelTable*>(h); }
uint64_t ref_two_level_groups(const void* h) {
    return static_cast<const wrs::TwoLevelTable*>(h)->groups();
}
uint64_t ref_two_level_group_begin(const void* h, uint64_t g) {
    return static_cast<const wrs::TwoLevelTable*>(h)->group_begin(g);
}
/* g < groups: local table g; g == groups: the top table.  Returns its size. */
uint64_t ref_two_level_buckets(const void* h, uint64_t g, void* out, double* mean) {
    const auto* t = static_cast<const wrs::TwoLevelTable*>(h);
    const wrs::AliasTable& a = g < t->groups() ? t->local(g) : t->top();
    if (out) std::memcpy(out, a.buckets().data(), a.size() * sizeof(wrs::alias_bucket));
    if (mean) *mean = a.bucket_mean();
    return a.size();
}
void ref_two_level_sample_many(const void* h, uint64_t seed, uint64_t k, unsigned workers,
                               uint32_t* out) {
    std::vector<uint32_t> v;
    static_cast<const wrs::TwoLevelTable*>(h)->sample_many(seed, k, workers, v);
    std::memcpy(out, v.data(), k * sizeof(uint32_t));
}

} // extern "C"
