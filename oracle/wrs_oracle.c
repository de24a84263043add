/*
 * oracle/wrs_oracle.c -- TEST INFRASTRUCTURE ONLY (see wrs_oracle.h).
 *
 * Plain-C restatement of the reference's PSA build and alias sampling.  The
 * floating-point operations are written in the reference's evaluation order
 * and compiled with -ffp-contract=off so every rounding step matches the
 * reference's x86-64 SSE2 build bit for bit.  Line citations are to
 * /root/reference/proj.
 */
#include "wrs_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- rng */

/* mix64: include/wrs/rng.hpp:16-20 */
uint64_t wo_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * UINT64_C(0xbf58476d1ce4e5b9);
    z = (z ^ (z >> 27)) * UINT64_C(0x94d049bb133111eb);
    return z ^ (z >> 31);
}

/* kGolden: rng.hpp:23 */
static const uint64_t kGolden = UINT64_C(0x9e3779b97f4a7c15);

/* RngStream(seed, stream): rng.hpp:36-37 */
wo_rng wo_rng_make(uint64_t seed, uint64_t stream) {
    wo_rng r;
    r.key = wo_mix64(wo_mix64(seed + kGolden) ^ wo_mix64(stream) ^ stream);
    r.ctr = 0;
    return r;
}

/* derive(salt): rng.hpp:40-45 */
wo_rng wo_rng_derive(const wo_rng* r, uint64_t salt) {
    wo_rng c;
    c.key = wo_mix64(r->key + wo_mix64(salt + kGolden));
    c.ctr = 0;
    return c;
}

/* next(): rng.hpp:47-50 */
uint64_t wo_rng_next(wo_rng* r) {
    r->ctr += kGolden;
    return wo_mix64(r->key + r->ctr);
}

/* uniform01(): rng.hpp:53-55 -- 53 random bits times 2^-53 */
double wo_rng_uniform01(wo_rng* r) {
    return (double)(wo_rng_next(r) >> 11) * 0x1.0p-53;
}

/* bounded(n): rng.hpp:63-66 -- high word of the 128-bit product */
uint64_t wo_rng_bounded(wo_rng* r, uint64_t n) {
    return (uint64_t)(((unsigned __int128)wo_rng_next(r) * n) >> 64);
}

/* `count` successive next() outputs of RngStream(seed, stream), or of its
 * derive(salt) child when salt >= 0. */
void wo_rng_outputs(uint64_t seed, uint64_t stream, int64_t salt, uint64_t count, uint64_t* out) {
    wo_rng r = wo_rng_make(seed, stream);
    if (salt >= 0)
        r = wo_rng_derive(&r, (uint64_t)salt);
    for (uint64_t i = 0; i < count; ++i)
        out[i] = wo_rng_next(&r);
}

/* --------------------------------------------------------- generators */

/* generate_uniform: weight_file.hpp:32-38 (stream 'genu') */
void wo_generate_uniform(uint64_t n, uint64_t seed, double* out) {
    wo_rng rng = wo_rng_make(seed, 0x67656e75u);
    for (uint64_t i = 0; i < n; ++i)
        out[i] = 1.0 - wo_rng_uniform01(&rng);
}

/* generate_powerlaw: weight_file.hpp:42-54 (stream 'genp'), (i+1)^-s then a
 * Fisher-Yates pass from the top. */
int wo_generate_powerlaw(uint64_t n, double s, uint64_t seed, double* out) {
    if (!(s >= 0.0) || !isfinite(s))
        return 1;
    wo_rng rng = wo_rng_make(seed, 0x67656e70u);
    for (uint64_t i = 0; i < n; ++i)
        out[i] = pow((double)(i + 1), -s);
    for (uint64_t i = n; i > 1; --i) {
        const uint64_t j = wo_rng_bounded(&rng, i);
        const double t = out[i - 1];
        out[i - 1] = out[j];
        out[j] = t;
    }
    return 0;
}

/* generate_lognormal: configs[3]'s weights -- NOT a reference generator (the
 * reference has none); the library's own, defined in
 * paper_1903_00227_b200/csrc/common.cuh (lognormal_weight) and restated
 * here operation for operation so the reference can be fed the same bytes:
 * item i takes outputs 2i+1, 2i+2 of RngStream(seed, 'logn'),
 * w = exp(sigma * sqrt(-2 log(1 - u1)) * cos(2 pi u2)), with log / cos / exp
 * evaluated by the same argument reductions and Horner series. */
static const double kLn2Hi = 0x1.62e42fefa3800p-1, kLn2Lo = 0x1.ef35793c76730p-45;

static double det_log(double x) {
    uint64_t b;
    memcpy(&b, &x, 8);
    int e = (int)((b >> 52) & 0x7ff) - 1023;
    b = (b & UINT64_C(0x000fffffffffffff)) | UINT64_C(0x3ff0000000000000);
    double m;
    memcpy(&m, &b, 8);
    if (m > 1.4142135623730951) {
        m = m * 0.5;
        e += 1;
    }
    const double s = (m - 1.0) / (m + 1.0), s2 = s * s;
    static const double c[13] = {1.0 / 25.0, 1.0 / 23.0, 1.0 / 21.0, 1.0 / 19.0, 1.0 / 17.0,
                                 1.0 / 15.0, 1.0 / 13.0, 1.0 / 11.0, 1.0 / 9.0,  1.0 / 7.0,
                                 1.0 / 5.0,  1.0 / 3.0,  1.0};
    double p = c[0];
    for (int k = 1; k < 13; ++k) p = p * s2 + c[k];
    const double de = (double)e;
    return de * kLn2Hi + (de * kLn2Lo + 2.0 * s * p);
}

static double det_cos2pi(double u) {
    double a = u - 0.5;
    a = a < 0.0 ? -a : a;
    double sign = -1.0;
    if (a > 0.25) {
        a = 0.5 - a;
        sign = 1.0;
    }
    const double t = a * 6.283185307179586, t2 = t * t;
    static const double c[13] = {1.0 / 620448401733239439360000.0, 1.0 / 1124000727777607680000.0,
                                 1.0 / 2432902008176640000.0,      1.0 / 6402373705728000.0,
                                 1.0 / 20922789888000.0,           1.0 / 87178291200.0,
                                 1.0 / 479001600.0,                1.0 / 3628800.0,
                                 1.0 / 40320.0,                    1.0 / 720.0,
                                 1.0 / 24.0,                       1.0 / 2.0,
                                 1.0};
    double p = c[0];
    for (int k = 1; k < 13; ++k) p = p * -t2 + c[k];
    return sign * p;
}

static double det_exp(double x) {
    const double kf = floor(x * 1.4426950408889634 + 0.5);
    const double r = (x - kf * kLn2Hi) - kf * kLn2Lo;
    static const double c[19] = {1.0 / 355687428096000.0, 1.0 / 20922789888000.0,
                                 1.0 / 1307674368000.0,   1.0 / 87178291200.0,
                                 1.0 / 6227020800.0,      1.0 / 479001600.0,
                                 1.0 / 39916800.0,        1.0 / 3628800.0,
                                 1.0 / 362880.0,          1.0 / 40320.0,
                                 1.0 / 5040.0,            1.0 / 720.0,
                                 1.0 / 120.0,             1.0 / 24.0,
                                 1.0 / 6.0,               0.5,
                                 1.0,                     1.0};
    double p = c[0];
    for (int k = 1; k < 18; ++k) p = p * r + c[k];
    const uint64_t eb = (uint64_t)((int64_t)kf + 1023) << 52;
    double scale;
    memcpy(&scale, &eb, 8);
    return p * scale;
}

void wo_generate_lognormal(uint64_t n, double sigma, uint64_t seed, double* out) {
    const wo_rng rng = wo_rng_make(seed, 0x6c6f676eu); /* 'logn' */
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t r1 = wo_mix64(rng.key + (2 * i + 1) * kGolden);
        const uint64_t r2 = wo_mix64(rng.key + (2 * i + 2) * kGolden);
        const double u1 = 1.0 - (double)(r1 >> 11) * 0x1.0p-53;
        const double u2 = (double)(r2 >> 11) * 0x1.0p-53;
        const double z = sqrt(-2.0 * det_log(u1)) * det_cos2pi(u2);
        out[i] = det_exp(sigma * z);
    }
}

/* ------------------------------------------------------------ weights */

/* pairwise_sum: weights.hpp:19-28 -- leaves of <= 32 summed left to right,
 * split at floor(n/2). */
double wo_pairwise_sum(const double* v, uint64_t n) {
    if (n <= 32) {
        double s = 0.0;
        for (uint64_t i = 0; i < n; ++i)
            s += v[i];
        return s;
    }
    const uint64_t half = n / 2;
    return wo_pairwise_sum(v, half) + wo_pairwise_sum(v + half, n - half);
}

/* WeightTable ctor: weights.hpp:32-46 */
int wo_weights_check(const double* w, uint64_t n, uint64_t* bad, double* total,
                     double* wmin, double* wmax) {
    if (n == 0) {
        if (bad)
            *bad = 0;
        return 1;
    }
    double mn = w[0], mx = w[0];
    for (uint64_t i = 0; i < n; ++i) {
        const double x = w[i];
        if (!isfinite(x) || x <= 0.0) {
            if (bad)
                *bad = i;
            return 1;
        }
        mn = x < mn ? x : mn;
        mx = x > mx ? x : mx;
    }
    if (total)
        *total = wo_pairwise_sum(w, n);
    if (wmin)
        *wmin = mn;
    if (wmax)
        *wmax = mx;
    return 0;
}

/* --------------------------------------------------------------- scan */

/* comp_sum (Neumaier): parallel.hpp:70-81 */
typedef struct {
    double hi, lo;
} cs_t;

static inline void cs_add(cs_t* s, double x) {
    const double t = s->hi + x;
    if (isfinite(t))
        s->lo += fabs(s->hi) >= fabs(x) ? (s->hi - t) + x : (x - t) + s->hi;
    s->hi = t;
}
static inline double cs_value(const cs_t* s) { return s->hi + s->lo; }

#define WO_SCAN_BLOCK 2048 /* kScanBlock: parallel.hpp:60 */

/* prefix_sums pass 1: parallel.hpp:110-115 */
void wo_scan_block_totals(const double* in, uint64_t n, double* totals) {
    const uint64_t nb = (n + WO_SCAN_BLOCK - 1) / WO_SCAN_BLOCK;
    for (uint64_t b = 0; b < nb; ++b) {
        const uint64_t lo = b * WO_SCAN_BLOCK;
        const uint64_t hi = lo + WO_SCAN_BLOCK < n ? lo + WO_SCAN_BLOCK : n;
        cs_t local = {0.0, 0.0};
        for (uint64_t i = lo; i < hi; ++i)
            cs_add(&local, in[i]);
        totals[b] = cs_value(&local);
    }
}

/* prefix_sums pass 2: parallel.hpp:116-121 (exclusive, in place) */
void wo_scan_carries(double* c, uint64_t nb) {
    cs_t acc = {0.0, 0.0};
    for (uint64_t b = 0; b < nb; ++b) {
        const double total = c[b];
        c[b] = cs_value(&acc);
        cs_add(&acc, total);
    }
}

/* prefix_sums: parallel.hpp:104-130 (pass 3 at :122-129) */
void wo_prefix_sums(const double* in, double* out, uint64_t n) {
    if (n == 0)
        return;
    const uint64_t nb = (n + WO_SCAN_BLOCK - 1) / WO_SCAN_BLOCK;
    double* carry = (double*)malloc(nb * sizeof(double));
    wo_scan_block_totals(in, n, carry);
    wo_scan_carries(carry, nb);
    for (uint64_t b = 0; b < nb; ++b) {
        const uint64_t lo = b * WO_SCAN_BLOCK;
        const uint64_t hi = lo + WO_SCAN_BLOCK < n ? lo + WO_SCAN_BLOCK : n;
        cs_t run = {0.0, 0.0};
        cs_add(&run, carry[b]);
        for (uint64_t i = lo; i < hi; ++i) {
            cs_add(&run, in[i]);
            out[i] = cs_value(&run);
        }
    }
    free(carry);
}

/* ---------------------------------------------------------- partition */

/* partition_items: alias.hpp:48-97.  The reference's 4096-item blocks only
 * parallelise a stable partition, so a single stable pass is the same
 * result (ascending index order inside both lists). */
int wo_partition_items(const double* w, uint64_t n, double total, wo_partition* p) {
    memset(p, 0, sizeof *p);
    const double wn = total / (double)n; /* :50 */
    p->wn = wn;
    uint64_t nl = 0;
    for (uint64_t i = 0; i < n; ++i)
        nl += (w[i] <= wn); /* ties are light, :60 */
    p->nl = nl;
    p->nh = n - nl;
    p->light = (uint32_t*)malloc((nl ? nl : 1) * sizeof(uint32_t));
    p->heavy = (uint32_t*)malloc((p->nh ? p->nh : 1) * sizeof(uint32_t));
    p->light_prefix = (double*)calloc(nl + 1, sizeof(double));
    p->heavy_prefix = (double*)calloc(p->nh + 1, sizeof(double));
    if (!p->light || !p->heavy || !p->light_prefix || !p->heavy_prefix)
        return 1;
    uint64_t li = 0, hi = 0;
    for (uint64_t i = 0; i < n; ++i) { /* :72-80 */
        if (w[i] <= wn)
            p->light[li++] = (uint32_t)i;
        else
            p->heavy[hi++] = (uint32_t)i;
    }
    /* exclusive_prefix: gather then prefix_sums into out+1, :82-95 */
    double* g = (double*)malloc((n ? n : 1) * sizeof(double));
    for (uint64_t i = 0; i < nl; ++i)
        g[i] = w[p->light[i]];
    wo_prefix_sums(g, p->light_prefix + 1, nl);
    for (uint64_t j = 0; j < p->nh; ++j)
        g[j] = w[p->heavy[j]];
    wo_prefix_sums(g, p->heavy_prefix + 1, p->nh);
    free(g);
    return 0;
}

void wo_partition_free(wo_partition* p) {
    free(p->light);
    free(p->heavy);
    free(p->light_prefix);
    free(p->heavy_prefix);
    memset(p, 0, sizeof *p);
}

/* --------------------------------------------------------------- split */

/* psa_split: alias.hpp:122-149.  Same binary search (same probe sequence),
 * so even a non-monotone f in floating point yields the reference's j. */
wo_split wo_psa_split(const wo_partition* p, const double* w, uint64_t n_prime) {
    const uint64_t nl = p->nl, nh = p->nh;
    const double target = (double)n_prime * p->wn; /* :125 */
    uint64_t lo = n_prime > nl ? n_prime - nl : 0;  /* :135 */
    uint64_t hi = n_prime < nh ? n_prime : nh;      /* :136 */
    while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        double f;
        if (mid >= nh)
            f = INFINITY; /* :130-131 */
        else
            f = (p->light_prefix[n_prime - mid] + p->heavy_prefix[mid]) + w[p->heavy[mid]];
        if (f > target)
            hi = mid;
        else
            lo = mid + 1;
    }
    wo_split s;
    s.heavy_count = lo;
    s.light_count = n_prime - lo;
    if (lo < nh) { /* :147 std::max(0.0, x) == (0.0 < x ? x : 0.0) */
        const double x = (w[p->heavy[lo]] + (p->light_prefix[n_prime - lo] + p->heavy_prefix[lo])) - target;
        s.spill = 0.0 < x ? x : 0.0;
    } else {
        s.spill = 0.0;
    }
    return s;
}

/* psa_plan: alias.hpp:214-238 */
int wo_psa_plan(const wo_partition* p, const double* w, uint64_t n, uint64_t P,
                wo_job* jobs) {
    uint64_t prev_l = 0, prev_j = 0;
    double carry = p->nh == 0 ? 0.0 : w[p->heavy[0]];
    for (uint64_t k = 0; k < P; ++k) {
        wo_split s;
        if (k + 1 == P) {
            s.light_count = p->nl;
            s.heavy_count = p->nh;
            s.spill = 0.0;
        } else {
            const uint64_t m = n * (k + 1);
            const uint64_t n_prime = m / P + (m % P != 0); /* :227 */
            s = wo_psa_split(p, w, n_prime);
        }
        if (s.light_count < prev_l || s.heavy_count < prev_j)
            return 1; /* :230-231 logic_error */
        jobs[k].light_lo = prev_l;
        jobs[k].light_hi = s.light_count;
        jobs[k].heavy_lo = prev_j;
        jobs[k].heavy_hi = s.heavy_count;
        jobs[k].spill = carry;
        prev_l = s.light_count;
        prev_j = s.heavy_count;
        carry = s.spill;
    }
    return 0;
}

/* ---------------------------------------------------------------- pack */

static inline double min_d(double a, double b) { return b < a ? b : a; } /* std::min */
static inline double max_d(double a, double b) { return a < b ? b : a; } /* std::max */

/* psa_pack: alias.hpp:160-209 */
void wo_psa_pack(const wo_partition* p, const double* w, const wo_job* job,
                 wo_bucket* buckets) {
    const uint64_t nh = p->nh;
    const double wn = p->wn;
#define HEAVY_AT(j) (p->heavy[(j) < nh - 1 ? (j) : nh - 1]) /* :164 */
    uint64_t i = job->light_lo;
    uint64_t j = job->heavy_lo;
    cs_t rem = {j < nh ? job->spill : INFINITY, 0.0}; /* :168 */
    for (;;) {
        if (cs_value(&rem) > wn) {
            if (i >= job->light_hi) { /* :172-184 */
                while (j < job->heavy_hi) {
                    const uint32_t idx = p->heavy[j];
                    buckets[idx].share = min_d(cs_value(&rem), wn);
                    buckets[idx].item = idx;
                    buckets[idx].alias = HEAVY_AT(j + 1);
                    if (j + 1 < nh)
                        cs_add(&rem, w[p->heavy[j + 1]] - wn);
                    else {
                        rem.hi = wn;
                        rem.lo = 0.0;
                    }
                    ++j;
                }
                return;
            }
            const uint32_t idx = p->light[i]; /* :186-189 */
            buckets[idx].share = w[idx];
            buckets[idx].item = idx;
            buckets[idx].alias = HEAVY_AT(j);
            cs_add(&rem, w[idx] - wn);
            ++i;
        } else {
            if (j >= job->heavy_hi) { /* :191-198 */
                for (; i < job->light_hi; ++i) {
                    const uint32_t idx = p->light[i];
                    buckets[idx].share = w[idx];
                    buckets[idx].item = idx;
                    buckets[idx].alias = HEAVY_AT(j);
                }
                return;
            }
            const uint32_t idx = p->heavy[j]; /* :200-206 */
            buckets[idx].share = max_d(0.0, min_d(cs_value(&rem), wn));
            buckets[idx].item = idx;
            buckets[idx].alias = HEAVY_AT(j + 1);
            if (j + 1 < nh)
                cs_add(&rem, w[p->heavy[j + 1]] - wn);
            else {
                rem.hi = INFINITY;
                rem.lo = 0.0;
            }
            ++j;
        }
    }
#undef HEAVY_AT
}

/* AliasTable(wt, psa, P): alias.hpp:246-257 + build_psa :411-419 +
 * fill_uniform_if_no_heavy :288-297 */
int wo_psa_build(const double* w, uint64_t n, uint64_t P, wo_bucket* buckets,
                 double* bucket_mean) {
    double total;
    if (wo_weights_check(w, n, NULL, &total, NULL, NULL))
        return 1;
    if (n > UINT32_MAX)
        return 2;
    if (P == 0)
        P = 1; /* std::max(1u, workers), :255 */
    const double wn = total / (double)n;
    if (bucket_mean)
        *bucket_mean = wn;
    memset(buckets, 0, n * sizeof(wo_bucket)); /* buckets_.resize(n) */
    int any_heavy = 0;
    for (uint64_t i = 0; i < n; ++i)
        if (w[i] > wn) {
            any_heavy = 1;
            break;
        }
    if (!any_heavy) {
        for (uint64_t i = 0; i < n; ++i) {
            buckets[i].share = w[i];
            buckets[i].item = (uint32_t)i;
            buckets[i].alias = (uint32_t)i;
        }
        return 0;
    }
    wo_partition part;
    if (wo_partition_items(w, n, total, &part)) {
        wo_partition_free(&part);
        return 1;
    }
    wo_job* jobs = (wo_job*)malloc(P * sizeof(wo_job));
    int rc = wo_psa_plan(&part, w, n, P, jobs);
    if (rc == 0)
        for (uint64_t k = 0; k < P; ++k)
            wo_psa_pack(&part, w, &jobs[k], buckets);
    free(jobs);
    wo_partition_free(&part);
    return rc ? 3 : 0;
}

/* -------------------------------------------------------------- sample */

/* worker_slice: parallel.hpp:37-43 */
static void worker_slice(uint64_t k, uint32_t workers, uint32_t wk, uint64_t* lo,
                         uint64_t* hi) {
    const uint64_t per = k / workers, rem = k % workers;
    *lo = per * wk + (wk < rem ? wk : rem);
    *hi = *lo + per + (wk < rem ? 1 : 0);
}

/* AliasTable::sample: alias.hpp:265-269 */
static inline uint32_t sample_one(const wo_bucket* b, uint64_t n, double wn, wo_rng* rng) {
    const wo_bucket* bk = &b[wo_rng_bounded(rng, n)];
    const double x = wo_rng_uniform01(rng) * wn;
    return x >= bk->share ? bk->alias : bk->item;
}

/* sample_many: alias.hpp:274-284 -- worker w draws its slice from
 * RngStream(seed, 'alia').derive(w). */
void wo_sample_many(const wo_bucket* b, uint64_t n, double wn, uint64_t seed,
                    uint64_t k, uint32_t workers, uint32_t* out) {
    wo_sample_range(b, n, wn, seed, k, workers, 0, k, out);
}

void wo_sample_range(const wo_bucket* b, uint64_t n, double wn, uint64_t seed,
                     uint64_t k, uint32_t workers, uint64_t q_lo, uint64_t q_hi,
                     uint32_t* out) {
    if (workers == 0)
        workers = 1;
    const wo_rng base = wo_rng_make(seed, 0x616c6961u);
    for (uint32_t wk = 0; wk < workers; ++wk) {
        uint64_t lo, hi;
        worker_slice(k, workers, wk, &lo, &hi);
        if (hi <= q_lo || lo >= q_hi)
            continue;
        wo_rng rng = wo_rng_derive(&base, wk);
        const uint64_t start = lo > q_lo ? lo : q_lo;
        const uint64_t end = hi < q_hi ? hi : q_hi;
        /* counter position: each earlier query consumed two outputs */
        rng.ctr = (start - lo) * 2 * kGolden;
        for (uint64_t q = start; q < end; ++q)
            out[q - q_lo] = sample_one(b, n, wn, &rng);
    }
}

/* TwoLevelTable::sample (two_level.hpp:66-69): group by the top table, then
 * the group's own table; sample_many (:71-81) with RngStream(seed, '2lvl'). */
void wo_two_level_sample_range(const wo_bucket* const* tables, const uint64_t* sizes,
                               const double* means, const uint64_t* bases, uint64_t groups,
                               const wo_bucket* top, double top_mean, uint64_t seed,
                               uint64_t k, uint32_t workers, uint64_t q_lo, uint64_t q_hi,
                               uint32_t* out) {
    if (workers == 0)
        workers = 1;
    const wo_rng base = wo_rng_make(seed, 0x326c766cu);
    for (uint32_t wk = 0; wk < workers; ++wk) {
        uint64_t lo, hi;
        worker_slice(k, workers, wk, &lo, &hi);
        if (hi <= q_lo || lo >= q_hi)
            continue;
        wo_rng rng = wo_rng_derive(&base, wk);
        const uint64_t start = lo > q_lo ? lo : q_lo;
        const uint64_t end = hi < q_hi ? hi : q_hi;
        rng.ctr = (start - lo) * 4 * kGolden; /* four outputs per earlier query */
        for (uint64_t q = start; q < end; ++q) {
            const uint32_t g = sample_one(top, groups, top_mean, &rng);
            out[q - q_lo] = (uint32_t)bases[g] + sample_one(tables[g], sizes[g], means[g], &rng);
        }
    }
}

/* Philox4x32-10: Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as
 * easy as 1, 2, 3" (SC'11) -- multipliers 0xD2511F53 / 0xCD9E8D57, Weyl key
 * increments 0x9E3779B9 / 0xBB67AE85, ten rounds. */
void wo_philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
        c[1] = (uint32_t)p1;
        c[3] = (uint32_t)p0;
        c[0] = n0;
        c[2] = n2;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

void wo_sample_philox_range(const wo_bucket* b, uint64_t n, double wn, uint64_t seed,
                            uint64_t q_lo, uint64_t q_hi, uint32_t* out) {
    for (uint64_t q = q_lo; q < q_hi; ++q) {
        uint32_t o[4] = {(uint32_t)q, (uint32_t)(q >> 32), 0u, 0u};
        wo_philox4x32_10(o, (uint32_t)seed, (uint32_t)(seed >> 32));
        const uint64_t r = ((uint64_t)o[1] << 32) | o[0];
        const uint64_t i = (uint64_t)(((unsigned __int128)r * n) >> 64);
        const uint64_t r2 = ((uint64_t)o[3] << 32) | o[2];
        const double x = ((double)(r2 >> 11) * 0x1.0p-53) * wn;
        out[q - q_lo] = x >= b[i].share ? b[i].alias : b[i].item;
    }
}

/* -------------------------------------------------------------- verify */

/* kahan_sum: verify.hpp:26-38; implied_masses: verify.hpp:43-54 */
void wo_implied_masses(const wo_bucket* b, uint64_t n, double wn, double* m) {
    double* c = (double*)calloc(n, sizeof(double));
    memset(m, 0, n * sizeof(double));
#define KADD(acc_s, acc_c, x)                                                        \
    do {                                                                             \
        const double y_ = (x) - (acc_c);                                             \
        const double t_ = (acc_s) + y_;                                              \
        (acc_c) = (t_ - (acc_s)) - y_;                                               \
        (acc_s) = t_;                                                                \
    } while (0)
    for (uint64_t i = 0; i < n; ++i) {
        KADD(m[b[i].item], c[b[i].item], b[i].share);
        KADD(m[b[i].alias], c[b[i].alias], wn - b[i].share);
    }
#undef KADD
    free(c);
}

/* max_relative_mass_error: verify.hpp:92-98 */
double wo_max_relative_mass_error(const double* m, const double* w, uint64_t n) {
    double worst = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        const double e = fabs(m[i] - w[i]) / w[i];
        worst = worst < e ? e : worst; /* std::max(worst, e) */
    }
    return worst;
}
