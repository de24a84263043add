// paper_1903_00227_b200/csrc/shard.cpp -- the multi-GPU pieces of the path
// that are pure host arithmetic: contiguous shard ranges (two_level.hpp:33-41)
// and the communication-free multinomial split of k over shards.
//
// Split: a binary divide-and-conquer over the shard range [a, b).  Node v
// splits its k between [a, mid) and [mid, b), mid = a + (b-a)/2, with
// binomial_split(RngStream(seed, 'shrd').derive(v), k, W_left, W_right)
// (binomial.hpp:161-170); children of v are 2v+1 and 2v+2.  Every rank runs
// the same descent from the same seed and the same allgathered totals, so all
// ranks agree on every shard's count without exchanging anything.  W_left and
// W_right are pairwise sums of the shard totals (weights.hpp:19-28), the
// totals being the shards' own bit-exact pairwise totals.
//
// The binomial sampler restates Hoermann's BTRD / CDF inversion exactly as
// the reference's binomial.hpp:24-153 evaluates it (same constants, same
// operation order, same RNG consumption), so a host replay with the
// reference's binomial_split reproduces every count (tests/test_shard.py).
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <limits>
#include <vector>

#include "engine.h"
#include "wrs_b200.h"

namespace {

struct Rng {  // RngStream (rng.hpp:32-82)
    uint64_t key, ctr = 0;
    uint64_t next() {
        ctr += wrsb::kGolden;
        return wrsb::mix64(key + ctr);
    }
    double uniform01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

// Stirling tail correction of log k! (binomial.hpp:24-35).
double stirling_fc(int64_t k) {
    static const double t[10] = {0.08106146679532726,  0.04134069595540929,
                                 0.02767792568499834,  0.02079067210376509,
                                 0.01664469118982119,  0.01387612882307075,
                                 0.01189670994589177,  0.01041126526197209,
                                 0.009255462182712733, 0.008330563433362871};
    if (k < 10) return t[k];
    const double r = 1.0 / static_cast<double>(k + 1);
    return (1.0 / 12 - (1.0 / 360 - (1.0 / 1260) * r * r) * r * r) * r;
}

// CDF walk for p <= 0.5 (binomial.hpp:37-63).
uint64_t by_inversion(Rng& rng, uint64_t n, double p) {
    const double q = 1.0 - p, s = p / q;
    const double a = static_cast<double>(n + 1) * s;
    const double r = std::pow(q, static_cast<double>(n));
    for (;;) {
        double u = rng.uniform01();
        uint64_t x = 0;
        double pm = r;
        bool valid = true;
        while (u > pm) {
            u -= pm;
            if (++x > n) {
                valid = false;
                break;
            }
            const double nx = (a / static_cast<double>(x) - s) * pm;
            if (nx < std::numeric_limits<double>::min() && nx < pm) return x > n ? n : x;
            pm = nx;
        }
        if (valid) return x;
    }
}

// BTRD for p <= 0.5, floor((n+1)p) >= 11 (binomial.hpp:66-136).
uint64_t by_btrd(Rng& rng, uint64_t n, double p) {
    const double nd = static_cast<double>(n);
    const int64_t m = static_cast<int64_t>(std::floor((nd + 1) * p));
    const double r = p / (1 - p), nr = (nd + 1) * r, npq = nd * p * (1 - p);
    const double sq = std::sqrt(npq);
    const double b = 1.15 + 2.53 * sq;
    const double a = -0.0873 + 0.0248 * b + 0.01 * p;
    const double c = nd * p + 0.5;
    const double alpha = (2.83 + 5.1 / b) * sq;
    const double vr = 0.92 - 4.2 / b;
    const double urvr = 0.86 * vr;
    for (;;) {
        double v = rng.uniform01(), u;
        if (v <= urvr) {
            u = v / vr - 0.43;
            return static_cast<uint64_t>(std::floor((2 * a / (0.5 - std::abs(u)) + b) * u + c));
        }
        if (v >= vr) {
            u = rng.uniform01() - 0.5;
        } else {
            u = v / vr - 0.93;
            u = (u < 0 ? -0.5 : 0.5) - u;
            v = rng.uniform01() * vr;
        }
        const double us = 0.5 - std::abs(u);
        const double kd = std::floor((2 * a / us + b) * u + c);
        if (kd < 0 || kd > nd) continue;
        const int64_t k = static_cast<int64_t>(kd);
        v = v * alpha / (a / (us * us) + b);
        const int64_t km = std::llabs(k - m);
        if (km <= 15) {
            double f = 1.0;
            if (m < k) {
                for (int64_t i = m + 1; i <= k; ++i) f *= nr / static_cast<double>(i) - r;
            } else if (m > k) {
                for (int64_t i = k + 1; i <= m; ++i) v *= nr / static_cast<double>(i) - r;
            }
            if (v <= f) return static_cast<uint64_t>(k);
            continue;
        }
        const double kmd = static_cast<double>(km);
        v = std::log(v);
        const double rho = (kmd / npq) * (((kmd / 3 + 0.625) * kmd + 1.0 / 6) / npq + 0.5);
        const double t = -kmd * kmd / (2 * npq);
        if (v < t - rho) return static_cast<uint64_t>(k);
        if (v > t + rho) continue;
        const double md = static_cast<double>(m);
        const double nm = nd - md + 1;
        const double h = (md + 0.5) * std::log((md + 1) / (r * nm)) + stirling_fc(m) +
                         stirling_fc(static_cast<int64_t>(nd - md));
        const double nk = nd - kd + 1;
        if (v <= h + (nd + 1) * std::log(nm / nk) + (kd + 0.5) * std::log(nk * r / (kd + 1)) -
                     stirling_fc(k) - stirling_fc(static_cast<int64_t>(nd - kd)))
            return static_cast<uint64_t>(k);
    }
}

uint64_t binomial(Rng& rng, uint64_t n, double p) {  // binomial.hpp:139-156
    if (n == 0 || p <= 0.0) return 0;
    if (p >= 1.0) return n;
    const bool flip = p > 0.5;
    const double ps = flip ? 1.0 - p : p;
    uint64_t x = (n < 32 || std::floor((static_cast<double>(n) + 1) * ps) < 11.0)
                     ? by_inversion(rng, n, ps)
                     : by_btrd(rng, n, ps);
    if (x > n) x = n;
    return flip ? n - x : x;
}

uint64_t binomial_split(Rng& rng, uint64_t k, double wl, double wr) {  // :161-170
    if (k == 0 || wl <= 0.0) return 0;
    if (wr <= 0.0) return k;
    return binomial(rng, k, wl / (wl + wr));
}

double pairwise(const double* v, uint64_t n) {  // weights.hpp:19-28
    if (n <= 32) {
        double s = 0.0;
        for (uint64_t i = 0; i < n; ++i) s += v[i];
        return s;
    }
    const uint64_t h = n / 2;
    return pairwise(v, h) + pairwise(v + h, n - h);
}

constexpr uint64_t kShardStream = 0x73687264u;  // "shrd"

void descend(const double* totals, uint64_t a, uint64_t b, uint64_t node, uint64_t root_key,
             uint64_t k, uint64_t* counts) {
    if (b - a == 1) {
        counts[a] = k;
        return;
    }
    const uint64_t mid = a + (b - a) / 2;
    Rng rng{wrsb::rng_derive(root_key, node)};
    const uint64_t kl = binomial_split(rng, k, pairwise(totals + a, mid - a),
                                       pairwise(totals + mid, b - mid));
    descend(totals, a, mid, 2 * node + 1, root_key, kl, counts);
    descend(totals, mid, b, 2 * node + 2, root_key, k - kl, counts);
}

}  // namespace

extern "C" {

void wrs_b200_shard_range(uint64_t n, uint64_t groups, uint64_t g, uint64_t* lo, uint64_t* hi) {
    if (!lo || !hi) return;
    if (groups == 0) groups = 1;
    if (groups > n) groups = n ? n : 1;
    const uint64_t block = n ? (n + groups - 1) / groups : 0;
    *lo = std::min<uint64_t>(n, g * block);
    *hi = std::min<uint64_t>(n, (g + 1) * block);
}

wrs_status wrs_b200_shard_counts(const double* totals, uint64_t groups, uint64_t seed, uint64_t k,
                                 uint64_t* counts) {
    if (!totals || !counts || groups == 0) return WRS_EINVAL;
    descend(totals, 0, groups, 0, wrsb::rng_key(seed, kShardStream), k, counts);
    return WRS_OK;
}

}  // extern "C"
