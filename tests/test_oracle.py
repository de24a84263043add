"""CPU: pin the oracle (oracle/wrs_oracle.c) against the reference's golden
vectors (tests/golden/, produced from the unmodified reference by
tests/golden/make_golden.py) and against the reference's own unit-test
expectations (test_alias.cpp, test_parallel.cpp, test_weights.cpp,
test_rng.cpp, test_stats.cpp)."""
import hashlib
import os

import numpy as np
import pytest

import oracle
from tests.stats_util import chi2_critical, chi_square

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def P():
    return oracle.port()


@pytest.fixture(scope="module")
def small():
    return np.load(os.path.join(GOLD, "psa_small.npz"))


def fixture_names(z):
    return sorted({k.split("/")[0] for k in z.files})


def test_golden_tables_all_fixtures(P, small):
    names = fixture_names(small)
    assert len(names) >= 25
    for name in names:
        w = small[f"{name}/w"]
        ok, _, total, _, _ = P.weights_check(w)
        assert ok and total == small[f"{name}/total"], name
        for jobs in (1, 2, 3, 4, 8):
            b, wn = P.psa_build(w, jobs)
            assert wn == small[f"{name}/P{jobs}/bucket_mean"], (name, jobs)
            assert b.tobytes() == small[f"{name}/P{jobs}/buckets"].tobytes(), (name, jobs)
            m = P.implied_masses(b, wn)
            assert m.tobytes() == small[f"{name}/P{jobs}/masses"].tobytes(), (name, jobs)


def test_golden_partition_and_plans(P, small):
    for name in fixture_names(small):
        if f"{name}/part/light" not in small.files:
            continue
        w = small[f"{name}/w"]
        part = P.partition(w)
        for k in ("light", "heavy", "light_prefix", "heavy_prefix"):
            assert part[k].tobytes() == small[f"{name}/part/{k}"].tobytes(), (name, k)
        for jobs in (2, 8):
            key = f"{name}/plan{jobs}/bounds"
            if key in small.files:
                b, s = P.psa_plan(w, jobs)
                assert np.array_equal(b, small[key]), (name, jobs)
                assert s.tobytes() == small[f"{name}/plan{jobs}/spill"].tobytes()


def test_golden_draws(P):
    d = np.load(os.path.join(GOLD, "draws_small.npz"))
    b, wn = P.psa_build(d["w"], 4)
    assert b.tobytes() == d["buckets"].tobytes()
    for W in (1, 3, 4, 8):
        assert np.array_equal(P.sample_many(b, wn, 99, 100001, W), d[f"seed99_W{W}"]), W
    assert np.array_equal(P.sample_many(b, wn, 100, 100001, 4), d["seed100_W4"])
    # any slice of the stream is reproducible on its own (counter RNG)
    full = d["seed99_W3"]
    assert np.array_equal(P.sample_range(b, wn, 99, 100001, 3, 33330, 66680), full[33330:66680])


def test_golden_rng(P):
    r = np.load(os.path.join(GOLD, "rng.npz"))
    assert np.array_equal(P.rng_outputs(42, 7, -1, 64), r["s42_st7"])
    assert np.array_equal(P.rng_outputs(9, 3, 123, 64), r["s9_st3_d123"])
    assert np.array_equal(P.rng_outputs(99, 0x616C6961, 0, 64), r["alia_s99_d0"])
    assert np.array_equal(P.rng_outputs(99, 0x616C6961, 3, 64), r["alia_s99_d3"])


def test_golden_medium_digests(P):
    m = np.load(os.path.join(GOLD, "psa_medium.npz"))
    gens = {"uniform_1e6_s42": lambda: P.generate_uniform(10**6, 42),
            "powerlaw1_1e6_s42": lambda: P.generate_powerlaw(10**6, 1.0, 42),
            "powerlaw05_2e5_s7": lambda: P.generate_powerlaw(200_000, 0.5, 7)}
    for tag, gen in gens.items():
        w = gen()
        assert sha(w) == str(m[f"{tag}/w_sha"]), tag
        ok, _, total, _, _ = P.weights_check(w)
        assert total == m[f"{tag}/total"]
        part = P.partition(w)
        assert sha(part["light"]) == str(m[f"{tag}/light_sha"])
        assert sha(part["heavy_prefix"]) == str(m[f"{tag}/heavy_prefix_sha"])
        jobs_keys = sorted({int(k.split("/")[1][1:]) for k in m.files
                            if k.startswith(tag + "/P")})
        for jobs in jobs_keys:
            b, wn = P.psa_build(w, jobs)
            assert sha(b) == str(m[f"{tag}/P{jobs}/buckets_sha"]), (tag, jobs)
            err = P.max_relative_mass_error(P.implied_masses(b, wn), w)
            assert err == m[f"{tag}/P{jobs}/max_rel_err"]


# ---- the reference's own unit expectations, on the oracle ------------------

def test_fixture_three_one(P):  # test_alias.cpp:56-71
    for jobs in (1, 2):
        b, wn = P.psa_build(np.array([3.0, 1, 1, 1]), jobs)
        assert np.all(b["item"] == np.arange(4))
        assert np.all(b["share"][1:] == 1.0) and np.all(b["alias"][1:] == 0)
        assert abs(b["share"][0] - 1.5) <= 1.5e-12


def test_tiny_mass_exact(P):  # test_alias.cpp:88-98
    b, wn = P.psa_build(np.array([1.0, 1e-12]), 2)
    m = P.implied_masses(b, wn)
    assert m[1] == 1e-12


def test_huge_heavy_filled_once(P):  # test_alias.cpp:173-193
    w = np.ones(100)
    w[0] = 100.0
    b, wn = P.psa_build(w, 8)
    assert int(np.sum(b["item"] == 0)) == 1
    bounds, _ = P.psa_plan(w, 8)
    assert np.all(bounds[:-1, 2] == bounds[:-1, 3])
    assert bounds[-1, 3] == bounds[-1, 2] + 1


def test_split_matches_linear_scan(P):  # test_alias.cpp:195-252
    rng = np.random.default_rng(0xABCD)
    for trial in range(40):
        n = 5 + int(rng.integers(36))
        w = 0.1 + rng.random(n) * np.where(rng.integers(4, size=n) == 0, 25.0, 1.0)
        if trial % 3 == 0:
            w[::3] = 1.0
        part = P.partition(w)
        nl, nh = part["light"].size, part["heavy"].size
        if nh == 0:
            continue
        for npr in range(1, n):
            lc, hc, spill = P.psa_split(w, npr)
            target = npr * part["wn"]
            expect = None
            for j in range(max(0, npr - nl), min(npr, nh) + 1):
                sig = part["light_prefix"][npr - j] + part["heavy_prefix"][j]
                nxt = w[part["heavy"][j]] if j < nh else np.inf
                if sig + nxt > target:
                    expect = j
                    break
            assert hc == expect and lc == npr - expect


def test_prefix_sums_accuracy_and_invariance(P):  # test_parallel.cpp:50-80
    rng = np.random.default_rng(7)
    x = rng.random(50_000) * 10.0 ** (rng.random(50_000) * 6 - 3)
    out = P.prefix_sums(x)
    acc = np.cumsum(x.astype(np.longdouble))
    assert np.all(np.abs(out - acc.astype(np.float64)) <= 1e-12 * acc.astype(np.float64))
    one = P.prefix_sums(np.array([2.5]))
    assert one[0] == 2.5


def test_weights_rules(P):  # test_weights.cpp:14-31
    for bad in ([1.0, 0.0], [1.0, -2.0], [1.0, np.nan], [np.inf]):
        assert not P.weights_check(np.array(bad))[0]
    ok, _, total, mn, mx = P.weights_check(np.array([4.0, 1.0, 2.0, 8.0]))
    assert ok and total == 15.0 and mn == 1.0 and mx == 8.0


def test_chi_square_quantile_pins():  # test_stats.cpp:10-29
    assert abs(chi2_critical(1, 1e-3) - 10.828) <= 10.828e-3
    assert abs(chi2_critical(9, 1e-3) - 27.877) <= 27.877e-3
    assert abs(chi2_critical(99, 1e-3) - 148.23) <= 148.23e-3
    assert chi_square([250] * 4, [0.25] * 4)[3]
    assert not chi_square([700, 100, 100, 100], [0.25] * 4)[3]


def test_oracle_draws_follow_weights(P):  # test_alias.cpp:269-284
    w = P.generate_powerlaw(50, 1.0, 3)
    b, wn = P.psa_build(w, 4)
    s = P.sample_many(b, wn, 99, 100001, 4)
    counts = np.bincount(s, minlength=50)
    assert chi_square(counts, w / w.sum())[3]


def test_golden_two_level(P):  # TwoLevelTable (two_level.hpp:26-81), reference-generated
    t = np.load(os.path.join(GOLD, "two_level.npz"))
    w = P.generate_powerlaw(3001, 1.0, 5)
    assert hashlib.sha256(w.tobytes()).hexdigest() == str(t["w_sha"])
    for G in (4, 7):
        tabs, means, bases, top, tm = P.two_level_build(w, G)
        assert np.array_equal(bases, t[f"G{G}/bases"])
        assert np.array_equal(means, t[f"G{G}/means"])
        assert top.tobytes() == t[f"G{G}/top"].tobytes() and tm == float(t[f"G{G}/top_mean"])
        assert hashlib.sha256(np.concatenate(tabs).tobytes()).hexdigest() == str(t[f"G{G}/tables_sha"])
        for W in (1, 3):
            got = P.two_level_sample_range(tabs, means, bases, top, tm, 7, 5001, W, 0, 5001)
            assert np.array_equal(got, t[f"G{G}/draws_s7_k5001_W{W}"])


def test_philox_known_answers(P):
    # Random123 kat_vectors for philox4x32-10 (Salmon et al., SC'11)
    kat = [((0, 0, 0, 0), (0, 0), (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
           ((0xffffffff,) * 4, (0xffffffff, 0xffffffff), (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
           ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0),
            (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1))]
    for ctr, key, want in kat:
        assert tuple(int(x) for x in P.philox4x32_10(ctr, key)) == want


def test_lognormal_generator_is_accurate_box_muller():
    """configs[3]'s own generator (common.cuh lognormal_weight, restated in
    the oracle): its fixed-sequence log / cos / exp agree with libm to a few
    ulps, on the same RngStream(seed, 'logn') outputs (2i+1, 2i+2)."""
    P = oracle.port()
    n, sigma, seed = 20000, 2.0, 42
    w = P.generate_lognormal(n, sigma, seed)
    r = P.rng_outputs(seed, 0x6C6F676E, -1, 2 * n).reshape(n, 2)
    u1 = 1.0 - (r[:, 0] >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    u2 = (r[:, 1] >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2 * np.pi * u2)
    ref = np.exp(sigma * z)
    assert np.max(np.abs(w - ref) / ref) < 1e-12
    assert abs(np.log(w).mean()) < 0.05 and abs(np.log(w).std() - sigma) < 0.05
    assert np.all(w > 0) and np.all(np.isfinite(w))
