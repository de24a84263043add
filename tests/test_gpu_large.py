"""Full-size parity pinned to the reference itself.

tests/golden/psa_large.npz holds digests the UNMODIFIED reference produced
(tests/golden/make_golden.py large / sweep_top, through oracle/_ref):
  * BASELINE configs[2]'s input generate_powerlaw(1e9, 1.0, 42)
    (weight_file.hpp:42-54) and its G-shard totals (two_level.hpp:33-51);
  * the PSA tables of shards g = 0 and g = 7 of G = 8 (1.25e8 items each) at
    three job counts (alias.hpp:411-419);
  * the configs[1] n = 1e8 uniform table at three job counts, including
    wrs_b200_default_jobs(1e8);
  * configs[4]'s n = 2^28 uniform and power-law 0.5 tables.
Here the same objects are produced on the device through the C ABI and
hashed.  A 1e9-draw chi-square on one G = 8 shard closes the statistical
check the north star asks for at that size.
"""
import hashlib
import os

import numpy as np
import pytest

import paper_1903_00227_b200 as wrs
from tests.stats_util import chi2_critical

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def sha(a) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(a).view(np.uint8).reshape(-1))
    return h.hexdigest()


@pytest.fixture(scope="module")
def Z():
    return np.load(os.path.join(GOLD, "psa_large.npz"))


@pytest.fixture(scope="module")
def PL(Z):
    """configs[2]'s 1e9 power-law vector, generated on the device."""
    W = wrs.Weights.generate("powerlaw", 1.0, 10**9, 42)
    yield W
    W.free()


def test_powerlaw_1e9_input_and_shard_totals(Z, PL):
    w = PL.values()
    assert np.array_equal(w[:16], Z["pl1_1e9_s42/w_head"])
    assert sha(w) == str(Z["pl1_1e9_s42/w_sha"])
    del w
    assert PL.total() == float(Z["pl1_1e9_s42/total"])
    n = 10**9
    for G in (2, 4, 8):
        ref = Z[f"pl1_1e9_s42/G{G}/totals"]
        for g in range(G):
            lo, hi = wrs.shard_range(n, G, g)
            S = wrs.Weights.from_device_ptr(PL.device_ptr() + 8 * lo, hi - lo, copy=False)
            assert S.total() == ref[g], (G, g)
            S.free()


@pytest.mark.parametrize("g", [0, 7])
def test_powerlaw_1e9_shard_tables(Z, PL, g):
    n = 10**9
    lo, hi = wrs.shard_range(n, 8, g)
    W = wrs.Weights.from_device_ptr(PL.device_ptr() + 8 * lo, hi - lo, copy=False)
    key = f"pl1_1e9_s42/G8/g{g}"
    assert W.total() == Z["pl1_1e9_s42/G8/totals"][g]
    for P in Z[f"{key}/jobs"]:
        S = wrs.Sampler.build_psa(W, int(P))
        assert S.bucket_mean == float(Z[f"{key}/P{P}/bucket_mean"]), P
        assert sha(S.buckets()) == str(Z[f"{key}/P{P}/buckets_sha"]), (g, P)
        if int(P) == wrs.default_jobs(hi - lo):
            # the reference's own mass error at this table (verify.hpp:92-98)
            _, worst = S.implied_masses()
            assert worst == float(Z[f"{key}/P{P}/max_rel_err"])
        S.free()
    W.free()


def test_powerlaw_1e9_shard_chi_square_1e9_draws(Z, PL):
    """1e9 draws from shard g = 7 of G = 8 (its default-P table, pinned
    above): Pearson chi-square with the reference policy (stats.hpp:35-79)."""
    import torch
    n, k = 10**9, 10**9
    lo, hi = wrs.shard_range(n, 8, 7)
    W = wrs.Weights.from_device_ptr(PL.device_ptr() + 8 * lo, hi - lo, copy=False)
    S = wrs.Sampler.build(W, "psa", 1)
    out = torch.empty(k, dtype=torch.int32, device="cuda")
    S.draw_device(77, k, 1, out)
    counts = torch.bincount(out.long(), minlength=hi - lo)
    del out
    wt = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
    wt.copy_(torch.from_numpy(W.values()))
    e = wt / W.total() * k
    big = e >= 5.0
    d = counts[big].double() - e[big]
    stat = float((d * d / e[big]).sum())
    cells = int(big.sum())
    pe = float(e[~big].sum())
    if pe > 0:
        stat += (float(counts[~big].sum()) - pe) ** 2 / pe
        cells += 1
    crit = chi2_critical(cells - 1, 1e-3)
    assert stat < crit, (stat, crit, cells)


def test_uniform_1e8_tables_at_three_job_counts(Z):
    W = wrs.Weights.generate("uniform", 0.0, 10**8, 42)
    assert int(wrs.default_jobs(10**8)) in [int(p) for p in Z["uniform_1e8_s42/jobs"]]
    for P in Z["uniform_1e8_s42/jobs"]:
        S = wrs.Sampler.build_psa(W, int(P))
        assert S.bucket_mean == float(Z[f"uniform_1e8_s42/P{P}/bucket_mean"])
        assert sha(S.buckets()) == str(Z[f"uniform_1e8_s42/P{P}/buckets_sha"]), P
        if int(P) == wrs.default_jobs(10**8):
            _, worst = S.implied_masses()
            assert worst == float(Z[f"uniform_1e8_s42/P{P}/max_rel_err"])
        S.free()


@pytest.mark.parametrize("tag,dist,param", [("uniform_2p28_s42", "uniform", 0.0),
                                            ("pl05_2p28_s42", "powerlaw", 0.5)])
def test_size_sweep_top_tables(Z, tag, dist, param):
    if f"{tag}/w_sha" not in Z.files:
        pytest.skip("psa_large.npz predates the sweep_top fixtures")
    W = wrs.Weights.generate(dist, param, 2**28, 42)
    assert sha(W.values()) == str(Z[f"{tag}/w_sha"])
    P = int(Z[f"{tag}/jobs"][0])
    S = wrs.Sampler.build_psa(W, P)
    assert S.bucket_mean == float(Z[f"{tag}/P{P}/bucket_mean"])
    assert sha(S.buckets()) == str(Z[f"{tag}/P{P}/buckets_sha"])


def test_draws_beyond_one_pass_bit_exact():
    """A draw of more than 2^30 samples takes region passes of up to 2^31
    draws when memory allows (fewer sweeps of the table): windows across the
    pass boundaries are bit-exact against the oracle, for W = 1 and W = 7."""
    import torch
    import oracle
    P = oracle.port()
    n, k = 20_000_003, (1 << 30) + 123_456_789
    W = wrs.Weights.generate("uniform", 0.0, n, 5)
    S = wrs.Sampler.build(W, "psa", 1)
    b = S.buckets()
    out = torch.empty(k, dtype=torch.int32, device="cuda")
    for Wk in (1, 7):
        S.draw_device(31, k, Wk, out)
        torch.cuda.synchronize()
        for lo in (0, (1 << 30) - 50_000, k - 100_000):
            ref = P.sample_range(b, S.bucket_mean, 31, k, Wk, lo, lo + 100_000)
            assert np.array_equal(out[lo:lo + 100_000].cpu().numpy().view(np.uint32), ref), (Wk, lo)


def test_draws_in_passes_beyond_2p31_bit_exact(monkeypatch):
    """3.3e9 draws take ONE region pass (slab positions and draw indices up
    to 2^32 - 1; draw_chunk_for): equal to the same draw in 2^30-draw passes,
    and windows around 2^31 and at the end bit-exact against the oracle."""
    import torch
    import oracle
    P = oracle.port()
    n, k = 10_000_019, 3_300_000_001
    W = wrs.Weights.generate("powerlaw", 0.5, n, 3)
    S = wrs.Sampler.build(W, "psa", 1)
    b = S.buckets()
    one = torch.empty(k, dtype=torch.int32, device="cuda")
    for Wk in (1, 5):
        S.draw_device(17, k, Wk, one)
        torch.cuda.synchronize()
        for lo in (0, (1 << 31) - 50_000, k - 100_000):
            ref = P.sample_range(b, S.bucket_mean, 17, k, Wk, lo, lo + 100_000)
            assert np.array_equal(one[lo:lo + 100_000].cpu().numpy().view(np.uint32), ref), (Wk, lo)
    monkeypatch.setenv("WRS_B200_DRAW_CHUNK", str(1 << 30))
    four = torch.empty(k, dtype=torch.int32, device="cuda")
    S.draw_device(17, k, 5, four)
    torch.cuda.synchronize()
    assert torch.equal(one, four)
