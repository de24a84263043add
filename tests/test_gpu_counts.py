"""GPU parity of the aggregated draws:
wrs_sample_with_replacement / wrs_b200_sampler_draw_counts return the
distinct items of sample_many(seed, k, workers) with their multiplicities,
items ascending -- exactly the histogram of the reference's own draws on the
same table (the oracle), on both the direct (L2-resident table) and the
region (HBM-resident table) plans, across chunked folds.

The reference's wrs_sample_with_replacement answers with its grouped sampler
(grouped.hpp:138-223), a different random stream: against it the parity is
distributional (the chi-square at full size below).
"""
import numpy as np
import pytest

import oracle
import paper_1903_00227_b200 as wrs
from tests.stats_util import chi2_critical

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    return oracle.port()


def histogram(draws):
    items, counts = np.unique(draws, return_counts=True)
    return items.astype(np.uint32), counts.astype(np.uint64)


def test_counts_match_oracle_draw_histogram(P):
    cases = [(1, 1000, 1, "one"), (2, 7, 1, "u"), (1000, 10**5, 1, "pl"),
             (65537, 300_001, 3, "pl"), (4097, 5, 16, "u"), (50_000, 2_000_000, 148, "ln")]
    rng = np.random.default_rng(5)
    for n, k, Wk, dist in cases:
        if dist == "one":
            w = np.array([3.0])
        elif dist == "u":
            w = P.generate_uniform(n, 9)
        elif dist == "pl":
            w = P.generate_powerlaw(n, 1.0, 4)
        else:
            w = np.exp(2.0 * rng.standard_normal(n))
        W = wrs.Weights.from_array(w)
        S = wrs.Sampler.build(W, "psa", 1)
        b = S.buckets()
        ref_items, ref_counts = histogram(P.sample_many(b, S.bucket_mean, 31, k, Wk))
        items, counts = S.draw_counts(31, k, Wk)
        assert np.array_equal(items, ref_items), (n, k, Wk)
        assert np.array_equal(counts, ref_counts), (n, k, Wk)
        assert int(counts.sum()) == k


def test_counts_zero_draws_and_module_entry(P):
    w = P.generate_uniform(1000, 2)
    W = wrs.Weights.from_array(w)
    S = wrs.Sampler.build(W, "psa", 1)
    items, counts = S.draw_counts(1, 0, 1)
    assert items.size == 0 and counts.size == 0
    # wrs_sample_with_replacement builds "psa" itself: the sampler's W=1 pairs
    i2, c2 = wrs.sample_with_replacement(W, 12345, 77, 4)
    i1, c1 = S.draw_counts(77, 12345, 1)
    assert np.array_equal(i1, i2) and np.array_equal(c1, c2)
    assert np.all(np.diff(i2.astype(np.int64)) > 0)


def test_sample_with_replacement_like_reference_capi():  # test_capi.cpp:80-112
    W = wrs.Weights.generate("powerlaw", 1.5, 200, 11)
    n, k = 200, 5000
    items, counts = wrs.sample_with_replacement(W, k, 9, 2)
    assert items.size <= n and np.all(items < n)
    assert np.unique(items).size == items.size
    assert int(counts.sum()) == k
    items2, counts2 = wrs.sample_with_replacement(W, k, 9, 7)  # workers do not matter
    assert np.array_equal(items2, items) and np.array_equal(counts2, counts)
    L = wrs.lib()
    import ctypes as C
    m = C.c_uint64()
    buf_i = np.empty(n, np.uint32)
    buf_c = np.empty(n, np.uint64)
    assert L.wrs_sample_with_replacement(None, k, 9, 1, buf_i.ctypes.data, buf_c.ctypes.data,
                                         C.byref(m)) == 1  # WRS_EINVAL


@pytest.mark.parametrize("chunk,shift", [(None, None), (3_000_001, None), (None, 22)])
def test_counts_region_plan_match_device_draws(P, chunk, shift, monkeypatch):
    """HBM-resident table (region plan); the device draws themselves are pinned
    bit-exact to the oracle in test_gpu_parity."""
    import torch
    if chunk:
        monkeypatch.setenv("WRS_B200_DRAW_CHUNK", str(chunk))
    if shift:  # 64-MB regions, the default above 2^27 buckets
        monkeypatch.setenv("WRS_B200_REGION_SHIFT", str(shift))
    n = 9_500_003
    w = P.generate_powerlaw(n, 0.5, 11)
    W = wrs.Weights.from_array(w)
    S = wrs.Sampler.build(W, "psa", 1)
    for k, Wk in ((6_000_011, 1), (7_000_000, 3)):
        out = torch.empty(k, dtype=torch.int32, device="cuda")
        S.draw_device(99, k, Wk, out)
        hist = torch.bincount(out.long(), minlength=n)
        nz = torch.nonzero(hist).flatten()
        d_items = torch.empty(min(k, n), dtype=torch.int32, device="cuda")
        d_counts = torch.empty(min(k, n), dtype=torch.int64, device="cuda")
        d_m = torch.zeros(1, dtype=torch.int64, device="cuda")
        S.draw_counts_device(99, k, Wk, d_items, d_counts, d_m)
        torch.cuda.synchronize()
        m = int(d_m.item())
        assert m == nz.numel(), (k, Wk)
        assert torch.equal(d_items[:m].long(), nz)
        assert torch.equal(d_counts[:m], hist[nz])
    # the host-output entry point agrees
    items, counts = S.draw_counts(5, 6_000_011, 2)
    ref = P.sample_many(S.buckets(), S.bucket_mean, 5, 6_000_011, 2)
    ri, rc = histogram(ref)
    assert np.array_equal(items, ri) and np.array_equal(counts, rc)


def test_counts_full_size_lognormal_chi_square():
    """Config 4 shape: n=1e8 lognormal(0, 2) weights, k=1e9 draws aggregated;
    counts sum to k, equal the histogram of the plain draws, and pass the
    reference's chi-square policy against w_i / W."""
    import torch
    n, k = 10**8, 10**9
    W = wrs.Weights.generate("lognormal", 2.0, n, 42)  # configs[3]'s generator
    wt = torch.from_numpy(W.values()).cuda()
    S = wrs.Sampler.build(W, "psa", 1)
    d_items = torch.empty(n, dtype=torch.int32, device="cuda")
    d_counts = torch.empty(n, dtype=torch.int64, device="cuda")
    d_m = torch.zeros(1, dtype=torch.int64, device="cuda")
    S.draw_counts_device(2024, k, 1, d_items, d_counts, d_m)
    torch.cuda.synchronize()
    m = int(d_m.item())
    items, counts = d_items[:m].long(), d_counts[:m]
    assert int(counts.sum()) == k
    assert bool((items[1:] > items[:-1]).all())
    out = torch.empty(k, dtype=torch.int32, device="cuda")
    S.draw_device(2024, k, 1, out)
    hist = torch.bincount(out.long(), minlength=n)
    del out
    assert torch.equal(hist[items], counts) and int((hist > 0).sum()) == m
    # chi-square with the reference policy (stats.hpp:35-79), on the device
    e = wt / wt.sum() * k
    big = e >= 5.0
    d = hist[big].double() - e[big]
    stat = float((d * d / e[big]).sum())
    cells = int(big.sum())
    pe = float(e[~big].sum())
    if pe > 0:
        stat += (float(hist[~big].sum()) - pe) ** 2 / pe
        cells += 1
    crit = chi2_critical(cells - 1, 1e-3)
    assert stat < crit, (stat, crit)
