"""GPU parity: the CUDA path (through the C ABI of libwrs_b200.so) against
the oracle and the reference's golden vectors.

Bar: buckets bit-exact (share, item, alias), bucket mean
bit-exact, every intermediate stage bit-exact, draws bit-exact -- all at the
same job count P, which is what the reference's table depends on.
"""
import hashlib
import os

import numpy as np
import pytest

import oracle
import paper_1903_00227_b200 as wrs
from tests.stats_util import chi_square
from tests.extreme import extreme_cases

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def P():
    return oracle.port()


def build(w, jobs=0, keep=False):
    W = wrs.Weights.from_array(w)
    return W, wrs.Sampler.build_psa(W, jobs, keep)


def assert_same_table(S, w, jobs, P):
    ob, own = P.psa_build(w, jobs)
    gb = S.buckets()
    assert S.bucket_mean == own
    if gb.tobytes() != ob.tobytes():
        bad = np.nonzero(gb.view(np.uint8).reshape(-1, 16).any(1) !=
                         ob.view(np.uint8).reshape(-1, 16).any(1))[0]
        diff = np.nonzero((gb["share"] != ob["share"]) | (gb["alias"] != ob["alias"]) |
                          (gb["item"] != ob["item"]))[0]
        raise AssertionError(f"n={w.size} P={jobs}: {diff.size} buckets differ, first "
                             f"{diff[:5]} gpu={gb[diff[:3]]} oracle={ob[diff[:3]]} {bad[:3]}")


# ---- golden vectors ------------------------------------------------------------

def test_golden_small_tables():
    z = np.load(os.path.join(GOLD, "psa_small.npz"))
    names = sorted({k.split("/")[0] for k in z.files})
    for name in names:
        w = z[f"{name}/w"]
        W = wrs.Weights.from_array(w)
        assert W.total() == z[f"{name}/total"], name
        for jobs in (1, 2, 3, 4, 8):
            S = wrs.Sampler.build_psa(W, jobs)
            assert S.bucket_mean == z[f"{name}/P{jobs}/bucket_mean"]
            assert S.buckets().tobytes() == z[f"{name}/P{jobs}/buckets"].tobytes(), (name, jobs)


def test_golden_draws_through_abi():
    d = np.load(os.path.join(GOLD, "draws_small.npz"))
    W = wrs.Weights.from_array(d["w"])
    S = wrs.Sampler.build(W, "psa-exact", 4)
    assert S.buckets().tobytes() == d["buckets"].tobytes()
    for Wk in (1, 3, 4, 8):
        assert np.array_equal(S.draw(99, 100001, Wk), d[f"seed99_W{Wk}"]), Wk
    assert np.array_equal(S.draw(100, 100001, 4), d["seed100_W4"])


def test_golden_medium_generators_and_tables():
    m = np.load(os.path.join(GOLD, "psa_medium.npz"))
    cases = {"uniform_1e6_s42": ("uniform", 0.0, 10**6, 42),
             "powerlaw1_1e6_s42": ("powerlaw", 1.0, 10**6, 42),
             "powerlaw05_2e5_s7": ("powerlaw", 0.5, 200_000, 7)}
    for tag, (dist, s, n, seed) in cases.items():
        W = wrs.Weights.generate(dist, s, n, seed)
        assert sha(W.values()) == str(m[f"{tag}/w_sha"]), tag
        assert W.total() == m[f"{tag}/total"]
        jobs_keys = sorted({int(k.split("/")[1][1:]) for k in m.files if k.startswith(tag + "/P")})
        assert wrs.default_jobs(n) in jobs_keys
        for jobs in jobs_keys:
            S = wrs.Sampler.build_psa(W, jobs)
            assert sha(S.buckets()) == str(m[f"{tag}/P{jobs}/buckets_sha"]), (tag, jobs)
        S = wrs.Sampler.build_psa(W, -(-n // 128))
        for Wk in (1, 8):
            s_ = S.draw(42, 10**6, Wk)
            assert sha(s_) == str(m[f"{tag}/draw_P{-(-n // 128)}_seed42_k1e6_W{Wk}_sha"])


# ---- per-stage parity ------------------------------------------------------------

def check_checkpoints(ck, prefix, x):
    """Checkpoint m holds the prefix chain's (hi, lo) state before element 16m
    of the list (k_scan_blocks_ckpt): continuing the chain from it with the
    same Neumaier adds (CompSumPos: all terms >= 0) must give exactly the
    oracle's prefix values prefix[16m + 1 .. 16m + 16] (parallel.hpp:122-129),
    stopping at block (2048) and list ends."""
    n = x.size
    m = ck.shape[0]
    assert m == -(-n // 16)
    hi, lo = ck[:, 0].copy(), ck[:, 1].copy()
    base = np.arange(m) * 16
    for e in range(16):
        pos = base + e
        live = (pos < n) & ((pos % 2048) >= (base % 2048))  # same block as the checkpoint
        live &= (pos // 2048) == (base // 2048)
        if not live.any():
            break
        xv = np.where(live, x[np.minimum(pos, n - 1)], 0.0)
        t = hi + xv
        big = hi >= xv
        a = np.where(big, hi, xv)
        b = np.where(big, xv, hi)
        lo = np.where(live, lo + ((a - t) + b), lo)
        hi = np.where(live, t, hi)
        val = hi + lo
        assert val[live].tobytes() == prefix[pos[live] + 1].tobytes(), e

@pytest.mark.parametrize("k2", ["split", "direct", "direct-lpw1", "direct-lpw32", "staged",
                                "staged-k1staged", "staged-k2bulk", "staged-nofuse",
                                "staged-fuse1", "staged-nokb"])
def test_stages_bit_exact(P, k2, monkeypatch):
    if k2.endswith("k1staged"):  # K1's staged form (the unstaged one is the default)
        monkeypatch.setenv("WRS_B200_K1", "staged")
        k2 = k2.split("-")[0]
    if k2.endswith("k2bulk"):  # K2a through TMA bulk copies (measured slower, opt-in)
        monkeypatch.setenv("WRS_B200_K2_BULK", "1")
        k2 = k2.split("-")[0]
    if k2.endswith("nofuse"):  # K2a, K2b and the checkpoint pass as three kernels
        monkeypatch.setenv("WRS_B200_K2_FUSE", "0")
        k2 = k2.split("-")[0]
    if k2.endswith("fuse1"):  # K2a on its own, K2b fused with the checkpoint pass
        monkeypatch.setenv("WRS_B200_K2_FUSE", "1")
        k2 = k2.split("-")[0]
    if k2.endswith("nokb"):  # the smem-staged K2a / K2c instead of the bulk-copy forms
        monkeypatch.setenv("WRS_B200_K2_KB", "0")
        k2 = k2.split("-")[0]
    # K2a/K2c have three forms (chains split over warps for a few blocks,
    # register-direct for small tables with 1..32 chains per warp, and the
    # large-table form above 2^25 items: bulk-copy rows with K2b fused into
    # the checkpoint pass); all must produce the same prefix arrays
    monkeypatch.setenv("WRS_B200_K2_SPLIT_MAX", str(2**62 if k2 == "split" else 0))
    monkeypatch.setenv("WRS_B200_K2_DIRECT_MAX", str(0 if k2 == "staged" else 2**62))
    if "lpw" in k2:
        monkeypatch.setenv("WRS_B200_K2_LPW", k2.split("lpw")[1])
    rng = np.random.default_rng(11)
    inputs = [P.generate_uniform(30011, 3), P.generate_powerlaw(20000, 1.0, 4),
              np.concatenate([np.full(5000, 1.0), rng.random(5000) + 0.5])]
    for w in inputs:
        for jobs in (1, 13, wrs.default_jobs(w.size), 977):
            W, S = build(w, jobs, keep=True)
            part = P.partition(w)
            nl, nh = S.stage("counts")
            assert (nl, nh) == (part["light"].size, part["heavy"].size)
            assert np.array_equal(S.stage("heavy"), part["heavy"])
            assert np.array_equal(S.stage("light_w"), w[part["light"]])
            assert np.array_equal(S.stage("heavy_w"), w[part["heavy"]])
            tot = np.concatenate([P.scan_block_totals(w[part["light"]]),
                                  P.scan_block_totals(w[part["heavy"]])])
            assert S.stage("block_totals").tobytes() == tot.tobytes()
            nbl = (part["light"].size + 2047) // 2048
            car = np.concatenate([P.scan_carries(tot[:nbl]), P.scan_carries(tot[nbl:])])
            assert S.stage("carries").tobytes() == car.tobytes()
            if k2 == "staged":  # checkpointed prefixes (large-table form)
                for name, pre, x in (("light_ckpt", part["light_prefix"], w[part["light"]]),
                                     ("heavy_ckpt", part["heavy_prefix"], w[part["heavy"]])):
                    check_checkpoints(S.stage(name).reshape(-1, 2), pre, x)
            else:
                assert S.stage("light_prefix").tobytes() == part["light_prefix"].tobytes()
                assert S.stage("heavy_prefix").tobytes() == part["heavy_prefix"].tobytes()
            if nh:
                bounds, spill = P.psa_plan(w, jobs)
                sl, sh, ss = S.stage("split_light"), S.stage("split_heavy"), S.stage("split_spill")
                assert np.array_equal(sl[1:], bounds[:, 1].astype(np.uint32))
                assert np.array_equal(sh[1:], bounds[:, 3].astype(np.uint32))
                assert ss[:-1].tobytes() == spill.tobytes()
                # K4a's list-order outputs = the oracle table read through the lists
                ob, _ = P.psa_build(w, jobs)
                # (the heavy rank each light was paired with; alias = heavy[min(rank, nh-1)])
                rk = S.stage("light_rank").astype(np.int64)
                assert np.array_equal(part["heavy"][np.minimum(rk, int(nh) - 1)],
                                      ob["alias"][part["light"]])
                assert np.all(np.diff(rk) >= 0)  # nondecreasing: K4b stages one id run per tile
                assert S.stage("heavy_share").tobytes() == ob["share"][part["heavy"]].tobytes()
            assert_same_table(S, w, jobs, P)


# ---- randomized table parity -------------------------------------------------------

def weight_cases(P):
    rng = np.random.default_rng(2024)
    yield "one", np.array([7.0])
    yield "two_tiny", np.array([1.0, 1e-12])
    yield "equal", np.full(1000, 0.25)
    yield "huge_heavy", np.concatenate([[1e6], np.ones(9999)])
    for n in (2, 3, 31, 32, 33, 100, 2047, 2048, 2049, 4095, 4096, 4097, 8193, 65537, 250_000):
        yield f"u{n}", P.generate_uniform(n, n + 1)
        yield f"pl1_{n}", P.generate_powerlaw(n, 1.0, n + 2)
    for n in (1000, 100_000):
        yield f"pl2_{n}", P.generate_powerlaw(n, 2.0, 5)
        yield f"pl05_{n}", P.generate_powerlaw(n, 0.5, 6)
        yield f"logn_{n}", np.exp(rng.normal(0.0, 2.0, n))
        t = np.ones(n)
        t[:: 50] = 9.0
        yield f"ties_{n}", t
        x = rng.random(n) + 0.5
        x[rng.random(n) < 0.5] = 1.0
        yield f"mixties_{n}", x
        yield f"skew_{n}", 10.0 ** rng.uniform(-12, 12, n)
        # sorted: whole 4096-item tiles of heavies (K4b's unstaged path) then of lights
        yield f"sorted_{n}", np.sort(rng.random(n) + 0.01)[::-1].copy()
    for i, w in enumerate(extreme_cases()):
        yield f"extreme{i}", w


def test_random_tables_bit_exact(P):
    for name, w in weight_cases(P):
        W = wrs.Weights.from_array(w)
        n = w.size
        for jobs in sorted({1, 3, wrs.default_jobs(n), max(1, n // 7), n, 2 * n + 1}):
            if jobs > 4 * 10**6:
                continue
            S = wrs.Sampler.build_psa(W, jobs)
            assert S.jobs == jobs
            assert_same_table(S, w, jobs, P)


def test_default_psa_is_reference_at_default_jobs(P):
    w = P.generate_uniform(300_000, 9)
    W = wrs.Weights.from_array(w)
    S = wrs.Sampler.build(W, "psa", 8)
    assert S.jobs == wrs.default_jobs(w.size)
    assert_same_table(S, w, S.jobs, P)
    S2 = wrs.Sampler.build(W, "psa-exact", 8)
    assert S2.jobs == 8
    assert_same_table(S2, w, 8, P)


# ---- draws ------------------------------------------------------------------------

def test_draws_bit_exact_random(P):
    import torch
    for n, k, Wk in ((1, 1000, 1), (17, 12345, 3), (1000, 10**6, 8), (100_000, 3 * 10**6 + 7, 13),
                     (4097, 5, 16), (1000, 7, 1000), (1000, 100_003, 65_536), (2, 10, 3)):
        w = P.generate_powerlaw(n, 1.0, 3) if n > 1 else np.array([2.0])
        W, S = build(w)
        b = S.buckets()
        ref = P.sample_many(b, S.bucket_mean, 77, k, Wk)
        assert np.array_equal(S.draw(77, k, Wk), ref), (n, k, Wk)
        out = torch.empty(k, dtype=torch.int32, device="cuda")
        S.draw_device(77, k, Wk, out)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint32), ref)


def test_draws_bit_exact_extreme_magnitudes(P):
    # totals >= 1e300 (guarded compensated add), infinite total (coin = u * inf),
    # subnormal weights; same cases the reference pins in test_ref_pins.py
    for w in extreme_cases():
        W, S = build(w, 3)
        assert_same_table(S, w, 3, P)
        for Wk in (1, 5):
            ref = P.sample_many(S.buckets(), S.bucket_mean, 9, 40001, Wk)
            assert np.array_equal(S.draw(9, 40001, Wk), ref), (w.size, Wk)


def test_draw_zero_and_workers_zero(P):
    W, S = build(P.generate_uniform(100, 1))
    assert S.draw(5, 0, 1).size == 0
    assert np.array_equal(S.draw(5, 1000, 0), S.draw(5, 1000, 1))  # capi.cpp:213


# ---- reference test_capi.cpp behaviour ----------------------------------------------

def test_capi_lifecycle_like_reference(tmp_path):  # test_capi.cpp:12-74
    w = np.array([3.0, 1, 1, 1])
    W = wrs.Weights.from_array(w)
    assert W.count() == 4 and np.array_equal(W.values(), w)
    with pytest.raises(wrs.WrsError) as e:
        wrs.Weights.from_array(np.array([1.0, -1.0]))
    assert e.value.status == 1 and "item 1" in e.value.message
    gen = wrs.Weights.generate("powerlaw", 1.5, 500, 42)
    path = str(tmp_path / "rt.wrs")
    gen.write(path)
    back = wrs.Weights.read(path)
    assert np.array_equal(back.values(), gen.values())
    with pytest.raises(wrs.WrsError) as e:
        wrs.Weights.read(str(tmp_path / "missing.wrs"))
    assert e.value.status == 2
    (tmp_path / "garbage.bin").write_bytes(b"not a weight file at all")
    with pytest.raises(wrs.WrsError) as e:
        wrs.Weights.read(str(tmp_path / "garbage.bin"))
    assert e.value.status == 3
    with pytest.raises(wrs.WrsError):
        wrs.Weights.generate("cauchy", 0, 10, 1)

    pl = wrs.Weights.generate("powerlaw", 2.0, 1000, 7)
    S = wrs.Sampler.build(pl, "psa", 4)
    assert S.verify_masses(1e-9) == 0
    out = S.draw(123, 10000, 2)
    assert out.max() < 1000
    assert np.array_equal(out, S.draw(123, 10000, 2))
    with pytest.raises(wrs.WrsError):
        wrs.Sampler.build(pl, "bogus", 1)


def test_bad_weight_file_payload(tmp_path):
    path = tmp_path / "bad.wrs"
    vals = np.array([1.0, 2.0, np.nan, 4.0])
    path.write_bytes(b"WRS1" + np.uint64(4).tobytes() + vals.tobytes())
    with pytest.raises(wrs.WrsError) as e:
        wrs.Weights.read(str(path))
    assert e.value.status == 3 and "weight 2" in e.value.message


# ---- full size (BASELINE config 2: n=1e8 uniform, k=1e9) ------------------------------

def test_full_size_table_and_draws(P):
    import torch
    n, k = 10**8, 10**9
    m = np.load(os.path.join(GOLD, "psa_medium.npz"))
    W = wrs.Weights.generate("uniform", 0.0, n, 42)
    w = W.values()
    assert sha(w) == str(m["uniform_1e8_s42/w_sha"])
    S = wrs.Sampler.build(W, "psa", 1)
    jobs = S.jobs
    # bytewise parity with the oracle at the same job count, full size
    ob, own = P.psa_build(w, jobs)
    gb = S.buckets()
    assert own == S.bucket_mean
    assert gb.tobytes() == ob.tobytes()
    # the reference's own verification oracle (verify.hpp:43-98)
    err = P.max_relative_mass_error(P.implied_masses(gb, own), w)
    assert err < 1e-7
    assert S.verify_masses(1e-7) == 0
    # 1e9 draws: bitwise on sampled windows, chi-square on everything
    out = torch.empty(k, dtype=torch.int32, device="cuda")
    for Wk in (1, 148):
        S.draw_device(2024, k, Wk, out)
        torch.cuda.synchronize()
        for lo in (0, 123_456_789, 499_999_000, k - 100_000):
            ref = P.sample_range(gb, own, 2024, k, Wk, lo, lo + 100_000)
            assert np.array_equal(out[lo:lo + 100_000].cpu().numpy().view(np.uint32), ref), (Wk, lo)
    counts = torch.bincount(out.long(), minlength=n)
    del out
    wt = torch.from_numpy(w).cuda()
    e = wt / wt.sum() * k
    big = e >= 5.0
    d = counts[big].double() - e[big]
    stat = float((d * d / e[big]).sum())
    cells = int(big.sum())
    pe = float(e[~big].sum())
    if pe > 0:
        stat += (float(counts[~big].sum()) - pe) ** 2 / pe
        cells += 1
    from tests.stats_util import chi2_critical
    crit = chi2_critical(cells - 1, 1e-3)
    assert stat < crit, (stat, crit)


# ---- region-ordered draw plan (table beyond L2) ---------------------------------------

@pytest.mark.parametrize("chunk,shift,rd,rows", [
    (None, None, "1", "32"), (3_000_001, None, "1", "32"), (None, 22, "1", "32"),
    (None, 19, "1", "32"), (None, None, "0", "32"), (None, 19, "0", "32"),
    (None, None, "1", "16"), (3_000_001, 19, "1", "64")])
def test_region_plan_draws_bit_exact(P, chunk, shift, rd, rows, monkeypatch):
    """rd: the unpermute's run staging -- bulk copies ("1", default) or the
    warp-wide LDGSTS form ("0"); rows: draws per scatter thread (32 default;
    16 / 64 the other scatter forms of the same tile)."""
    import torch
    monkeypatch.setenv("WRS_B200_RD_BULK", rd)
    monkeypatch.setenv("WRS_B200_SCATTER_ROWS", rows)
    if chunk:
        monkeypatch.setenv("WRS_B200_DRAW_CHUNK", str(chunk))
    if shift:  # 64-MB regions (the default above 2^27 buckets) / many small regions
        monkeypatch.setenv("WRS_B200_REGION_SHIFT", str(shift))
    n = 9_500_003  # 152 MB table: region plan
    w = P.generate_powerlaw(n, 0.5, 11)
    W, S = build(w)
    b = S.buckets()
    for k, Wk in ((6_000_011, 1), (7_000_000, 3), (6_500_001, 148)):
        ref = P.sample_many(b, S.bucket_mean, 99, k, Wk)
        out = torch.empty(k, dtype=torch.int32, device="cuda")
        S.draw_device(99, k, Wk, out)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint32), ref), (k, Wk)
    # host output path (chunked D2H) through the reference ABI call
    assert np.array_equal(S.draw(5, 6_000_011, 2), P.sample_many(b, S.bucket_mean, 5, 6_000_011, 2))


@pytest.mark.parametrize("side", ["0", "1"])
def test_double_buffered_rebuild_then_draw_on_other_stream(P, side, monkeypatch):
    """wrs_b200_sampler_double_buffer: the first rebuild writes the second
    (uninitialised) table on its own stream while a draw issued right after it
    on another stream must wait for it; then pipelined rebuild/draw rounds.
    side = "1": each draw's first scatter runs on the side stream, under the
    rebuild (WRS_B200_SIDE_SCATTER)."""
    import torch
    monkeypatch.setenv("WRS_B200_SIDE_SCATTER", side)
    n, k = 3_000_017, 4_000_003
    w = P.generate_uniform(n, 17)
    W, S = build(w)
    ref = P.sample_many(S.buckets(), S.bucket_mean, 5, k, 1)
    S.double_buffer()
    a, b = torch.cuda.Stream(), torch.cuda.Stream()
    out = torch.empty(k, dtype=torch.int32, device="cuda")
    for i in range(3):
        S.rebuild_async(a)
        S.draw_device(5, k, 1, out, b)
        b.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint32), ref), i
    S.check()
    assert_same_table(S, w, S.jobs, P)


def test_weight_validation_like_reference():  # test_weights.cpp:14-21, weights.hpp:32-41
    for bad, item in ((np.array([], np.float64), None), (np.array([1.0, 0.0]), 1),
                      (np.array([1.0, -2.0]), 1), (np.array([1.0, np.nan]), 1),
                      (np.array([np.inf]), 0), (np.array([2.0, 3.0, -np.inf, 1.0]), 2)):
        with pytest.raises(wrs.WrsError) as e:
            wrs.Weights.from_array(bad)
        assert e.value.status == 1, bad
        if item is None:
            assert "need at least one item" in e.value.message
        else:
            assert f"item {item} is not finite and positive" in e.value.message
    W = wrs.Weights.from_array(np.array([4.0, 1.0, 2.0, 8.0]))  # test_weights.cpp:23-31
    assert W.total() == 15.0 and W.count() == 4


def test_samples_follow_the_weights(P):  # test_alias.cpp:254-286
    from tests.stats_util import chi_square
    W = wrs.Weights.from_array(np.array([3.0, 1, 1, 1]))
    S = wrs.Sampler.build(W, "psa-exact", 2)
    counts = np.bincount(S.draw(0xC0FFEE, 400_000, 1), minlength=4)
    assert chi_square(counts, [0.5, 1 / 6, 1 / 6, 1 / 6])[3]
    w = P.generate_powerlaw(50, 1.0, 3)
    S = wrs.Sampler.build(wrs.Weights.from_array(w), "psa-exact", 4)
    a, b = S.draw(99, 100_001, 4), S.draw(99, 100_001, 4)
    assert np.array_equal(a, b) and not np.array_equal(a, S.draw(100, 100_001, 4))
    assert chi_square(np.bincount(a, minlength=50), w / w.sum())[3]


def test_implied_masses_on_device_bit_exact(P):  # verify.hpp:43-54, 92-98
    rng = np.random.default_rng(12)
    cases = [np.array([3.0, 1, 1, 1]), np.full(64, 0.5), np.array([1.0, 1e-12]), np.array([7.0])]
    w = np.ones(100)
    w[0] = 100.0
    cases.append(w)  # one heavy aliased by every other bucket (test_alias.cpp:173-193)
    cases += [P.generate_powerlaw(100_003, 1.0, 2), rng.random(250_000) + 1e-9,
              np.exp(3.0 * rng.standard_normal(77_777))]
    for w in cases:
        for jobs in (0, 1, 7):
            W, S = build(w, jobs)
            m, worst = S.implied_masses()
            ref = P.implied_masses(S.buckets(), S.bucket_mean)
            assert m.tobytes() == ref.tobytes(), (w.size, jobs)
            assert worst == P.max_relative_mass_error(ref, w), (w.size, jobs)


def test_powerlaw_device_deal_matches_reference_generator(P):  # weight_file.hpp:42-54
    for n, s_, seed in ((1, 1.0, 3), (2, 1.0, 3), (3, 0.5, 9), (1000, 1.0, 1), (65537, 2.0, 5),
                        (1_000_003, 0.5, 42), (4_000_000, 1.0, 7)):
        W = wrs.Weights.generate("powerlaw", s_, n, seed)
        assert np.array_equal(W.values(), P.generate_powerlaw(n, s_, seed)), (n, s_, seed)
    # shard slices of the global deal
    n = 300_007
    full = P.generate_powerlaw(n, 1.0, 11)
    for lo, hi in ((0, 1000), (150_000, 300_007), (1, 2)):
        Wr = wrs.Weights.generate_range("powerlaw", 1.0, n, lo, hi, 11)
        assert np.array_equal(Wr.values(), full[lo:hi])


def test_philox_mode_replays_on_the_table(P):  # north star: Philox uniforms, replayed
    import torch
    for n, k, seed in ((1, 1000, 3), (1000, 200_001, 9), (100_003, 3_000_001, 2**40 + 7),
                       (9_500_003, 6_000_011, 11)):  # the last one takes the region plan
        w = P.generate_powerlaw(n, 0.5, 11) if n > 1 else np.array([2.0])
        W, S = build(w)
        b = S.buckets()
        out = torch.empty(k, dtype=torch.int32, device="cuda")
        S.draw_philox_device(seed, k, out)
        torch.cuda.synchronize()
        got = out.cpu().numpy().view(np.uint32)
        for lo, hi in ((0, min(k, 100_000)), (max(0, k - 50_000), k)):
            assert np.array_equal(got[lo:hi], P.sample_philox_range(b, S.bucket_mean, seed, lo, hi)), (n, lo)


@pytest.mark.parametrize("tt", [512, 1024])
def test_region_plan_larger_tiles_bit_exact(P, tt, monkeypatch):
    """Tables with many regions use 8192- / 16384-draw tiles (forced here on a
    4-region table, with a chunk that splits the draws, so the bigger tiles'
    scatter, run table and unpermute are checked end to end)."""
    import torch
    monkeypatch.setenv("WRS_B200_TILE_THREADS", str(tt))
    n = 9_500_003
    w = P.generate_powerlaw(n, 0.5, 13)
    W, S = build(w)
    b = S.buckets()
    for k, Wk, chunk in ((6_000_011, 1, None), (7_000_000, 3, 2_500_001)):
        if chunk:
            monkeypatch.setenv("WRS_B200_DRAW_CHUNK", str(chunk))
        out = torch.empty(k, dtype=torch.int32, device="cuda")
        S.draw_device(31, k, Wk, out)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint32),
                              P.sample_many(b, S.bucket_mean, 31, k, Wk)), (tt, k, Wk)
        items, counts = S.draw_counts(31, k, Wk)
        ri, rc = np.unique(P.sample_many(b, S.bucket_mean, 31, k, Wk), return_counts=True)
        assert np.array_equal(items, ri) and np.array_equal(counts, rc)


@pytest.mark.parametrize("ov_cap", [2_000_000, 4096])
def test_region_plan_slab_redirect_and_overflow(P, ov_cap, monkeypatch):
    """Slabs shrunk below the draws they receive (WRS_B200_TEST_SLAB_CAP):
    runs that do not fit go to the overflow slab (ov_cap large: the gather
    must stop at the first run that did not fit, never reading the unwritten
    tail of the slab) or overflow it too (ov_cap tiny: the unpermute recomputes
    the chunk directly).  Draws and counts stay bit-exact either way."""
    import torch
    monkeypatch.setenv("WRS_B200_PLAN", "r")
    monkeypatch.setenv("WRS_B200_REGION_SHIFT", "16")   # 16 regions of 2^16 buckets
    monkeypatch.setenv("WRS_B200_TEST_SLAB_CAP", "100000")
    monkeypatch.setenv("WRS_B200_TEST_OV_CAP", str(ov_cap))
    n, k = 1_000_003, 2_000_011  # ~125k draws per region: a fifth of every slab redirected
    w = P.generate_powerlaw(n, 0.5, 3)
    W, S = build(w)
    b = S.buckets()
    for Wk in (1, 5):
        ref = P.sample_many(b, S.bucket_mean, 31, k, Wk)
        out = torch.empty(k, dtype=torch.int32, device="cuda")
        S.draw_device(31, k, Wk, out)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint32), ref), Wk
        items, counts = S.draw_counts(31, k, Wk)
        ri, rc = np.unique(ref, return_counts=True)
        assert np.array_equal(items, ri) and np.array_equal(counts, rc), Wk


def test_lognormal_device_generator_matches_oracle(P):
    """configs[3]'s weights: wrs_weights_generate("lognormal", sigma, ...) on
    the device equals the oracle's restatement byte for byte (whole vector and
    a shard's slice), so the CPU reference can be fed the same input."""
    n = 1_000_003
    ref = P.generate_lognormal(n, 2.0, 42)
    W = wrs.Weights.generate("lognormal", 2.0, n, 42)
    assert W.values().tobytes() == ref.tobytes()
    S = wrs.Weights.generate_range("lognormal", 2.0, n, 123_457, 654_321, 42)
    assert S.values().tobytes() == ref[123_457:654_321].tobytes()


def test_c_client_through_the_reference_abi(tmp_path):
    """tests/capi_client.c: a plain C program against include/wrs.h, linked
    to libwrs_b200.so (the reference client flow, test_capi.cpp:12-112)."""
    import subprocess
    from tests.test_capi_host import build_capi_client
    exe = build_capi_client(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, cwd=str(tmp_path))
    assert r.returncode == 0, r.stderr
    assert "capi client ok" in r.stdout


def test_masses_agree_with_reference_vose_and_sweep(P):
    """the reference's other builders as extra oracles.  The
    GPU PSA table, the reference's Build::vose and Build::sweep tables
    (alias.hpp:299-409, run through oracle/_ref) are different tables whose
    implied masses (verify.hpp:43-54) must all reproduce w_i within the
    reference's own tolerance, and agree with each other."""
    R = oracle.ref()
    if R is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(3)
    cases = [P.generate_uniform(200_003, 1), P.generate_powerlaw(100_000, 1.0, 2),
             np.exp(rng.normal(0.0, 2.0, 50_000)), np.concatenate([[1e6], np.ones(9999)])]
    for w in cases:
        W = wrs.Weights.from_array(w)
        S = wrs.Sampler.build(W, "psa", 1)
        gm, worst = S.implied_masses()
        assert worst < 1e-9
        for method in ("vose", "sweep"):
            b, wn = R.build_method(w, method)
            rm = R.implied_masses(b, wn)
            assert np.max(np.abs(rm - w) / w) < 1e-9, method
            assert np.max(np.abs(rm - gm) / w) < 2e-9, method


def test_psa_exact_env_gives_the_reference_table(P, monkeypatch):
    """WRS_B200_PSA_EXACT=1: an unmodified client's wrs_sampler_build(w, "psa",
    workers) gets the reference's AliasTable(wt, psa, workers) and stream."""
    monkeypatch.setenv("WRS_B200_PSA_EXACT", "1")
    w = P.generate_powerlaw(50_000, 1.0, 3)
    W = wrs.Weights.from_array(w)
    S = wrs.Sampler.build(W, "psa", 8)
    assert S.jobs == 8
    assert_same_table(S, w, 8, P)


def test_host_output_draws_span_several_copy_chunks(P):
    """wrs_sampler_draw into host memory copies out in 2^26-draw chunks while
    the next chunk draws: more than one chunk, a ragged last one, both plans
    (region plan on a 150-MB table) equal the device draw, itself pinned to
    the oracle by the tests above."""
    import torch
    k = (1 << 26) * 2 + 12_345
    for n in (1_000_003, 9_500_003):
        w = P.generate_uniform(n, 23)
        W, S = build(w)
        host = S.draw(31, k, 3)
        dev = torch.empty(k, dtype=torch.int32, device="cuda")
        S.draw_device(31, k, 3, dev)
        torch.cuda.synchronize()
        assert np.array_equal(host, dev.cpu().numpy().view(np.uint32)), n
        ref = P.sample_many(S.buckets(), S.bucket_mean, 31, 1_000_000, 3)
        assert np.array_equal(S.draw(31, 1_000_000, 3), ref)


@pytest.mark.parametrize("n", [12_000_000, 16_777_216, 50_000_000])
def test_wave_fit_default_jobs_tables_bit_exact(P, n):
    """Default job counts folded into whole K4a waves (non-power-of-two jobs
    of 212 / 296 / 880 items at these n) give the oracle's table at that P,
    for uniform and power-law weights; every one of the three draws checked
    on a window."""
    import torch
    P_ = wrs.default_jobs(n)
    assert P_ < 56832 and -(-n // P_) not in (128, 256, 512)  # one wave of stretched jobs
    for w in (P.generate_uniform(n, 3), P.generate_powerlaw(n, 0.5, 4)):
        W, S = build(w)
        assert S.jobs == P_
        assert_same_table(S, w, P_, P)
        k = 3_000_000
        out = torch.empty(k, dtype=torch.int32, device="cuda")
        S.draw_device(11, k, 1, out)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint32),
                              P.sample_many(S.buckets(), S.bucket_mean, 11, k, 1))
        S.free()
        W.free()


def test_concurrent_host_threads_build_draw_free(P):
    """Host threads each running upload -> build -> draw into host memory ->
    free through the ABI at once (the e2e bench's two lanes): a free waits
    for its own sampler's streams only (SyncedFrees, alloc.cpp), so a block
    another thread gets back from the cache must hold no in-flight work.
    Every draw equals the same job run alone."""
    import threading
    k = (1 << 26) + 4_321  # two copy chunks
    cases = [(P.generate_uniform(2_000_003 + 7 * j, 40 + j), 50 + j) for j in range(3)]
    want = []
    for w, seed in cases:
        W, S = build(w)
        want.append(S.draw(seed, k, 2))
        S.free()
        W.free()
    bad = []

    def lane(j):
        w, seed = cases[j]
        for _ in range(4):
            W, S = build(w)
            got = S.draw(seed, k, 2)
            S.free()
            W.free()
            if not np.array_equal(got, want[j]):
                bad.append(j)

    ths = [threading.Thread(target=lane, args=(j,)) for j in range(3)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not bad


def test_free_after_draw_on_caller_stream_waits_for_it(P):
    """A sampler whose draw ran on the caller's stream is freed without
    synchronising that stream: the free must still wait for the draw
    (ext_stream -> device-wide wait) before its table goes back to the cache
    and the next sampler of the same size overwrites it."""
    import torch
    n, k = 3_000_017, 1 << 27
    w1, w2 = P.generate_uniform(n, 61), P.generate_powerlaw(n, 1.0, 62)
    W, S = build(w1)
    want = S.draw(63, 1 << 20, 1)
    out = torch.empty(k, dtype=torch.int32, device="cuda")
    st = torch.cuda.Stream()
    S.draw_device(63, k, 1, out, stream=st.cuda_stream)
    S.free()
    W.free()
    W2, S2 = build(w2)  # same sizes: reuses the freed blocks
    torch.cuda.synchronize()
    assert np.array_equal(out[: 1 << 20].cpu().numpy().view(np.uint32), want)
    S2.free()
    W2.free()
