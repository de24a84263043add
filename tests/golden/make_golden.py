"""Generate tests/golden/*.npz from the UNMODIFIED reference.

Run in the build container (needs /root/reference, compiled by oracle/Makefile
into oracle/_ref/libwrs_ref.so):

    make -C oracle && PYTHONPATH=. python tests/golden/make_golden.py

Every fixture below is produced by the reference's own code paths through
ref_shim.cpp: WeightTable / pairwise_sum (weights.hpp:19-46),
generate_uniform / generate_powerlaw (weight_file.hpp:32-54),
AliasTable(wt, Build::psa, P) (alias.hpp:246-257, 411-419) and its detail::
pieces, AliasTable::sample_many (alias.hpp:274-284), implied_masses
(verify.hpp:43-54), prefix_sums (parallel.hpp:104-130) and RngStream
(rng.hpp:32-82).  The hand-written weight vectors are the reference tests'
own fixtures (cited per entry).  Large outputs are stored as SHA-256 digests
of their little-endian bytes.
"""
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
import oracle  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    R = oracle.ref()
    if R is None:
        raise SystemExit("oracle/_ref/libwrs_ref.so missing: run make -C oracle first")

    # --- hand fixtures (tests/test_alias.cpp) -----------------------------
    hand = {
        "three_one": ([3, 1, 1, 1], "test_alias.cpp:56-71"),
        "two_heavies": ([4, 4, 1, 1, 1, 1], "test_alias.cpp:73-75"),
        "single": ([7.0], "test_alias.cpp:77-86"),
        "tiny_mass": ([1.0, 1e-12], "test_alias.cpp:88-98"),
        "uniform16": ([0.25] * 16, "test_alias.cpp:100-108"),
        "fig1_13": ([5.0, 0.5, 1.2, 3.0, 0.3, 0.9, 2.2, 0.4, 1.1, 0.6, 4.0, 0.8, 0.7],
                    "test_alias.cpp:135-171"),
        "huge_heavy": ([100.0] + [1.0] * 99, "test_alias.cpp:173-193"),
        "ties401": ([9.0 if i % 50 == 0 else 1.0 for i in range(401)], "test_alias.cpp:117-121"),
        "sum15": ([4.0, 1.0, 2.0, 8.0], "test_weights.cpp:23-31"),
    }
    tables = {}
    for name, (w, cite) in hand.items():
        w = np.array(w, np.float64)
        tables[name] = (w, cite)
    # random mixes (test_alias.cpp:110-122 sizes, generator seeds fixed here)
    for n in (2, 3, 5, 17, 64, 1000):
        tables[f"uniform_{n}"] = (R.generate_uniform(n, 1000 + n), "test_alias.cpp:112-113")
        tables[f"pl05_{n}"] = (R.generate_powerlaw(n, 0.5, 2000 + n), "test_alias.cpp:114")
        tables[f"pl2_{n}"] = (R.generate_powerlaw(n, 2.0, 3000 + n), "test_alias.cpp:115")
    tables["pl1_333"] = (R.generate_powerlaw(333, 1.0, 5), "test_alias.cpp:124-133")

    out = {}
    for name, (w, cite) in tables.items():
        out[f"{name}/w"] = w
        ok, total, _, _ = R.weights_check(w)
        assert ok
        out[f"{name}/total"] = np.float64(total)
        for P in (1, 2, 3, 4, 8):
            b, wn = R.psa_build(w, P)
            out[f"{name}/P{P}/buckets"] = b
            out[f"{name}/P{P}/bucket_mean"] = np.float64(wn)
            out[f"{name}/P{P}/masses"] = R.implied_masses(b, wn)
        if w.size >= 2:
            part = R.partition(w)
            for k in ("light", "heavy", "light_prefix", "heavy_prefix"):
                out[f"{name}/part/{k}"] = part[k]
            for P in (2, 8):
                try:
                    bnd, sp = R.psa_plan(w, P)
                    out[f"{name}/plan{P}/bounds"] = bnd
                    out[f"{name}/plan{P}/spill"] = sp
                except RuntimeError:
                    pass
    np.savez_compressed(os.path.join(HERE, "psa_small.npz"), **out)

    # --- draws (test_alias.cpp:269-284): powerlaw(50, 1.0, 3), psa(4) ------
    d = {}
    w = R.generate_powerlaw(50, 1.0, 3)
    t = R.table(w, 4)
    b, wn = t.buckets()
    d["w"] = w
    d["buckets"] = b
    d["bucket_mean"] = np.float64(wn)
    for W in (1, 3, 4, 8):
        s = t.sample_many(99, 100001, W)
        d[f"seed99_W{W}"] = s
    d["seed100_W4"] = t.sample_many(100, 100001, 4)
    np.savez_compressed(os.path.join(HERE, "draws_small.npz"), **d)

    medium(R)

    # --- rng known answers (rng.hpp) ----------------------------------------
    rng_and_two_level(R)
    print("golden fixtures written to", HERE)


def medium(R):
    """Medium tables at GPU-sized job counts (incl. wrs_b200_default_jobs(n):
    jobs of 32 items at these n): digests only."""
    m = {}
    for tag, w in (("uniform_1e6_s42", R.generate_uniform(10**6, 42)),
                   ("powerlaw1_1e6_s42", R.generate_powerlaw(10**6, 1.0, 42)),
                   ("powerlaw05_2e5_s7", R.generate_powerlaw(200_000, 0.5, 7))):
        m[f"{tag}/w_sha"] = sha(w)
        m[f"{tag}/w_head"] = w[:16].copy()
        ok, total, _, _ = R.weights_check(w)
        m[f"{tag}/total"] = np.float64(total)
        part = R.partition(w)
        m[f"{tag}/nl"] = np.uint64(part["light"].size)
        m[f"{tag}/light_sha"] = sha(part["light"])
        m[f"{tag}/heavy_sha"] = sha(part["heavy"])
        m[f"{tag}/light_prefix_sha"] = sha(part["light_prefix"])
        m[f"{tag}/heavy_prefix_sha"] = sha(part["heavy_prefix"])
        n = w.size
        for P in sorted({8, -(-n // 1024), -(-n // 512), -(-n // 256), -(-n // 128),
                         -(-n // 32)}):
            b, wn = R.psa_build_jobs(w, P, 8)
            m[f"{tag}/P{P}/buckets_sha"] = sha(b)
            m[f"{tag}/P{P}/bucket_mean"] = np.float64(wn)
            masses = R.implied_masses(b, wn)
            m[f"{tag}/P{P}/max_rel_err"] = np.float64(np.max(np.abs(masses - w) / w))
            if P == -(-n // 128):
                tb = b
                twn = wn
        # draws from the last table: seed 42, k=1e6, W in {1, 8}
        for W in (1, 8):
            from oracle import port
            s = port().sample_many(tb, twn, 42, 10**6, W)
            m[f"{tag}/draw_P{-(-n // 128)}_seed42_k1e6_W{W}_sha"] = sha(s)
    # generators at bench sizes (digests)
    m["uniform_1e8_s42/w_sha"] = sha(R.generate_uniform(10**8, 42))
    np.savez_compressed(os.path.join(HERE, "psa_medium.npz"), **m)


def rng_and_two_level(R):
    r = {}
    r["s42_st7"] = R.rng_outputs(42, 7, -1, 64)
    r["s9_st3_d123"] = R.rng_outputs(9, 3, 123, 64)
    r["alia_s99_d0"] = R.rng_outputs(99, 0x616C6961, 0, 64)
    r["alia_s99_d3"] = R.rng_outputs(99, 0x616C6961, 3, 64)
    np.savez_compressed(os.path.join(HERE, "rng.npz"), **r)
    two_level(R)


def two_level(R):
    """TwoLevelTable(wt, psa, 1, G).sample_many (two_level.hpp:26-81) over
    generate_powerlaw(3001, 1.0, 5): the routed-draw pins."""
    t = {}
    w = R.generate_powerlaw(3001, 1.0, 5)
    t["w_sha"] = sha(w)
    for G in (4, 7):
        tabs, means, bases, top, top_mean, T = R.two_level(w, G)
        t[f"G{G}/bases"] = bases
        t[f"G{G}/means"] = means
        t[f"G{G}/top"] = top
        t[f"G{G}/top_mean"] = np.float64(top_mean)
        t[f"G{G}/tables_sha"] = sha(np.concatenate(tabs))
        for W in (1, 3):
            t[f"G{G}/draws_s7_k5001_W{W}"] = T.draw(7, 5001, W)
    np.savez_compressed(os.path.join(HERE, "two_level.npz"), **t)


def default_jobs(n: int) -> int:
    """wrs_b200_default_jobs (engine.h): the job count "psa" uses."""
    j = 32
    while j < 1024 and 2 * j <= n // 49152:
        j *= 2
    lanes = 148 * 12 * 32  # K4a's resident jobs: stretch jobs when the last wave is < half full
    waves, last = divmod(-(-n // j), lanes)
    if waves >= 1 and last > 0 and (j < 1024 or last < lanes // 2):
        j = -(-n // (waves * lanes))
    return max(1, -(-n // j))


def large(R):
    """Full-size pins (VERDICT r1 "next" #1): reference-build digests of
    BASELINE configs[2]'s input generate_powerlaw(1e9, 1.0, 42)
    (weight_file.hpp:42-54), its G-shard totals (two_level.hpp:33-51: each a
    WeightTable over the contiguous block), the PSA tables of shards g = 0 and
    g = 7 of G = 8 at several job counts (alias.hpp:411-419 via the detail::
    pieces), and the configs[1] n = 1e8 uniform table at the job counts of
    1024-, 512- and 2048-item jobs.  Needs ~40 GB of host memory and a few
    minutes; writes psa_large.npz."""
    m = {}
    n = 10**9
    w = R.generate_powerlaw(n, 1.0, 42)
    m["pl1_1e9_s42/w_sha"] = sha(w)
    m["pl1_1e9_s42/w_head"] = w[:16].copy()
    m["pl1_1e9_s42/total"] = np.float64(R.pairwise_sum(w))
    for G in (2, 4, 8):
        block = -(-n // G)
        m[f"pl1_1e9_s42/G{G}/totals"] = np.array(
            [R.pairwise_sum(w[g * block:min(n, (g + 1) * block)]) for g in range(G)], np.float64)
    block = -(-n // 8)
    for g in (0, 7):
        ws = np.ascontiguousarray(w[g * block:min(n, (g + 1) * block)])
        m[f"pl1_1e9_s42/G8/g{g}/w_sha"] = sha(ws)
        ns = ws.size
        Ps = sorted({default_jobs(ns), -(-ns // 512), -(-ns // 2048)})
        m[f"pl1_1e9_s42/G8/g{g}/jobs"] = np.array(Ps, np.uint64)
        for P in Ps:
            b, wn = R.psa_build_jobs(ws, P, 8)
            m[f"pl1_1e9_s42/G8/g{g}/P{P}/buckets_sha"] = sha(b)
            m[f"pl1_1e9_s42/G8/g{g}/P{P}/bucket_mean"] = np.float64(wn)
            if P == default_jobs(ns):
                masses = R.implied_masses(b, wn)
                m[f"pl1_1e9_s42/G8/g{g}/P{P}/max_rel_err"] = np.float64(
                    np.max(np.abs(masses - ws) / ws))
                del masses
            del b
        del ws
        print("shard", g, "done", flush=True)
    del w
    n = 10**8
    w = R.generate_uniform(n, 42)
    Ps = sorted({default_jobs(n), -(-n // 512), -(-n // 2048)})
    m["uniform_1e8_s42/jobs"] = np.array(Ps, np.uint64)
    for P in Ps:
        b, wn = R.psa_build_jobs(w, P, 8)
        m[f"uniform_1e8_s42/P{P}/buckets_sha"] = sha(b)
        m[f"uniform_1e8_s42/P{P}/bucket_mean"] = np.float64(wn)
        if P == default_jobs(n):
            masses = R.implied_masses(b, wn)
            m[f"uniform_1e8_s42/P{P}/max_rel_err"] = np.float64(np.max(np.abs(masses - w) / w))
    print("uniform 1e8 done", flush=True)
    np.savez_compressed(os.path.join(HERE, "psa_large.npz"), **m)


def sweep_top(R):
    """BASELINE configs[4]'s largest sizes that fit this host: n = 2^28
    uniform and power-law s = 0.5 (seed 42) tables at the default job count,
    appended to psa_large.npz (2^30 needs ~60 GB of host memory here)."""
    path = os.path.join(HERE, "psa_large.npz")
    m = dict(np.load(path))
    n = 2**28
    for tag, w in (("uniform_2p28_s42", lambda: R.generate_uniform(n, 42)),
                   ("pl05_2p28_s42", lambda: R.generate_powerlaw(n, 0.5, 42))):
        w = w()
        m[f"{tag}/w_sha"] = sha(w)
        P = default_jobs(n)
        m[f"{tag}/jobs"] = np.array([P], np.uint64)
        b, wn = R.psa_build_jobs(w, P, 8)
        h = hashlib.sha256()
        h.update(memoryview(b).cast("B"))
        m[f"{tag}/P{P}/buckets_sha"] = h.hexdigest()
        m[f"{tag}/P{P}/bucket_mean"] = np.float64(wn)
        del b, w
        print(tag, "done", flush=True)
    np.savez_compressed(path, **m)


if __name__ == "__main__":
    if sys.argv[1:] == ["large"]:
        large(oracle.ref())
        sweep_top(oracle.ref())
    elif sys.argv[1:] == ["sweep_top"]:
        sweep_top(oracle.ref())
    elif sys.argv[1:] == ["two_level"]:
        two_level(oracle.ref())
    elif sys.argv[1:] == ["medium"]:
        medium(oracle.ref())
    else:
        main()
