"""Small-n workload for the checked build (scripts/gpu_checked.sh;
compute-sanitizer itself is closed on the GPU pool).

Exercises every kernel family of libwrs_b200.so at sizes where the
sanitizers finish in minutes, and checks each result against the oracle so a
sanitizer run is also a parity run:
  * the PSA build with every K2 form (split / direct / staged), several job
    counts (incl. P > n), uniform / power-law / ties / no-heavy inputs, and
    the guarded (W >= 1e300) chains;
  * draws on the direct and the region plan (region plan forced on a small
    table with 2^16-bucket regions), W in {1, 3}, the Philox mode, the slab
    redirect path (shrunken slabs);
  * aggregated draws (region + direct), routed two-level draws, device
    implied masses, the device power-law deal, the double-buffered rebuild
    with a draw on another stream.
Test infrastructure: imports oracle/ only as the checker.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_1903_00227_b200 as wrs  # noqa: E402


def check_table(S, w, P, port):
    ob, own = port.psa_build(w, P)
    assert S.bucket_mean == own
    assert S.buckets().tobytes() == ob.tobytes(), (w.size, P)
    return ob, own


def main():
    import torch
    torch.cuda.set_device(0)
    port = oracle.port()
    rng = np.random.default_rng(5)
    cases = [port.generate_uniform(20011, 1), port.generate_powerlaw(30000, 1.0, 2),
             np.full(777, 0.5), np.concatenate([[1e6], np.ones(4999)]),
             np.where(rng.random(9000) < 0.5, 1.0, rng.random(9000) + 0.5),
             np.array([1e300, 2e300, 3e300, 1.0])]
    big = "9223372036854775807"
    # staged = the large-table forms: bulk-copy K2a + fused K2b/K2c (default),
    # bulk-copy with a separate K2b, and the smem-staged kernels
    forms = {"split": (big, big, {}), "direct": ("0", big, {}), "staged": ("0", "0", {}),
             "staged-nofuse": ("0", "0", {"WRS_B200_K2_FUSE": "0"}),
             "staged-fuse1": ("0", "0", {"WRS_B200_K2_FUSE": "1"}),
             "staged-nokb": ("0", "0", {"WRS_B200_K2_KB": "0"})}
    for form, (smax, dmax, extra) in forms.items():
        os.environ["WRS_B200_K2_SPLIT_MAX"] = smax
        os.environ["WRS_B200_K2_DIRECT_MAX"] = dmax
        for e in ("WRS_B200_K2_FUSE", "WRS_B200_K2_KB"):
            os.environ.pop(e, None)
        os.environ.update(extra)
        for w in cases:
            for P in (1, 7, wrs.default_jobs(w.size), w.size + 3):
                W = wrs.Weights.from_array(w)
                S = wrs.Sampler.build_psa(W, P, keep_workspace=(P == 7))
                check_table(S, w, P, port)
                S.free()
                W.free()
        print("build", form, "ok", flush=True)
    for k in ("WRS_B200_K2_SPLIT_MAX", "WRS_B200_K2_DIRECT_MAX", "WRS_B200_K2_FUSE", "WRS_B200_K2_KB"):
        os.environ.pop(k, None)

    # draws: direct plan, then the region plan forced on 2^16-bucket regions
    w = port.generate_powerlaw(300_007, 0.5, 9)
    W = wrs.Weights.from_array(w)
    S = wrs.Sampler.build(W, "psa", 1)
    ob, own = check_table(S, w, S.jobs, port)
    k = 400_009
    out = torch.empty(k, dtype=torch.int32, device="cuda")
    for plan in ("d", "r"):
        os.environ["WRS_B200_PLAN"] = plan
        os.environ["WRS_B200_REGION_SHIFT"] = "16"
        for Wk in (1, 3):
            S.draw_device(11, k, Wk, out)
            torch.cuda.synchronize()
            assert np.array_equal(out.cpu().numpy().view(np.uint32),
                                  port.sample_many(ob, own, 11, k, Wk)), (plan, Wk)
            items, counts = S.draw_counts(11, k, Wk)
            ri, rc = np.unique(port.sample_many(ob, own, 11, k, Wk), return_counts=True)
            assert np.array_equal(items, ri) and np.array_equal(counts, rc), (plan, Wk)
        S.draw_philox_device(5, k, out)
        torch.cuda.synchronize()
        got = out.cpu().numpy().view(np.uint32)
        assert np.array_equal(got, port.sample_philox_range(ob, own, 5, 0, k)), plan
        print("draws", plan, "ok", flush=True)
    # slab redirect (region plan): shrunken slabs, large overflow slab
    os.environ["WRS_B200_TEST_SLAB_CAP"] = "4096"
    os.environ["WRS_B200_TEST_OV_CAP"] = "1000000"
    S.draw_device(12, k, 1, out)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().view(np.uint32), port.sample_many(ob, own, 12, k, 1))
    for e in ("WRS_B200_TEST_SLAB_CAP", "WRS_B200_TEST_OV_CAP", "WRS_B200_PLAN",
              "WRS_B200_REGION_SHIFT"):
        os.environ.pop(e)
    print("slab redirect ok", flush=True)

    # implied masses on the device
    m, worst = S.implied_masses()
    assert m.tobytes() == port.implied_masses(ob, own).tobytes()

    # double-buffered rebuild, draw on another stream
    S.double_buffer()
    a, b = torch.cuda.Stream(), torch.cuda.Stream()
    ref = port.sample_many(ob, own, 3, k, 1)
    for _ in range(2):
        S.rebuild_async(a)
        S.draw_device(3, k, 1, out, b)
        b.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint32), ref)
    S.check()
    print("double buffer ok", flush=True)

    # routed two-level draws
    tabs, means, bases, top, tm = port.two_level_build(w[:50_000], 8)
    dt = [torch.from_numpy(t.view(np.uint8).copy()).cuda() for t in tabs]
    dtop = torch.from_numpy(top.view(np.uint8).copy()).cuda()
    kk = 60_000
    o2 = torch.empty(kk, dtype=torch.int32, device="cuda")
    wrs.wrs.two_level_draw_device(dt, [t.size for t in tabs], means, bases, dtop, tm, 7, 0, kk,
                                  kk, 3, o2)
    torch.cuda.synchronize()
    assert np.array_equal(o2.cpu().numpy().view(np.uint32),
                          port.two_level_sample_range(tabs, means, bases, top, tm, 7, kk, 3, 0, kk))
    print("two-level ok", flush=True)

    # device power-law deal
    Wp = wrs.Weights.generate("powerlaw", 1.0, 100_003, 8)
    assert np.array_equal(Wp.values(), port.generate_powerlaw(100_003, 1.0, 8))
    bad, line = wrs.check_failures()
    print(f"device index-check violations: {bad} (first at line {line})", flush=True)
    assert bad <= 0, (bad, line)
    print("sanitize cases: all ok", flush=True)


if __name__ == "__main__":
    main()
