"""CPU: the C-ABI library loads, exports exactly what include/*.h declares,
and its host-only logic (status names, argument checks, stubs, job count,
shard ranges, the binomial k-split) behaves like the reference.  No compute
call is made here (no GPU in this container)."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

import oracle
import paper_1903_00227_b200 as wrs
from paper_1903_00227_b200.wrs import SIGNATURES, WRS_EINVAL, lib
from tests.conftest import cuda_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in ("wrs.h", "wrs_b200.h"):
        text = open(os.path.join(ROOT, "include", h)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names |= set(re.findall(r"WRS_API[^;(]*?\b(wrs_\w+)\s*\(", text))
    return names


def test_every_declared_symbol_is_exported_and_bound():
    names = declared_symbols()
    assert len(names) >= 40
    L = lib()
    for n in names:
        assert hasattr(L, n), n
    assert names == set(SIGNATURES), names ^ set(SIGNATURES)


def test_reference_abi_surface_is_complete():
    # every entry point of the reference header wrs.h:36-134
    ref_names = {"wrs_last_error", "wrs_status_name", "wrs_weights_from_array",
                 "wrs_weights_generate", "wrs_weights_read", "wrs_weights_write",
                 "wrs_weights_count", "wrs_weights_values", "wrs_weights_free",
                 "wrs_sampler_build", "wrs_sampler_verify_masses", "wrs_sampler_draw",
                 "wrs_sampler_free", "wrs_sample_with_replacement",
                 "wrs_sample_without_replacement", "wrs_permutation", "wrs_subset_sample",
                 "wrs_reservoir_create", "wrs_reservoir_push", "wrs_reservoir_items",
                 "wrs_reservoir_threshold", "wrs_reservoir_free", "wrs_verify"}
    assert ref_names <= declared_symbols()


def test_status_names():  # test_capi.cpp:76-79
    assert wrs.status_name(0) == "WRS_OK"
    assert wrs.status_name(4) == "WRS_EVERIFY"
    assert wrs.status_name(99) == "WRS_UNKNOWN"


def test_null_arguments_are_einval():  # capi.cpp:104-105,151-152,208-209
    L = lib()
    h = C.c_void_p()
    assert L.wrs_weights_from_array(None, 2, C.byref(h)) == WRS_EINVAL
    assert "null" in wrs.last_error()
    assert L.wrs_sampler_build(None, b"psa", 1, 0, C.byref(h)) == WRS_EINVAL
    assert L.wrs_sampler_draw(None, 1, 1, 1, None) == WRS_EINVAL
    assert L.wrs_sample_with_replacement(None, 1, 1, 1, None, None, None) == WRS_EINVAL
    assert L.wrs_b200_sampler_draw_counts(None, 1, 1, 1, None, None, None) == WRS_EINVAL
    assert L.wrs_b200_sampler_draw_counts_device(None, 1, 1, 1, None, None, None,
                                                 None) == WRS_EINVAL
    assert L.wrs_weights_count(None) == 0
    assert L.wrs_weights_values(None) is None


def test_out_of_path_entry_points_are_stubbed():
    L = lib()
    h = C.c_void_p()
    assert L.wrs_permutation(None, 1, 1, None) == WRS_EINVAL
    assert L.wrs_reservoir_create(1, 1, 1, C.byref(h)) == WRS_EINVAL and not h.value
    assert math.isnan(L.wrs_reservoir_threshold(None))
    assert L.wrs_verify(b"all", 1, 0) == WRS_EINVAL
    assert "not part of the B200 PSA path" in wrs.last_error()


def test_default_job_count():
    # jobs of J = pow2_floor(n / 49152) items clamped to [32, 1024], stretched
    # to fill whole K4a waves (148 * 12 * 32 = 56832 jobs each) when jobs are
    # below the 1024 cap, or the last wave would be less than half full
    # (engine.h default_job_items)
    assert wrs.default_jobs(1) == 1
    assert wrs.default_jobs(32) == 1
    assert wrs.default_jobs(33) == 2
    assert wrs.default_jobs(10**6) == -(-10**6 // 32)            # < one wave
    assert wrs.default_jobs(1 << 22) == -(-(1 << 22) // 74)       # 1.15 waves of J = 64 -> 1
    assert wrs.default_jobs(1 << 24) == -(-(1 << 24) // 296)      # 1.15 waves of J = 256 -> 1
    assert wrs.default_jobs(12_000_000) == -(-12_000_000 // 212)  # 1.65 waves of J = 128 -> 1
    assert wrs.default_jobs(10**8) == -(-10**8 // 1024)           # J = 1024, last wave 72 % full: kept
    assert wrs.default_jobs(125_000_000) == -(-125_000_000 // 1100)  # 2.15 waves -> 2
    assert wrs.default_jobs(1 << 28) == (1 << 28) // 1024         # 4.61 waves: kept
    assert wrs.default_jobs(1 << 30) == -(-(1 << 30) // 1050)     # 18.45 waves -> 18
    for n in (1 << 24, 125_000_000, 1 << 30, 10**9):
        P = wrs.default_jobs(n)
        assert P % 56832 == 0 or P % 56832 >= 28416 or P < 56832, n


def test_shard_ranges_match_two_level_blocks():  # two_level.hpp:33-41
    for n, G in ((103, 7), (10**9, 8), (10, 4), (5, 8)):
        los = [wrs.shard_range(n, G, g) for g in range(G)]
        block = -(-n // min(G, n))
        for g, (lo, hi) in enumerate(los):
            assert lo == min(n, g * block) and hi == min(n, (g + 1) * block)
        assert los[0][0] == 0 and max(hi for _, hi in los) == n


def _replay_counts(R, P, totals, seed, k):
    """Host replay of the k-split DC tree with the reference's binomial_split."""
    G = len(totals)
    counts = [0] * G

    def rec(a, b, node, kk):
        if b - a == 1:
            counts[a] = kk
            return
        mid = a + (b - a) // 2
        wl = P.pairwise_sum(np.array(totals[a:mid]))
        wr = P.pairwise_sum(np.array(totals[mid:b]))
        kl = R.binomial_split(seed, 0x73687264, node, kk, wl, wr)
        rec(a, mid, 2 * node + 1, kl)
        rec(mid, b, 2 * node + 2, kk - kl)

    rec(0, G, 0, k)
    return counts


def test_shard_counts_sum_and_reproduce():
    totals = np.array([5.0e8, 1.0e8, 3.3e8, 0.2e8, 7.1e8, 2.0e8, 1.0e8, 4.4e8])
    for k in (0, 1, 17, 10**6, 10**10):
        c = wrs.shard_counts(totals, 42, k)
        assert int(c.sum()) == k
        assert np.array_equal(c, wrs.shard_counts(totals, 42, k))
    R = oracle.ref()
    if R is None:
        pytest.skip("reference build absent")
    P = oracle.port()
    for seed in (1, 42, 7777):
        for k in (5, 31, 1000, 10**7, 10**10):
            for G in (1, 2, 3, 8):
                c = wrs.shard_counts(totals[:G], seed, k)
                assert list(c) == _replay_counts(R, P, list(totals[:G]), seed, k), (seed, k, G)


@pytest.mark.skipif(cuda_available(), reason="checks the no-GPU failure mode")
def test_compute_calls_fail_loudly_without_gpu():
    with pytest.raises(wrs.WrsError) as e:
        wrs.Weights.from_array(np.array([1.0, 2.0]))
    assert e.value.status in (wrs.wrs.WRS_EINTERNAL, wrs.wrs.WRS_ENOMEM)


def test_nccl_loads_lazily_for_the_multi_gpu_path():
    """libwrs_b200.so has no link-time NCCL dependency; the multi-GPU calls
    dlopen libnccl.so.2 (here: the system NCCL) and can make a job's unique
    id without a GPU."""
    import subprocess
    deps = subprocess.run(["ldd", wrs.wrs.LIB_PATH], capture_output=True, text=True).stdout
    assert "nccl" not in deps
    ok, version = wrs.nccl_available()
    assert ok and version >= 22700, version
    a, b = wrs.nccl_unique_id(), wrs.nccl_unique_id()
    assert len(a) == 128 and a != b


def test_multi_calls_validate_arguments():
    L = lib()
    h = C.c_void_p()
    assert L.wrs_b200_multi_create(None, 10, 0, 1, None, C.byref(h)) == wrs.wrs.WRS_EINVAL
    assert L.wrs_b200_multi_set_totals(None, None) == wrs.wrs.WRS_EINVAL
    assert L.wrs_b200_multi_exchange(None, None) == wrs.wrs.WRS_EINVAL
    assert L.wrs_b200_multi_counts(None, 1, 1, None) == wrs.wrs.WRS_EINVAL
    assert L.wrs_b200_multi_shard(None) is None
    L.wrs_b200_multi_free(None)


def build_capi_client(tmp_dir) -> str:
    """Compile tests/capi_client.c (plain C, include/wrs.h) and link it to
    libwrs_b200.so the way a reference client links libwrs."""
    import subprocess
    exe = os.path.join(str(tmp_dir), "capi_client")
    libdir = os.path.dirname(wrs.wrs.LIB_PATH)
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "capi_client.c"), "-o", exe, "-L", libdir,
                    "-l:libwrs_b200.so", f"-Wl,-rpath,{libdir}"], check=True)
    return exe


def test_c_client_links_and_fails_loudly_without_gpu(tmp_path):
    import subprocess
    from tests.conftest import cuda_available
    if cuda_available():
        pytest.skip("GPU present: test_gpu_parity runs the client for real")
    exe = build_capi_client(tmp_path)
    r = subprocess.run([exe, "--no-gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "capi client ok" in r.stdout
