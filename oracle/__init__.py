"""TEST INFRASTRUCTURE ONLY -- ctypes handles on the two CPU checkers.

``port()``  -> oracle/liboracle.so, the plain-C restatement (wrs_oracle.c).
``ref()``   -> oracle/_ref/libwrs_ref.so, the unmodified reference headers
               behind ref_shim.cpp (None when it was not built, e.g. on a box
               where /root/reference never existed and no prebuilt copy came
               along).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline leg may
import this package; the product (paper_1903_00227_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libwrs_ref.so")

BUCKET_DTYPE = np.dtype([("share", "<f8"), ("item", "<u4"), ("alias", "<u4")])

_port = None
_ref = None

u64 = C.c_uint64
f64 = C.c_double
vp = C.c_void_p


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class _Split(C.Structure):
    _fields_ = [("light_count", u64), ("heavy_count", u64), ("spill", f64)]


class _Job(C.Structure):
    _fields_ = [("light_lo", u64), ("light_hi", u64), ("heavy_lo", u64),
                ("heavy_hi", u64), ("spill", f64)]


class _Partition(C.Structure):
    _fields_ = [("nl", u64), ("nh", u64), ("light", vp), ("heavy", vp),
                ("light_prefix", vp), ("heavy_prefix", vp), ("wn", f64)]


def port() -> "Port":
    global _port
    if _port is None:
        if not os.path.exists(PORT_SO):
            build()
        _port = Port(C.CDLL(PORT_SO))
    return _port


def ref():
    global _ref
    if _ref is None and os.path.exists(REF_SO):
        _ref = Ref(C.CDLL(REF_SO))
    return _ref


class Port:
    """Plain-C restatement of the reference path (wrs_oracle.c)."""

    def __init__(self, lib):
        self.lib = lib
        lib.wo_mix64.restype = u64
        lib.wo_mix64.argtypes = [u64]
        lib.wo_rng_outputs.argtypes = [u64, u64, C.c_int64, u64, vp]
        lib.wo_pairwise_sum.restype = f64
        lib.wo_pairwise_sum.argtypes = [vp, u64]
        lib.wo_weights_check.argtypes = [vp, u64, vp, vp, vp, vp]
        lib.wo_generate_uniform.argtypes = [u64, u64, vp]
        lib.wo_generate_lognormal.argtypes = [u64, f64, u64, vp]
        lib.wo_generate_powerlaw.argtypes = [u64, f64, u64, vp]
        lib.wo_prefix_sums.argtypes = [vp, vp, u64]
        lib.wo_scan_block_totals.argtypes = [vp, u64, vp]
        lib.wo_scan_carries.argtypes = [vp, u64]
        lib.wo_partition_items.argtypes = [vp, u64, f64, C.POINTER(_Partition)]
        lib.wo_partition_free.argtypes = [C.POINTER(_Partition)]
        lib.wo_psa_split.restype = _Split
        lib.wo_psa_split.argtypes = [C.POINTER(_Partition), vp, u64]
        lib.wo_psa_plan.argtypes = [C.POINTER(_Partition), vp, u64, u64, C.POINTER(_Job)]
        lib.wo_psa_build.argtypes = [vp, u64, u64, vp, C.POINTER(f64)]
        lib.wo_sample_many.argtypes = [vp, u64, f64, u64, u64, C.c_uint32, vp]
        lib.wo_sample_range.argtypes = [vp, u64, f64, u64, u64, C.c_uint32, u64, u64, vp]
        lib.wo_implied_masses.argtypes = [vp, u64, f64, vp]
        lib.wo_two_level_sample_range.argtypes = [vp, vp, vp, vp, u64, vp, f64, u64, u64,
                                                  C.c_uint32, u64, u64, vp]
        lib.wo_philox4x32_10.argtypes = [vp, C.c_uint32, C.c_uint32]
        lib.wo_sample_philox_range.argtypes = [vp, u64, f64, u64, u64, u64, vp]
        lib.wo_max_relative_mass_error.restype = f64
        lib.wo_max_relative_mass_error.argtypes = [vp, vp, u64]

    # generators ----------------------------------------------------------
    def generate_uniform(self, n: int, seed: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        self.lib.wo_generate_uniform(n, seed, _ptr(out))
        return out

    def generate_lognormal(self, n: int, sigma: float, seed: int) -> np.ndarray:
        """configs[3]'s weights (the library's own generator, restated)."""
        out = np.empty(n, np.float64)
        self.lib.wo_generate_lognormal(n, C.c_double(sigma), seed, _ptr(out))
        return out

    def generate_powerlaw(self, n: int, s: float, seed: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        if self.lib.wo_generate_powerlaw(n, s, seed, _ptr(out)):
            raise ValueError("power law exponent must be finite and >= 0")
        return out

    # weights -------------------------------------------------------------
    def pairwise_sum(self, w: np.ndarray) -> float:
        w = np.ascontiguousarray(w, np.float64)
        return self.lib.wo_pairwise_sum(_ptr(w), w.size)

    def weights_check(self, w: np.ndarray):
        """(ok, bad_index, total, min, max)"""
        w = np.ascontiguousarray(w, np.float64)
        bad, tot, mn, mx = u64(), f64(), f64(), f64()
        rc = self.lib.wo_weights_check(_ptr(w), w.size, C.byref(bad), C.byref(tot),
                                       C.byref(mn), C.byref(mx))
        return rc == 0, bad.value, tot.value, mn.value, mx.value

    # scan ----------------------------------------------------------------
    def prefix_sums(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty_like(x)
        self.lib.wo_prefix_sums(_ptr(x), _ptr(out), x.size)
        return out

    def scan_block_totals(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty((x.size + 2047) // 2048, np.float64)
        self.lib.wo_scan_block_totals(_ptr(x), x.size, _ptr(out))
        return out

    def scan_carries(self, totals: np.ndarray) -> np.ndarray:
        c = np.array(totals, np.float64, copy=True)
        self.lib.wo_scan_carries(_ptr(c), c.size)
        return c

    # partition / plan / build --------------------------------------------
    def partition(self, w: np.ndarray):
        """dict(light, heavy, light_prefix, heavy_prefix, wn)"""
        w = np.ascontiguousarray(w, np.float64)
        ok, _, total, _, _ = self.weights_check(w)
        assert ok
        p = _Partition()
        self.lib.wo_partition_items(_ptr(w), w.size, total, C.byref(p))
        nl, nh = p.nl, p.nh
        res = dict(
            light=np.ctypeslib.as_array(C.cast(p.light, C.POINTER(C.c_uint32)), (max(nl, 1),))[:nl].copy(),
            heavy=np.ctypeslib.as_array(C.cast(p.heavy, C.POINTER(C.c_uint32)), (max(nh, 1),))[:nh].copy(),
            light_prefix=np.ctypeslib.as_array(C.cast(p.light_prefix, C.POINTER(C.c_double)), (nl + 1,)).copy(),
            heavy_prefix=np.ctypeslib.as_array(C.cast(p.heavy_prefix, C.POINTER(C.c_double)), (nh + 1,)).copy(),
            wn=p.wn, total=total)
        self.lib.wo_partition_free(C.byref(p))
        return res

    def psa_plan(self, w: np.ndarray, P: int):
        """(bounds[P,4] u64, spill[P] f64) or raises RuntimeError on the
        reference's logic_error."""
        w = np.ascontiguousarray(w, np.float64)
        ok, _, total, _, _ = self.weights_check(w)
        assert ok
        p = _Partition()
        self.lib.wo_partition_items(_ptr(w), w.size, total, C.byref(p))
        jobs = (_Job * P)()
        rc = self.lib.wo_psa_plan(C.byref(p), _ptr(w), w.size, P, jobs)
        self.lib.wo_partition_free(C.byref(p))
        if rc:
            raise RuntimeError("alias split boundaries must be nondecreasing")
        b = np.array([[j.light_lo, j.light_hi, j.heavy_lo, j.heavy_hi] for j in jobs], np.uint64)
        s = np.array([j.spill for j in jobs], np.float64)
        return b, s

    def psa_split(self, w: np.ndarray, n_prime: int):
        w = np.ascontiguousarray(w, np.float64)
        ok, _, total, _, _ = self.weights_check(w)
        p = _Partition()
        self.lib.wo_partition_items(_ptr(w), w.size, total, C.byref(p))
        s = self.lib.wo_psa_split(C.byref(p), _ptr(w), n_prime)
        self.lib.wo_partition_free(C.byref(p))
        return s.light_count, s.heavy_count, s.spill

    def psa_build(self, w: np.ndarray, P: int):
        """(buckets structured array, bucket_mean)"""
        w = np.ascontiguousarray(w, np.float64)
        out = np.zeros(w.size, BUCKET_DTYPE)
        wn = f64()
        rc = self.lib.wo_psa_build(_ptr(w), w.size, P, _ptr(out), C.byref(wn))
        if rc:
            raise ValueError(f"wo_psa_build failed rc={rc}")
        return out, wn.value

    # sampling / verify ---------------------------------------------------
    def sample_many(self, buckets, wn: float, seed: int, k: int, workers: int) -> np.ndarray:
        out = np.empty(k, np.uint32)
        self.lib.wo_sample_many(_ptr(buckets), buckets.size, wn, seed, k, workers, _ptr(out))
        return out

    def sample_range(self, buckets, wn, seed, k, workers, q_lo, q_hi) -> np.ndarray:
        out = np.empty(q_hi - q_lo, np.uint32)
        self.lib.wo_sample_range(_ptr(buckets), buckets.size, wn, seed, k, workers,
                                 q_lo, q_hi, _ptr(out))
        return out

    def implied_masses(self, buckets, wn: float) -> np.ndarray:
        out = np.empty(buckets.size, np.float64)
        self.lib.wo_implied_masses(_ptr(buckets), buckets.size, wn, _ptr(out))
        return out

    def philox4x32_10(self, ctr, key):
        c = np.array(ctr, np.uint32)
        self.lib.wo_philox4x32_10(_ptr(c), int(key[0]), int(key[1]))
        return c

    def sample_philox_range(self, buckets, wn, seed, q_lo, q_hi) -> np.ndarray:
        out = np.empty(q_hi - q_lo, np.uint32)
        self.lib.wo_sample_philox_range(_ptr(buckets), buckets.size, wn, seed, q_lo, q_hi,
                                        _ptr(out))
        return out

    def two_level_build(self, w, groups: int):
        """TwoLevelTable(wt, psa, 1, groups) (two_level.hpp:30-58) restated:
        contiguous groups of ceil(n/groups), P=1 psa tables per group and over
        the group totals.  Returns (tables, means, bases, top, top_mean)."""
        w = np.ascontiguousarray(w, np.float64)
        n = w.size
        groups = min(groups, n)
        block = -(-n // groups)
        groups = -(-n // block)
        bases = [min(n, g * block) for g in range(groups + 1)]
        tables, means, totals = [], [], []
        for g in range(groups):
            wg = w[bases[g]:bases[g + 1]]
            b, m = self.psa_build(wg, 1)
            tables.append(b)
            means.append(m)
            totals.append(self.pairwise_sum(wg))
        top, top_mean = self.psa_build(np.array(totals), 1)
        return tables, np.array(means), np.array(bases[:-1], np.uint64), top, top_mean

    def two_level_sample_range(self, tables, means, bases, top, top_mean, seed, k, workers,
                               q_lo, q_hi) -> np.ndarray:
        G = len(tables)
        ptrs = (C.c_void_p * G)(*[t.ctypes.data for t in tables])
        sizes = np.array([t.size for t in tables], np.uint64)
        means = np.ascontiguousarray(means, np.float64)
        bases = np.ascontiguousarray(bases, np.uint64)
        out = np.empty(q_hi - q_lo, np.uint32)
        self.lib.wo_two_level_sample_range(ptrs, _ptr(sizes), _ptr(means), _ptr(bases), G,
                                           _ptr(top), top_mean, seed, k, workers, q_lo, q_hi,
                                           _ptr(out))
        return out

    def max_relative_mass_error(self, masses, w) -> float:
        w = np.ascontiguousarray(w, np.float64)
        return self.lib.wo_max_relative_mass_error(_ptr(masses), _ptr(w), w.size)

    def mix64(self, z: int) -> int:
        return self.lib.wo_mix64(z)

    def rng_outputs(self, seed, stream, salt, count) -> np.ndarray:
        out = np.empty(count, np.uint64)
        self.lib.wo_rng_outputs(seed, stream, salt, count, _ptr(out))
        return out


class Ref:
    """The unmodified reference headers (ref_shim.cpp)."""

    def __init__(self, lib):
        self.lib = lib
        lib.ref_weights_check.argtypes = [vp, u64, vp, vp, vp]
        lib.ref_pairwise_sum.restype = f64
        lib.ref_pairwise_sum.argtypes = [vp, u64]
        lib.ref_prefix_sums.argtypes = [vp, vp, u64, C.c_uint]
        lib.ref_generate_uniform.argtypes = [u64, u64, vp]
        lib.ref_generate_powerlaw.argtypes = [u64, f64, u64, vp]
        lib.ref_rng_outputs.restype = u64
        lib.ref_rng_outputs.argtypes = [u64, u64, C.c_int64, u64, vp]
        lib.ref_psa_build.argtypes = [vp, u64, C.c_uint, vp, C.POINTER(f64)]
        lib.ref_psa_build_jobs.argtypes = [vp, u64, u64, C.c_uint, vp, C.POINTER(f64)]
        lib.ref_partition.argtypes = [vp, u64, vp, vp, vp, vp, vp, vp, vp]
        lib.ref_psa_plan.argtypes = [vp, u64, u64, vp, vp]
        lib.ref_table_new.restype = vp
        lib.ref_table_new.argtypes = [vp, u64, C.c_uint]
        lib.ref_table_free.argtypes = [vp]
        lib.ref_table_buckets.argtypes = [vp, vp, C.POINTER(f64)]
        lib.ref_table_sample_many.argtypes = [vp, u64, u64, C.c_uint, vp]
        lib.ref_build_method.argtypes = [vp, u64, C.c_int, vp, C.POINTER(f64)]
        lib.ref_wt_new.restype = vp
        lib.ref_wt_new.argtypes = [vp, u64]
        lib.ref_wt_free.argtypes = [vp]
        lib.ref_table_from_wt.restype = vp
        lib.ref_table_from_wt.argtypes = [vp, C.c_uint]
        lib.ref_outbuf_new.restype = vp
        lib.ref_outbuf_new.argtypes = [u64]
        lib.ref_outbuf_free.argtypes = [vp]
        lib.ref_outbuf_data.restype = vp
        lib.ref_outbuf_data.argtypes = [vp]
        lib.ref_table_sample_into.argtypes = [vp, u64, u64, C.c_uint, vp]
        lib.ref_implied_masses.argtypes = [vp, u64, f64, vp]
        lib.ref_binomial_split.restype = u64
        lib.ref_binomial_split.argtypes = [u64, u64, C.c_int64, u64, f64, f64]
        lib.ref_two_level_group_totals.restype = u64
        lib.ref_two_level_group_totals.argtypes = [vp, u64, u64, vp]
        lib.ref_two_level_new.restype = vp
        lib.ref_two_level_new.argtypes = [vp, u64, u64]
        lib.ref_two_level_free.argtypes = [vp]
        lib.ref_two_level_groups.restype = u64
        lib.ref_two_level_groups.argtypes = [vp]
        lib.ref_two_level_group_begin.restype = u64
        lib.ref_two_level_group_begin.argtypes = [vp, u64]
        lib.ref_two_level_buckets.restype = u64
        lib.ref_two_level_buckets.argtypes = [vp, u64, vp, C.POINTER(f64)]
        lib.ref_two_level_sample_many.argtypes = [vp, u64, u64, C.c_uint, vp]

    def generate_uniform(self, n, seed):
        out = np.empty(n, np.float64)
        self.lib.ref_generate_uniform(n, seed, _ptr(out))
        return out

    def generate_powerlaw(self, n, s, seed):
        out = np.empty(n, np.float64)
        if self.lib.ref_generate_powerlaw(n, s, seed, _ptr(out)):
            raise ValueError("bad exponent")
        return out

    def weights_check(self, w):
        w = np.ascontiguousarray(w, np.float64)
        t, a, b = f64(), f64(), f64()
        rc = self.lib.ref_weights_check(_ptr(w), w.size, C.byref(t), C.byref(a), C.byref(b))
        return rc == 0, t.value, a.value, b.value

    def pairwise_sum(self, w):
        w = np.ascontiguousarray(w, np.float64)
        return self.lib.ref_pairwise_sum(_ptr(w), w.size)

    def prefix_sums(self, x, workers=4):
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty_like(x)
        self.lib.ref_prefix_sums(_ptr(x), _ptr(out), x.size, workers)
        return out

    def rng_outputs(self, seed, stream, salt, count):
        out = np.empty(count, np.uint64)
        self.lib.ref_rng_outputs(seed, stream, salt, count, _ptr(out))
        return out

    def psa_build(self, w, workers):
        """AliasTable(wt, psa, workers) -- one OS thread per job."""
        w = np.ascontiguousarray(w, np.float64)
        out = np.zeros(w.size, BUCKET_DTYPE)
        wn = f64()
        if self.lib.ref_psa_build(_ptr(w), w.size, workers, _ptr(out), C.byref(wn)):
            raise ValueError("reference build failed")
        return out, wn.value

    def build_method(self, w, method: str):
        """AliasTable(wt, Build::vose | Build::sweep) of the reference."""
        w = np.ascontiguousarray(w, np.float64)
        out = np.zeros(w.size, BUCKET_DTYPE)
        wn = f64()
        if self.lib.ref_build_method(_ptr(w), w.size, {"vose": 0, "sweep": 1}[method], _ptr(out),
                                     C.byref(wn)):
            raise ValueError("reference build failed")
        return out, wn.value

    def psa_build_jobs(self, w, P, threads=8):
        """detail:: pieces at job count P over `threads` threads."""
        w = np.ascontiguousarray(w, np.float64)
        out = np.zeros(w.size, BUCKET_DTYPE)
        wn = f64()
        if self.lib.ref_psa_build_jobs(_ptr(w), w.size, P, threads, _ptr(out), C.byref(wn)):
            raise ValueError("reference build failed")
        return out, wn.value

    def partition(self, w):
        w = np.ascontiguousarray(w, np.float64)
        nl, nh, wn = u64(), u64(), f64()
        self.lib.ref_partition(_ptr(w), w.size, C.byref(nl), C.byref(nh), None, None,
                               None, None, C.byref(wn))
        L = np.empty(nl.value, np.uint32)
        H = np.empty(nh.value, np.uint32)
        Lp = np.empty(nl.value + 1, np.float64)
        Hp = np.empty(nh.value + 1, np.float64)
        self.lib.ref_partition(_ptr(w), w.size, C.byref(nl), C.byref(nh), _ptr(L), _ptr(H),
                               _ptr(Lp), _ptr(Hp), C.byref(wn))
        return dict(light=L, heavy=H, light_prefix=Lp, heavy_prefix=Hp, wn=wn.value)

    def psa_plan(self, w, P):
        w = np.ascontiguousarray(w, np.float64)
        b = np.empty((P, 4), np.uint64)
        s = np.empty(P, np.float64)
        rc = self.lib.ref_psa_plan(_ptr(w), w.size, P, _ptr(b), _ptr(s))
        if rc == 2:
            raise RuntimeError("alias split boundaries must be nondecreasing")
        if rc:
            raise ValueError("reference plan failed")
        return b, s

    def table(self, w, workers):
        return RefTable(self, w, workers)

    def implied_masses(self, buckets, wn):
        out = np.empty(buckets.size, np.float64)
        self.lib.ref_implied_masses(_ptr(buckets), buckets.size, wn, _ptr(out))
        return out

    def binomial_split(self, seed, stream, salt, k, wl, wr):
        return self.lib.ref_binomial_split(seed, stream, salt, k, wl, wr)

    def two_level(self, w, groups):
        """The reference TwoLevelTable(wt, psa, 1, groups): (tables, means,
        bases, top, top_mean, draw) with draw(seed, k, workers)."""
        w = np.ascontiguousarray(w, np.float64)
        h = self.lib.ref_two_level_new(_ptr(w), w.size, groups)
        if not h:
            raise ValueError("reference two-level build failed")
        try:
            G = self.lib.ref_two_level_groups(h)

            def buckets(g):
                m = f64()
                size = self.lib.ref_two_level_buckets(h, g, None, C.byref(m))
                b = np.empty(size, BUCKET_DTYPE)
                self.lib.ref_two_level_buckets(h, g, _ptr(b), C.byref(m))
                return b, m.value
            tabs = [buckets(g) for g in range(G)]
            top, top_mean = buckets(G)
            bases = np.array([self.lib.ref_two_level_group_begin(h, g) for g in range(G)],
                             np.uint64)
        except Exception:
            self.lib.ref_two_level_free(h)
            raise
        lib = self.lib

        class _T:
            def draw(self_, seed, k, workers):
                out = np.empty(k, np.uint32)
                lib.ref_two_level_sample_many(h, seed, k, workers, _ptr(out))
                return out

            def __del__(self_):
                lib.ref_two_level_free(h)
        t = _T()
        return ([b for b, _ in tabs], np.array([m for _, m in tabs]), bases, top, top_mean, t)

    def two_level_group_totals(self, w, groups):
        w = np.ascontiguousarray(w, np.float64)
        out = np.empty(max(1, groups), np.float64)
        g = self.lib.ref_two_level_group_totals(_ptr(w), w.size, groups, _ptr(out))
        return out[:g]


class RefTable:
    def __init__(self, ref: Ref, w, workers):
        self.ref = ref
        w = np.ascontiguousarray(w, np.float64)
        self.n = w.size
        self.h = ref.lib.ref_table_new(_ptr(w), w.size, workers)
        if not self.h:
            raise ValueError("reference table build failed")

    def buckets(self):
        out = np.zeros(self.n, BUCKET_DTYPE)
        wn = f64()
        self.ref.lib.ref_table_buckets(self.h, _ptr(out), C.byref(wn))
        return out, wn.value

    def sample_many(self, seed, k, workers):
        out = np.empty(k, np.uint32)
        self.ref.lib.ref_table_sample_many(self.h, seed, k, workers, _ptr(out))
        return out

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_table_free(self.h)
            self.h = None
