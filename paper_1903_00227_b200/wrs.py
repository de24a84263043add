"""ctypes binding of libwrs_b200.so -- the reference's C ABI (include/wrs.h)
plus the B200 extensions (include/wrs_b200.h).

The classes mirror the reference's handle model (capi.cpp: wrs_weights,
wrs_sampler) so the tests read like the reference's own test_capi.cpp.  There
is no Python or CPU compute here: every method is one ABI call into the CUDA
library, and loading fails loudly when the library is missing.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# WRS_B200_LIB selects another build of the same library (A/B experiments)
LIB_PATH = os.environ.get("WRS_B200_LIB") or os.path.join(HERE, "libwrs_b200.so")

WRS_OK, WRS_EINVAL, WRS_EIO, WRS_EFORMAT, WRS_EVERIFY, WRS_ENOMEM, WRS_EINTERNAL = range(7)
KEEP_WORKSPACE = 1
CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy

BUCKET_DTYPE = np.dtype([("share", "<f8"), ("item", "<u4"), ("alias", "<u4")])

u64, f64, u32, vp = C.c_uint64, C.c_double, C.c_uint32, C.c_void_p

# every symbol include/wrs.h and include/wrs_b200.h declare, with ctypes types
SIGNATURES = {
    "wrs_last_error": (C.c_char_p, []),
    "wrs_status_name": (C.c_char_p, [C.c_int]),
    "wrs_weights_from_array": (C.c_int, [vp, u64, C.POINTER(vp)]),
    "wrs_weights_generate": (C.c_int, [C.c_char_p, f64, u64, u64, C.POINTER(vp)]),
    "wrs_weights_read": (C.c_int, [C.c_char_p, C.POINTER(vp)]),
    "wrs_weights_write": (C.c_int, [vp, C.c_char_p]),
    "wrs_weights_count": (u64, [vp]),
    "wrs_weights_values": (vp, [vp]),
    "wrs_weights_free": (None, [vp]),
    "wrs_sampler_build": (C.c_int, [vp, C.c_char_p, C.c_uint, u64, C.POINTER(vp)]),
    "wrs_sampler_verify_masses": (C.c_int, [vp, f64]),
    "wrs_sampler_draw": (C.c_int, [vp, u64, u64, C.c_uint, vp]),
    "wrs_sampler_free": (None, [vp]),
    "wrs_sample_with_replacement": (C.c_int, [vp, u64, u64, C.c_uint, vp, vp, C.POINTER(u64)]),
    "wrs_sample_without_replacement": (C.c_int, [vp, u64, u64, C.c_uint, vp]),
    "wrs_permutation": (C.c_int, [vp, u64, C.c_uint, vp]),
    "wrs_subset_sample": (C.c_int, [vp, u64, C.c_uint, vp, vp]),
    "wrs_reservoir_create": (C.c_int, [u64, C.c_uint, u64, C.POINTER(vp)]),
    "wrs_reservoir_push": (C.c_int, [vp, vp, vp, u64]),
    "wrs_reservoir_items": (C.c_int, [vp, vp, vp, vp]),
    "wrs_reservoir_threshold": (f64, [vp]),
    "wrs_reservoir_free": (None, [vp]),
    "wrs_verify": (C.c_int, [C.c_char_p, u64, C.c_int]),
    "wrs_b200_default_jobs": (u64, [u64]),
    "wrs_b200_release_cache": (u64, []),
    "wrs_b200_check_failures": (C.c_int64, [C.POINTER(C.c_uint)]),
    "wrs_b200_weights_from_device": (C.c_int, [vp, u64, C.c_int, C.POINTER(vp)]),
    "wrs_b200_weights_generate_range": (C.c_int, [C.c_char_p, f64, u64, u64, u64, u64,
                                                  C.POINTER(vp)]),
    "wrs_b200_weights_total": (f64, [vp]),
    "wrs_b200_weights_device": (vp, [vp]),
    "wrs_b200_sampler_build_psa": (C.c_int, [vp, u64, C.c_uint, C.POINTER(vp)]),
    "wrs_b200_sampler_jobs": (u64, [vp]),
    "wrs_b200_sampler_size": (u64, [vp]),
    "wrs_b200_sampler_bucket_mean": (f64, [vp]),
    "wrs_b200_sampler_total": (f64, [vp]),
    "wrs_b200_sampler_device_buckets": (vp, [vp]),
    "wrs_b200_sampler_copy_buckets": (C.c_int, [vp, vp]),
    "wrs_b200_sampler_rebuild_async": (C.c_int, [vp, vp]),
    "wrs_b200_sampler_check": (C.c_int, [vp]),
    "wrs_b200_sampler_double_buffer": (C.c_int, [vp]),
    "wrs_b200_sampler_implied_masses": (C.c_int, [vp, vp, C.POINTER(f64)]),
    "wrs_b200_sampler_draw_device": (C.c_int, [vp, u64, u64, C.c_uint, vp, vp]),
    "wrs_b200_sampler_stage": (C.c_int, [vp, C.c_char_p, vp, u64, C.POINTER(u64)]),
    "wrs_b200_set_timing": (C.c_int, [C.c_int]),
    "wrs_b200_sampler_stage_times": (C.c_int, [vp, C.POINTER(C.c_float), C.c_int]),
    "wrs_b200_shard_range": (None, [u64, u64, u64, C.POINTER(u64), C.POINTER(u64)]),
    "wrs_b200_shard_counts": (C.c_int, [vp, u64, u64, u64, vp]),
    "wrs_b200_shard_seed": (u64, [u64, u64]),
    "wrs_b200_sampler_draw_shard_device": (C.c_int, [vp, u64, u64, u64, u64, vp, vp]),
    "wrs_b200_sampler_draw_counts": (C.c_int, [vp, u64, u64, C.c_uint, vp, vp, C.POINTER(u64)]),
    "wrs_b200_sampler_draw_philox_device": (C.c_int, [vp, u64, u64, vp, vp]),
    "wrs_b200_two_level_draw_device": (C.c_int, [vp, vp, vp, vp, u64, vp, f64, u64, u64, u64,
                                                 u64, C.c_uint, vp, vp]),
    "wrs_b200_sampler_ipc_handle": (C.c_int, [vp, vp]),
    "wrs_b200_ipc_open": (C.c_int, [vp, C.POINTER(vp)]),
    "wrs_b200_ipc_close": (C.c_int, [vp]),
    "wrs_b200_sampler_draw_counts_device": (C.c_int, [vp, u64, u64, C.c_uint, vp, vp, vp, vp]),
    "wrs_b200_nccl_available": (C.c_int, [C.POINTER(C.c_int)]),
    "wrs_b200_nccl_unique_id": (C.c_int, [vp]),
    "wrs_b200_multi_create": (C.c_int, [vp, u64, u32, u32, vp, C.POINTER(vp)]),
    "wrs_b200_multi_create_local": (C.c_int, [vp, u32, u64, vp]),
    "wrs_b200_multi_set_totals": (C.c_int, [vp, vp]),
    "wrs_b200_multi_exchange": (C.c_int, [vp, vp]),
    "wrs_b200_multi_rebuild_async": (C.c_int, [vp, vp]),
    "wrs_b200_multi_totals": (C.c_int, [vp, vp]),
    "wrs_b200_multi_counts": (C.c_int, [vp, u64, u64, vp]),
    "wrs_b200_multi_draw_device": (C.c_int, [vp, u64, u64, vp, vp, C.POINTER(u64)]),
    "wrs_b200_multi_top_buckets": (C.c_int, [vp, vp, C.POINTER(f64)]),
    "wrs_b200_multi_shard": (vp, [vp]),
    "wrs_b200_multi_free": (None, [vp]),
}

_lib = None


class WrsError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{status_name(status)}: {message}")
        self.status = status
        self.message = message


def lib() -> C.CDLL:
    """Load libwrs_b200.so; raise if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} missing: build it with `make -C paper_1903_00227_b200/csrc` "
                "or __graft_entry__.build(); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def status_name(status: int) -> str:
    return lib().wrs_status_name(status).decode()


def last_error() -> str:
    return lib().wrs_last_error().decode()


def _check(status: int) -> None:
    if status != WRS_OK:
        raise WrsError(status, last_error())


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(vp)


def _dev_ptr(t) -> int:
    """Device pointer of a torch tensor (or an int)."""
    return t if isinstance(t, int) else t.data_ptr()


def _stream_ptr(stream, out=None) -> int | None:
    """cudaStream_t for a call.  With no explicit stream and a torch tensor as
    the output, the tensor's current torch stream is used, so the library's
    writes are ordered with torch's own use (and reuse) of that memory."""
    if stream is None:
        if out is None or not hasattr(out, "device"):
            return None  # the handle's own stream
        import torch
        stream = torch.cuda.current_stream(out.device)
    h = stream if isinstance(stream, int) else stream.cuda_stream
    # torch's default stream is the legacy stream (handle 0); NULL means "the
    # handle's own stream" to the ABI, so name the legacy stream explicitly
    return h if h else CUDA_STREAM_LEGACY


def default_jobs(n: int) -> int:
    return lib().wrs_b200_default_jobs(n)


class Weights:
    """wrs_weights handle (reference capi.cpp:33-35 / WeightTable)."""

    def __init__(self, handle):
        self.h = handle

    @classmethod
    def from_array(cls, w) -> "Weights":
        w = np.ascontiguousarray(w, dtype=np.float64)
        h = vp()
        _check(lib().wrs_weights_from_array(_ptr(w), w.size, C.byref(h)))
        return cls(h)

    @classmethod
    def generate(cls, dist: str, param: float, n: int, seed: int) -> "Weights":
        h = vp()
        _check(lib().wrs_weights_generate(dist.encode(), param, n, seed, C.byref(h)))
        return cls(h)

    @classmethod
    def generate_range(cls, dist: str, param: float, n_total: int, lo: int, hi: int,
                       seed: int) -> "Weights":
        """B200 extension: items [lo, hi) of generate(dist, param, n_total, seed)."""
        h = vp()
        _check(lib().wrs_b200_weights_generate_range(dist.encode(), param, n_total, lo, hi,
                                                     seed, C.byref(h)))
        return cls(h)

    @classmethod
    def read(cls, path: str) -> "Weights":
        h = vp()
        _check(lib().wrs_weights_read(os.fsencode(path), C.byref(h)))
        return cls(h)

    @classmethod
    def from_device(cls, tensor, copy: bool = True) -> "Weights":
        """B200 extension: weights already in HBM (a float64 CUDA tensor)."""
        h = vp()
        _check(lib().wrs_b200_weights_from_device(_dev_ptr(tensor), tensor.numel(),
                                                  1 if copy else 0, C.byref(h)))
        obj = cls(h)
        obj._keepalive = tensor
        return obj

    @classmethod
    def from_device_ptr(cls, ptr: int, n: int, copy: bool = True) -> "Weights":
        """B200 extension: n float64 weights at device address ptr (e.g. a
        slice of another handle's device_ptr()); copy=False borrows them."""
        h = vp()
        _check(lib().wrs_b200_weights_from_device(vp(ptr), n, 1 if copy else 0, C.byref(h)))
        return cls(h)

    def write(self, path: str) -> None:
        _check(lib().wrs_weights_write(self.h, os.fsencode(path)))

    def count(self) -> int:
        return lib().wrs_weights_count(self.h)

    def values(self) -> np.ndarray:
        p = lib().wrs_weights_values(self.h)
        if not p:
            raise WrsError(WRS_EINTERNAL, last_error())
        return np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_double)), (self.count(),)).copy()

    def total(self) -> float:
        return lib().wrs_b200_weights_total(self.h)

    def device_ptr(self) -> int:
        return lib().wrs_b200_weights_device(self.h)

    def free(self) -> None:
        if self.h:
            lib().wrs_weights_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Sampler:
    """wrs_sampler handle (reference capi.cpp:37-49, AliasTable)."""

    def __init__(self, handle, weights: Weights):
        self.h = handle
        self.weights = weights

    @classmethod
    def build(cls, weights: Weights, algo: str = "psa", workers: int = 1, groups: int = 0):
        h = vp()
        _check(lib().wrs_sampler_build(weights.h, algo.encode(), workers, groups, C.byref(h)))
        return cls(h, weights)

    @classmethod
    def build_psa(cls, weights: Weights, jobs: int = 0, keep_workspace: bool = False):
        h = vp()
        _check(lib().wrs_b200_sampler_build_psa(weights.h, jobs,
                                                KEEP_WORKSPACE if keep_workspace else 0,
                                                C.byref(h)))
        return cls(h, weights)

    # reference surface ----------------------------------------------------
    def verify_masses(self, rel_tol: float) -> int:
        return lib().wrs_sampler_verify_masses(self.h, rel_tol)

    def draw(self, seed: int, count: int, workers: int = 1, out: np.ndarray | None = None):
        if out is None:
            out = np.empty(count, np.uint32)
        _check(lib().wrs_sampler_draw(self.h, seed, count, workers, _ptr(out)))
        return out

    def draw_into(self, seed: int, count: int, workers: int, out_ptr: int) -> None:
        """wrs_sampler_draw with a raw pointer (pinned host or device)."""
        _check(lib().wrs_sampler_draw(self.h, seed, count, workers, out_ptr))

    # B200 extensions -------------------------------------------------------
    @property
    def jobs(self) -> int:
        return lib().wrs_b200_sampler_jobs(self.h)

    @property
    def size(self) -> int:
        return lib().wrs_b200_sampler_size(self.h)

    @property
    def bucket_mean(self) -> float:
        return lib().wrs_b200_sampler_bucket_mean(self.h)

    @property
    def total(self) -> float:
        return lib().wrs_b200_sampler_total(self.h)

    def buckets(self) -> np.ndarray:
        out = np.empty(self.size, BUCKET_DTYPE)
        _check(lib().wrs_b200_sampler_copy_buckets(self.h, _ptr(out)))
        return out

    def device_buckets(self) -> int:
        return lib().wrs_b200_sampler_device_buckets(self.h)

    def rebuild_async(self, stream=None) -> None:
        _check(lib().wrs_b200_sampler_rebuild_async(self.h, _stream_ptr(stream)))

    def check(self) -> None:
        _check(lib().wrs_b200_sampler_check(self.h))

    def implied_masses(self) -> tuple[np.ndarray, float]:
        """(per-item implied masses, max relative error vs the weights),
        verify.hpp:43-54, 92-98, computed on the device."""
        out = np.empty(self.size, np.float64)
        worst = f64()
        _check(lib().wrs_b200_sampler_implied_masses(self.h, _ptr(out), C.byref(worst)))
        return out, worst.value

    def double_buffer(self) -> None:
        """wrs_b200_sampler_double_buffer: rebuilds write a second table."""
        _check(lib().wrs_b200_sampler_double_buffer(self.h))

    def draw_device(self, seed: int, count: int, workers: int, out, stream=None) -> None:
        _check(lib().wrs_b200_sampler_draw_device(self.h, seed, count, workers,
                                                  _dev_ptr(out), _stream_ptr(stream, out)))

    def draw_shard_device(self, seed: int, shard: int, count: int, base: int, out,
                          stream=None) -> None:
        _check(lib().wrs_b200_sampler_draw_shard_device(self.h, seed, shard, count, base,
                                                        _dev_ptr(out), _stream_ptr(stream, out)))

    def draw_philox_device(self, seed: int, count: int, out, stream=None) -> None:
        """Philox draw mode (wrs_b200_sampler_draw_philox_device)."""
        _check(lib().wrs_b200_sampler_draw_philox_device(self.h, seed, count, _dev_ptr(out),
                                                         _stream_ptr(stream, out)))

    def draw_counts(self, seed: int, k: int, workers: int = 1) -> tuple[np.ndarray, np.ndarray]:
        """Distinct items of draw(seed, k, workers) (ascending) and their counts."""
        cap = max(min(k, self.size), 1)
        items = np.empty(cap, np.uint32)
        counts = np.empty(cap, np.uint64)
        m = u64()
        _check(lib().wrs_b200_sampler_draw_counts(self.h, seed, k, workers, _ptr(items),
                                                  _ptr(counts), C.byref(m)))
        return items[:m.value], counts[:m.value]

    def draw_counts_device(self, seed: int, k: int, workers: int, items, counts, n_unique,
                           stream=None) -> None:
        """Device outputs (torch int32 / int64 tensors of min(k, n), n_unique: int64[1])."""
        _check(lib().wrs_b200_sampler_draw_counts_device(
            self.h, seed, k, workers, _dev_ptr(items), _dev_ptr(counts), _dev_ptr(n_unique),
            _stream_ptr(stream, items)))

    def stage(self, name: str) -> np.ndarray:
        dtypes = {"counts": np.uint64, "heavy": np.uint32, "light_rank": np.uint32,
                  "heavy_share": np.float64,
                  "light_w": np.float64, "heavy_w": np.float64, "light_prefix": np.float64,
                  "heavy_prefix": np.float64, "light_ckpt": np.float64, "heavy_ckpt": np.float64, "block_totals": np.float64,
                  "carries": np.float64, "split_light": np.uint32, "split_heavy": np.uint32,
                  "split_spill": np.float64}
        nbytes = u64()
        _check(lib().wrs_b200_sampler_stage(self.h, name.encode(), None, 0, C.byref(nbytes)))
        dt = np.dtype(dtypes[name])
        out = np.empty(nbytes.value // dt.itemsize, dt)
        _check(lib().wrs_b200_sampler_stage(self.h, name.encode(), _ptr(out), nbytes.value,
                                            C.byref(nbytes)))
        return out

    def stage_times(self) -> list[float]:
        buf = (C.c_float * 8)()
        k = lib().wrs_b200_sampler_stage_times(self.h, buf, 8)
        return [buf[i] for i in range(k)]

    def free(self) -> None:
        if self.h:
            lib().wrs_sampler_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def nccl_available() -> tuple[bool, int]:
    """(libnccl.so.2 loadable, its version code)."""
    v = C.c_int()
    return bool(lib().wrs_b200_nccl_available(C.byref(v))), v.value


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(lib().wrs_b200_nccl_unique_id(buf))
    return bytes(buf)


class _BorrowedSampler(Sampler):
    """A sampler handle owned by something else (never freed here)."""

    def free(self) -> None:
        self.h = None


class MultiSampler:
    """wrs_b200_multi handle: one rank's part of the C++-owned multi-GPU
    sampler (shard table, NCCL all-gather of the shard totals, top table,
    binomial k-split, this rank's draws with global ids)."""

    def __init__(self, handle, shard: "Weights"):
        self.h = handle
        self.shard_weights = shard
        self.sampler = _BorrowedSampler(lib().wrs_b200_multi_shard(handle), shard)

    @classmethod
    def create(cls, shard: "Weights", n_total: int, rank: int, ranks: int,
               nccl_id: bytes | None) -> "MultiSampler":
        h = vp()
        idp = C.c_char_p(nccl_id) if nccl_id is not None else None
        _check(lib().wrs_b200_multi_create(shard.h, n_total, rank, ranks, idp, C.byref(h)))
        return cls(h, shard)

    @classmethod
    def create_local(cls, shards: list, n_total: int) -> list:
        G = len(shards)
        hs = (vp * G)(*[w.h for w in shards])
        out = (vp * G)()
        _check(lib().wrs_b200_multi_create_local(hs, G, n_total, out))
        return [cls(vp(out[g]), shards[g]) for g in range(G)]

    def set_totals(self, totals) -> None:
        t = np.ascontiguousarray(totals, np.float64)
        _check(lib().wrs_b200_multi_set_totals(self.h, _ptr(t)))

    def exchange(self, stream=None) -> None:
        _check(lib().wrs_b200_multi_exchange(self.h, _stream_ptr(stream)))

    def rebuild_async(self, stream=None) -> None:
        _check(lib().wrs_b200_multi_rebuild_async(self.h, _stream_ptr(stream)))

    def totals(self, ranks: int) -> np.ndarray:
        out = np.empty(ranks, np.float64)
        _check(lib().wrs_b200_multi_totals(self.h, _ptr(out)))
        return out

    def counts(self, seed: int, k: int, ranks: int) -> np.ndarray:
        out = np.empty(ranks, np.uint64)
        _check(lib().wrs_b200_multi_counts(self.h, seed, k, _ptr(out)))
        return out

    def draw_device(self, seed: int, k: int, out, stream=None) -> int:
        c = u64()
        _check(lib().wrs_b200_multi_draw_device(self.h, seed, k, _dev_ptr(out),
                                                _stream_ptr(stream, out), C.byref(c)))
        return c.value

    def top_buckets(self, ranks: int) -> tuple[np.ndarray, float]:
        out = np.empty(ranks, BUCKET_DTYPE)
        m = f64()
        _check(lib().wrs_b200_multi_top_buckets(self.h, _ptr(out), C.byref(m)))
        return out, m.value

    def free(self) -> None:
        if self.h:
            lib().wrs_b200_multi_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def check_failures() -> tuple[int, int]:
    """(device index-check violations so far, first offending line); (-1, 0)
    in the normal build (the checks exist only in libwrs_b200_checked.so)."""
    line = C.c_uint()
    return int(lib().wrs_b200_check_failures(C.byref(line))), line.value


def release_cache() -> int:
    """wrs_b200_release_cache: return the library's cached device buffers."""
    return int(lib().wrs_b200_release_cache())


def set_timing(on: bool) -> None:
    lib().wrs_b200_set_timing(1 if on else 0)


def shard_range(n: int, groups: int, g: int) -> tuple[int, int]:
    lo, hi = u64(), u64()
    lib().wrs_b200_shard_range(n, groups, g, C.byref(lo), C.byref(hi))
    return lo.value, hi.value


def shard_counts(totals, seed: int, k: int) -> np.ndarray:
    t = np.ascontiguousarray(totals, np.float64)
    out = np.empty(t.size, np.uint64)
    _check(lib().wrs_b200_shard_counts(_ptr(t), t.size, seed, k, _ptr(out)))
    return out


def sample_with_replacement(weights: Weights, k: int, seed: int,
                            workers: int = 1) -> tuple[np.ndarray, np.ndarray]:
    """wrs_sample_with_replacement: (items, counts) of k draws, items ascending."""
    n = weights.count()
    cap = max(min(k, n), 1)
    items = np.empty(cap, np.uint32)
    counts = np.empty(cap, np.uint64)
    m = u64()
    _check(lib().wrs_sample_with_replacement(weights.h, k, seed, workers, _ptr(items),
                                             _ptr(counts), C.byref(m)))
    return items[:m.value], counts[:m.value]


def two_level_draw_device(tables, sizes, means, bases, top, top_mean: float, seed: int,
                          q_begin: int, q_end: int, k: int, workers: int, out,
                          stream=None) -> None:
    """wrs_b200_two_level_draw_device: outputs [q_begin, q_end) of
    TwoLevelTable::sample_many(seed, k, workers) into `out` (device).
    `tables` / `top`: device pointers (ints) or CUDA tensors."""
    G = len(tables)
    ptrs = (vp * G)(*[t if isinstance(t, int) else _dev_ptr(t) for t in tables])
    sz = np.ascontiguousarray(sizes, np.uint64)
    mn = np.ascontiguousarray(means, np.float64)
    bs = np.ascontiguousarray(bases, np.uint64)
    tp = top if isinstance(top, int) else _dev_ptr(top)
    _check(lib().wrs_b200_two_level_draw_device(ptrs, _ptr(sz), _ptr(mn), _ptr(bs), G, tp,
                                                top_mean, seed, q_begin, q_end, k, workers,
                                                _dev_ptr(out), _stream_ptr(stream, out)))


def ipc_handle(sampler: "Sampler") -> bytes:
    buf = (C.c_char * 64)()
    _check(lib().wrs_b200_sampler_ipc_handle(sampler.h, buf))
    return bytes(buf)


def ipc_open(handle: bytes) -> int:
    p = vp()
    _check(lib().wrs_b200_ipc_open(C.c_char_p(handle), C.byref(p)))
    return p.value


def ipc_close(ptr: int) -> None:
    _check(lib().wrs_b200_ipc_close(vp(ptr)))


def shard_seed(seed: int, shard: int) -> int:
    return lib().wrs_b200_shard_seed(seed, shard)
