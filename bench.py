#!/usr/bin/env python
"""Benchmark of the hot path: PSA alias-table build + bulk alias sampling.

Workload (BASELINE.json configs[1]): n = 1e8 float64 weights, Uniform(0,1]
from the reference generator with seed 42, resident in HBM; one step =
  (1) a full PSA build over them (K0 total, K1 partition, K2a/b/c compensated
      block scans, K3 split searches, K4 pack -> 16-B buckets), then
  (2) k = 1e9 with-replacement draws (K5) into a device buffer.
value = (n + k) / step time, in G(items+samples)/s, whole job.  The two
halves are reported separately under "build" and "sample" with their own
rooflines.  N > 1 (torchrun): weak scaling -- every rank owns a contiguous
shard of N*1e8 items, builds it, all-gathers the shard totals (NCCL), derives
its sample count from the communication-free binomial split and draws it.

--impl reference: the reference's own CPU implementation (oracle/_ref, i.e.
the unmodified /root/reference headers; the C restatement when that build is
absent) on this host's cores, same metric and config.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_ITEMS = 10**8
K_SAMPLES = 10**9
C2_ITEMS = 10**9    # BASELINE configs[2]
C2_DRAWS = 10**10
SEED = 42
METRIC = "alias build Gitems/s + sample Gsamples/s at 1/2/4/8 B200; % HBM roofline"
UNIT = "G(items+samples)/s"
BUILD_BYTES_PER_ITEM = 72   # SURVEY.md §8(d) minus K0 (W comes with the weights, as the
                            # reference's WeightTable): K1 20 + K2 24 + K4 28
SAMPLE_BYTES_PER_DRAW = 36  # one 32-B sector gather + one 4-B index store
KERNELS_PER_STEP = 10       # build: k_reset_scalars, k_partition_direct, k_carry_ckpt (K2
                            # fused), k_split, k_pack, k_assemble; draw: k_region_scatter
                            # (full tiles + the partial last tile: 1e9 is not a multiple of
                            # 8192), _gather, _unpermute (profiles/r02f_launch_list.txt)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--items", dest="n", type=int, default=N_ITEMS, help="items per GPU")
    ap.add_argument("--draws", dest="k", type=int, default=K_SAMPLES, help="draws per GPU")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-aggregate", action="store_true")
    ap.add_argument("--c2-items", type=int, default=C2_ITEMS, help="configs[2] items in total")
    ap.add_argument("--c2-draws", type=int, default=C2_DRAWS, help="configs[2] draws in total")
    ap.add_argument("--no-config1", action="store_true", help="N > 1: skip configs[1] weak")
    ap.add_argument("--no-config2", action="store_true", help="N = 1: skip configs[2]")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def traffic_per_unit():
    """dram bytes per unit (item / sample) from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock + throttle reasons via NVML during the timed region."""

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons)}


def host_cpu() -> dict:
    """CPU model, sockets, NUMA nodes, physical cores and usable threads of
    this host (stated next to every CPU number)."""
    model, sockets, cores = "unknown", set(), set()
    try:
        phys = None
        for line in open("/proc/cpuinfo"):
            k, _, v = line.partition(":")
            k, v = k.strip(), v.strip()
            if k == "model name" and model == "unknown":
                model = v
            elif k == "physical id":
                phys = v
                sockets.add(v)
            elif k == "core id":
                cores.add((phys, v))
    except OSError:
        pass
    try:
        numa = len([d for d in os.listdir("/sys/devices/system/node") if d.startswith("node")
                    and d[4:].isdigit()])
    except OSError:
        numa = 1
    return {"model": model, "sockets": max(1, len(sockets)), "numa_nodes": max(1, numa),
            "physical_cores": len(cores) or None, "hw_threads": os.cpu_count(),
            "usable_threads": host_threads()}


def host_threads() -> int:
    """std::thread::hardware_concurrency() as this process may use it."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ------------------------------------------------------------- CPU arm
def cpu_reference(n: int, k: int, reps: int, w=None, t1_draws: int = 10**8) -> dict:
    """The reference's CPU path on this host, as BASELINE.md's CPU baseline
    plan states it: the WeightTable is built outside the timed region;
    AliasTable(wt, Build::psa, T) is timed alone (bucket allocation and first
    touch included, alias.hpp:246-257); sample_many(seed, k, T, out) over ALL
    k draws into a pre-sized vector (alias.hpp:271-284); median of `reps`,
    with T = hardware_concurrency.  A T = 1 leg follows: one build and
    t1_draws draws (a bounded sample: a full single-thread 1e9-draw run takes
    about a minute), reported as rates.  Runs oracle/_ref (the unmodified
    reference headers); the C restatement (kind "port", one thread) only
    where that build is absent."""
    import numpy as np
    import oracle
    R = oracle.ref()
    T = host_threads()
    if w is None:
        w = (R or oracle.port()).generate_uniform(n, SEED)
    if R is None:
        P = oracle.port()
        tb, td = [], []
        out = np.empty(k, np.uint32)
        for _ in range(reps):
            t0 = time.perf_counter()
            b, wn = P.psa_build(w, 1)
            tb.append(time.perf_counter() - t0)
            t0 = time.perf_counter()
            P.lib.wo_sample_many(b.ctypes.data, n, wn, SEED, k, 1, out.ctypes.data)
            td.append(time.perf_counter() - t0)
        bs, ds = statistics.median(tb), statistics.median(td)
        return {"kind": "port", "cores": 1, "build_s": bs, "draw_s": ds, "step_s": bs + ds,
                "build_s_all": tb, "draw_s_all": td, "w": w}
    L = R.lib
    wt = L.ref_wt_new(w.ctypes.data, n)  # WeightTable: validation + pairwise total, untimed
    assert wt, "reference WeightTable rejected the weights"
    tb, td = [], []
    h = None
    try:
        for _ in range(reps):
            if h:
                L.ref_table_free(h)
            t0 = time.perf_counter()
            h = L.ref_table_from_wt(wt, T)
            tb.append(time.perf_counter() - t0)
        ob = L.ref_outbuf_new(k)  # pre-sized: allocation and first touch excluded
        try:
            for i in range(reps):
                t0 = time.perf_counter()
                L.ref_table_sample_into(h, SEED + i, k, T, ob)
                td.append(time.perf_counter() - t0)
        finally:
            L.ref_outbuf_free(ob)
        L.ref_table_free(h)
        h = None
        # T = 1: one build, a bounded draw sample
        t0 = time.perf_counter()
        h = L.ref_table_from_wt(wt, 1)
        b1 = time.perf_counter() - t0
        k1 = min(k, t1_draws)
        ob = L.ref_outbuf_new(k1)
        try:
            t0 = time.perf_counter()
            L.ref_table_sample_into(h, SEED, k1, 1, ob)
            d1 = time.perf_counter() - t0
        finally:
            L.ref_outbuf_free(ob)
    finally:
        if h:
            L.ref_table_free(h)
        L.ref_wt_free(wt)
    bs, ds = statistics.median(tb), statistics.median(td)
    return {"kind": "reference", "cores": T, "build_s": bs, "draw_s": ds, "step_s": bs + ds,
            "build_s_all": tb, "draw_s_all": td,
            "t1": {"cores": 1, "build_s": b1, "build_gitems_per_s": n / b1 / 1e9,
                   "draws": k1, "draw_s": d1, "gsamples_per_s": k1 / d1 / 1e9,
                   "sample": f"one AliasTable(wt, psa, 1) over n={n}; sample_many(seed, {k1}, 1)"},
            "w": w}


def cpu_baseline_obj(n: int, k: int, reps: int, d: dict) -> dict:
    T = d["cores"]
    out = {"value": (n + k) / d["step_s"] / 1e9, "unit": UNIT, "cores": T, "kind": d["kind"],
           "host": host_cpu(),
           "sample": (f"median of {reps}: AliasTable(wt, psa, {T}) over n={n} (WeightTable built "
                      f"untimed; bucket allocation + first touch timed, alias.hpp:251) + "
                      f"sample_many(seed, {k}, {T}) into a pre-sized vector -- the full workload, "
                      f"no extrapolation"),
           "build_s": d["build_s"], "draw_s": d["draw_s"],
           "build_gitems_per_s": n / d["build_s"] / 1e9,
           "gsamples_per_s": k / d["draw_s"] / 1e9}
    if "t1" in d:
        out["t1"] = d["t1"]
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # torchrun N>1: rank 0 alone runs the CPU arm
    world = args.gpus
    import oracle
    oracle.build() if not os.path.exists(oracle.PORT_SO) else None
    R = oracle.ref()
    if world == 1:
        # configs[1] in full: n = 1e8 uniform, k = 1e9
        n, k = workload(args)
        w = (R or oracle.port()).generate_uniform(n, SEED)
        cfg, scaling = config_obj(1), "weak"
        data = "synthetic: reference generate_uniform(n, 42)"
        sample = None
    else:
        # configs[2] (n = 1e9 power-law, k = 1e10) as a bounded sample: the
        # reference's own generator at n = 1e8 and k = 1e9 per step (the
        # full configuration takes ~35 s per step on 16 host threads); the
        # metric is a rate, so the sample's rate stands for the whole
        n, k = args.c2_items // 10, args.c2_draws // 10
        w = (R or oracle.port()).generate_powerlaw(n, 1.0, SEED)
        cfg, scaling = config_obj(2, world), "strong"
        data = "synthetic: reference generate_powerlaw(1e8, 1.0, 42) (bounded sample of configs[2])"
        sample = (f"bounded sample of configs[2]: AliasTable(generate_powerlaw({n}, 1.0, 42), "
                  f"psa, T) + sample_many({k}) per step (the full n=1e9 / k=1e10 at this rate)")
    # one "step" = build + all k draws, median over the timed steps; the
    # warm-up steps run the same work untimed
    if args.warmup:
        cpu_reference(n, k, 1, w=w, t1_draws=0)
    d = cpu_reference(n, k, max(1, args.steps), w=w)
    d.pop("w")
    value = (n + k) / d["step_s"] / 1e9
    cb = cpu_baseline_obj(n, k, max(1, args.steps), d)
    if sample:
        cb["sample"] = sample
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": d["step_s"] * 1e3,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": data, "config": cfg, "cpu_baseline": cb,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def workload(args) -> tuple[int, int]:
    return args.n, args.k


def config_obj(which: int, world: int = 1) -> dict:
    """The same keys in both arms (the driver compares them)."""
    if which == 1:
        return {"workload": "BASELINE configs[1]: n=1e8 uniform(0,1] f64 per GPU, psa build + "
                            "1e9 with-replacement draws per GPU",
                "n_per_gpu": N_ITEMS, "k_per_gpu": K_SAMPLES,
                "parallelism": f"shard{world}" if world > 1 else "single",
                "l2": "no flush: weights 0.8 GB, table 1.6 GB, output 4 GB > 126 MB L2"}
    return {"workload": "BASELINE configs[2]: n=1e9 power-law s=1 f64 (reference generator, "
                        "shuffled, seed 42) sharded contiguously over the GPUs; per-shard psa "
                        "tables + top table over the shard totals; 1e10 with-replacement draws "
                        "split multinomially across the GPUs (strong scaling)",
            "n_total": C2_ITEMS, "k_total": C2_DRAWS, "parallelism": f"shard{world}",
            "l2": "no flush: weights 8 GB, tables 16 GB, output 40 GB in total > 126 MB L2"}


# ------------------------------------------------------------- GPU arm
class Ctx:
    """What every GPU leg needs: torch, the library, the rank layout."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist

        import paper_1903_00227_b200 as wrs
        self.args, self.torch, self.dist, self.wrs = args, torch, dist, wrs
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.backend = os.environ.get("WRS_BENCH_BACKEND", "nccl")  # gloo: 1-GPU smoke of N>1
        if self.backend != "nccl":
            self.local %= torch.cuda.device_count()
        torch.cuda.set_device(self.local)
        if self.world > 1:
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            else:
                dist.init_process_group(self.backend)
        self.dev = torch.device("cuda", self.local)
        self.stream = torch.cuda.Stream(self.dev)

    def timed(self, fn, reps):
        """mean device ms of fn() on the stream, each call bracketed by events"""
        torch = self.torch
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(reps)]
        torch.cuda.synchronize()
        for a, b in evs:
            with torch.cuda.stream(self.stream):
                a.record(self.stream)
                fn()
                b.record(self.stream)
        torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in evs) / reps

    def max_over_ranks(self, vals):
        if self.world == 1:
            return list(vals)
        torch = self.torch
        mdev = self.dev if self.backend == "nccl" else torch.device("cpu")
        m = torch.tensor(list(vals), dtype=torch.float64, device=mdev)
        self.dist.all_reduce(m, op=self.dist.ReduceOp.MAX)
        return m.tolist()

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()


def rooflines(n_local, k_local, build_ms, draw_ms):
    hbm, hbm_kind = peaks()
    tr = traffic_per_unit()
    build_gbs = BUILD_BYTES_PER_ITEM * n_local / (build_ms * 1e-3) / 1e9
    draw_gbs = SAMPLE_BYTES_PER_DRAW * k_local / (draw_ms * 1e-3) / 1e9

    def traffic(key, units):
        v = tr.get(key)
        return None if v is None else v * units

    build = {"gitems_per_s": n_local / (build_ms * 1e-3) / 1e9, "ms": build_ms,
             "roofline": {"bound": "hbm", "achieved": build_gbs, "peak": hbm,
                          "peak_kind": hbm_kind, "unit": "GB/s", "frac": build_gbs / hbm,
                          "bytes_per_item": BUILD_BYTES_PER_ITEM,
                          "traffic": traffic("build_bytes_per_item", n_local)}}
    draw = {"bound": "hbm",
            "kernel": "draw stage: k_region_scatter + k_region_gather + k_region_unpermute",
            "achieved": draw_gbs, "peak": hbm, "peak_kind": hbm_kind, "unit": "GB/s",
            "frac": draw_gbs / hbm, "bytes_per_sample": SAMPLE_BYTES_PER_DRAW,
            "traffic": traffic("draw_bytes_per_sample", k_local)}
    return build, draw


def config1(ctx, weak_world: int):
    """BASELINE configs[1] (n = 1e8 uniform, k = 1e9 per GPU).  weak_world > 1:
    every rank owns a shard of weak_world * 1e8 items and draws its share of
    weak_world * 1e9 (weak scaling; totals gathered with torch.distributed)."""
    args, torch, wrs = ctx.args, ctx.torch, ctx.wrs
    world, rank, stream = weak_world, ctx.rank, ctx.stream
    n_total, k_total = args.n * world, args.k * world
    lo, hi = wrs.shard_range(n_total, world, rank)
    W = wrs.Weights.generate_range("uniform", 0.0, n_total, lo, hi, SEED)
    n_local = hi - lo
    if world > 1:
        from paper_1903_00227_b200.sharded import ShardedSampler
        shard = ShardedSampler(W, n_total, rank, world)
        S = shard.sampler
        cap = int(shard.counts(SEED, k_total).max()) + 1024
    else:
        shard = None
        S = wrs.Sampler.build(W, "psa", 1)
        cap = args.k
    out = torch.empty(cap, dtype=torch.int32, device=ctx.dev)

    def step():
        with torch.cuda.stream(stream):
            # rebuild on the library's high-priority stream (ordered behind
            # `stream`), then the draw (its scatter, which does not read the
            # table, may overlap the rebuild with WRS_B200_SIDE_SCATTER=1;
            # measured no faster, so the default runs it after)
            S.rebuild_async(stream)
            if shard is not None:
                from paper_1903_00227_b200.sharded import default_gather
                shard.totals = default_gather(W.total())
                return shard.draw_device(SEED, k_total, out, stream)
            S.draw_device(SEED, args.k, 1, out, stream)
            return args.k

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    S.check()
    # isolated halves for the rooflines (not the headline): build alone, the
    # per-kernel stage breakdown, draws alone against a fixed table
    build_ms = ctx.timed(lambda: S.rebuild_async(stream), max(args.steps, 3))
    wrs.set_timing(True)
    S.rebuild_async(stream)
    torch.cuda.synchronize()
    stage_ms = S.stage_times()
    wrs.set_timing(False)
    S.rebuild_async(stream)  # re-arm the untimed path
    if shard is None:
        draw_ms = ctx.timed(lambda: S.draw_device(SEED, args.k, 1, out, stream), max(args.steps, 3))
    else:
        draw_ms = ctx.timed(lambda: shard.draw_device(SEED, k_total, out, stream),
                            max(args.steps, 3))
    S.check()

    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.barrier()
    torch.cuda.synchronize()
    with ClockSampler(ctx.local) as clocks:
        t0.record(stream)
        for _ in range(args.steps):
            step()
        t1.record(stream)
        torch.cuda.synchronize()
    ctx.barrier()
    S.check()
    ms_step = t0.elapsed_time(t1) / args.steps
    ms_step, build_ms, draw_ms = ctx.max_over_ranks([ms_step, build_ms, draw_ms])
    build, draw_roof = rooflines(n_local, k_total / world, build_ms, draw_ms)
    build["jobs"] = S.jobs
    build["stages_ms"] = dict(zip(["K1_partition", "K2a_block_totals", "K2b_carries",
                                   "K2c_prefix_checkpoints", "K3_splits", "K4a_pack",
                                   "K4b_assemble"], [round(x, 4) for x in stage_ms]))
    res = {
        "value": (n_total + k_total) / (ms_step * 1e-3) / 1e9, "ms_per_step": ms_step,
        "scaling": "weak", "config": config_obj(1, world),
        "data": "synthetic: reference generate_uniform(n_total, 42) generated on device",
        "overlap": "each step = rebuild then draw, stream-ordered; build/sample below are "
                   "each timed alone",
        "build": build,
        "sample": {"gsamples_per_s": k_total / world / (draw_ms * 1e-3) / 1e9, "ms": draw_ms},
        "roofline": draw_roof,
        "gpu_launches": KERNELS_PER_STEP * args.steps,
        "clocks": clocks.summary(),
    }
    del out, S, shard, W
    torch.cuda.synchronize()
    wrs.release_cache()
    return res


def draw_launches(k: int) -> int:
    """Draw kernels of one k-draw call (region plan, 8192-draw tiles): per
    region pass a scatter (+ a one-CTA launch for a partial last tile), a
    gather and an unpermute; passes as sample_kernels.cu draw_chunk_for makes
    them (equal passes of up to 3.5e9 draws beyond 2^30)."""
    if k <= 1 << 30:
        passes = [k]
    else:
        p = -(-k // 3_500_000_000)
        c = -(-k // p)
        passes = [c] * (p - 1) + [k - c * (p - 1)]
    return sum(3 + (1 if c % 8192 else 0) for c in passes)


def config2(ctx):
    """BASELINE configs[2]: n = 1e9 power-law s = 1 weights (the reference
    generator: (i+1)^-1 dealt by its Fisher-Yates, seed 42), sharded
    contiguously over the N ranks; k = 1e10 draws split multinomially across
    the ranks -- strong scaling, the north star's multi-GPU target.  One step
    = every rank rebuilds its shard table, the shard totals are all-gathered
    over NCCL by the library (wrs_b200_multi_exchange), every rank derives
    the same k-split and draws its share from its own table (global ids)."""
    args, torch, wrs = ctx.args, ctx.torch, ctx.wrs
    from paper_1903_00227_b200.sharded import multi_create
    world, rank, stream = ctx.world, ctx.rank, ctx.stream
    n_total, k_total = args.c2_items, args.c2_draws
    lo, hi = wrs.shard_range(n_total, world, rank)
    W = wrs.Weights.generate_range("powerlaw", 1.0, n_total, lo, hi, SEED)
    wrs.release_cache()
    M = multi_create(W, n_total, rank, world)
    nccl = M.has_comm
    counts = M.counts(SEED, k_total, world)
    out = torch.empty(max(int(counts.max()), 1), dtype=torch.int32, device=ctx.dev)

    def step():
        with torch.cuda.stream(stream):
            M.rebuild_async(stream)
            if nccl:
                M.exchange(stream)  # ncclAllGather of the G shard totals
            return M.draw_device(SEED, k_total, out, stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    M.sampler.check()
    build_ms = ctx.timed(lambda: M.rebuild_async(stream), max(args.steps, 3))
    draw_ms = ctx.timed(lambda: M.draw_device(SEED, k_total, out, stream), max(args.steps, 3))
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.barrier()
    torch.cuda.synchronize()
    k_mine = 0
    with ClockSampler(ctx.local) as clocks:
        t0.record(stream)
        for _ in range(args.steps):
            k_mine += step()
        t1.record(stream)
        torch.cuda.synchronize()
    ctx.barrier()
    M.sampler.check()
    ms_step = t0.elapsed_time(t1) / args.steps
    ms_step, build_ms, draw_ms = ctx.max_over_ranks([ms_step, build_ms, draw_ms])
    build, draw_roof = rooflines(hi - lo, int(counts.max()), build_ms, draw_ms)
    res = {
        "value": (n_total + k_total) / (ms_step * 1e-3) / 1e9, "ms_per_step": ms_step,
        "scaling": "strong", "config": config_obj(2, world),
        "data": "synthetic: reference generate_powerlaw(1e9, 1.0, 42) (device deal, bit-exact)",
        "exchange": "wrs_b200_multi_exchange: ncclAllGather of the shard totals (library-owned "
                    "communicator)" if nccl else "totals gathered by torch.distributed",
        "per_rank": {"items": hi - lo, "draws_max": int(counts.max()), "draws_min": int(counts.min()),
                     "build_ms_max": build_ms, "draw_ms_max": draw_ms,
                     "build": build, "draw_roofline": draw_roof},
        "gpu_launches": (6 + draw_launches(int(counts.max())) + (1 if nccl else 0)) * args.steps,
        "clocks": clocks.summary(),
    }
    del out
    M.free()
    W.free()
    torch.cuda.synchronize()
    wrs.release_cache()
    return res


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    ctx = Ctx(args)
    world, rank = ctx.world, ctx.rank
    head = {"metric": METRIC, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "vs_baseline": None, "dtype": "f64"}
    if world == 1:
        # N = 1: BASELINE configs[1], the configuration the roofline targets
        # are stated on; configs[2] on this one GPU is the strong-scaling
        # curve's first point ("config2")
        result = dict(head, **config1(ctx, 1))
        if not args.no_config2:
            result["config2"] = config2(ctx)
    else:
        # N > 1: BASELINE configs[2], strong scaling over the N ranks (the
        # north star's multi-GPU target); configs[1] weak scaling beside it
        result = dict(head, **config2(ctx))
        if not args.no_config1:
            result["config1_weak"] = config1(ctx, world)
    lo, hi = ctx.wrs.shard_range(args.n * world, world, rank)

    # ---- aggregated draws (BASELINE configs[3] shape, on this GPU) ------------
    if world == 1 and not args.no_aggregate:
        result["aggregate"] = aggregate(args, ctx.wrs, ctx.torch, ctx.dev, ctx.stream)

    # ---- end to end through the C ABI with host buffers ---------------------
    if not args.no_e2e:
        if world == 1:
            result["e2e"] = e2e(args, ctx.wrs, ctx.torch, world, rank, lo, hi, args.n, args.k)
        else:
            result["e2e"] = e2e_multi(ctx)

    if rank == 0 and world == 1 and not args.no_cpu:
        # the reference on this host's cores: 3 builds + 3 full k-draw runs
        # (~10 s on 16 threads) and the T = 1 leg (~10 s)
        d = cpu_reference(args.n, args.k, 3)
        d.pop("w")
        result["cpu_baseline"] = cpu_baseline_obj(args.n, args.k, 3, d)
    if world > 1:
        ctx.dist.barrier()
        ctx.dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result))


def e2e_multi(ctx):
    """configs[2] end to end at N ranks through the public API with host
    buffers: every step each rank copies its shard of the weights from pinned
    host memory (wrs_weights_from_array), builds its multi-GPU handle (shard
    table; the totals gathered with the caller's process group), draws its
    share of k and copies it back to pinned host memory.  Max over ranks."""
    args, torch, wrs = ctx.args, ctx.torch, ctx.wrs
    from paper_1903_00227_b200.sharded import default_gather
    world, rank = ctx.world, ctx.rank
    n_total, k_total = args.c2_items, args.c2_draws
    lo, hi = wrs.shard_range(n_total, world, rank)
    Wd = wrs.Weights.generate_range("powerlaw", 1.0, n_total, lo, hi, SEED)
    host_w = torch.empty(hi - lo, dtype=torch.float64, pin_memory=True)
    host_w.numpy()[:] = Wd.values()
    totals = default_gather(Wd.total())
    Wd.free()
    wrs.release_cache()
    cnt = int(wrs.shard_counts(totals, SEED, k_total)[rank])
    host_out = torch.empty(max(cnt, 1), dtype=torch.int32, pin_memory=True)
    dev_out = torch.empty(max(cnt, 1), dtype=torch.int32, device=ctx.dev)
    times = []
    for i in range(1 + max(1, min(args.steps, 3))):
        ctx.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        W = wrs.Weights.from_array(host_w.numpy())
        M = wrs.MultiSampler.create(W, n_total, rank, world, None)
        M.set_totals(default_gather(W.total()))
        M.draw_device(SEED, k_total, dev_out, ctx.stream)
        with torch.cuda.stream(ctx.stream):
            host_out.copy_(dev_out, non_blocking=True)
        ctx.stream.synchronize()
        checksum = int(host_out[-1])
        t1 = time.perf_counter()
        M.free()
        W.free()
        if i:
            times.append(t1 - t0)
    sec = ctx.max_over_ranks([statistics.median(times)])[0]
    return {"value": (n_total + k_total) / sec / 1e9, "unit": UNIT,
            "h2d_bytes_per_step": 8 * (hi - lo), "d2h_bytes_per_step": 4 * cnt,
            "ms_per_step": sec * 1e3,
            "api": "wrs_weights_from_array + wrs_b200_multi_create/set_totals + "
                   "wrs_b200_multi_draw_device + D2H", "checksum_last": checksum}


def aggregate(args, wrs, torch, dev, stream):
    """BASELINE configs[3] on one GPU: n lognormal(0, 2) weights, k draws
    aggregated to (item, count) pairs (wrs_b200_sampler_draw_counts_device):
    the same alias draws as the main line, counted instead of written."""
    n, k = args.n, args.k
    W = wrs.Weights.generate("lognormal", 2.0, n, SEED)  # common.cuh, restated in the oracle
    S = wrs.Sampler.build(W, "psa", 1)
    cap = min(n, k)
    items = torch.empty(cap, dtype=torch.int32, device=dev)
    counts = torch.empty(cap, dtype=torch.int64, device=dev)
    m = torch.zeros(1, dtype=torch.int64, device=dev)
    for _ in range(2):
        S.draw_counts_device(SEED, k, 1, items, counts, m, stream)
    torch.cuda.synchronize()
    reps = max(args.steps, 3)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        S.draw_counts_device(SEED, k, 1, items, counts, m, stream)
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    nu = int(m.item())
    assert int(counts[:nu].sum()) == k
    return {"workload": "BASELINE configs[3] on 1 GPU: n=%d lognormal(0,2) f64 weights "
                        "(the library's Box-Muller generator on RngStream(seed, 'logn'), seed %d; "
                        "oracle twin wo_generate_lognormal), k=%d draws -> (item, count) pairs"
                        % (n, SEED, k),
            "gsamples_per_s": k / (ms * 1e-3) / 1e9, "ms": ms, "n_unique": nu,
            "gpu_launches": 8}


def e2e(args, wrs, torch, world, rank, lo, hi, n_total, k_total):
    """wrs_weights_from_array(host) -> wrs_sampler_build("psa") ->
    wrs_sampler_draw(host out): every step copies the weights H2D and the
    draws D2H (pinned host memory), allocations included."""
    import numpy as np
    n = hi - lo
    Wd = wrs.Weights.generate_range("uniform", 0.0, n_total, lo, hi, SEED)
    host_w = torch.empty(n, dtype=torch.float64, pin_memory=True)
    host_w.numpy()[:] = Wd.values()
    Wd.free()
    k = args.k
    host_out = torch.empty(k, dtype=torch.int32, pin_memory=True)
    steps = max(1, min(args.steps, 5))
    times, phases = [], []
    for i in range(1 + steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        W = wrs.Weights.from_array(host_w.numpy())
        ta = time.perf_counter()
        S = wrs.Sampler.build(W, "psa", 1)
        tb = time.perf_counter()
        S.draw_into(SEED, k, 1, host_out.data_ptr())
        checksum = int(host_out[-1])  # the step's result read on the host
        t1 = time.perf_counter()
        S.free()
        W.free()
        if i:
            times.append(t1 - t0)
            phases.append((ta - t0, tb - ta, t1 - tb))
    serial = statistics.median(times)
    ph = phases[times.index(serial)] if serial in times else phases[-1]
    sec, lanes_ms = e2e_lanes(wrs, torch, host_w, k, steps, checksum)
    if world > 1:
        import torch.distributed as dist
        tdev = "cuda" if dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor([sec, serial], dtype=torch.float64, device=tdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sec, serial = (float(x) for x in t.tolist())
    return {"value": (n_total + k * world) / sec / 1e9, "unit": UNIT,
            "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 4 * k, "ms_per_step": sec * 1e3,
            "api": "wrs_weights_from_array + wrs_sampler_build(psa) + wrs_sampler_draw",
            "pipeline": "2 host threads, each running whole steps (upload, build, draw + "
                        "download, free) through the C ABI with its own pinned output; one "
                        "lane's weight upload overlaps the other's draw download (PCIe is full "
                        "duplex); value = all steps / wall time of both lanes",
            "lane_steps_ms": lanes_ms,  # [upload, build, draw+download, free]
            "serial": {"value": (n_total + k * world) / serial / 1e9, "ms_per_step": serial * 1e3,
                       "phases_ms": {"weights_from_array_h2d": ph[0] * 1e3,
                                     "build": ph[1] * 1e3, "draw_d2h": ph[2] * 1e3}},
            "checksum_last": checksum}


def e2e_lanes(wrs, torch, host_w, k, steps, checksum):
    """The e2e step sequence on two host threads ("lanes"); ctypes releases
    the GIL for each call and the library frees a lane's buffers after
    synchronising only that lane's streams, so the lanes overlap.  Lane 1
    starts once lane 0's first upload returned, so the uploads interleave
    with the other lane's downloads.  Every step's last draw is checked
    against the serial run's (same seed, same weights)."""
    import threading
    per_lane = [2, max(8, steps)]  # warm-up round, timed round (8: the start-up
    # upload and the drain of the last download spread over 16 steps)
    outs = [torch.empty(k, dtype=torch.int32, pin_memory=True) for _ in range(2)]
    start = threading.Barrier(2)
    uploaded = threading.Event()
    lane_ms = [[], []]
    errors = []

    def lane(j, steps):
        try:
            out = outs[j]
            start.wait()
            if j:
                uploaded.wait()
            for _ in range(steps):
                t = [time.perf_counter()]
                W = wrs.Weights.from_array(host_w.numpy())
                uploaded.set()
                t.append(time.perf_counter())
                S = wrs.Sampler.build(W, "psa", 1)
                t.append(time.perf_counter())
                S.draw_into(SEED, k, 1, out.data_ptr())
                if int(out[-1]) != checksum:
                    raise RuntimeError("lane %d: draw differs from the serial run" % j)
                t.append(time.perf_counter())
                S.free()
                W.free()
                t.append(time.perf_counter())
                # (upload, build, draw + download, free) per step
                lane_ms[j].append([round((b - a) * 1e3, 2) for a, b in zip(t, t[1:])])
        except BaseException as e:  # surfaced below
            errors.append(e)
            uploaded.set()

    # one untimed round to warm both lanes' allocations
    for timed in (False, True):
        ths = [threading.Thread(target=lane, args=(j, per_lane[timed])) for j in range(2)]
        uploaded.clear()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        t1 = time.perf_counter()
        if errors:
            raise errors[0]
        if not timed:
            for ms in lane_ms:
                ms.clear()
    return (t1 - t0) / (2 * per_lane[1]), lane_ms


if __name__ == "__main__":
    main()
