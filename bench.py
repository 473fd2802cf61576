#!/usr/bin/env python3
"""Benchmark of the enumeration hot path (one JSON line on stdout, rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl reference]

A *step* is one complete search of the workload's example set: every cost level is enumerated on the device
until the minimal separating formula is found (or the cost cap is hit).

* N = 1 (default): BASELINE.json's second configuration -- "the paper's running example with the default cost
  function" -- which SURVEY.md section 8(d) maps onto the paper's 7+7-trace LTL example (``spec2``: 142,066,187
  candidates, 16,258,320 unique CMs, witness of cost 16).
* N > 1: ONE search sharded over the N GPUs (owner-sharded dedup set, candidates routed to their hash owners,
  paper_2504_18943_b200/dist.py): strong scaling, so the default workload is one with seconds of work,
  ``c3-16`` (BASELINE configs[2]'s example set exhaustively to cost 16); the line also carries the same search on
  ONE GPU of the same box (``single_gpu``), so every N > 1 line is a self-contained scaling point.
  Without torchrun's environment ``--gpus N`` starts the N ranks itself (torch.distributed.run, 127.0.0.1).

Numbers on the line:

* ``value``         unique CMs per second, device-resident: the specification is already on the GPU, K searches are
                    timed with CUDA events on the engine's stream (max over ranks);
* ``e2e``           the same metric through the public API ``synthesize(spec, config)`` with host inputs, a fresh
                    store per step, host<->device copies (counted by the handle that ran the search) and the
                    witness read-back inside the timed region (wall clock, max over ranks);
* ``roofline``      the construction+dedup kernels: algorithmic bytes over their CUDA-event time,
                    against the measured HBM copy peak;
* ``cpu_baseline``  the reference's own CPU implementation (``oracle/_ref``: the unmodified ``ltlsynth`` package,
                    installed there by ``__graft_entry__.build()``; else the C port ``oracle/ltl_oracle.c``) timed on
                    this host on a bounded sample of the same workload;
* ``workloads``     (N = 1) BASELINE configs[2], [3], [4] in short device-resident runs: ``c3-fill`` (<= 128-bit CMs
                    until the set cannot grow), ``c4-1024`` (1024-bit CMs), ``c5-12`` (LTL, 128-byte CMs, cost 12) and
                    ``c5-fill`` (the same until the device is full: cost 13, 536 M CMs).

``--impl reference`` times the reference's CPU implementation alone (rank 0; the other ranks exit).
Only that leg and ``cpu_baseline`` touch ``oracle/``; the measured product path never does.
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "unique_cs_per_s"
UNIT = "unique CS/s"
# per workload: cost cap and mode of the GPU search; `sample_cost` = cost cap of the bounded CPU sample
# (chosen so that one CPU step takes seconds); `base` = the example set when the name is a variant
WORKLOADS = {
    "spec2": dict(max_cost=16, exhaustive=False, sample_cost=13),
    "c3": dict(max_cost=13, exhaustive=True, sample_cost=11),
    # BASELINE configs[2]: "<= 128-bit CS, enumerated until the cache fills HBM on 1 GPU": cost 17 stores 639 M CMs;
    # cost 18 would need a hash set beyond 2^32 slots and ends the run with "memory budget exhausted"
    "c3-fill": dict(max_cost=18, exhaustive=True, sample_cost=11, base="c3"),
    "c3-16": dict(max_cost=16, exhaustive=True, sample_cost=11, base="c3"),
    "c1": dict(max_cost=14, exhaustive=False, sample_cost=14),
    "spec1": dict(max_cost=10, exhaustive=True, sample_cost=10),
    "c5": dict(max_cost=10, exhaustive=True, sample_cost=9),
    "c5-12": dict(max_cost=12, exhaustive=True, sample_cost=9, base="c5"),
    # BASELINE configs[4] until the device is full: cost 13 stores 536.5 M CMs of 128 bytes (68.7 GB of rows, 114 GB in
    # all); cost 14 would need a hash set beyond 2^32 slots and ends the run with "memory budget exhausted"
    "c5-fill": dict(max_cost=14, exhaustive=True, sample_cost=9, base="c5"),
    "c4-512": dict(max_cost=10, exhaustive=True, sample_cost=9),
    "c4-1024": dict(max_cost=10, exhaustive=True, sample_cost=9),
    "c4-1024-11": dict(max_cost=11, exhaustive=True, sample_cost=9, base="c4-1024"),
}
DEFAULT_WORKLOAD = {1: "spec2"}
DEFAULT_SHARDED_WORKLOAD = "c3-16"
EXTRA_WORKLOADS = ("c3-fill", "c4-1024-11", "c5-12", "c5-fill")
# regex front-end (BASELINE configs[1]-[3] as literally worded): name -> exhaustive levels built
# (re-c2 is BASELINE configs[2] "enumerated until the cache fills": cost 20 stores 352 M sequences; cost 21 would need
# a hash set beyond 2^32 slots and ends the run with "memory budget exhausted", like c3-fill / c5-fill)
REGEX_WORKLOADS = {"re-email": 13, "re-c2": 21, "re-c3": 13}
OPERATORS = "not,next,future,and,until"


def regex_arm(name: str, max_cost: int, seed: int, device: int, steps: int, warmup: int) -> dict:
    """One regex workload of the `workloads` table: exhaustive levels 1..max_cost through the regex front-end's store
    (paper_2504_18943_b200.regex.RegexStore), host wall clock around the level loop (every level ends with a
    device-to-host read of its counters)."""
    import torch

    from paper_2504_18943_b200 import regex as rx
    from paper_2504_18943_b200.workloads import regex_workload

    spec = regex_workload(name, seed)
    times, unique, constructed, stats = [], 0, 0, None
    for it in range(warmup + steps):
        store = rx.RegexStore(spec, device=device)
        try:
            torch.cuda.synchronize(device)
            t0 = time.perf_counter()
            unique = constructed = reached = 0
            sizes = []
            for c in range(1, max_cost + 1):
                status, n_new, _, built = store.expand(c, exhaustive=True)
                unique, constructed = unique + n_new, constructed + built
                sizes.append(n_new)
                if status != 0:
                    break
                reached = c
            torch.cuda.synchronize(device)
            if it >= warmup:
                times.append(time.perf_counter() - t0)
            stats, n_bits, entries = store.device_stats(), store.ix.n_bits, len(store.ix.splits)
        finally:
            store.close()
    ms = 1e3 * sum(times) / len(times)
    # the same byte count per candidate as for LTL; the unary operators (? and *) read every stored row but
    # those of the last level once each.  The concatenation is bound by its integer work, not by these bytes (DESIGN 11).
    level_sizes = [lv for lv in sizes]
    alg = algorithmic_bytes(stats["key_bytes"], constructed, unique, 2 * sum(level_sizes[:-1]))
    peak, _ = measured_peaks()
    frac = alg / (stats["enumerate_ms"] * 1e-3) / 1e9 / peak if stats["enumerate_ms"] > 0 else None
    return {"ms_per_step": ms, "roofline_frac": frac, "unique_per_s": unique / (ms * 1e-3), "constructed_per_s": constructed / (ms * 1e-3),
            "unique_per_step": unique, "constructed_per_step": constructed, "max_cost_reached": reached,
            "cs_bits": n_bits, "guide_entries": entries, "cm_bytes": stats["row_bytes"], "device_bytes": stats["device_bytes"],
            "kernel_ms_per_step": stats["enumerate_ms"], "finalize_ms_per_step": stats["finalize_ms"], "steps": steps, "warmup": warmup,
            "grammar": "regex (literal, ?, *, concatenation, union; unit costs); parity unpinned: the reference has no regex synthesiser"}


def measured_peaks() -> tuple[float, str]:
    path = ROOT / "MEASURED_PEAKS.json"
    if path.exists():
        return float(json.loads(path.read_text())["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)"
    return 6650.0, "fallback of B200_PROFILING.md (MEASURED_PEAKS.json absent)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._pump, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _pump(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()

    def summary(self) -> dict:
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[2:]) if v.lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def algorithmic_bytes(key_bytes: int, constructed: int, unique: int, unary_candidates: int) -> float:
    """B_cand = K*(r + 1 + 2u) + P*u, summed over the run's candidates.
    r = 1 for unary candidates (one operand row read each), ~0 for tiled binary ones;
    P = 8 (the winning ordinal this engine stores per entry)."""
    return key_bytes * (unary_candidates + constructed + 2 * unique) + 8 * unique


def workload_config(name: str, seed: int) -> dict:
    wl = WORKLOADS[name]
    return {"workload": name, "seed": seed, "operators": OPERATORS, "max_cost": wl["max_cost"], "exhaustive": wl["exhaustive"]}


# ---- the reference's CPU implementation -------------------------------------------------------------------------

def cpu_reference(name: str, seed: int, repeats: int, warmup: int) -> dict:
    """Times the reference's CPU enumerator on a bounded sample of workload `name` (cost cap `sample_cost`):
    `warmup` untimed runs, then `repeats` timed ones.  oracle/_ref (the unmodified reference, all host threads:
    its own benchmark protocol, pkg/scripts/benchmark_throughput.py:28-40) when it is installed, else the
    single-core C port.  -> dict(kind, cores, times, unique, constructed, sample)."""
    from paper_2504_18943_b200 import workloads

    wl = WORKLOADS[name]
    spec = workloads.named_workload(wl.get("base", name), seed)
    ref_dir = ROOT / "oracle" / "_ref"
    times, unique, constructed = [], 0, 0
    if (ref_dir / "ltlsynth" / "engine.py").exists():
        sys.path.insert(0, str(ref_dir))
        try:
            import ltlsynth
            from paper_2504_18943_b200.traces import serialize_specification

            rspec = ltlsynth.parse_specification(serialize_specification(spec))
            cores = os.cpu_count() or 1
            cfg = ltlsynth.EngineConfig(max_cost=wl["sample_cost"], exhaustive=wl["exhaustive"], threads=cores,
                                        time_budget_s=3600.0, memory_budget_mb=1 << 20)
            for step in range(warmup + repeats):
                t0 = time.perf_counter()
                res = ltlsynth.synthesize(rspec, cfg)
                if step >= warmup:
                    times.append(time.perf_counter() - t0)
                unique, constructed = res.stats.unique, res.stats.constructed
            kind, what = "reference", f"oracle/_ref: unmodified ltlsynth {getattr(ltlsynth, '__version__', '0.1.0')}, threads={cores}"
        finally:
            sys.path.remove(str(ref_dir))
    else:
        import oracle

        oracle.build()
        cores = 1
        for step in range(warmup + repeats):
            t0 = time.perf_counter()
            res = oracle.synthesize(spec, max_cost=wl["sample_cost"], exhaustive=wl["exhaustive"], time_budget_s=3600.0,
                                    memory_budget_mb=1 << 20)
            if step >= warmup:
                times.append(time.perf_counter() - t0)
            unique, constructed = res.unique, res.constructed
        kind, what = "port", "oracle/ltl_oracle.c on one host core (oracle/_ref is not installed)"
    sample = (f"{name} cost levels 1..{wl['sample_cost']} of {wl['max_cost']}: {constructed} candidates, {unique} unique CMs "
              f"per step ({what})")
    return dict(kind=kind, cores=cores, times=times, unique=unique, constructed=constructed, sample=sample)


def run_reference(args, rank: int) -> int:
    if rank != 0:
        return 0
    ref = cpu_reference(args.workload, args.seed, args.steps, args.warmup)
    per_step = sum(ref["times"]) / len(ref["times"])
    value = ref["unique"] / per_step
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": workload_config(args.workload, args.seed),
        "constructed_per_s": ref["constructed"] / per_step,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": ref["cores"], "kind": ref["kind"], "sample": ref["sample"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# ---- launching N ranks ----------------------------------------------------------------------------------------

def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def respawn_under_torchrun(args) -> int:
    """`bench.py --gpus N` outside torchrun: start the N ranks here (one process per GPU) and pass their output on."""
    if not getattr(args, "selftest_cpu", False):
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:  # say so in the line's own format instead of N tracebacks from the ranks
            print(json.dumps({"metric": METRIC, "n_gpus": args.gpus, "error": f"--gpus {args.gpus} needs {args.gpus} CUDA devices, this box has {have}"}))
            return 1
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), str(ROOT / "bench.py"), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "WARN")
    return subprocess.call(cmd, env=env)


# ---- one device-resident measurement ---------------------------------------------------------------------------

def search_loop(store, cfg, expand):
    """One search on a store that is already on the device -> (stats, (separator id, cost) or None)."""
    from paper_2504_18943_b200 import engine

    store.reset()
    stats, found = engine.RunStats(), None
    stats.levels_built = 0  # (levels whose candidates were constructed: a level that ran out of memory is not one)
    for cost in range(1, cfg.max_cost + 1):
        stats.max_cost_reached = cost
        try:
            _, sep = expand(store, cost, cfg, stats)
        except engine._BudgetExceeded:  # the cache filled the device: the search ends here (outcome "exhausted")
            break
        stats.levels_built = cost
        if sep is not None and found is None:
            found = (sep, cost)
            if not cfg.exhaustive:
                break
    return stats, found


def device_arm(name, seed, device, stream, steps, warmup, expand, sync, clocks_index=None):
    """K searches of workload `name`, specification resident in HBM, timed with CUDA events on `stream`."""
    import torch

    from paper_2504_18943_b200 import engine, workloads

    wl = WORKLOADS[name]
    spec = workloads.named_workload(wl.get("base", name), seed)
    cfg = engine.EngineConfig(max_cost=wl["max_cost"], exhaustive=wl["exhaustive"], time_budget_s=3600.0,
                              memory_budget_mb=1 << 20, device=device)
    store = engine.CandidateStore(spec, device=device, stream=stream.cuda_stream)
    try:
        for _ in range(warmup):
            stats, found = search_loop(store, cfg, expand)
        before = store.device_stats()
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sync()
        sampler = ClockSampler(clocks_index) if clocks_index is not None else None
        if sampler:
            sampler.__enter__()
        start.record(stream)
        for _ in range(steps):
            stats, found = search_loop(store, cfg, expand)
        stop.record(stream)
        sync()
        if sampler:
            sampler.__exit__()
        after = store.device_stats()
        out = dict(spec=spec, cfg=cfg, stats=stats, found=found, device_ms=start.elapsed_time(stop), before=before, after=after,
                   clocks=sampler.summary() if sampler else None, levels=[store.level(c).n for c in range(1, stats.levels_built + 1)])
        out["witness"] = None
        if found:
            from paper_2504_18943_b200 import to_text

            out["witness"] = to_text(engine.reconstruct(store, found[0]), spec.alphabet)
        return out
    finally:
        store.close()


def kernel_numbers(arm, steps) -> dict:
    """Per-step kernel figures of a device arm and the roofline fraction of its construction+dedup kernels."""
    before, after, stats = arm["before"], arm["after"], arm["stats"]
    enum_ms = (after["enumerate_ms"] - before["enumerate_ms"]) / steps
    unary = 3 * sum(arm["levels"][:-1])  # not, next, future over every level but the last
    alg = algorithmic_bytes(after["key_bytes"], stats.constructed, stats.unique, unary)
    peak, peak_src = measured_peaks()
    achieved = alg / (enum_ms * 1e-3) / 1e9 if enum_ms > 0 else 0.0
    return dict(enum_ms=enum_ms, fin_ms=(after["finalize_ms"] - before["finalize_ms"]) / steps,
                tiny_ms=(after.get("tiny_ms", 0.0) - before.get("tiny_ms", 0.0)) / steps,
                enum_launches=(after["enumerate_launches"] - before["enumerate_launches"]) // steps,
                launches=(after["kernel_launches"] - before["kernel_launches"]) // steps,
                alg_bytes=alg, achieved=achieved, peak=peak, peak_src=peak_src, frac=achieved / peak)


def main() -> int:
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS))
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the `workloads` table (N = 1)")
    ap.add_argument("--selftest-cpu", action="store_true",
                    help="launch check without GPUs: the sharded protocol over gloo with the numpy shard engine of tests/")
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")

    under_launcher = "WORLD_SIZE" in os.environ and "RANK" in os.environ
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        args.workload = args.workload or "spec2"
        return run_reference(args, rank)
    if args.gpus > 1 and not under_launcher:
        return respawn_under_torchrun(args)
    if under_launcher and world != args.gpus:
        if rank == 0:
            print(f"bench.py: --gpus {args.gpus} but the launcher started {world} ranks; measuring {world}", file=sys.stderr)
    if args.selftest_cpu:
        return selftest_cpu(args, rank, world)
    args.warmup = max(args.warmup, 3)
    args.workload = args.workload or (DEFAULT_WORKLOAD[1] if world == 1 else DEFAULT_SHARDED_WORKLOAD)

    import torch
    import torch.distributed as dist

    from paper_2504_18943_b200 import _native, engine, to_text, workloads
    from paper_2504_18943_b200 import dist as pdist
    from paper_2504_18943_b200.traces import smallest_lane_dtype

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device: the engine has no CPU path")
    torch.cuda.set_device(local_rank)
    distributed = world > 1
    if distributed:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    def barrier():
        if distributed:
            dist.barrier()
        torch.cuda.synchronize()

    def reduce_over_ranks(x: float, op) -> float:
        if not distributed:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=op)
        return float(t.item())

    stream = torch.cuda.current_stream()
    single = lambda store, cost, cfg, stats: engine.expand_level(store, cost, cfg.operators, config=cfg, stats=stats)
    sharded = lambda store, cost, cfg, stats: pdist.sharded_expand_level(store, cost, cfg.operators, cfg, stats)

    # ---- device-resident arm
    arm = device_arm(args.workload, args.seed, local_rank, stream, args.steps, args.warmup, sharded if distributed else single,
                     barrier, clocks_index=local_rank)
    device_ms = reduce_over_ranks(arm["device_ms"], dist.ReduceOp.MAX if distributed else None)
    spec, cfg, stats = arm["spec"], arm["cfg"], arm["stats"]
    k = kernel_numbers(arm, args.steps)
    launches = int(reduce_over_ranks(float(k["launches"]), dist.ReduceOp.SUM if distributed else None))

    # ---- end-to-end arm: public API, host inputs, fresh store per step; the copies are counted by the handle
    run_api = (lambda: pdist.synthesize_sharded(spec, cfg)) if distributed else (lambda: engine.synthesize(spec, cfg))
    for _ in range(2):
        res = run_api()
    barrier()
    h2d = d2h = 0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        res = run_api()
        h2d += res.device_stats["h2d_bytes"]
        d2h += res.device_stats["d2h_bytes"]
    torch.cuda.synchronize()
    e2e_s = reduce_over_ranks(time.perf_counter() - t0, dist.ReduceOp.MAX if distributed else None)

    # ---- N > 1: the same search on ONE GPU of this box (rank 0 alone), so that the line is a scaling point by itself
    single_gpu = None
    if distributed:
        if rank == 0:
            one = device_arm(args.workload, args.seed, local_rank, stream, max(1, min(args.steps, 3)), 1, single, torch.cuda.synchronize)
            n1 = max(1, min(args.steps, 3))
            single_gpu = {"ms_per_step": one["device_ms"] / n1, "value": one["stats"].unique * n1 / (one["device_ms"] * 1e-3),
                          "unit": UNIT, "steps": n1, "unique_per_step": one["stats"].unique}
        barrier()

    extra = None
    if not distributed and not args.no_extra and args.workload == DEFAULT_WORKLOAD[1]:
        extra = {}
        for name in EXTRA_WORKLOADS:
            _native.load().ltlb200_trim(local_rank)
            try:
                a = device_arm(name, args.seed, local_rank, stream, 2, 2, single, torch.cuda.synchronize)
            except Exception as err:  # noqa: BLE001  (a workload that does not fit this device is reported, not fatal)
                extra[name] = {"error": str(err)[:200]}
                continue
            kk = kernel_numbers(a, 2)
            extra[name] = {"ms_per_step": a["device_ms"] / 2, "unique_per_s": a["stats"].unique * 2 / (a["device_ms"] * 1e-3),
                           "constructed_per_s": a["stats"].constructed * 2 / (a["device_ms"] * 1e-3),
                           "unique_per_step": a["stats"].unique, "constructed_per_step": a["stats"].constructed,
                           "max_cost_reached": a["stats"].max_cost_reached, "cm_bytes": a["after"]["row_bytes"],
                           "device_bytes": a["after"]["device_bytes"], "kernel_ms_per_step": kk["enum_ms"],
                           "finalize_ms_per_step": kk["fin_ms"], "tiny_levels_ms_per_step": kk["tiny_ms"],
                           "roofline_frac": kk["frac"], "steps": 2, "warmup": 2}
        for name, max_cost in REGEX_WORKLOADS.items():
            _native.load().ltlb200_trim(local_rank)
            try:
                extra[name] = regex_arm(name, max_cost, args.seed, local_rank, 2, 2)
            except Exception as err:  # noqa: BLE001
                extra[name] = {"error": str(err)[:200]}
        _native.load().ltlb200_trim(local_rank)

    if rank != 0:
        if distributed:
            dist.destroy_process_group()
        return 0

    after = arm["after"]
    key_bytes, table_slots, device_bytes = after["key_bytes"], after["table_slots"], after["device_bytes"]
    slot_bytes = 32 if key_bytes == 16 else 8
    # DRAM bytes the enumerate kernels actually moved in one search: from the committed ncu pass of
    # this workload (dram__bytes_read.sum + dram__bytes_write.sum summed over the enumerate launches)
    traffic, traffic_src = None, None
    profs = sorted((ROOT / "profiles").glob(f"r*_dram_{args.workload}.json"))  # the latest committed pass
    if profs:
        pj = json.loads(profs[-1].read_text())
        traffic, traffic_src = pj["enumerate_dram_bytes"], f"profiles/{profs[-1].name} (bytes per search over {pj['enumerate_launches']} enumerate launches)"
    # measured ceiling of the probe's access pattern on this device (random 32-byte slots, 256-bit loads)
    probe = None
    tool = ROOT / "tools" / "random_probe_bench"
    if tool.exists() and not distributed:
        try:
            mb = max(128, int(table_slots * slot_bytes >> 20))
            out = subprocess.run([str(tool), str(mb)], capture_output=True, text=True, timeout=60).stdout
            rates = [float(line.split(":")[1].split()[0]) for line in out.splitlines() if "probes/ns" in line]
            if rates:
                probe = {"table_mb": mb, "ceiling_probes_per_ns": max(rates),
                         "kernel_candidates_per_ns": stats.constructed / (k["enum_ms"] * 1e6) if k["enum_ms"] > 0 else None}
        except (OSError, subprocess.SubprocessError, ValueError):
            probe = None
    config = workload_config(args.workload, args.seed)
    config.update({
        "cm_bytes": after["row_bytes"],
        "parallelism": (f"one search over {world} GPUs: pair space tile-sharded, dedup set owner-sharded, per level one NCCL "
                        "all-to-all of candidate records to their hash owners, one all-reduce of the winners bitmap, one "
                        "all-gather of the winners") if distributed else "single GPU",
        "l2": f"working set {device_bytes >> 20} MiB (hash set {table_slots * slot_bytes >> 20} MiB) exceeds the 126 MB L2; no flush needed",
    })
    lane = "lane_bits"
    kernel_name = (f"narrow_level_kernel<{lane}, op> + narrow_small_level_kernel<{lane}> (construction + separation check + hash-set dedup)"
                   if key_bytes == 16 else
                   f"wide2_level_kernel<{lane}, op> + wide2_small_level_kernel<{lane}> (construction + separation check + hash-set dedup)")
    if distributed:
        kernel_name = ("narrow_route_kernel + narrow_probe_kernel" if key_bytes == 16 else "wide2_route_kernel + wide_import_kernel") + \
            " (construction + routing to hash owners; owner-side dedup)"
    line = {
        "metric": METRIC,
        "value": stats.unique * args.steps / (device_ms * 1e-3),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": device_ms / args.steps,
        "higher_is_better": True,
        "scaling": "strong" if distributed else "weak",
        "vs_baseline": None,
        "dtype": "u%d" % (8 * smallest_lane_dtype(spec.max_length).itemsize),
        "data": "synthetic",
        "config": config,
        "time_to_solution_ms": device_ms / args.steps,
        "constructed_per_s": stats.constructed * args.steps / (device_ms * 1e-3),
        "unique_per_step": stats.unique,
        "constructed_per_step": stats.constructed,
        "witness": arm["witness"],
        "e2e": {
            "value": stats.unique * args.steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d // args.steps),
            "d2h_bytes_per_step": int(d2h // args.steps), "time_to_solution_ms": 1e3 * e2e_s / args.steps,
            "api": ("paper_2504_18943_b200.dist.synthesize_sharded(spec, EngineConfig)" if distributed
                    else "paper_2504_18943_b200.engine.synthesize(spec, EngineConfig)"),
            "bytes_source": "ltlb200_stats.h2d_bytes / d2h_bytes of the handles that ran the timed searches",
            "witness": to_text(res.formula, spec.alphabet) if res.formula is not None else None,
        },
        "gpu_launches": int(launches * args.steps),
        "clocks": arm["clocks"],
        "roofline": {
            "bound": "hbm", "achieved": k["achieved"], "peak": k["peak"], "unit": "GB/s", "frac": k["frac"],
            "traffic": traffic, "kernel": kernel_name,
            "launches_per_step": int(k["enum_launches"]), "kernel_ms_per_step": k["enum_ms"], "finalize_ms_per_step": k["fin_ms"],
            "tiny_levels_ms_per_step": k["tiny_ms"],
            "algorithmic_bytes_per_step": k["alg_bytes"], "peak_source": k["peak_src"],
            "traffic_source": traffic_src,
            "random_probe": probe,
            "note": "the dedup probe is one random 32-byte sector per candidate; the ceiling for that access pattern "
                    "(tools/random_probe_bench.cu, 37-40 probes/ns = 1.2 TB/s of useful sectors for 2-8 GiB tables) is "
                    "what bounds the kernel, not the copy bandwidth used as `peak`",
        },
    }
    if single_gpu is not None:
        line["single_gpu"] = single_gpu
    if extra is not None:
        line["workloads"] = extra
    if not args.no_cpu_baseline:
        ref = cpu_reference(args.workload, args.seed, 3, 1)  # one warm-up, best of three (the reference's own protocol)
        best = min(ref["times"])
        line["cpu_baseline"] = {
            "value": ref["unique"] / best, "unit": UNIT, "cores": ref["cores"], "kind": ref["kind"],
            "constructed_per_s": ref["constructed"] / best,
            "sample": ref["sample"] + f", best of 3 = {best:.2f} s",
        }
    print(json.dumps(line), flush=True)
    if distributed:
        dist.destroy_process_group()
    return 0


def selftest_cpu(args, rank: int, world: int) -> int:
    """`bench.py --gpus N --selftest-cpu`: proves that the launch path starts N ranks and that they run the sharded
    protocol together -- gloo instead of NCCL, the numpy shard engine of tests/ instead of the CUDA engine.
    Not a measurement: the line says so."""
    import torch.distributed as dist

    sys.path.insert(0, str(ROOT / "tests"))
    from cpu_shard_engine import CpuShardEngine

    from paper_2504_18943_b200 import dist as pdist
    from paper_2504_18943_b200 import engine, to_text, workloads

    if world > 1:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("gloo", rank=0, world_size=1, init_method=f"tcp://127.0.0.1:{free_port()}")
    pdist.REPLICATE_BELOW = 0
    spec = workloads.spec1()
    t0 = time.perf_counter()
    res = pdist.synthesize_sharded(spec, engine.EngineConfig(), store_factory=CpuShardEngine)
    elapsed = time.perf_counter() - t0
    pids = [None] * world
    dist.all_gather_object(pids, os.getpid())
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"impl": "selftest-cpu-shards", "n_gpus": world, "processes": len(set(pids)), "backend": "gloo",
                          "witness": to_text(res.formula, spec.alphabet), "unique_per_step": res.stats.unique,
                          "ms_per_step": 1e3 * elapsed, "note": "launch check, not a measurement"}), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
