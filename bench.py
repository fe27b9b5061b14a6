#!/usr/bin/env python3
"""Benchmark: subsets expanded/sec and time-to-reset-threshold of the exact
bidirectional-BFS search on random binary n=300 (BASELINE.json configs[2]).

One "step" = one exact solve of the workload automaton through the C-ABI
(sw_solve_exact).  `value` = engine expansions (Σ k·|L| over the
list steps + Σ k·|slice| over DFS levels — identical integers for the GPU and
the reference) ÷ the engine's device time (CUDA events on the engine's stream,
heuristic bound R supplied so the hot path is isolated).  `e2e` = the same
metric through the public call with host buffers and the adaptive heuristic
included (solve_exact(aut) from a host transition table, result word read back).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1 (torchrun): ONE solve of the workload partitioned over the N GPUs by hash
ownership (sw_solve_exact_dist over NCCL) — `value` is the job's
expansions over the max-over-ranks device time (strong scaling).
--impl reference: the reference's own CPU engine (oracle/_ref, built from
/root/reference) on the same workload, bounded samples, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = "random:300,2,0"
METRIC = "subsets expanded/sec"
UNIT = "subsets/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", default=WORKLOAD)
    p.add_argument("--cpu-seconds", type=float, default=20.0,
                   help="bounded CPU-baseline sample (seconds of reference engine work)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-ref-full", action="store_true",
                   help="skip the one complete reference solve (time to threshold, ~2 min)")
    return p.parse_args()


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device),
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 5 + i and s[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ------------------------------------------------------------ distributed
def dist_setup(gpus: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(world, x: float) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(world, x: float) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


# ------------------------------------------------------------ frontier exchange (N>1)
def exchange_probe(n: int, world: int, rank: int, rows: int = 1 << 20, reps: int = 3):
    """Hash-ownership exchange of one generated level (SURVEY §8(e),
    distributed.owner_exchange_dedupe): every rank holds `rows` sets at the
    frontier density (drawn from one shared pool, so duplicates span ranks),
    regroups them by owner on the device, ONE NCCL all-to-all carries them to
    their owners, the owners dedupe.  Reported: max-over-ranks device time and
    the bytes that crossed NVLink (rows sent to other ranks x (8W+4))."""
    import numpy as np
    import torch
    from paper_2207_05495_b200 import distributed, native as sw
    W = sw.W(n)
    pool_rng = np.random.default_rng(12345)
    pool = pool_rng.integers(0, 2**63, size=(rows, W), dtype=np.int64).view(np.uint64)
    for _ in range(3):  # density ~1/16 per bit
        pool &= pool_rng.integers(0, 2**63, size=(rows, W), dtype=np.int64).view(np.uint64) << np.uint64(1)
    if n % 64:
        pool[:, -1] &= ~np.uint64(0) << np.uint64(64 - n % 64)
    mine = pool[np.random.default_rng(rank + 1).integers(0, rows, rows)]
    cards = np.bitwise_count(mine).sum(axis=1).astype(np.int32)
    tw = torch.from_numpy(mine.reshape(-1).view(np.int64).copy()).cuda()
    tc = torch.from_numpy(cards).cuda()
    distributed.owner_exchange_dedupe(n, tw, tc)  # warm-up (NCCL channels, pools)
    times, sent, kept = [], 0, 0
    for _ in range(reps):
        barrier(world)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ow, oc, sent = distributed.owner_exchange_dedupe(n, tw, tc)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        kept = oc.numel()
    ms = max_over_ranks(world, statistics.median(times))
    total_sent = sum_over_ranks(world, float(sent))
    return {"rows_per_rank": rows, "ms": ms, "nvlink_bytes_per_rank": sent,
            "nvlink_bytes_total": total_sent,
            "nvlink_gbs": total_sent / (ms / 1e3) / 1e9 if ms > 0 else None,
            "kept_total": sum_over_ranks(world, float(kept)),
            "note": "device partition + NCCL all_to_all_single (counts, rows, cards) + owner "
                    "hash dedupe, CUDA events on the current stream, max over ranks"}


# ------------------------------------------------------------ cpu baseline
def reference_sample(spec: str, upper_bound: int, seconds: float):
    """The reference's own engine (oracle/_ref) on a bounded prefix of the
    workload: (expansions, seconds, iterations, status)."""
    from oracle import ref as R
    kind, _, args = spec.partition(":")
    n, k, seed = (int(x) for x in args.split(","))
    d = R.random_automaton(n, k, seed)
    t = time.perf_counter()
    s = R.solve_instrumented(n, k, d, upper_bound=upper_bound, max_seconds=seconds)
    wall = time.perf_counter() - t
    return s.expansions_phase1 + s.expansions_dfs, s.engine_seconds or wall, s.iterations, s.status


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def reference_full_solve(spec: str):
    """One complete reference solve_exact (heuristic included, the CLI's timed
    region, tools/synchro.cpp:210-212): (seconds, threshold)."""
    from oracle import ref as R
    kind, _, args = spec.partition(":")
    n, k, seed = (int(x) for x in args.split(","))
    d = R.random_automaton(n, k, seed)
    t = time.perf_counter()
    s = R.solve_exact(n, k, d)
    return time.perf_counter() - t, s.threshold


def cpu_baseline(spec, upper_bound, seconds, full=True):
    e, s, it, st = reference_sample(spec, upper_bound, seconds)
    out = {"value": e / s if s > 0 else None, "unit": UNIT, "cores": 1, "kind": "reference",
           "sample": (f"PREFIX of the workload: reference solve_exact engine (oracle/_ref, -O3) "
                      f"on {spec} with upper_bound={upper_bound}, first {it} iterations in "
                      f"{s:.1f} s ({'complete' if st == 0 else 'stopped at the sample budget'}; "
                      f"no DFS phase) — its rate exceeds the full solve's, so ratios against it "
                      f"are lower bounds; single-threaded by construction (SPEC.md:418); "
                      f"host {cpu_model()}")}
    if full:
        wall, thr = reference_full_solve(spec)
        out["time_to_threshold_s"] = wall
        out["time_to_threshold_note"] = (f"one complete reference solve_exact of {spec} "
                                         f"(heuristic + engine, threshold {thr}) on the same host")
    return out


# -------------------------------------------------------------- our arm
def flush_l2(dev: int):
    import torch
    buf = getattr(flush_l2, "buf", None)
    if buf is None:
        buf = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{dev}")
        flush_l2.buf = buf
    buf.zero_()
    torch.cuda.synchronize(dev)


def run_ours(args, world, rank, local):
    import torch
    from paper_2207_05495_b200 import native as sw
    if sw.device_count() < 1:
        raise SystemExit("no CUDA device: the B200 data plane has no CPU fallback")
    torch.cuda.set_device(local)
    aut = sw.from_spec(args.workload)
    nvlink = []
    if world > 1:
        # ONE partitioned solve over the N GPUs (hash ownership):
        # NCCL communicator, per-level all-to-all to the owners, all-gathers
        # for containment, all-reduced statistics, DFS shares + MIN.
        from paper_2207_05495_b200 import distributed
        comm = distributed.make_comm("nccl")

        def solve(**kw):
            r, sent = distributed.solve_exact_partitioned(aut, comm, device=local, **kw)
            nvlink.append(sent)
            return r
    else:
        def solve(**kw):
            return sw.solve_exact(aut, device=local, **kw)
    # Heuristic bound R once (the reference computes the same R, bit-identical).
    R = solve().upper_bound
    W = (aut.n + 63) // 64
    exp_bytes_per_child = 8 * W / aut.k + 8 * W + 4  # parent/k + child + card

    for _ in range(max(3, args.warmup)):
        solve(upper_bound=R, timing=True)

    flush_l2(local)
    barrier(world)
    torch.cuda.synchronize()
    results = []
    nvlink.clear()
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush_l2(local)  # between timed steps: L2 flushed (device time excludes the flush)
            results.append(solve(upper_bound=R, timing=True))
    torch.cuda.synchronize()
    barrier(world)
    dev_s = sum(r.engine_device_ms for r in results) / 1e3
    dev_s_max = max_over_ranks(world, dev_s)
    expansions = results[0].expansions
    # the partitioned solve reports global counts on every rank: the job's units
    total_units = float(sum(r.expansions for r in results))
    value = total_units / dev_s_max
    nvlink_sent = sum_over_ranks(world, float(sum(nvlink))) / max(1, args.steps) if world > 1 else 0
    launches = sum(r.kernel_launches for r in results)
    exp_children = sum(r.expansions for r in results)
    exp_ms = sum(r.expand_kernel_ms for r in results)
    for r in results:
        assert r.threshold == results[0].threshold

    # e2e: public call, host transition table in, threshold + word out, heuristic included.
    e2e = []
    for _ in range(2):  # untimed warm-up of the public path (first use of the heuristic kernels)
        solve(track_word=True)
    for _ in range(max(1, min(args.steps, 3))):
        flush_l2(local)
        barrier(world)
        t = time.perf_counter()
        r = solve(track_word=True)
        e2e.append((time.perf_counter() - t, r))
    e2e_s = max_over_ranks(world, sum(x[0] for x in e2e))
    e2e_units = float(sum(x[1].expansions for x in e2e))
    last = e2e[-1][1]
    assert last.word is not None and len(last.word) == last.threshold and sw.is_reset_word(aut, last.word)

    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    roof_peak = json.load(open(peaks_path))["hbm_gbs"] if os.path.exists(peaks_path) else 6650.0
    peak_src = ("MEASURED_PEAKS.json hbm_gbs (measured copy, burst)" if os.path.exists(peaks_path)
                else "fallback 6650 GB/s (B200_PROFILING.md)")
    achieved = exp_children * exp_bytes_per_child / (exp_ms / 1e3) / 1e9 if exp_ms > 0 else None
    engine_ms = sum(r.engine_device_ms for r in results)
    cont_ms = sum(r.contain_kernel_ms for r in results)
    cont_bytes = sum(r.contain_bytes for r in results)
    cont_gbs = cont_bytes / (cont_ms / 1e3) / 1e9 if cont_ms > 0 else None
    # HBM-scale microbenchmarks of the north-star kernels (2^24
    # random subsets at the measured frontier density, under the workload automaton).
    mb_count, mb_density = 1 << 24, 0.077
    mb_exp_ms = sw.bench_expand(aut, mb_count, mb_density, seed=1, inverse=False, iters=5)
    mb_pre_ms = sw.bench_expand(aut, mb_count, mb_density, seed=1, inverse=True, iters=5)
    mb_exp_gbs = mb_count * aut.k * exp_bytes_per_child / (mb_exp_ms / 1e3) / 1e9
    mb_pre_gbs = mb_count * aut.k * exp_bytes_per_child / (mb_pre_ms / 1e3) / 1e9
    dd_ms, dd_unique = sw.bench_dedupe(aut.n, mb_count, mb_density, seed=1, dup_fraction=0.1, iters=3)
    ls_ms, _ = sw.bench_dedupe(aut.n, mb_count, mb_density, seed=1, dup_fraction=0.1, iters=2,
                               lex_sort=True)
    # Containment as work rather than bytes: one untimed solve with
    # the traversal counters on; node visits + range-scan pair tests per second of
    # the timed traversal, against the INT32 logic ceiling.
    cs = solve(upper_bound=R, contain_stats=True)
    cont_ms_solve = cont_ms / len(results)
    logic_rate = ((cs.contain_visits + cs.contain_pairs) / (cont_ms_solve / 1e3)
                  if cont_ms_solve > 0 else None)
    logic_ceiling = 148 * 128 * 1.965e9 / 10  # SMs x INT32 lanes x clock / ~10 LOP3 per W=5 test
    row = 8 * W + 4
    dd_bytes = mb_count * row + dd_unique * row
    traffic = dram_traffic(W, cont_bytes / len(results))  # read every candidate once + write survivors once
    dd_gbs = dd_bytes / (dd_ms / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": dev_s_max * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (SplitMix64 random automaton, automaton.hpp:159-164)",
        "config": arm_config(args.workload, aut.n, aut.k, R, world, results[0].threshold,
                             expansions),
        "time_to_threshold_s": statistics.median(x[0] for x in e2e),
        "engine_time_s": dev_s_max / args.steps,
        "e2e": {"value": e2e_units / e2e_s, "unit": UNIT,
                "h2d_bytes_per_step": int(statistics.mean(x[1].h2d_bytes for x in e2e)),
                "d2h_bytes_per_step": int(statistics.mean(x[1].d2h_bytes for x in e2e)),
                "time_to_threshold_s": statistics.median(x[0] for x in e2e),
                "note": "sw_solve_exact from a host delta table, adaptive heuristic included, "
                        "word read back and verified"},
        # Dominant kernel of the step: the containment traversal (self-reduction,
        # meet check, DFS queries).  Algorithmic bytes = every key and query row
        # read once; it is a latency-bound tree walk (ncu: L1/TEX-throughput bound,
        # profiles/), so its HBM fraction is small by nature.
        "roofline": {"bound": "hbm", "kernel": "containment traversal (contain_pool_kernel marking "
                                                "+ trie_pool_kernel existence queries)",
                     "achieved": cont_gbs, "peak": roof_peak, "unit": "GB/s",
                     "frac": (cont_gbs / roof_peak) if cont_gbs else None,
                     "traffic": traffic["contain"], "traffic_note": traffic["contain_note"],
                     "share_of_step": cont_ms / engine_ms if engine_ms else None,
                     "bytes_per_unit": f"{row} B per key/query row", "peak_source": peak_src,
                     "logic": {"unit": "node visits + pair tests /s", "achieved": logic_rate,
                               "ceiling": logic_ceiling,
                               "frac": logic_rate / logic_ceiling if logic_rate else None,
                               "visits_per_solve": cs.contain_visits,
                               "pair_tests_per_solve": cs.contain_pairs,
                               "ceiling_source": "SURVEY §8(d): 148 SMs x 128 INT32 ops/clk x "
                                                 "1.965 GHz / ~10 LOP3 per W=5 pair test"}},
        # North-star kernels at HBM scale (2^24 parents, n=300, density 0.077).
        "roofline_expand": {"bound": "hbm", "kernel": "expand_sliced_kernel",
                            "achieved": mb_exp_gbs, "achieved_preimage": mb_pre_gbs,
                            "peak": roof_peak, "unit": "GB/s", "frac": mb_exp_gbs / roof_peak,
                            "frac_preimage": mb_pre_gbs / roof_peak,
                            "bytes_per_unit": exp_bytes_per_child,
                            "ms_per_launch": mb_exp_ms, "children_per_launch": mb_count * aut.k,
                            "traffic": traffic["expand"],
                            "traffic_preimage": traffic["expand_preimage"],
                            "algorithmic_bytes_per_launch": mb_count * aut.k * exp_bytes_per_child,
                            "in_engine_achieved": achieved,
                            "in_engine_share_of_step": exp_ms / engine_ms if engine_ms else None},
        "roofline_dedupe": {"bound": "hbm", "kernel": "dd_single_kernel (one pass: hash claim in a "
                                                       "32-bit L2-sized table + warp-tile block "
                                                       "reservation; untagged frontier dedupe)",
                            "achieved": dd_gbs, "peak": roof_peak, "unit": "GB/s",
                            "frac": dd_gbs / roof_peak, "ms_per_call": dd_ms,
                            "traffic": traffic["dedupe"], "algorithmic_bytes_per_launch": dd_bytes,
                            "sets": mb_count, "unique": dd_unique,
                            "lex_sort_dedupe_ms": ls_ms,
                            "lex_sort_dedupe_frac": dd_bytes / (ls_ms / 1e3) / 1e9 / roof_peak,
                            "bytes_per_unit": f"{row} B read per candidate + {row} B per survivor"},
        "gpu_launches": launches,
    }
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.workload, R, args.cpu_seconds,
                                            full=not args.no_ref_full)
        if line["cpu_baseline"].get("time_to_threshold_s"):
            line["e2e"]["vs_reference_time_to_threshold"] = (
                line["cpu_baseline"]["time_to_threshold_s"] / line["e2e"]["time_to_threshold_s"])
    if world > 1:
        line["nvlink_bytes_per_solve"] = nvlink_sent
        line["nvlink_gbs"] = nvlink_sent / (dev_s_max / args.steps) / 1e9 if dev_s_max else None
        try:
            line["exchange"] = exchange_probe(aut.n, world, rank)
        except Exception as e:  # the partitioned-solve numbers above stand on their own
            line["exchange"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    line["clocks"] = clocks.summary()
    if rank == 0:
        print(json.dumps(line), flush=True)


def dram_traffic(W, cont_bytes_per_solve):
    """roofline.traffic: DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per
    launch from the committed ncu captures of the same kernels on the same workload
    (profiles/r01_dram_traffic.json, made by scripts/traffic_summary.py), or None."""
    path = os.path.join(ROOT, "profiles", "r02_dram_traffic.json")
    if not os.path.exists(path):
        path = os.path.join(ROOT, "profiles", "r01_dram_traffic.json")
    out = {"contain": None, "contain_note": None, "expand": None, "expand_preimage": None,
           "dedupe": None}
    if not os.path.exists(path):
        return out
    t = json.load(open(path))
    # the containment traversal: radix-tree marking + trie existence queries
    cont = [v for k, v in t.items()
            if k.startswith(f"contain_pool_kernel<{W},") or f"trie_pool_kernel<{W}," in k]
    if cont:
        launches = sum(v["launches"] for v in cont)
        tb = sum(v["traffic_bytes_per_launch"] * v["launches"] for v in cont)
        out["contain"] = tb / launches
        out["contain_note"] = (f"ncu over one solve's {launches} traversal launches "
                               f"({cont[0]['source']}); algorithmic bytes per launch "
                               f"{cont_bytes_per_solve / launches:.3g}")
    for key, name in (("expand", f"expand_sliced_kernel<{W}, 0, 1>"),
                      ("expand_preimage", f"expand_sliced_kernel<{W}, 1, 1>"),
                      ("dedupe", f"dd_single_kernel<{W}")):
        hit = [v for k, v in t.items() if name in k]
        if hit:
            out[key] = hit[0]["traffic_bytes_per_launch"]
    return out


def arm_config(workload, n, k, R, world, threshold=None, expansions=None):
    """The `config` both arms print (the driver compares the arms on it)."""
    if threshold is None or expansions is None:  # bit-identical across implementations
        gold = os.path.join(ROOT, "tests", "golden", "solve_" + workload.replace("random:", "random_")
                            .replace(",", "_") + ".json")
        if os.path.exists(gold):
            g = json.load(open(gold))
            threshold = g["threshold"]
            expansions = g["expansions_phase1"] + g["expansions_dfs"]
    return {"workload": f"{workload} exact solve (engine; heuristic bound R={R} precomputed, "
                        "bit-identical to the reference's)",
            "n": n, "k": k, "threshold": threshold, "expansions_per_solve": expansions,
            "l2": "flushed between timed steps (512 MiB write; device time excludes it)",
            "parallelism": (f"one solve partitioned over {world} GPUs by hash ownership (NCCL)"
                            if world > 1 else "single GPU")}


def run_reference(args, world, rank):
    if rank != 0:
        return
    from oracle import ref as R
    if not R.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    kind, _, rest = args.workload.partition(":")
    n, k, seed = (int(x) for x in rest.split(","))
    d = R.random_automaton(n, k, seed)
    ub = R.adaptive(n, k, d)[0]
    per_step = max(3.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        reference_sample(args.workload, ub, min(per_step, 3.0))
    tot_e, tot_s, its = 0, 0.0, 0
    for _ in range(args.steps):
        e, s, it, st = reference_sample(args.workload, ub, per_step)
        tot_e += e
        tot_s += s
        its = it
    value = tot_e / tot_s
    full_s, full_thr = (None, None) if args.no_ref_full else reference_full_solve(args.workload)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_s * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (SplitMix64 random automaton)",
        "config": dict(arm_config(args.workload, n, k, ub, world),
                       reference_step=f"PREFIX: the first {its} iterations of the solve per step "
                                      f"(phase 1 only, no DFS; a {per_step:.0f} s budget) — the "
                                      "reference's full solve runs ~10^2 s, so a step is a "
                                      "bounded sample; its rate exceeds the full solve's"),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "reference",
                         "sample": f"PREFIX: reference engine on {args.workload}, first {its} "
                                   f"iterations per step ({per_step:.0f} s budget); "
                                   f"single-threaded by construction; host {cpu_model()}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if full_s is not None:
        line["time_to_threshold_s"] = full_s
        line["cpu_baseline"]["time_to_threshold_s"] = full_s
        line["cpu_baseline"]["time_to_threshold_note"] = (
            f"one complete reference solve_exact of {args.workload} (heuristic + engine, "
            f"threshold {full_thr}), same host, after the timed steps")
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":  # CPU arm: rank 0 alone works, no process group needed
        run_reference(args, int(os.environ.get("WORLD_SIZE", "1")),
                      int(os.environ.get("RANK", "0")))
        return
    world, rank, local = dist_setup(args.gpus)
    run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
