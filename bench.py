#!/usr/bin/env python
"""Benchmark of the B-ADMM barycenter hot path (arXiv 1510.00012, Alg. 4) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload 5] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (driver launch for N > 1)

A "step" is one full round of the centroid update for every cluster:
ad2_barycenter_init (sort, cost, rho, Pi2 init) -> T/tau x (ad2_badmm_step(tau);
ad2_update_support()) -> ad2_objective (device->host read of the result).  Inputs are resident
in HBM when the timed region starts (value); e2e repeats the step from pinned host buffers
through the same C ABI with the host<->device copies inside the timed region.

metric: B-ADMM plan-entry-iterations/s = sum_k m*m_k * T / step time, all ranks (whole job).
Members are sharded over ranks (entry-balanced contiguous shards, fixed total N: strong
scaling); the per-cluster w/x partial sums are NCCL all-reduced inside libad2.
The state (Pi1, Pi2, Lambda, C: 41 GB at cfg5) is far larger than L2, so no flush is needed.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1510_00012_b200 import workloads as wl  # noqa: E402
from paper_1510_00012_b200.sharding import shard_bounds  # noqa: E402

METRIC = "B-ADMM plan-entry-iterations/sec"
UNIT = "entry-iter/s"
CACHE = os.environ.get("AD2_BENCH_CACHE", "/dev/shm/ad2_bench")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------------------------------ data

def load_bundle(cfg: int, rank: int, world: int, barrier) -> wl.Bundle:
    """Rank 0 generates the seeded bundle (or finds it cached in /dev/shm); other ranks load it."""
    path = os.path.join(CACHE, f"cfg{cfg}_seed0_v1")
    keys = ["offsets", "supports", "weights", "labels", "x0", "w0"]
    done = os.path.join(path, "meta.json")
    if rank == 0 and not os.path.exists(done):
        t = time.time()
        b = wl.make_config(cfg)
        log(f"[bench] generated {b.name} in {time.time() - t:.1f}s")
        try:
            os.makedirs(path, exist_ok=True)
            for k in keys:
                np.save(os.path.join(path, k + ".npy"), getattr(b, k))
            json.dump({"name": b.name, "d": b.d, "m": b.m, "K": b.K, "dtype": b.dtype}, open(done + ".tmp", "w"))
            os.replace(done + ".tmp", done)
        except OSError as e:
            log(f"[bench] cache write failed: {e}")
        barrier()
        return b
    barrier()
    if not os.path.exists(done):        # no shared cache: the seeded generator is deterministic
        return wl.make_config(cfg)
    meta = json.load(open(done))
    arrs = {k: np.load(os.path.join(path, k + ".npy")) for k in keys}
    sched = wl.make_config(cfg, N=64, K=1).sched if cfg != 1 else wl.make_config(1).sched
    return wl.Bundle(meta["name"], meta["d"], meta["m"], meta["K"], dtype=meta["dtype"], sched=sched, **arrs)


# ------------------------------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi's start-up (NVML init) holds driver locks for tens to hundreds of ms: let it
            # finish before the caller's timed region starts (it stalled short configs' rounds)
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.02)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------------------------ ours

def run_ours(args, rank, world, local_rank, dist_on=False):
    import torch
    import torch.distributed as dist
    from paper_1510_00012_b200 import ad2
    from paper_1510_00012_b200.sharding import bootstrap_nccl

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    barrier = (lambda: dist.barrier(device_ids=[local_rank])) if dist_on else (lambda: None)
    b = load_bundle(args.workload, rank, world, barrier)
    s = b.sched
    T, tau = s.T, s.tau
    bounds = shard_bounds(b.offsets, world)
    mine = b.subset(np.arange(bounds[rank], bounds[rank + 1])) if dist_on else b
    entries_local = mine.entries()
    entries_total = b.entries()
    stream = torch.cuda.current_stream(dev)
    ctx = ad2.Context(local_rank, stream.cuda_stream)
    ctx.set_state_mode(args.state_mode)
    if args.tc_cost >= 0:
        ctx.set_tc_cost(args.tc_cost)
    if dist_on:
        bootstrap_nccl(ctx)

    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    D = dict(offsets=t(mine.offsets), supports=t(mine.supports), weights=t(mine.weights), labels=t(mine.labels),
             x0=t(b.x0), w0=t(b.w0))
    obj_box = {}

    sched_ev = []                                      # events around step/update (SURVEY.md §8(d) metric)

    prof_box = {"arm": False}

    def step(arr, mem, after_init=None):
        ctx.init(arr["offsets"], arr["supports"], arr["weights"], arr["labels"], arr["x0"], arr["w0"], b.K, b.m,
                 s.rho0, s.eps, s.rule, mem=mem, dtype=b.dtype, cost_mode=args.cost_mode)
        if after_init is not None:
            after_init()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        arm = prof_box["arm"]
        prof_box["arm"] = False
        ad2.run_schedule(ctx, T, tau, before_last_step=(lambda: ctx.set_profiling(2)) if arm else None)
        e1.record(stream)
        sched_ev.append((e0, e1))
        obj_box["obj"] = ctx.objective()               # device -> host read of the result (syncs)

    def timed(fn, K, W, before_last=None):
        for _ in range(W):
            fn()
        barrier()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = ctx.info()["launches"]
        e0.record(stream)
        for k in range(K):
            if before_last is not None and k == K - 1:
                before_last()
            fn()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        ms = e0.elapsed_time(e1) / K
        launches = ctx.info()["launches"] - l0
        if dist_on:
            x = torch.tensor([ms], device=dev, dtype=torch.float64)
            dist.all_reduce(x, op=dist.ReduceOp.MAX)
            ms = float(x.item())
        return ms, launches

    # the iteration kernels of the LAST step(tau) of the last timed round run with event-record nodes
    # around every launch (live, in-graph, inside the timed region); the other steps run the
    # plain graph, so the instrumentation costs the timed region almost nothing
    ctx.set_profiling(0)
    with ClockSampler(local_rank) as clk:
        ms, launches = timed(lambda: step(D, "device"), args.steps, args.warmup,
                             before_last=lambda: prof_box.update(arm=True))
    sched_ms = float(np.mean([a.elapsed_time(z) for a, z in sched_ev[-args.steps:]]))
    launch_ms, step_graph_ms = ctx.prof_read()
    info = ctx.info()
    value = entries_total * T / (ms / 1e3)

    # dominant kernel: the fused iteration kernel (launches 1..n-1 of each step graph)
    fused = launch_ms[1:-1] if len(launch_ms) > 2 else launch_ms
    avg_fused_ms = float(np.mean(fused))
    # algorithmic bytes per entry-iteration: read + write of the plan state and
    # Lambda (16 B fp32, 32 B fp64), plus the read of a cached C (variants 3 / 0 keep C in HBM)
    es = 8 if b.dtype == "f64" else 4
    bytes_per_entry = 4 * es + (es if info["variant"] in (0, 3) else 0)
    gz = args.state_mode == 1 and info["variant"] == 2 and tau >= 3
    if gz:
        # compressed state: the middle passes (GMID) read the anchor G and read + write U (3 x es per
        # entry) and read + write the per-member log-factors (m per member, one per point)
        bytes_per_entry = 3 * es + 2 * es * (mine.N * b.m + mine.n) / max(1, entries_local)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = bytes_per_entry * entries_local / (avg_fused_ms / 1e3) / 1e9
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        for rec in (prof if isinstance(prof, list) else [prof]):
            if rec.get("workload") == b.name and rec.get("kernel_variant") == ("gmid" if gz else "fused"):
                traffic = rec.get("dram_bytes_per_launch")
    except (OSError, ValueError):
        pass
    # the profiled graph is one step(tau); a round runs T/tau of them
    iter_share = float(np.sum(launch_ms)) * (T // tau) / ms if ms > 0 else None

    # the other state representation on the same box (§13 of DESIGN.md), reported beside the headline:
    # variant 2 only (the compressed passes exist there), same workload, same timing rules
    alt = None
    if info["variant"] == 2 and tau >= 3 and not args.no_alt:
        other = 1 - args.state_mode
        ctx.set_state_mode(other)
        with ClockSampler(local_rank) as clk_alt:
            ms_alt, _ = timed(lambda: step(D, "device"), args.steps, max(3, args.warmup),
                              before_last=lambda: prof_box.update(arm=True))
        lm_alt, _ = ctx.prof_read()
        dom = lm_alt[1:-1] if len(lm_alt) > 2 else lm_alt
        bpe_alt = (3 * es + 2 * es * (mine.N * b.m + mine.n) / max(1, entries_local)) if other == 1 else 4 * es
        ach_alt = bpe_alt * entries_local / (float(np.mean(dom)) / 1e3) / 1e9
        alt = {"state": ["exact (Pi1, Lambda)", "epoch-anchored compressed (G, U, log-factors)"][other],
               "value": entries_total * T / (ms_alt / 1e3), "unit": UNIT, "ms_per_step": ms_alt,
               "kernel": "k_badmm_tma<" + ("GMID" if other == 1 else "FUSED") + ">",
               "avg_launch_ms": float(np.mean(dom)), "bytes_per_entry": bpe_alt, "achieved_gbs": ach_alt,
               "frac": ach_alt / peak, "clocks": clk_alt.summary(),
               "parity": "exact path" if other == 0 else
               "north_star tolerances except x of centroid rows with w_i < 1e-8 (eps-decided; DESIGN.md 13)"}
        ctx.set_state_mode(args.state_mode)

    # e2e: the same step through the C ABI from pinned host buffers (H2D inside the timed region)
    e2e = None
    if not args.no_e2e:
        H = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in
             dict(offsets=mine.offsets, supports=mine.supports, weights=mine.weights, labels=mine.labels,
                  x0=b.x0, w0=b.w0).items()}
        xo = torch.empty(b.x0.shape, dtype=H["x0"].dtype).pin_memory()
        wo = torch.empty(b.w0.shape, dtype=H["w0"].dtype).pin_memory()

        # pipelined like a stream of batches: during timed step i (i < K) the next step's inputs are
        # copied on the library's copy stream (ad2_prefetch) while step i computes; the warm-up
        # step prefetches nothing, so every timed step's own host->device copy is inside the
        # timed region (step 1's synchronously, steps 2..K's overlapped with steps 1..K-1)
        k_e2e = max(1, args.steps)
        calls = {"n": 0}

        use_pf = not os.environ.get("AD2_BENCH_NO_PREFETCH")

        def prefetch_next():
            c = calls["n"]
            if use_pf and 1 <= c < k_e2e:
                ctx.prefetch(H["offsets"], H["supports"], H["weights"], H["labels"], dtype=b.dtype,
                             cost_mode=args.cost_mode)

        def step_host():
            step(H, "host", prefetch_next)
            ctx.centroids_into(xo, wo, mem="host")
            calls["n"] += 1

        ctx.set_profiling(0)
        ms_e2e, _ = timed(step_host, k_e2e, 1)
        h2d = sum(v.numel() * v.element_size() for v in H.values())
        d2h = xo.numel() * xo.element_size() + wo.numel() * wo.element_size() + 2 * 8 * b.K
        e2e = {"value": entries_total * T / (ms_e2e / 1e3), "unit": UNIT, "ms_per_step": ms_e2e,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "h2d_overlap": "next step's inputs prefetched during the current step (ad2_prefetch)"}

    if rank != 0:
        return
    cpu = None
    if world == 1 and not args.no_cpu:
        cpu = cpu_baseline(b, budget_s=args.cpu_budget)
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32" if b.dtype == "f32" else "f64", "data": "synthetic",
        "config": {"workload": b.name, "N": b.N, "K": b.K, "m": b.m, "d": b.d, "T": T, "tau": tau,
                   "entries_per_iter": entries_total, "step": "1 round: init + T/tau x (step(tau), update_support) + objective",
                   "parallelism": f"dp{world} (members sharded, NCCL all-reduce of per-cluster partials)",
                   "l2": "inputs larger than L2 (state %.1f GB)" % (info["state_bytes"] / 1e9),
                   "cost_build": ["fp32", "tcgen05-bf16"][args.cost_mode],
                   "state": ["exact (Pi1, Lambda)", "epoch-anchored compressed (G, U, log-factors)"][args.state_mode],
                   "kernel_variant": {3: "wide", 2: "tma", 1: "warp", 0: "generic"}[info["variant"]]},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": {3: "k_badmm_wide", 2: "k_badmm_tma", 1: "k_badmm_warp", 0: "k_badmm_generic"}[info["variant"]]
                     + ("<GMID>" if gz else "<FUSED>") + " (one B-ADMM iteration: phase 2 of t-1 + phase 1 of t)",
                     "bytes_per_entry": bytes_per_entry, "entries_per_launch": entries_local,
                     "avg_launch_ms": avg_fused_ms, "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback",
                     "iteration_kernels_share_of_step": iter_share},
        # the profiled graph is one step(tau) (tau iterations in tau or tau + 1 launches); a round runs T/tau
        "iter_only": {"value": entries_total * T / ((np.sum(launch_ms) * (T // tau)) / 1e3),
                      "note": "iteration kernels only (event-timed), excluding consensus/init/objective"},
        "steps_and_updates": {"value": entries_total * T / (sched_ms / 1e3), "ms": sched_ms,
                              "note": "SURVEY.md 8(d) definition: ad2_badmm_step + ad2_update_support only "
                                      "(value above is the whole round incl. init and objective)"},
        "e2e": e2e,
        "alt_state_mode": alt,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------------------------------ oracle

_NCORES = None


def host_cores() -> int:
    """All host cores the oracle's OpenMP runtime offers, read ONCE before any oracle call (a call
    with nthreads = k sets the OpenMP thread count for the rest of the process)."""
    global _NCORES
    if _NCORES is None:
        import oracle
        _NCORES = oracle.max_threads()
    return _NCORES


def cpu_baseline(b: wl.Bundle, budget_s: float = 15.0, n_clusters=None, one_thread=True):
    """The fp64 oracle (Alg. 4 as written, OpenMP over members) on a bounded sample of the same
    workload: whole clusters 0, 1, ... with the full schedule until about budget_s of host time
    (or exactly n_clusters when given, for repeatable reference steps), on every host core; then
    (one_thread) the 1-thread rate on a small sample."""
    import oracle
    ncores = host_cores()
    s = b.sched
    t_all, entries, members, c = 0.0, 0, 0, 0
    while c < b.K:
        mem = np.nonzero(b.labels == c)[0]
        sub = b.subset(mem)
        t = time.time()
        oracle.badmm_centroid(b.x0[c], b.w0[c], sub.offsets, sub.supports, sub.weights, s.T, s.tau, s.rule, s.rho0,
                              s.eps, 1e-5, nthreads=ncores, want_state=False)
        t_all += time.time() - t
        entries += b.m * sub.n
        members += sub.N
        c += 1
        if (n_clusters is not None and c >= n_clusters) or (n_clusters is None and t_all >= budget_s):
            break
    out = {"value": entries * s.T / t_all, "unit": UNIT, "cores": ncores, "kind": "oracle",
           "sample": f"clusters 0..{c - 1} of {b.name}: {members} members ({entries} plan entries), T={s.T}, "
                     f"tau={s.tau}, fp64, {t_all:.1f}s", "n_clusters": c, "cpu_model": cpu_model()}
    if n_clusters is None and one_thread:
        # the 1-thread rate on the first members of cluster 0, ~2 s
        mem = np.nonzero(b.labels == 0)[0]
        k = max(1, min(len(mem), int(len(mem) * min(1.0, 2.0 / max(t_all / c, 1e-3)) / max(1, ncores))))
        sub = b.subset(mem[:k])
        t = time.time()
        oracle.badmm_centroid(b.x0[0], b.w0[0], sub.offsets, sub.supports, sub.weights, s.T, s.tau, s.rule, s.rho0,
                              s.eps, 1e-5, nthreads=1, want_state=False)
        out["value_1thread"] = b.m * sub.n * s.T / (time.time() - t)
        out["sample_1thread"] = f"first {k} members of cluster 0, 1 thread"
    return out


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args, rank, world):
    """--impl reference: the fp64 oracle as it stands, on the host cores, rank 0 only."""
    if rank != 0:
        return
    b = load_bundle(args.workload, 0, 1, lambda: None)
    # each reference step: the same bounded sample (whole clusters), sized so the run stays short
    probe = cpu_baseline(b, budget_s=max(2.0, args.cpu_budget / max(1, args.steps + args.warmup)), one_thread=False)
    nc = probe["n_clusters"]
    for _ in range(max(0, args.warmup - 1)):
        cpu_baseline(b, n_clusters=nc)
    t = time.time()
    vals = [cpu_baseline(b, n_clusters=nc) for _ in range(args.steps)]
    ms = (time.time() - t) / max(1, args.steps) * 1e3
    v = float(np.mean([x["value"] for x in vals]))
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": b.name, "N": b.N, "K": b.K, "m": b.m, "d": b.d, "T": b.sched.T, "tau": b.sched.tau},
           "cpu_baseline": {"kind": "oracle", "cores": vals[-1]["cores"], "sample": vals[-1]["sample"], "value": v},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", type=int, default=5, help="BASELINE.json config (1-based)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-alt", action="store_true", help="skip the other state representation's measurement")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--cost-mode", type=int, default=0, help="0: fp32 cost build, 1: bf16 tcgen05 (cached-cost kernels)")
    ap.add_argument("--tc-cost", type=int, default=-1,
                    help="1/0: tensor-core / FFMA2 dot products in the variant-2 cost (ad2_set_tc_cost); -1: library default")
    ap.add_argument("--state-mode", type=int, default=0,
                    help="0: exact Pi1/Lambda state, 1: epoch-anchored compressed state (ad2_set_state_mode)")
    ap.add_argument("--dist", action="store_true",
                    help="use the multi-GPU path (torch.distributed + NCCL communicator in libad2) even with 1 rank")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    dist_on = world > 1 or args.dist
    if dist_on:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    run_ours(args, rank, world, local_rank, dist_on)
    if dist_on:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
