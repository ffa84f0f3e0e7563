#!/usr/bin/env python3
"""Benchmark of the batched controller-evaluation hot path (BASELINE.json north_star).

Metric: simulated tenant-ticks/s (tenant-tick = one tenant advanced through one 1-s engine tick,
SURVEY.md section 8(d)).  Workload at N=1: BASELINE.json configs[1] = C2, the 2-node 16-GPU
cluster scenario with the 8-tenant mix under the full controller (dynamic MIG + PCIe-aware
placement + MPS/cgroup guardrails), 256 seeds (scenarios/c2_cluster16.yaml).  Weak scaling: each
rank runs its own block of 256 seeds; NCCL (torch.distributed) only reduces the per-seed SLO-miss
histogram and gathers per-seed focus rows at the end, like SURVEY.md 8(e).

  python bench.py [--gpus N --steps K --warmup W]          # the B200 engine
  python bench.py --impl reference [--steps K --warmup W]   # the reference CPU engine (oracle/_ref)

One JSON line on rank 0.  `value` = tenant-ticks / device time of the engine kernels (CUDA events
on the engine stream; scenario + seeds resident, arrival records generated on device); `e2e` =
the same metric through the C-ABI call a user makes (host packing, H2D, kernels, D2H of all
results) by host wall clock.
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

SCENARIO = os.path.join(ROOT, "scenarios", "c2_cluster16.yaml")
SEEDS_PER_GPU = 256
WORKLOAD = ("C2 c2-cluster16: 2 hosts x 8 GPUs (4 PCIe roots/host, GPUs 6-7 MPS), 8 tenants "
            "(3x t1-inference, llm-ttft, 2x t2-etl, 2x t3-train), full controller, 1800 s horizon, 256 seeds/GPU")
METRIC = "simulated tenant-ticks/s (C2 2-node 16-GPU 8-tenant full-controller sweep)"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def run_reference(args):
    """Reference arm: the unmodified reference engine (oracle/_ref, built from /root/reference
    sources) with its own std::async replica fan-out over all host cores."""
    world, rank, _ = _dist()
    if rank != 0:
        return
    import ctypes

    from tests._libs import oracle, scenario_json

    lib = oracle()
    cores = os.cpu_count() or 1
    n_rep = max(cores, 8)  # one fan-out batch over every core: the bounded per-step sample
    sj = scenario_json(SCENARIO)
    ov = (ctypes.c_char_p * 1)(None)
    walls = []
    for i in range(args.warmup + args.steps):
        w = lib.ref_run_batch(sj, ov, 1, 1 + 1000 * i, n_rep, cores, b"ta", None, None, None, None)
        if w < 0:
            raise RuntimeError(lib.ref_last_error().decode())
        if i >= args.warmup:
            walls.append(w)
    ticks = n_rep * 8 * 1800
    value = ticks * len(walls) / sum(walls)
    sample = f"{n_rep} C2 replicas (seeds block) per step, std::async fan-out on {cores} threads"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tenant-ticks/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * sum(walls) / len(walls),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (scenario-v1 C2, reference RNG streams)",
        "config": {"workload": WORKLOAD, "scenario": "scenarios/c2_cluster16.yaml", "seeds_per_step": n_rep},
        "cpu_baseline": {"value": value, "unit": "tenant-ticks/s", "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "tenant-ticks/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_sample():
    """The reference (oracle/_ref) timed on this box's host cores on a bounded C2 sample."""
    import ctypes

    from tests._libs import oracle, scenario_json

    lib = oracle()
    cores = os.cpu_count() or 1
    n_rep = max(cores, 8)
    w = lib.ref_run_batch(scenario_json(SCENARIO), (ctypes.c_char_p * 1)(None), 1, 900001, n_rep, cores, b"ta",
                          None, None, None, None)
    if w < 0:
        return None
    return {"value": n_rep * 8 * 1800 / w, "unit": "tenant-ticks/s", "cores": cores, "kind": "reference",
            "sample": f"{n_rep} C2 replicas, one std::async fan-out batch on {cores} threads, {w:.1f} s wall"}


def run_engine(args):
    import numpy as np

    world, rank, local = _dist()
    import torch

    dist = None
    n_dev = torch.cuda.device_count()
    device = local % max(n_dev, 1)
    # NCCL over NVLink when every rank owns a GPU; gloo only when ranks share a device (test boxes)
    coll_dev = "cuda" if n_dev >= world else "cpu"
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(device)
        dist.init_process_group("nccl" if coll_dev == "cuda" else "gloo")
    from paper_2508_20274_b200 import Engine

    eng = Engine(device)
    sid = eng.load_scenario(SCENARIO)
    T = len(eng.tenant_ids(sid))
    seeds = [1 + rank * SEEDS_PER_GPU + i for i in range(SEEDS_PER_GPU)]

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        eng.run_batch(sid, seeds).close()
    clocks = ClockSampler(device)
    clocks.start()
    barrier()
    t0 = time.perf_counter()
    dev_ms = gen_ms = des_ms = sel_ms = 0.0
    ticks = completions = arrivals = samples = launches = 0
    last = None
    for _ in range(args.steps):
        res = eng.run_batch(sid, seeds)
        t = res.timing
        dev_ms += t["total_device_ms"]
        gen_ms += t["gen_ms"]
        des_ms += t["des_ms"]
        sel_ms += t["select_ms"]
        ticks += t["tenant_ticks"]
        completions += t["completions"]
        arrivals += t["arrivals"]
        samples += t["select_samples"]
        launches += 6 * t["waves"]
        if last is not None:
            last.close()
        last = res
    barrier()
    wall_s = time.perf_counter() - t0
    clk = clocks.stop()
    # per-seed focus rows + SLO-miss histogram of the last step: the only cross-GPU data (8(e))
    from paper_2508_20274_b200 import sharding

    focus = last.tenant_ids.index("ta")
    thr = []
    for run in last.rows:  # summed over tenants in id order, as harness.cpp:194-196
        s = 0.0
        for x in run["throughput_hz"]:
            s += float(x)
        thr.append(s)
    rows = np.stack([last.rows[:, focus]["p99_ms"], last.rows[:, focus]["miss_rate"], np.array(thr)], 1)
    all_rows, hist, cis = sharding.reduce_rows(rows, dist, device=coll_dev)
    if dist:
        tt = torch.tensor([dev_ms, wall_s], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dev_ms, wall_s = float(tt[0]), float(tt[1])
        cnt = torch.tensor([ticks, completions, arrivals, samples], dtype=torch.int64, device=coll_dev)
        dist.all_reduce(cnt)
        ticks, completions, arrivals, samples = [int(x) for x in cnt.tolist()]
    if rank != 0:
        last.close()
        if dist:
            dist.destroy_process_group()
        return
    hbm, peak_kind = _peaks()
    # dominant kernel = replica DES; algorithmic bytes per SURVEY 8(d): 48 B per completion
    # (32 B arrival record read + 16 B completion written)
    des_s = des_ms / 1000.0
    des_gbs = 48.0 * completions / des_s / 1e9 if des_s > 0 else 0.0
    sel_gbs = 8.0 * samples / (sel_ms / 1000.0) / 1e9 if sel_ms > 0 else 0.0
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", "des_kernel_traffic.json")
    if os.path.exists(tr_path):
        with open(tr_path) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    value = ticks / (dev_ms / 1000.0)
    sat = None
    if args.c4_seeds > 0:
        # Secondary, outside the timed region: the saturated regime (BASELINE configs[3] shape,
        # 4-variant ablation on default.yaml) where thousands of replicas fill every SM.
        from paper_2508_20274_b200 import Variant

        c4 = eng.load_scenario(os.path.join(ROOT, "tests", "golden", "scenarios", "default.yaml"))
        vs = [Variant("static", False, False, False, False), Variant("mig-only", True, True, False, False),
              Variant("placement-only", True, False, True, False), Variant("full", True, True, True, True)]
        r4 = eng.run_batch(c4, list(range(1, args.c4_seeds + 1)), vs)
        t4 = r4.timing
        sat = {"workload": f"C4-shape ablation: default.yaml x 4 variants x {args.c4_seeds} seeds",
               "replicas": int(t4["replicas"]), "tenant_ticks_per_s": t4["tenant_ticks"] / (t4["total_device_ms"] / 1e3),
               "device_ms": t4["total_device_ms"], "des_ms": t4["des_ms"], "waves": int(t4["waves"]),
               "completions_per_s": t4["completions"] / (t4["total_device_ms"] / 1e3)}
        r4.close()
    h2d = 8 * SEEDS_PER_GPU + 4 * SEEDS_PER_GPU + 2 * (SEEDS_PER_GPU + 1) * 8
    d2h = int(last.timing["replicas"]) * (T * (48 + 32) + 24 + 16 * 2 * 8)
    cpu = None if args.no_cpu_baseline else cpu_baseline_sample()
    line = {
        "metric": METRIC, "value": value, "unit": "tenant-ticks/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (scenario-v1 C2 inputs, reference RNG streams)",
        "config": {"workload": WORKLOAD, "scenario": "scenarios/c2_cluster16.yaml", "seeds_per_gpu": SEEDS_PER_GPU,
                   "variant": "full", "parallelism": f"seed-sharded x{world}", "l2": "inputs_larger_than_L2 "
                   "(per-step arrival records ~5 GB regenerated on device each step)"},
        "e2e": {"value": ticks / wall_s, "unit": "tenant-ticks/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "kernel": "des_kernel_reg" if T <= 10 else "des_kernel", "achieved": des_gbs, "peak": hbm, "unit": "GB/s",
                     "frac": des_gbs / hbm, "traffic": traffic, "peak_kind": peak_kind,
                     "note": "replica DES is latency/issue bound (one sequential event loop per warp); "
                             "48 B algorithmic per completion"},
        "kernels": {"gen_ms_per_step": gen_ms / args.steps, "des_ms_per_step": des_ms / args.steps,
                    "select_ms_per_step": sel_ms / args.steps, "select_GBps": sel_gbs, "select_frac": sel_gbs / hbm,
                    "completions": completions, "arrivals": arrivals, "select_samples": samples},
        "clocks": clk,
        "cpu_baseline": cpu,
        "outcome": {"focus_tenant": "ta", "seeds": int(len(all_rows)), "p99_ci_ms": cis[0], "miss_ci": cis[1],
                    "miss_histogram_nonzero_bins": int((hist > 0).sum())},
        "saturated_regime": sat,
    }
    print(json.dumps(line), flush=True)
    last.close()
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--c4-seeds", type=int, default=1024, help="seeds of the secondary saturated-regime run (0: off)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_engine(args)


if __name__ == "__main__":
    main()
