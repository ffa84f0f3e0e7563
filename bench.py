#!/usr/bin/env python3
"""Benchmark of the batched controller-evaluation hot path (BASELINE.json north_star).

Metric: simulated tenant-ticks/s (tenant-tick = one tenant advanced through one 1-s engine tick,
SURVEY.md section 8(d)).  Workload at N=1: BASELINE.json configs[3] = C4, the largest config that
fits one GPU: the ablation sweep default.yaml x {static, mig-only, placement-only, full controller}
x 16,384 seeds (/root/reference/proj/src/harness.cpp:45-53, 114-216) with per-variant SLO-miss-rate
histograms -- 65,536 replicas, 354 M tenant-ticks per step.  Weak scaling: each rank runs its own
block of 16,384 seeds x 4 variants; torch.distributed (NCCL over NVLink) only reduces the per-seed
miss-rate histogram, the per-(variant, tenant) latency histograms and counters, and gathers the
per-seed focus rows at the end of each step.

  python bench.py [--gpus N --steps K --warmup W]          # the B200 engine
  python bench.py --impl reference [--steps K --warmup W]   # the reference CPU engine (oracle/_ref)

One JSON line on rank 0.  `value` = tenant-ticks / device time of the engine kernels (CUDA events
on the engine stream, max over ranks; scenario + seeds resident, arrival records generated on
device); `e2e` = the same metric through the C-ABI call a user makes (host packing, H2D of seeds and
scenario tables, kernels, D2H of every RunResult) plus the cross-rank reduction, by host wall clock.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SCENARIO = os.path.join(ROOT, "tests", "golden", "scenarios", "default.yaml")
SCENARIO_REL = "tests/golden/scenarios/default.yaml"
SEEDS_PER_GPU = 16384
# BASELINE configs[3] variant set, harness.cpp:45-53 flags (enabled, mig, placement, guardrails)
C4_VARIANTS = [("static", False, False, False, False), ("mig-only", True, True, False, False),
               ("placement-only", True, False, True, False), ("full", True, True, True, True)]
WORKLOAD = ("C4 ablation sweep (BASELINE configs[3]): default.yaml (1 host, 8 GPUs, 3 tenants, 1800 s horizon) x "
            "{static MIG, MIG-only, placement-only, full controller} x 16384 seeds/GPU, SLO-miss-rate histograms")
METRIC = "simulated tenant-ticks/s (C4 ablation: default.yaml x 4 controller variants x 16k seeds)"
C2_SCENARIO = os.path.join(ROOT, "scenarios", "c2_cluster16.yaml")


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


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
                                          "--format=csv,noheader,nounits", "-lms", "500"],
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


def _ref_overrides():
    import ctypes

    keys = ("enabled", "enable_mig", "enable_placement", "enable_guardrails")
    ov = [json.dumps(dict(zip(keys, v[1:]))).encode() for v in C4_VARIANTS]
    return (ctypes.c_char_p * len(ov))(*ov)


def _ref_sample(lib, sj, per_variant: int, seed_base: int, cores: int) -> float:
    """One reference fan-out over the 4-variant C4 mix: per_variant contiguous seeds per variant, jobs
    = variants x seeds in std::async batches of `cores` (harness.cpp:156-176).  Returns wall s."""
    w = lib.ref_run_batch(sj, _ref_overrides(), len(C4_VARIANTS), seed_base, per_variant, cores, b"t1", None, None,
                          None, None)
    if w < 0:
        raise RuntimeError(lib.ref_last_error().decode())
    return w


def run_reference(args):
    """Reference arm: the unmodified reference engine (oracle/_ref, built from /root/reference
    sources) with its own std::async replica fan-out over all host cores, on the same 4-variant C4 mix
    (a contiguous seed block per step, extrapolated linearly: per-replica cost is seed-independent
    in distribution)."""
    world, rank, _ = _dist()
    if rank != 0:
        return
    from tests._libs import oracle, scenario_json

    lib = oracle()
    cores = os.cpu_count() or 1
    # one fan-out batch of nproc jobs per variant per step, the seed block advancing every step, so
    # the timed steps together cover steps x nproc contiguous seeds per variant (>= 8 x nproc at
    # the driver's --steps 20) while the whole run stays within a few minutes
    per_variant = args.ref_seeds or cores
    sj = scenario_json(SCENARIO)
    T = len(json.loads(sj)["tenants"])
    walls = []
    for i in range(args.warmup + args.steps):
        w = _ref_sample(lib, sj, per_variant, 1 + (i * per_variant) % SEEDS_PER_GPU, cores)
        if i >= args.warmup:
            walls.append(w)
    n_rep = per_variant * len(C4_VARIANTS)
    ticks = n_rep * T * 1800
    value = ticks * len(walls) / sum(walls)
    sample = (f"{per_variant} contiguous seeds x 4 variants = {n_rep} replicas per step (seed block advancing per step: "
              f"{per_variant * args.steps} seeds per variant over the timed steps) of the {SEEDS_PER_GPU}-seed C4 job, "
              f"extrapolated linearly; std::async fan-out on {cores} threads of {_cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tenant-ticks/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * sum(walls) / len(walls),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (scenario-v1 default.yaml, reference RNG streams)",
        "config": {"workload": WORKLOAD, "scenario": SCENARIO_REL, "variants": [v[0] for v in C4_VARIANTS],
                   "seeds_per_variant_per_step": per_variant, "nproc": cores, "cpu_model": _cpu_model()},
        "cpu_baseline": {"value": value, "unit": "tenant-ticks/s", "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "tenant-ticks/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_sample(per_variant: int):
    """The reference (oracle/_ref) timed on this box's host cores on a bounded sample of the same C4
    mix (one fan-out of per_variant seeds x 4 variants)."""
    from tests._libs import oracle, scenario_json

    lib = oracle()
    cores = os.cpu_count() or 1
    sj = scenario_json(SCENARIO)
    T = len(json.loads(sj)["tenants"])
    try:
        w = _ref_sample(lib, sj, per_variant, 1, cores)
    except RuntimeError:
        return None
    n_rep = per_variant * len(C4_VARIANTS)
    return {"value": n_rep * T * 1800 / w, "unit": "tenant-ticks/s", "cores": cores, "kind": "reference",
            "sample": f"{per_variant} seeds x 4 C4 variants = {n_rep} replicas, one std::async fan-out on {cores} "
                      f"threads of {_cpu_model()}, {w:.1f} s wall (extrapolated linearly)"}


def _focus_rows(res, focus):
    import numpy as np

    f = res.tenant_ids.index(focus)
    thr = np.zeros(res.rows.shape[0])
    for i in range(res.rows.shape[1]):  # summed over tenants in id order, as harness.cpp:194-196
        thr = thr + res.rows[:, i]["throughput_hz"]
    return np.stack([res.rows[:, f]["p99_ms"], res.rows[:, f]["miss_rate"], thr], 1)


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
        if n_dev < world:  # ranks share devices (test boxes): split each device's HBM between them
            share = -(-world // max(n_dev, 1))
            os.environ.setdefault("MIGSIM_MEM_FRACTION", str(0.70 / share))
        dist.init_process_group("nccl" if coll_dev == "cuda" else "gloo")
    from paper_2508_20274_b200 import Engine, Variant, sharding

    eng = Engine(device)
    sid = eng.load_scenario(SCENARIO)
    tids = eng.tenant_ids(sid)
    T = len(tids)
    vs = [Variant(*v) for v in C4_VARIANTS]
    n_seeds = args.seeds
    seeds = sharding.seed_block(rank, world, n_seeds)
    focus = "t1"  # harness.cpp:80-87 pick_focus_tenant on default.yaml (smallest slo_tail_ms)

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def step():
        """One pass of the hot path over the C4 batch, through the public API, + the end-of-step
        cross-rank reduction (per variant: miss-rate histogram + focus rows; per (variant, tenant):
        latency histograms + completion/miss counters)."""
        res = eng.run_batch(sid, seeds, vs)
        rows = _focus_rows(res, focus)
        lat, cnt = sharding.reduce_tenant_hists(res.latency_hist(), res.tenant_counts(), dist, device=coll_dev)
        per_var = [sharding.reduce_rows(rows[v * n_seeds:(v + 1) * n_seeds], dist, device=coll_dev)
                   for v in range(len(vs))]
        t = dict(res.timing)
        res.close()
        return t, per_var, lat, cnt

    for _ in range(args.warmup):
        step()
    clocks = ClockSampler(device)
    clocks.start()
    barrier()
    t0 = time.perf_counter()
    acc = {k: 0.0 for k in ("total_device_ms", "gen_ms", "des_ms", "select_ms", "tenant_ticks", "completions",
                            "arrivals", "select_samples", "kernel_launches", "h2d_bytes", "d2h_bytes", "events",
                            "waves")}
    last = None
    for _ in range(args.steps):
        t, per_var, lat, cnt = step()
        for k in acc:
            acc[k] += t[k]
        last = (t, per_var, lat, cnt)
    barrier()
    wall_s = time.perf_counter() - t0
    clk = clocks.stop()
    dev_ms = acc["total_device_ms"]
    if dist:
        tt = torch.tensor([dev_ms, wall_s, acc["des_ms"], acc["select_ms"], acc["gen_ms"]], dtype=torch.float64,
                          device=coll_dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dev_ms, wall_s = float(tt[0]), float(tt[1])
        acc["des_ms"], acc["select_ms"], acc["gen_ms"] = float(tt[2]), float(tt[3]), float(tt[4])
        keys = ("tenant_ticks", "completions", "arrivals", "select_samples", "kernel_launches")
        cnt_t = torch.tensor([int(acc[k]) for k in keys], dtype=torch.int64, device=coll_dev)
        dist.all_reduce(cnt_t)
        for k, x in zip(keys, cnt_t.tolist()):
            acc[k] = x
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    t_last, per_var, lat, cnt = last
    hbm, peak_kind = _peaks()
    steps = args.steps
    # dominant kernel = replica DES; algorithmic bytes per SURVEY 8(d): 48 B per completion
    # (32 B arrival record read + 16 B completion written); DES device time over the timed region
    des_s = acc["des_ms"] / 1000.0
    des_gbs = 48.0 * acc["completions"] / des_s / 1e9 if des_s > 0 else 0.0
    sel_gbs = 8.0 * acc["select_samples"] / (acc["select_ms"] / 1000.0) / 1e9 if acc["select_ms"] > 0 else 0.0
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", "des_kernel_traffic.json")
    if os.path.exists(tr_path):
        with open(tr_path) as f:
            tj = json.load(f)
        # ncu per-launch DRAM bytes of the captured launch, and its ratio to the algorithmic 48 B per
        # completion applied to this run's DES launches (one launch per wave)
        ratio = tj["dram_bytes_per_launch"] / tj["algorithmic_bytes_per_launch"]
        alg_launch = 48.0 * acc["completions"] / max(1, acc["waves"])
        traffic = {"dram_bytes_per_launch": ratio * alg_launch, "algorithmic_bytes_per_launch": alg_launch,
                   "dram_over_algorithmic": ratio, "captured_kernel": tj.get("kernel"),
                   "captured_workload": tj.get("workload"), "source": tj.get("source")}
    value = acc["tenant_ticks"] / (dev_ms / 1000.0)
    sec = None
    if args.c2_seeds > 0:
        # Secondary, outside the timed region: C2 (BASELINE configs[1]) 256 seeds, full controller
        c2 = eng.load_scenario(C2_SCENARIO)
        r2 = eng.run_batch(c2, list(range(1, args.c2_seeds + 1)))
        t2 = r2.timing
        sec = {"workload": f"C2 c2_cluster16.yaml, full controller, {args.c2_seeds} seeds (BASELINE configs[1])",
               "tenant_ticks_per_s": t2["tenant_ticks"] / (t2["total_device_ms"] / 1e3),
               "e2e_tenant_ticks_per_s": t2["tenant_ticks"] / (t2["wall_ms"] / 1e3),
               "device_ms": t2["total_device_ms"], "des_ms": t2["des_ms"]}
        r2.close()
    cpu = None if args.no_cpu_baseline else cpu_baseline_sample(args.cpu_seeds or 2 * (os.cpu_count() or 1))
    outcome = {}
    for v, (all_rows, hist, cis) in zip(vs, per_var):
        outcome[v.name] = {"seeds": int(len(all_rows)), "t1_p99_ci_ms": cis[0], "t1_miss_ci": cis[1],
                           "miss_histogram_nonzero_bins": int((hist > 0).sum())}
    vi = {v.name: i for i, v in enumerate(vs)}
    from paper_2508_20274_b200.api import hist_bin_edges

    edges = hist_bin_edges()
    for name, i in vi.items():
        # pooled t1 tail over all seeds (and ranks) from the reduced histogram, exact to the bin
        ft = tids.index(focus)
        outcome[name]["t1_pooled_p99_bin_ms"], outcome[name]["t1_pooled_p999_bin_ms"] = (
            list(b) for b in sharding.pooled_quantiles(lat[i, ft], edges, (0.99, 0.999)))
        outcome[name]["window_completions"] = {tid: int(cnt[i, k, 1]) for k, tid in enumerate(tids)}
        outcome[name]["window_misses"] = {tid: int(cnt[i, k, 2]) for k, tid in enumerate(tids)}
    line = {
        "metric": METRIC, "value": value, "unit": "tenant-ticks/s", "n_gpus": world, "steps": steps,
        "warmup": args.warmup, "ms_per_step": dev_ms / steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (scenario-v1 default.yaml inputs, reference RNG streams)",
        "config": {"workload": WORKLOAD, "scenario": SCENARIO_REL, "variants": [v.name for v in vs],
                   "seeds_per_gpu": n_seeds, "replicas_per_gpu": n_seeds * len(vs),
                   "parallelism": f"seed-sharded x{world}",
                   "l2": "inputs_larger_than_L2 (per-wave arrival records, tens of GB, regenerated on device)"},
        "e2e": {"value": acc["tenant_ticks"] / wall_s, "unit": "tenant-ticks/s",
                "h2d_bytes_per_step": int(t_last["h2d_bytes"]), "d2h_bytes_per_step": int(t_last["d2h_bytes"]),
                "note": "wall clock around the C-ABI call (host packing, H2D, kernels, D2H of every RunResult) "
                        "+ the cross-rank reduction, max over ranks"},
        "gpu_launches": int(acc["kernel_launches"]),
        "roofline": {"bound": "hbm", "kernel": {0: "des_kernel_reg" if T <= 10 else "des_kernel", 1: "des_simt_kernel",
                                                2: "des_kernel_reg_occ"}[int(t_last["des_form"])], "achieved": des_gbs,
                     "peak": hbm, "unit": "GB/s", "frac": des_gbs / hbm, "traffic": traffic, "peak_kind": peak_kind,
                     "note": "replica DES is latency/issue bound (one sequential event loop per warp); "
                             "48 B algorithmic per completion"},
        "kernels": {"gen_ms_per_step": acc["gen_ms"] / steps, "des_ms_per_step": acc["des_ms"] / steps,
                    "select_ms_per_step": acc["select_ms"] / steps, "select_GBps": sel_gbs, "select_frac": sel_gbs / hbm,
                    "completions": int(acc["completions"]), "arrivals": int(acc["arrivals"]),
                    "select_samples": int(acc["select_samples"]), "waves_per_step": int(t_last["waves"]),
                    "des_blocks_per_sm": int(t_last["des_blocks_per_sm"]),
                    "des_smem_bytes": int(t_last["des_smem_bytes"])},
        "clocks": clk,
        "cpu_baseline": cpu,
        "outcome": outcome,
        "secondary": sec,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--seeds", type=int, default=SEEDS_PER_GPU, help="seeds per variant per GPU (C4: 16384)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seeds", type=int, default=0, help="seeds per variant of the cpu_baseline sample (0: 2 x nproc)")
    ap.add_argument("--ref-seeds", type=int, default=0, help="reference arm: seeds per variant per step (0: nproc)")
    ap.add_argument("--c2-seeds", type=int, default=256, help="seeds of the secondary C2 run (0: off)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_engine(args)


if __name__ == "__main__":
    main()
