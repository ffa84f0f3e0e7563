"""Seed sweeps for the large BASELINE configs (C4: 4-variant ablation x 16k seeds with SLO-miss
histograms; C5: 10^6 seeds x 64 tenants), sharded over the GPUs of one box.

The reference runs such sweeps as harness jobs = variants x seeds fanned out over std::async
(harness.cpp:114-216, jobs row-major variant x seed).  Here each rank takes a contiguous seed block
(sharding.seed_block / split_seeds), runs all variants of it as GPU batches (the engine streams the
replicas through HBM in waves), and the end-of-run reduction is the only cross-GPU traffic
(sharding.reduce_rows: NCCL all-reduce of the integer miss-rate histogram + all-gather of the
per-seed focus rows, CIs summed in seed order exactly like harness.cpp:32-43).

  torchrun --nproc-per-node 8 -m paper_2508_20274_b200.sweep --scenario tests/golden/scenarios/default.yaml \\
      --variants ablation --seeds 16384                    # C4
  torchrun --nproc-per-node 8 -m paper_2508_20274_b200.sweep --scenario scenarios/c5_mc64.yaml \\
      --variants full --seeds 1000000 --chunk 8192          # C5
"""
from __future__ import annotations

import argparse
import json
import os
import time
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import sharding
from .api import HIST_BINS, Engine, Variant, ablation_variants, main_variants, scenario_spec


def focus_rows(res, focus: str) -> np.ndarray:
    """[runs, 3] = (focus p99_ms, focus miss_rate, throughput summed over tenants in id order) --
    the per-seed values harness.cpp:178-197 aggregates."""
    f = res.tenant_ids.index(focus)
    thr = np.zeros(res.rows.shape[0])
    for i in range(res.rows.shape[1]):  # id order, like the std::map iteration
        thr = thr + res.rows[:, i]["throughput_hz"]
    return np.stack([res.rows[:, f]["p99_ms"], res.rows[:, f]["miss_rate"], thr], 1)


def default_focus(path: str) -> str:
    """harness.cpp:80-87 pick_focus_tenant: the smallest tail SLO after presets, first in file
    order on ties."""
    best = None
    for t in scenario_spec(path)["tenants"]:
        if best is None or t["slo_tail_ms"] < best["slo_tail_ms"]:
            best = t
    return best["id"]


def run_sweep(path: str, variants: Sequence[Variant], seeds: Sequence[int], focus: Optional[str] = None,
              dist=None, device: int = 0, chunk: int = 0, coll_device: str = "cpu") -> Dict:
    """Run `variants` x `seeds` (this rank's block) and reduce across ranks.

    Returns per variant: all seeds' focus rows (global seed order), the summed 1e-3-bin miss-rate
    histogram, CIs (p99, miss, throughput), plus device/wall timing of this rank."""
    eng = Engine(device)
    sid = eng.load_scenario(path)
    focus = focus or default_focus(path)
    T = len(eng.tenant_ids(sid))
    chunk = chunk or len(seeds) or 1
    out = {"scenario": path, "focus_tenant": focus, "variants": [], "tenant_ticks": 0, "device_ms": 0.0,
           "completions": 0}
    t0 = time.perf_counter()
    for v in variants:
        rows = []
        lat = np.zeros((1, T, HIST_BINS), np.int64)
        cnt = np.zeros((1, T, 3), np.int64)
        for c0 in range(0, len(seeds), chunk):
            part = list(seeds[c0:c0 + chunk])
            res = eng.run_batch(sid, part, [v])
            rows.append(focus_rows(res, focus))
            lat += res.latency_hist()
            cnt += res.tenant_counts()
            out["tenant_ticks"] += int(res.timing["tenant_ticks"])
            out["device_ms"] += float(res.timing["total_device_ms"])
            out["completions"] += int(res.timing["completions"])
            res.close()
        local = np.concatenate(rows, 0) if rows else np.zeros((0, 3))
        all_rows, hist, cis = sharding.reduce_rows(local, dist, device=coll_device)
        lat, cnt = sharding.reduce_tenant_hists(lat, cnt, dist, device=coll_device)
        out["variants"].append({"name": v.name, "seeds": int(all_rows.shape[0]), "p99_ci": cis[0], "miss_ci": cis[1],
                                "throughput_ci": cis[2], "miss_histogram": hist, "rows": all_rows,
                                "latency_hist": lat[0], "tenant_counts": cnt[0]})
    out["wall_s"] = time.perf_counter() - t0
    out["tenants"] = T
    out["tenant_ids"] = eng.tenant_ids(sid)
    eng.close()
    return out


def _variants(name: str) -> List[Variant]:
    if name == "ablation":
        return ablation_variants()
    if name == "main":
        return main_variants()
    if name == "full":
        return [Variant("full", True, True, True, True)]
    if name == "c4":  # BASELINE configs[3]: static / MIG-only / placement-only / full controller
        return [v for v in ablation_variants() if v.name in ("static", "mig-only", "placement-only", "full")]
    raise ValueError(f"unknown variant set '{name}' (ablation | main | full | c4)")


def main(argv=None) -> None:
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--scenario", required=True)
    ap.add_argument("--variants", default="ablation")
    ap.add_argument("--seeds", type=int, default=16384, help="total seeds (strong scaling over ranks)")
    ap.add_argument("--seed-base", type=int, default=1)
    ap.add_argument("--focus", default=None)
    ap.add_argument("--chunk", type=int, default=0, help="seeds per GPU batch (0: all of the rank's block)")
    ap.add_argument("--out", default=None, help="write the rank-0 summary JSON here")
    args = ap.parse_args(argv)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    coll = "cpu"
    if world > 1:
        import torch
        import torch.distributed as dist

        n_dev = torch.cuda.device_count()
        coll = "cuda" if n_dev >= world else "cpu"
        if coll == "cuda":
            torch.cuda.set_device(local)
        dist.init_process_group("nccl" if coll == "cuda" else "gloo")
    seeds = list(range(args.seed_base, args.seed_base + args.seeds))
    mine = sharding.split_seeds(seeds, rank, world)
    import torch

    device = local % max(torch.cuda.device_count(), 1)
    res = run_sweep(args.scenario, _variants(args.variants), mine, args.focus, dist, device, args.chunk, coll)
    if dist is not None:
        import torch

        t = torch.tensor([res["device_ms"], res["wall_s"]], dtype=torch.float64, device=coll)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res["device_ms"], res["wall_s"] = float(t[0]), float(t[1])
        c = torch.tensor([res["tenant_ticks"], res["completions"]], dtype=torch.int64, device=coll)
        dist.all_reduce(c)
        res["tenant_ticks"], res["completions"] = int(c[0]), int(c[1])
    if rank == 0:
        from .api import hist_bin_edges

        edges = hist_bin_edges()
        summary = {
            "scenario": args.scenario, "focus_tenant": res["focus_tenant"], "ranks": world, "seeds": args.seeds,
            "tenant_ticks": res["tenant_ticks"], "completions": res["completions"],
            "device_ms_max_over_ranks": res["device_ms"], "wall_s": res["wall_s"],
            "tenant_ticks_per_s": res["tenant_ticks"] / (res["device_ms"] / 1e3) if res["device_ms"] else None,
            "variants": [{"name": v["name"], "seeds": v["seeds"], "p99_ci": v["p99_ci"], "miss_ci": v["miss_ci"],
                          "throughput_ci": v["throughput_ci"],
                          "tenant_counts": {tid: [int(x) for x in v["tenant_counts"][i]]
                                            for i, tid in enumerate(res["tenant_ids"])},
                          "latency_hist_total": int(v["latency_hist"].sum()),
                          # pooled p50/p95/p99/p999 over every seed's window latencies, exact to the bin
                          "pooled_quantile_bins_ms": {
                              tid: {name: list(b) for name, b in zip(("p50", "p95", "p99", "p999"),
                                                                       sharding.pooled_quantiles(v["latency_hist"][i], edges))}
                              for i, tid in enumerate(res["tenant_ids"])},
                          "miss_histogram_nonzero": {int(i): int(x) for i, x in enumerate(v["miss_histogram"]) if x}}
                         for v in res["variants"]],
        }
        text = json.dumps(summary)
        print(text, flush=True)
        if args.out:
            with open(args.out, "w") as fh:
                fh.write(text + "\n")
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
