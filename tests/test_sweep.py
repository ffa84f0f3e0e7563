"""Seed sweeps (BASELINE configs C4/C5 driver, paper_2508_20274_b200/sweep.py): per-seed focus
rows, the 1e-3-bin SLO-miss histogram and harness CIs equal the reference replicas aggregated the
way harness.cpp:178-204 does; the 2-rank path (gloo, both ranks on cuda:0) equals 1 rank."""
import os
import socket

import numpy as np
import pytest

from oracle import restate
from tests._libs import GOLDEN_SCENARIOS, ref_run

pytestmark = pytest.mark.gpu

PATH = GOLDEN_SCENARIOS[1]  # llm.yaml: short, controller active


def _ref_rows(variant, seeds, focus):
    ov = dict(enabled=variant.enabled, enable_mig=variant.enable_mig, enable_placement=variant.enable_placement,
              enable_guardrails=variant.enable_guardrails)
    rows = []
    for s in seeds:
        t = ref_run(PATH, s, ov)[0]["summary"]["tenants"]
        thr = 0.0
        for tid in sorted(t):
            thr += t[tid]["throughput_hz"]
        rows.append((t[focus]["p99_ms"], t[focus]["miss_rate"], thr))
    return np.array(rows)


def test_sweep_matches_reference_replicas():
    from paper_2508_20274_b200 import ablation_variants, sharding
    from paper_2508_20274_b200.sweep import default_focus, run_sweep

    seeds = list(range(31, 39))
    vs = ablation_variants()[:2]
    out = run_sweep(PATH, vs, seeds, chunk=3)
    focus = default_focus(PATH)
    assert out["focus_tenant"] == focus == "llm"
    for v, got in zip(vs, out["variants"]):
        ref = _ref_rows(v, seeds, focus)
        assert (got["rows"].view(np.uint64) == ref.view(np.uint64)).all(), v.name
        assert (got["miss_histogram"] == sharding.miss_histogram(ref[:, 1])).all()
        for k, key in enumerate(("p99_ci", "miss_ci", "throughput_ci")):
            assert tuple(got[key]) == restate.confidence_interval(list(ref[:, k]))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, seeds, out):
    import torch.distributed as dist

    from paper_2508_20274_b200 import ablation_variants, sharding
    from paper_2508_20274_b200.sweep import run_sweep

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = run_sweep(PATH, ablation_variants()[:1], sharding.split_seeds(seeds, rank, world), dist=dist)
    v = res["variants"][0]
    out[rank] = (v["rows"], v["miss_histogram"], v["p99_ci"])
    dist.destroy_process_group()


def test_sweep_two_ranks_equals_one():
    import torch.multiprocessing as mp

    from paper_2508_20274_b200 import ablation_variants
    from paper_2508_20274_b200.sweep import run_sweep

    seeds = list(range(1, 11))
    one = run_sweep(PATH, ablation_variants()[:1], seeds)["variants"][0]
    mgr = mp.Manager()
    out = mgr.dict()
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, seeds, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    for r in range(2):
        rows, hist, ci = out[r]
        assert (rows.view(np.uint64) == one["rows"].view(np.uint64)).all()
        assert (hist == one["miss_histogram"]).all()
        assert tuple(ci) == tuple(one["p99_ci"])
