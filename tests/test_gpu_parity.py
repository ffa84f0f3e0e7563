"""GPU parity: the sm_100a engine through its C-ABI vs the compiled reference, bit-exact.

Outputs compared (north_star bar): action sequences (kind, tenant, target, t_s, placement detail,
p99/EMA at decision, breach windows, obs counters, pauses, rollbacks), percentile values (nearest
rank -> indices bit-exact), SLO-miss and completion counts, end states, stability flags and notes.
FP64 values are required bit-identical (stricter than the 1e-9 relative the spec allows).
"""
import ctypes
import os

import numpy as np
import pytest

from oracle import restate
from tests._libs import CONFIG_DIR, CONFIG_SCENARIOS, GOLDEN_SCENARIOS, diff_results, oracle, ref_run, scenario_json

pytestmark = pytest.mark.gpu

VARIANTS = [
    ("full", dict(enabled=True, enable_mig=True, enable_placement=True, enable_guardrails=True)),
    ("mig-only", dict(enabled=True, enable_mig=True, enable_placement=False, enable_guardrails=False)),
    ("placement-only", dict(enabled=True, enable_mig=False, enable_placement=True, enable_guardrails=False)),
    ("guards-only", dict(enabled=True, enable_mig=False, enable_placement=False, enable_guardrails=True)),
    ("static", dict(enabled=False, enable_mig=False, enable_placement=False, enable_guardrails=False)),
]


def _variants():
    from paper_2508_20274_b200 import Variant

    return [Variant(n, **v) for n, v in VARIANTS]


@pytest.mark.parametrize("path", GOLDEN_SCENARIOS + CONFIG_SCENARIOS)
def test_scenarios_all_variants(engine, path):
    """Every shipped scenario + C1..C3, 5-variant ablation grid x 3 seeds in ONE batched call."""
    fast = "stability" not in path and "c2" not in path
    seeds = [1, 2, 3] if fast else [1]
    sid = engine.load_scenario(path)
    res = engine.run_batch(sid, seeds, _variants())
    try:
        for vi, (name, ov) in enumerate(VARIANTS):
            if not fast and name not in ("full", "static"):
                continue
            for si, seed in enumerate(seeds):
                ref, _ = ref_run(path, seed, ov)
                mine = res.run(vi * len(seeds) + si)
                assert diff_results(ref, mine) == [], (name, seed)
    finally:
        res.close()


def test_many_seeds_default(engine):
    """32 seeds of default.yaml in one wave vs the reference (summaries + action logs)."""
    path = GOLDEN_SCENARIOS[0]
    sid = engine.load_scenario(path)
    seeds = list(range(100, 132))
    res = engine.run_batch(sid, seeds)
    try:
        for i in range(0, 32, 4):
            ref, _ = ref_run(path, seeds[i])
            assert diff_results(ref, res.run(i)) == []
    finally:
        res.close()


@pytest.mark.parametrize("path", [GOLDEN_SCENARIOS[1], CONFIG_SCENARIOS[2], GOLDEN_SCENARIOS[0]])
def test_per_completion_records(engine, path):
    """keep_completions: every CompletionRecord (engine.hpp:47-57) bit-exact, plus the p999
    extension against a nearest-rank restatement over the reference's window samples."""
    sid = engine.load_scenario(path)
    res = engine.run_batch(sid, [5], keep_completions=True)
    try:
        comps = res.completions(0)
        run = res.run(0)
        ref, rc = ref_run(path, 5, keep_completions=True)
        ids = res.tenant_ids
        for ti, tid in enumerate(ids):
            mine = comps[comps[:, 0] == ti]
            sel = rc["tenant"] == ti
            assert len(mine) == sel.sum()
            order = np.argsort(rc["seq"][sel], kind="stable")
            for col, key in ((2, "done"), (3, "total"), (4, "compute"), (5, "transfer"), (6, "noise")):
                a = rc[key][sel][order]
                b = mine[:, col]
                assert (a.view(np.uint64) == b.view(np.uint64)).all(), (tid, key)
            ms = ref["summary"]["measure_start_s"]
            win = rc["total"][sel][rc["done"][sel] >= ms]
            if len(win):
                assert run["tenants"][tid]["p999_ms"] == restate.nearest_rank(win.tolist(), 0.999)
    finally:
        res.close()


def test_single_replica_api(engine):
    """paper_2508_20274_b200.run_scenario mirrors engine::run_scenario (engine.hpp:117)."""
    from paper_2508_20274_b200 import run_scenario

    path = GOLDEN_SCENARIOS[1]
    mine = run_scenario(path, seed=9)
    ref, _ = ref_run(path, 9)
    assert diff_results(ref, mine) == []


def test_audit_invariants_hold_on_gpu_runs(engine):
    """audit::audit_run (audit.cpp:52-122), the reference's own code, over the GPU logs == over the
    reference logs (both clean).  More cases in test_gpu_parity_wide.py."""
    from tests._libs import ref_audit_gpu, ref_audit_ref

    path = GOLDEN_SCENARIOS[0]
    sid = engine.load_scenario(path)
    res = engine.run_batch(sid, [3])
    mine = res.run(0)
    res.close()
    assert ref_audit_gpu(path, mine) == ref_audit_ref(path, 3) == []


def test_c5_64_tenants(engine):
    """C5 shape: 64 tenants on 32 GPUs, exhaustive try_move scoring over all GPUs; controller rings
    spill to global memory at this size."""
    path = os.path.join(CONFIG_DIR, "c5_mc64.yaml")
    sid = engine.load_scenario(path)
    res = engine.run_batch(sid, [1])
    try:
        ref, _ = ref_run(path, 1)
        assert len(ref["actions"]) > 100
        assert diff_results(ref, res.run(0)) == []
    finally:
        res.close()


@pytest.mark.parametrize("plan", ["e1", "e2"])
def test_run_plan_matches_reference_harness(engine, plan):
    """harness::run_plan (harness.cpp:114-216): per-seed focus p99/miss, summed throughput and the
    population-sigma CIs summed in seed order, vs reference replicas aggregated by the restatement."""
    path = GOLDEN_SCENARIOS[1]
    exp = engine.run_plan(plan, path, seeds=3, seed_base=11)
    from paper_2508_20274_b200 import ablation_variants, main_variants

    variants = main_variants() if plan == "e1" else ablation_variants()
    assert [v["name"] for v in exp["variants"]] == [v.name for v in variants]
    assert exp["focus_tenant"] == "llm"
    for v, ve in zip(variants, exp["variants"]):
        ov = dict(enabled=v.enabled, enable_mig=v.enable_mig, enable_placement=v.enable_placement,
                  enable_guardrails=v.enable_guardrails)
        p99, miss, thr = [], [], []
        for seed in (11, 12, 13):
            ref, _ = ref_run(path, seed, ov)
            t = ref["summary"]["tenants"]
            p99.append(t["llm"]["p99_ms"])
            miss.append(t["llm"]["miss_rate"])
            s = 0.0
            for tid in sorted(t):
                s += t[tid]["throughput_hz"]
            thr.append(s)
        assert ve["seeds"] == [11, 12, 13]
        assert ve["p99_ms"] == p99 and ve["miss_rate"] == miss and ve["throughput_hz"] == thr
        for key, vals in (("p99_ci", p99), ("miss_ci", miss), ("throughput_ci", thr)):
            m, h = restate.confidence_interval(vals)
            assert ve[key] == {"mean": m, "half_width": h}
