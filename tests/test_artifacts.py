"""Run artifacts byte-identical to the reference's writers.

engine::run_scenario(spec, RunOptions{seed, out_dir, write_traces=true}) writes requests.csv,
counters.csv, fabric.csv (engine.cpp:279-288, :503, :744-775; trace.cpp:24-96, "%.9g"),
actions.jsonl and summary.json (engine.cpp:889-892; trace.cpp:98-203, nlohmann ordered_json).
The oracle is the reference itself (oracle/_ref, its own trace.cpp).  CPU tests drive the engine
logic through the test-only host harness (tests/native/hostsim.cpp); GPU tests drive the product
C-ABI (migsim_gpu_run_scenario).  Acceptance C5 (acceptance.cpp: byte-identical artifacts across
two runs of one seed) is checked on the GPU path too.
"""
import filecmp
import os

import pytest

from tests._libs import CONFIG_SCENARIOS, GOLDEN_SCENARIOS, hostsim, oracle, scenario_json

FILES = ("requests.csv", "counters.csv", "fabric.csv", "actions.jsonl", "summary.json")


def _ref_artifacts(path, seed, out_dir, traces=True):
    lib = oracle()
    assert lib.ref_run_artifacts(scenario_json(path), None, seed, str(out_dir).encode(), int(traces)) == 0, \
        lib.ref_last_error()


def _same_files(a, b, names):
    bad = []
    for f in names:
        pa, pb = os.path.join(a, f), os.path.join(b, f)
        if not os.path.exists(pb):
            bad.append((f, "missing"))
        elif not filecmp.cmp(pa, pb, shallow=False):
            with open(pa, "rb") as x, open(pb, "rb") as y:
                la, lb = x.read().split(b"\n"), y.read().split(b"\n")
            first = next((i for i, (u, v) in enumerate(zip(la, lb)) if u != v), min(len(la), len(lb)))
            bad.append((f, first, la[first][:120] if first < len(la) else b"<eof>",
                        lb[first][:120] if first < len(lb) else b"<eof>"))
    return bad


CPU_CASES = [(p, 1) for p in GOLDEN_SCENARIOS + CONFIG_SCENARIOS[:1]] + [(GOLDEN_SCENARIOS[1], 4)]


@pytest.mark.parametrize("path,seed", CPU_CASES, ids=[f"{os.path.basename(p)}-s{s}" for p, s in CPU_CASES])
def test_host_harness_artifacts_byte_identical(tmp_path, path, seed):
    ref, mine = tmp_path / "ref", tmp_path / "mine"
    _ref_artifacts(path, seed, ref)
    p = hostsim().hostsim_run_artifacts(path.encode(), seed, str(mine).encode())
    assert p, hostsim().hostsim_last_error()
    hostsim().hostsim_free(p)
    assert sorted(os.listdir(ref)) == sorted(FILES)
    assert _same_files(ref, mine, FILES) == []


GPU_CASES = [(p, s) for p in GOLDEN_SCENARIOS for s in (1, 2)] + [(p, 1) for p in CONFIG_SCENARIOS]


@pytest.mark.gpu
@pytest.mark.parametrize("path,seed", GPU_CASES, ids=[f"{os.path.basename(p)}-s{s}" for p, s in GPU_CASES])
def test_gpu_artifacts_byte_identical(engine, tmp_path, path, seed):
    ref, mine = tmp_path / "ref", tmp_path / "mine"
    _ref_artifacts(path, seed, ref)
    sid = engine.load_scenario(path)
    res = engine.run_scenario(sid, seed, out_dir=str(mine), write_traces=True)
    assert res["seed"] == seed
    assert _same_files(ref, mine, FILES) == []


@pytest.mark.gpu
def test_gpu_artifacts_without_traces_and_determinism(engine, tmp_path):
    """write_traces=false writes only actions.jsonl + summary.json (engine.cpp:282); two runs of
    one seed are byte-identical (acceptance C5)."""
    path = GOLDEN_SCENARIOS[0]
    ref, a, b = tmp_path / "ref", tmp_path / "a", tmp_path / "b"
    _ref_artifacts(path, 7, ref, traces=False)
    sid = engine.load_scenario(path)
    engine.run_scenario(sid, 7, out_dir=str(a), write_traces=False)
    engine.run_scenario(sid, 7, out_dir=str(b), write_traces=False)
    assert sorted(os.listdir(a)) == sorted(os.listdir(ref)) == ["actions.jsonl", "summary.json"]
    assert _same_files(ref, a, ["actions.jsonl", "summary.json"]) == []
    assert _same_files(a, b, ["actions.jsonl", "summary.json"]) == []


# ---- harness plans: experiment.json / summary.csv / per-job artifacts, render_report ----------

def _ref_plan(plan, path, seeds, seed_base, out_dir, tmp_path):
    """harness::run_plan of the reference (PlanOptions with out_dir); returns experiment json."""
    import ctypes
    import json

    jpath = tmp_path / "scenario.json"
    jpath.write_bytes(scenario_json(path))
    lib = oracle()
    p = lib.ref_run_plan(plan.encode(), str(jpath).encode(), seeds, seed_base, None,
                         str(out_dir).encode() if out_dir else None, 0)
    assert p, lib.ref_last_error()
    try:
        return json.loads(ctypes.string_at(p).decode())
    finally:
        lib.ref_free(p)


def test_render_report_matches_reference(tmp_path):
    """render_report (harness.cpp:285-313) is host code: our C-ABI formats the reference's own
    experiment.json exactly like the reference (no GPU needed)."""
    import ctypes
    import json

    from paper_2508_20274_b200 import render_report

    exp = _ref_plan("e1", GOLDEN_SCENARIOS[1], 2, 5, None, tmp_path)
    text = json.dumps(exp)
    lib = oracle()
    p = lib.ref_render_report(text.encode())
    assert p, lib.ref_last_error()
    ref = ctypes.string_at(p).decode()
    lib.ref_free(p)
    assert render_report(text) == ref
    assert "vs static" in ref


@pytest.mark.gpu
@pytest.mark.parametrize("plan", ["e1", "e2", "e3", "llm"])
def test_gpu_plan_artifacts_match_reference(engine, tmp_path, plan):
    """run_plan with out_dir: summary.csv and every <variant>/seed<N>/ file byte-identical to the
    reference harness; experiment.json identical except the wall-clock field."""
    import json

    path = GOLDEN_SCENARIOS[1]
    ref_dir, my_dir = tmp_path / "ref", tmp_path / "mine"
    _ref_plan(plan, path, 3, 21, ref_dir, tmp_path)
    mine = engine.run_plan(plan, path, seeds=3, seed_base=21, out_dir=str(my_dir))
    assert _same_files(ref_dir, my_dir, ["summary.csv"]) == []
    rj = json.loads((ref_dir / "experiment.json").read_text())
    mj = json.loads((my_dir / "experiment.json").read_text())
    rj.pop("wall_s"), mj.pop("wall_s"), mine.pop("wall_s")
    assert rj == mj == mine
    runs = 0
    for v in os.listdir(ref_dir):
        if not (ref_dir / v).is_dir():
            continue
        for sd in os.listdir(ref_dir / v):
            assert _same_files(ref_dir / v / sd, my_dir / v / sd, ["actions.jsonl", "summary.json"]) == []
            runs += 1
    assert runs == 3 * len(mine["variants"])
