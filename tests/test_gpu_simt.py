"""GPU parity of the SIMT DES (one thread per replica, des_simt_kernel) forced on small batches with
MIGSIM_DES=simt -- the form large batches (the C4 headline) run in -- bit-exact against the compiled
reference, plus identity with the warp form on a larger batch."""
import os

import numpy as np
import pytest

from tests._libs import CONFIG_SCENARIOS, GOLDEN_SCENARIOS, diff_results, ref_run
from tests.fuzz_scenarios import make_scenario
from tests.test_gpu_parity_wide import ABLATION, _check_batch

pytestmark = pytest.mark.gpu


@pytest.fixture
def simt(monkeypatch):
    monkeypatch.setenv("MIGSIM_DES", "simt")


@pytest.mark.parametrize("path", GOLDEN_SCENARIOS[:2] + GOLDEN_SCENARIOS[3:] + CONFIG_SCENARIOS)
def test_simt_scenarios_ablation(engine, simt, path):
    seeds = [1, 2] if "c2" not in path else [1]
    _check_batch(engine, path, seeds, ABLATION)


def test_simt_stability_full(engine, simt):
    _check_batch(engine, GOLDEN_SCENARIOS[2], [1], ABLATION[:1])


def test_simt_fuzz(engine, simt, tmp_path):
    for seed in list(range(700, 730)) + [9000, 9001, 9002]:
        p = tmp_path / f"s{seed}.yaml"
        p.write_text(make_scenario(seed, wide=seed >= 9000))
        _check_batch(engine, str(p), [seed % 4 + 1, seed % 4 + 2, seed % 4 + 3], None)


def test_simt_per_completion_records(engine, simt):
    path = GOLDEN_SCENARIOS[1]
    sid = engine.load_scenario(path)
    res = engine.run_batch(sid, [5, 6], keep_completions=True)
    try:
        for i, seed in enumerate((5, 6)):
            comps = res.completions(i)
            ref, rc = ref_run(path, seed, keep_completions=True)
            assert diff_results(ref, res.run(i)) == []
            for ti in range(len(res.tenant_ids)):
                mine = comps[comps[:, 0] == ti]
                sel = rc["tenant"] == ti
                order = np.argsort(rc["seq"][sel], kind="stable")
                for col, key in ((2, "done"), (3, "total"), (4, "compute"), (5, "transfer"), (6, "noise")):
                    assert (rc[key][sel][order].view(np.uint64) == mine[:, col].view(np.uint64)).all()
    finally:
        res.close()


def test_simt_artifacts_with_traces(engine, simt, tmp_path):
    from tests.test_artifacts import FILES, _ref_artifacts, _same_files

    path = GOLDEN_SCENARIOS[0]
    ref, mine = tmp_path / "ref", tmp_path / "mine"
    _ref_artifacts(path, 2, ref)
    sid = engine.load_scenario(path)
    engine.run_scenario(sid, 2, out_dir=str(mine), write_traces=True)
    assert _same_files(ref, mine, FILES) == []


def test_simt_equals_warp_form(engine, monkeypatch):
    """Both DES forms over the same 4-variant batch of 512 default.yaml replicas: identical rows and
    action logs."""
    from paper_2508_20274_b200 import Variant

    vs = [Variant(n, **ov) for n, ov in ABLATION if n != "guards-only"]
    sid = engine.load_scenario(GOLDEN_SCENARIOS[0])
    outs = {}
    for mode in ("warp", "simt"):
        monkeypatch.setenv("MIGSIM_DES", mode)
        res = engine.run_batch(sid, list(range(1, 129)), vs)
        assert (res.timing["des_form"] == 1) == (mode == "simt")
        outs[mode] = (res.rows.copy(), [res.run(k)["actions"] for k in range(0, res.n_runs, 7)])
        res.close()
    assert (outs["warp"][0].view(np.uint8) == outs["simt"][0].view(np.uint8)).all()
    assert outs["warp"][1] == outs["simt"][1]
