"""GPU parity of the register-capped DES (des_kernel_reg_occ, 64 registers, 32 resident warps/SM) --
the form saturated batches such as the C4 headline run in -- forced on small batches with
MIGSIM_DES_REGS=capped, bit-exact against the compiled reference, plus identity with the uncapped
kernel on a 4-variant batch."""
import numpy as np
import pytest

from tests._libs import CONFIG_SCENARIOS, GOLDEN_SCENARIOS
from tests.fuzz_scenarios import make_scenario
from tests.test_gpu_parity_wide import ABLATION, _check_batch

pytestmark = pytest.mark.gpu


@pytest.fixture
def capped(monkeypatch):
    monkeypatch.setenv("MIGSIM_DES_REGS", "capped")


@pytest.mark.parametrize("path", GOLDEN_SCENARIOS + CONFIG_SCENARIOS)
def test_capped_scenarios_ablation(engine, capped, path):
    seeds = [1, 2] if "c2" not in path else [1]
    _check_batch(engine, path, seeds, ABLATION)


def test_capped_fuzz(engine, capped, tmp_path):
    for seed in list(range(740, 770)):
        p = tmp_path / f"s{seed}.yaml"
        p.write_text(make_scenario(seed))
        _check_batch(engine, str(p), [seed % 4 + 1, seed % 4 + 2], None)


def test_capped_equals_uncapped(engine, monkeypatch):
    """Both register forms over the same 4-variant batch of default.yaml replicas: identical rows,
    action logs and per-(variant, tenant) latency histograms."""
    from paper_2508_20274_b200 import Variant

    vs = [Variant(n, **ov) for n, ov in ABLATION if n != "guards-only"]
    sid = engine.load_scenario(GOLDEN_SCENARIOS[0])
    outs = {}
    for mode in ("full", "capped"):
        monkeypatch.setenv("MIGSIM_DES_REGS", mode)
        res = engine.run_batch(sid, list(range(1, 193)), vs)
        assert (res.timing["des_form"] == 2) == (mode == "capped")
        outs[mode] = (res.rows.copy(), [res.run(k)["actions"] for k in range(0, res.n_runs, 5)],
                      res.latency_hist().copy())
        res.close()
    assert (outs["full"][0].view(np.uint8) == outs["capped"][0].view(np.uint8)).all()
    assert outs["full"][1] == outs["capped"][1]
    assert (outs["full"][2] == outs["capped"][2]).all()
