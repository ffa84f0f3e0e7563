"""Differential fuzzing: randomly generated scenario-v1 documents (tests/fuzz_scenarios.py) run
through the reference engine and through ours -- the CPU-compiled engine logic here, the CUDA
kernels on the GPU -- with bit-exact comparison of every output.  The corpus exercises every
ActionKind (guardrail io/mps, expire, move, mig_up/down, rollback, none), deterministic clocks,
zero-byte transfers, phase and square-wave thinning, MPS devices and drain timeouts."""
import collections

import pytest

from tests._libs import diff_results, hostsim_run, ref_run
from tests.fuzz_scenarios import make_scenario

CPU_SEEDS = range(0, 120)
GPU_SEEDS = range(500, 560)


def _write(tmp_path, seed):
    p = tmp_path / f"fuzz{seed}.yaml"
    p.write_text(make_scenario(seed))
    return str(p)


def test_fuzz_engine_logic_cpu(tmp_path):
    kinds = collections.Counter()
    for seed in CPU_SEEDS:
        path = _write(tmp_path, seed)
        run_seed = seed % 7 + 1
        ref, _ = ref_run(path, run_seed)
        for a in ref["actions"]:
            kinds[a["kind"]] += 1
        assert diff_results(ref, hostsim_run(path, run_seed)) == [], seed
    # the corpus must keep exercising the controller's whole action vocabulary
    for k in ("guardrail_io_throttle", "guardrail_expire", "move", "mig_up", "mig_down", "rollback", "none"):
        assert kinds[k] > 0, k


@pytest.mark.gpu
def test_fuzz_gpu(engine, tmp_path):
    for seed in GPU_SEEDS:
        path = _write(tmp_path, seed)
        sid = engine.load_scenario(path)
        res = engine.run_batch(sid, [seed % 5 + 1, seed % 5 + 2])
        try:
            for i, run_seed in enumerate((seed % 5 + 1, seed % 5 + 2)):
                ref, _ = ref_run(path, run_seed)
                d = diff_results(ref, res.run(i))
                assert d == [], (seed, run_seed, d[:8])
        finally:
            res.close()


WIDE_SEEDS = range(9000, 9030)


def test_fuzz_wide_engine_logic_cpu(tmp_path):
    """11-40 tenants: the event slots live in shared memory (T > 10) on the device."""
    for seed in WIDE_SEEDS[:6]:
        p = tmp_path / f"wide{seed}.yaml"
        p.write_text(make_scenario(seed, wide=True))
        ref, _ = ref_run(str(p), seed % 3 + 1)
        assert diff_results(ref, hostsim_run(str(p), seed % 3 + 1)) == [], seed


@pytest.mark.gpu
def test_fuzz_wide_gpu(engine, tmp_path):
    for seed in WIDE_SEEDS:
        p = tmp_path / f"wide{seed}.yaml"
        p.write_text(make_scenario(seed, wide=True))
        sid = engine.load_scenario(str(p))
        seeds = [seed % 3 + 1, seed % 3 + 2]
        res = engine.run_batch(sid, seeds)
        try:
            for i, s in enumerate(seeds):
                ref, _ = ref_run(str(p), s)
                assert diff_results(ref, res.run(i)) == [], (seed, s)
        finally:
            res.close()
