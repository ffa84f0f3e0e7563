"""GPU: the compiled drop-in.  The reference's own C++ API, linked against the B200 shim
(paper_2508_20274_b200/shim/migsim_ref_shim.cpp: engine::run_scenario + harness::run_plan over
the C-ABI, specs crossing in memory via migsim_gpu_load_spec), against the unmodified reference
in the same process (oracle/_ref/shim_parity: every RunResult / ExperimentResult field bit-exact),
and the reference's unmodified tests/acceptance.cpp run on GPU output vs on its own CPU output
(oracle/_ref/acceptance_gpu vs acceptance_cpu, /root/reference/proj/tests/acceptance.cpp:212-556).

The binaries are built where /root/reference is mounted (oracle/Makefile `shim`, called by
__graft_entry__.build()) and travel prebuilt to the GPU box."""
import os
import re
import subprocess

import pytest

from oracle.json_scenarios import write_dir
from tests._libs import CONFIG_SCENARIOS, GOLDEN_SCENARIOS, ROOT

pytestmark = pytest.mark.gpu

BIN = os.path.join(ROOT, "oracle", "_ref")


@pytest.fixture(scope="module")
def jscen(tmp_path_factory):
    return write_dir(str(tmp_path_factory.mktemp("jscen")), GOLDEN_SCENARIOS + CONFIG_SCENARIOS)


def _run(args, cwd=None, timeout=1500):
    exe = os.path.join(BIN, args[0])
    assert os.path.exists(exe), f"{exe} missing: build with `make -C oracle shim` where /root/reference is mounted"
    p = subprocess.run([exe] + args[1:], cwd=cwd, capture_output=True, text=True, timeout=timeout)
    return p.returncode, p.stdout + p.stderr


@pytest.mark.parametrize("name,seed,n,keep", [("default.yaml", 1, 3, ""), ("llm.yaml", 5, 2, "keep"),
                                              ("c2_cluster16.yaml", 9, 1, ""), ("unstable.yaml", 2, 1, ""),
                                              ("c1_single_host.yaml", 3, 1, "keep")])
def test_shim_run_scenario_bit_exact(jscen, name, seed, n, keep):
    rc, out = _run(["shim_parity", "run", os.path.join(jscen, name), str(seed), str(n)] + ([keep] if keep else []))
    assert rc == 0 and out.strip().splitlines()[-1].startswith("OK"), out[-3000:]


@pytest.mark.parametrize("plan,name", [("e1", "default.yaml"), ("e2", "default.yaml"), ("e3", "default.yaml"),
                                       ("llm", "llm.yaml")])
def test_shim_run_plan_bit_exact(jscen, plan, name):
    rc, out = _run(["shim_parity", "plan", plan, os.path.join(jscen, name), "3"])
    assert rc == 0 and out.strip().splitlines()[-1].startswith("OK"), out[-3000:]


def test_shim_in_memory_spec_edits(jscen):
    rc, out = _run(["shim_parity", "spec", os.path.join(jscen, "default.yaml")])
    assert rc == 0 and out.strip().splitlines()[-1].startswith("OK"), out[-3000:]


def _verdicts(text):
    return {m.group(1): m.group(2) for m in re.finditer(r"^(C\d+)\s+(PASS|FAIL)", text, re.M)}


def test_reference_acceptance_on_gpu_output(jscen, tmp_path):
    """acceptance.cpp C1-C10 on GPU results: the same verdict per criterion as the reference's own
    CPU run (C10 fails in the reference too)."""
    (tmp_path / "gpu").mkdir()
    (tmp_path / "cpu").mkdir()
    rc_g, out_g = _run(["acceptance_gpu", jscen], cwd=str(tmp_path / "gpu"))
    rc_c, out_c = _run(["acceptance_cpu", jscen], cwd=str(tmp_path / "cpu"))
    vg, vc = _verdicts(out_g), _verdicts(out_c)
    assert len(vc) == 10 and vg == vc, f"gpu:\n{out_g}\ncpu:\n{out_c}"
    assert all(vg[c] == "PASS" for c in ("C4", "C5", "C6", "C7", "C8", "C9")), out_g
    # the criteria lines carry the same statistics except wall times
    strip = lambda s: re.sub(r"wall [0-9.e+-]+s", "wall", s)  # noqa: E731
    lines = lambda s: [strip(x) for x in s.splitlines() if re.match(r"^C\d+ ", x)]  # noqa: E731
    assert lines(out_g) == lines(out_c), f"gpu:\n{out_g}\ncpu:\n{out_c}"
