"""CPU coverage of the audit bridge used on GPU logs (tests._libs.ref_audit_gpu): the reference's own
audit::audit_run (audit.cpp:52-122) over an engine RunResult JSON -- here produced by the host
harness of the engine logic -- returns exactly what it returns over the reference's own run."""
import pytest

from tests._libs import GOLDEN_SCENARIOS, hostsim_run, ref_audit_gpu, ref_audit_ref
from tests.fuzz_scenarios import make_scenario


@pytest.mark.parametrize("seed", [1, 2])
def test_audit_bridge_default(seed):
    for ov in (None, dict(enabled=True, enable_mig=True, enable_placement=False, enable_guardrails=False)):
        mine = hostsim_run(GOLDEN_SCENARIOS[0], seed, ov)
        assert ref_audit_gpu(GOLDEN_SCENARIOS[0], mine, ov) == ref_audit_ref(GOLDEN_SCENARIOS[0], seed, ov) == []


def test_audit_bridge_flags_identically_on_fuzz(tmp_path):
    flagged = 0
    for seed in range(300, 312):
        p = tmp_path / f"f{seed}.yaml"
        p.write_text(make_scenario(seed))
        a = ref_audit_gpu(str(p), hostsim_run(str(p), 1))
        assert a == ref_audit_ref(str(p), 1), seed
        flagged += bool(a)
