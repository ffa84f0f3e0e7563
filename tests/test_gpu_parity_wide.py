"""GPU parity on the configurations the bench and the scaling claims run (round-2 pinning).

Every comparison is bit-exact against the compiled reference (oracle/_ref), like test_gpu_parity.py:
  * C2 (bench shape): 16 seeds spread over 1..2048 (the seed range an 8-GPU weak-scaling run of
    256 seeds/GPU covers) under the full controller, plus all 5 ablation variants for 2 seeds;
  * C4 (the N=1 headline): default.yaml x {static, mig-only, placement-only, full}, seeds spread
    over 1..16384 in one batch;
  * C5: 8 seeds of the 64-tenant Monte Carlo scenario (T = 64 is the engine's hard limit);
  * random 41-64-tenant scenarios (tests/fuzz_scenarios.py xwide);
  * the reference's audit::audit_run (audit.cpp:52-122) over GPU action logs == over its own logs;
  * wave splitting (max_wave_replicas 1 / 3 / auto) and mixed per-variant ring strides (e3 knobs)
    give identical results.
Reference runs execute on every host core (tests._libs.ref_runs_parallel).
"""
import os

import numpy as np
import pytest

from tests._libs import (CONFIG_DIR, CONFIG_SCENARIOS, GOLDEN_SCENARIOS, diff_results, ref_audit_gpu, ref_audit_ref,
                         ref_runs_parallel)
from tests.fuzz_scenarios import make_scenario

pytestmark = pytest.mark.gpu

ABLATION = [
    ("full", dict(enabled=True, enable_mig=True, enable_placement=True, enable_guardrails=True)),
    ("mig-only", dict(enabled=True, enable_mig=True, enable_placement=False, enable_guardrails=False)),
    ("placement-only", dict(enabled=True, enable_mig=False, enable_placement=True, enable_guardrails=False)),
    ("guards-only", dict(enabled=True, enable_mig=False, enable_placement=False, enable_guardrails=True)),
    ("static", dict(enabled=False, enable_mig=False, enable_placement=False, enable_guardrails=False)),
]
C4 = [v for v in ABLATION if v[0] in ("static", "mig-only", "placement-only", "full")]


def _variants(spec):
    from paper_2508_20274_b200 import Variant

    return [Variant(n, **v) for n, v in spec]


def _check_batch(engine, path, seeds, variants):
    """One batched GPU call over variants x seeds, every run diffed against the reference."""
    sid = engine.load_scenario(path)
    res = engine.run_batch(sid, seeds, _variants(variants) if variants else None)
    try:
        jobs = [(path, s, ov) for _, ov in (variants or [("as-is", None)]) for s in seeds]
        refs = ref_runs_parallel(jobs)
        bad = []
        for k, ref in enumerate(refs):
            d = diff_results(ref, res.run(k))
            if d:
                bad.append((jobs[k][1], jobs[k][2], d[:4]))
        assert bad == []
        return res.rows.copy()
    finally:
        res.close()


C2_SEEDS = [1, 2, 3, 64, 129, 256, 257, 511, 700, 1024, 1025, 1300, 1536, 1800, 2047, 2048]


def test_c2_seeds_across_weak_scaling_range(engine):
    _check_batch(engine, CONFIG_SCENARIOS[1], C2_SEEDS, [ABLATION[0]])


def test_c2_all_ablation_variants(engine):
    _check_batch(engine, CONFIG_SCENARIOS[1], [7, 1500], ABLATION)


def test_c4_headline_mix(engine):
    """The bench headline's replica mix (BASELINE configs[3]): 4 variants, seeds across 1..16384."""
    _check_batch(engine, GOLDEN_SCENARIOS[0], [1, 4096, 9999, 16384], C4)


def test_c5_eight_seeds(engine):
    _check_batch(engine, os.path.join(CONFIG_DIR, "c5_mc64.yaml"), list(range(1, 9)), None)


XWIDE_SEEDS = range(9100, 9116)


def test_fuzz_41_to_64_tenants(engine, tmp_path):
    for seed in XWIDE_SEEDS:
        p = tmp_path / f"xwide{seed}.yaml"
        p.write_text(make_scenario(seed, xwide=True))
        _check_batch(engine, str(p), [seed % 3 + 1, seed % 3 + 2], None)


AUDIT_CASES = [(GOLDEN_SCENARIOS[0], s, n, ov) for s in (1, 2, 3) for n, ov in ABLATION] + \
              [(GOLDEN_SCENARIOS[1], s, n, ov) for s in (1, 2) for n, ov in ABLATION[:1] + ABLATION[-1:]]


def test_reference_audit_on_gpu_logs(engine):
    """Acceptance C4 (acceptance.cpp:212-235) on GPU output: the reference's audit_run over every
    E1/E2-style run of default.yaml (and llm.yaml) gives the same verdict as over the reference's
    own run -- clean in every case."""
    for path, seed, name, ov in AUDIT_CASES:
        from paper_2508_20274_b200 import Variant

        sid = engine.load_scenario(path)
        res = engine.run_batch(sid, [seed], [Variant(name, **ov)])
        mine = res.run(0)
        res.close()
        assert ref_audit_gpu(path, mine, ov) == ref_audit_ref(path, seed, ov) == [], (path, seed, name)


def test_reference_audit_flags_same_issues_on_fuzz(engine, tmp_path):
    """Aggressive fuzz controllers (short dwell, cooldown 0) -- the audit verdicts, including any
    flagged issues, are identical for the GPU logs and the reference logs."""
    n_issue_runs = 0
    for seed in range(300, 340):
        p = tmp_path / f"f{seed}.yaml"
        p.write_text(make_scenario(seed))
        sid = engine.load_scenario(str(p))
        res = engine.run_batch(sid, [1])
        mine = res.run(0)
        res.close()
        a, b = ref_audit_gpu(str(p), mine), ref_audit_ref(str(p), 1)
        assert a == b, seed
        n_issue_runs += bool(a)
    print(f"audit: {n_issue_runs} of 40 fuzz runs flag issues (identically on both engines)")


def test_wave_split_and_mixed_ring_strides_identical(engine):
    """Same batch with max_wave_replicas 1, 3 and auto: identical rows, actions and pauses (buffer
    reuse across waves); the e3 knobs give variants different dwell/validation ring sizes in one
    batch (ring stride = max over variants)."""
    from paper_2508_20274_b200 import Variant

    path = GOLDEN_SCENARIOS[1]
    vs = [Variant("dwell=128", dwell_obs=128, cooldown_obs=64), Variant("dwell=512", dwell_obs=512, cooldown_obs=256),
          Variant("interval=2s", sample_interval_s=2.0), Variant("v=16", validation_obs=16)]
    sid = engine.load_scenario(path)
    outs = []
    for w in (1, 3, 0):
        res = engine.run_batch(sid, [3, 4, 5], vs, max_wave_replicas=w)
        outs.append((res.rows.copy(), [res.run(k) for k in range(res.n_runs)]))
        res.close()
    for rows, runs in outs[1:]:
        assert (rows.view(np.uint8) == outs[0][0].view(np.uint8)).all()
        assert runs == outs[0][1]
    ovs = [dict(dwell_obs=128, cooldown_obs=64), dict(dwell_obs=512, cooldown_obs=256), dict(sample_interval_s=2.0),
           dict(validation_obs=16)]
    refs = ref_runs_parallel([(path, s, ov) for ov in ovs for s in (3, 4, 5)])
    for k, ref in enumerate(refs):
        assert diff_results(ref, outs[0][1][k]) == [], k


def test_invalid_variant_knobs_raise(engine):
    """Only None keeps the scenario value: dwell_obs=0 / sample_interval_s=0 reach
    ControllerConfig::validate and fail like the reference (model.cpp:184-206)."""
    from paper_2508_20274_b200 import ConfigError, Variant

    sid = engine.load_scenario(GOLDEN_SCENARIOS[1])
    for bad in (Variant("d0", dwell_obs=0), Variant("s0", sample_interval_s=0.0), Variant("v0", validation_obs=0),
                Variant("c-1", cooldown_obs=-1)):
        with pytest.raises(ConfigError):
            engine.run_batch(sid, [1], [bad])
