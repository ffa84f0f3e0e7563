"""GPU unit parity of the individual kernels: glibc-exact device math, the arrival-stream
generator, and the nearest-rank radix select."""
import ctypes
import json

import numpy as np
import pytest

from oracle import restate
from tests._libs import CONFIG_SCENARIOS, GOLDEN_SCENARIOS, oracle, scenario_json
from tests.test_host_logic import LIBM, _math_inputs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fn", [0, 1, 2])
def test_device_libm_bit_exact(engine, fn):
    rng = np.random.default_rng(7 + fn)
    x = np.ascontiguousarray(_math_inputs(400000, rng))
    y = np.ascontiguousarray(rng.uniform(0.5, 3.0, len(x))) if fn == 2 else None
    if fn == 2:
        x = np.ascontiguousarray(np.abs(x))
    out = np.zeros_like(x)
    lib = engine._lib
    lib.migsim_gpu_libm.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_size_t, ctypes.c_char_p, ctypes.c_size_t]
    err = ctypes.create_string_buffer(512)
    assert lib.migsim_gpu_libm(engine._h, fn, x.ctypes.data, None if y is None else y.ctypes.data, out.ctypes.data,
                               len(x), err, 512) == 0, err.value
    sample = slice(None, None, 7)
    xs = x[sample]
    ref = (np.array([LIBM.pow(a, b) for a, b in zip(xs, y[sample])]) if fn == 2
           else np.array([[LIBM.log, LIBM.exp][fn](a) for a in xs]))
    o = out[sample]
    same = (o.view(np.uint64) == ref.view(np.uint64)) | (np.isnan(o) & np.isnan(ref))
    assert same.all(), (xs[~same][:4], o[~same][:4], ref[~same][:4])


def test_device_fmod_fast_exact(engine):
    """the event loop's schedule phase (fmod_fast, arrivals.h sched_active) vs C fmod, on the device"""
    from tests.test_host_logic import _fmod_inputs

    x, y = _fmod_inputs(400000, np.random.default_rng(12))
    out = np.zeros_like(x)
    lib = engine._lib
    lib.migsim_gpu_libm.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_size_t, ctypes.c_char_p, ctypes.c_size_t]
    err = ctypes.create_string_buffer(512)
    assert lib.migsim_gpu_libm(engine._h, 3, x.ctypes.data, y.ctypes.data, out.ctypes.data, len(x), err, 512) == 0
    ref = np.fmod(x, y)
    same = (out.view(np.uint64) == ref.view(np.uint64)) | (np.isnan(out) & np.isnan(ref))
    assert same.all(), (x[~same][:5], y[~same][:5], out[~same][:5], ref[~same][:5])


def _arrivals_match(engine, path, seeds):
    """Every tenant's device arrival records (time, bytes, service multiplier, noise) equal the
    reference's ArrivalGen stream (workload.cpp:103-157) bit for bit."""
    lib = engine._lib
    lib.migsim_gpu_arrivals.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64, ctypes.c_int32,
                                        ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64),
                                        ctypes.c_char_p, ctypes.c_size_t]
    sid = engine.load_scenario(path)
    ids = engine.tenant_ids(sid)
    spec = json.loads(ctypes.string_at(oracle().ref_scenario_dump(scenario_json(path), b"x")).decode())
    total = 0
    for seed in seeds:
        for ti, tid in enumerate(ids):
            cap = 2_000_000
            ref = np.zeros((cap, 4))
            n = oracle().ref_generate_arrivals(scenario_json(path), tid.encode(), seed, spec["duration_s"],
                                               ref.ctypes.data, cap)
            mine = np.zeros((cap, 4))
            m = ctypes.c_int64()
            err = ctypes.create_string_buffer(512)
            assert lib.migsim_gpu_arrivals(engine._h, sid, seed, ti, mine.ctypes.data, cap, ctypes.byref(m), err,
                                           512) == 0, err.value
            assert m.value == n, (path, tid, seed)
            assert (ref[:n].view(np.uint64) == mine[:n].view(np.uint64)).all(), (path, tid, seed)
            total += n
    return total


def test_device_arrivals_fuzz(engine, tmp_path):
    """The generator's speculative scan / call walk / ordered clock over the fuzz corpus: gamma shapes
    below and above 1 (arrival_cv 0.5-1.5: the pow boost on and off), deterministic clocks, phase and
    square-wave thinning, size mixes, service and noise marks; 3 seeds per scenario."""
    from tests.fuzz_scenarios import make_scenario

    total = 0
    for k in range(80):
        path = str(tmp_path / f"a{k}.yaml")
        with open(path, "w") as f:
            f.write(make_scenario(7000 + k, wide=k % 4 == 3))
        total += _arrivals_match(engine, path, (1 + k % 7, 40 + k, 1000 + 3 * k))
    assert total > 0


@pytest.mark.parametrize("path", GOLDEN_SCENARIOS + CONFIG_SCENARIOS)
def test_device_arrivals_bit_exact(engine, path):
    _arrivals_match(engine, path, (1, 23))


def test_select_matches_nearest_rank(engine):
    rng = np.random.default_rng(11)
    segs = [
        np.zeros(0),
        np.array([3.5]),
        np.array([2.0, 2.0, 2.0, 2.0]),
        rng.lognormal(1.0, 1.0, 1000),
        rng.lognormal(0.5, 0.3, 58_640),
        np.round(rng.uniform(0, 50, 200_000), 1),  # heavy ties
        rng.normal(0.0, 1.0, 5000),  # negative values too
        np.full(3000, 7.25),
        np.concatenate([np.full(5000, 1.0), [1e300, -1e-300, 0.0]]),
    ]
    qs = [0.0, 0.01, 0.5, 0.95, 0.99, 0.999, 1.0]
    out, ms = engine.select(segs, qs)
    for s, row in zip(segs, out):
        for q, v in zip(qs, row):
            expect = restate.nearest_rank(s.tolist(), q) if len(s) else 0.0
            assert v == expect, (len(s), q, v, expect)
    assert ms > 0


def test_select_many_segments_shared_groups(engine):
    """Many large segments where several quantiles land in the same digit group (bimodal data with
    heavy ties, like a deterministic-service tenant's latencies): exercises concurrent refinement
    of quantiles that share a group -- the pattern that once raced on the shared quantile state."""
    rng = np.random.default_rng(558)
    segs = []
    for k in range(300):
        n = int(rng.integers(4097, 30_000))
        lo = np.round(2.45 + rng.exponential(0.01, n), 4)
        hi = np.round(7.6 + rng.exponential(0.5, n), 3)
        pick = rng.random(n) < rng.choice([0.005, 0.01, 0.012, 0.02])
        segs.append(np.where(pick, hi, lo))
    qs = [0.5, 0.95, 0.99, 0.999]
    out, _ = engine.select(segs, qs)
    for s, row in zip(segs, out):
        srt = np.sort(s)
        n = len(s)
        for q, v in zip(qs, row):
            r = min(max(int(np.ceil(q * n)), 1), n) - 1
            assert v == srt[r], (n, q, v, srt[r])


@pytest.mark.parametrize("name", ["c2_cluster16.yaml", "default.yaml", "c5_mc64.yaml"])
def test_select_variants_agree_with_sorted_completions(engine, monkeypatch, name):
    """All three summary-select paths -- the default producer-histogram one-pass select, the
    two-pass digit select (MIGSIM_SELECT=two-pass) and the TMA/DSMEM cluster select
    (MIGSIM_SELECT=cluster) -- return exactly the nearest-rank p50/p95/p99/p999 of the sorted
    measurement-window latencies (engine.cpp:800-816) for every (replica, tenant)."""
    import os

    from tests._libs import CONFIG_DIR, SCEN_DIR

    path = os.path.join(CONFIG_DIR if name.startswith("c") else SCEN_DIR, name)
    sid = engine.load_scenario(path)
    seeds = list(range(1, 9)) if not name.startswith("c5") else [1, 2]
    runs = {}
    for mode in ("default", "two-pass", "cluster"):
        if mode == "default":
            monkeypatch.delenv("MIGSIM_SELECT", raising=False)
        else:
            monkeypatch.setenv("MIGSIM_SELECT", mode)
        runs[mode] = engine.run_batch(sid, seeds, keep_completions=(mode == "default"))
    a = runs["default"]
    try:
        ms = a.run(0)["measure_start_s"]
        for i in range(len(seeds)):
            comp = a.completions(i)
            for t in range(a.n_tenants):
                v = np.sort(comp[(comp[:, 0] == t) & (comp[:, 2] >= ms), 3])
                n = len(v)
                assert n == a.rows[i, t]["completed_window"]
                for q, k in ((0.5, "p50_ms"), (0.95, "p95_ms"), (0.99, "p99_ms"), (0.999, "p999_ms")):
                    if n:
                        r = min(max(int(np.ceil(q * n)), 1), n) - 1
                        assert a.rows[i, t][k] == v[r], (i, t, k)
        for mode in ("two-pass", "cluster"):
            for k in ("p50_ms", "p95_ms", "p99_ms", "p999_ms"):
                assert (a.rows[k].view(np.uint64) == runs[mode].rows[k].view(np.uint64)).all(), (mode, k)
    finally:
        for r in runs.values():
            r.close()
