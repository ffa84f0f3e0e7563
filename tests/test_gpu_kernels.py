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


@pytest.mark.parametrize("path", GOLDEN_SCENARIOS + CONFIG_SCENARIOS)
def test_device_arrivals_bit_exact(engine, path):
    lib = engine._lib
    lib.migsim_gpu_arrivals.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64, ctypes.c_int32,
                                        ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64),
                                        ctypes.c_char_p, ctypes.c_size_t]
    sid = engine.load_scenario(path)
    ids = engine.tenant_ids(sid)
    spec = json.loads(ctypes.string_at(oracle().ref_scenario_dump(scenario_json(path), b"x")).decode())
    for seed in (1, 23):
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
            assert m.value == n
            assert (ref[:n].view(np.uint64) == mine[:n].view(np.uint64)).all(), (tid, seed)


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


def test_cluster_select_matches_two_pass(engine, monkeypatch):
    """The one-HBM-pass cluster select (MIGSIM_SELECT=cluster: TMA bulk loads, DSMEM histogram and
    gather) returns exactly the two-pass kernel's p50/p95/p99/p999 on every segment of a wave."""
    import os

    from tests._libs import CONFIG_DIR

    path = os.path.join(CONFIG_DIR, "c2_cluster16.yaml")
    sid = engine.load_scenario(path)
    seeds = list(range(1, 17))
    a = engine.run_batch(sid, seeds)
    monkeypatch.setenv("MIGSIM_SELECT", "cluster")
    b = engine.run_batch(sid, seeds)
    try:
        for k in ("p50_ms", "p95_ms", "p99_ms", "p999_ms"):
            assert (a.rows[k].view(np.uint64) == b.rows[k].view(np.uint64)).all(), k
        assert (a.rows["completed_window"] == b.rows["completed_window"]).all()
    finally:
        a.close()
        b.close()
