"""Pin the oracle: CPU restatements (oracle/restate.py) against the reference's own known-answer
tests and against the compiled reference itself (oracle/_ref)."""
import ctypes
import math

import numpy as np
import pytest

from oracle import restate
from tests._libs import oracle

# ---- fabric (test_fabric.cpp:38-77 KATs, fabric.cpp:31-87) ---------------------------------


def _ref_alloc(flows, cap, wf):
    lib = oracle()
    n = len(flows)
    w = np.array([f[0] for f in flows], np.float64)
    c = np.array([-1.0 if f[1] is None else f[1] for f in flows], np.float64)
    g = np.zeros(n, np.float64)
    res = ctypes.c_double()
    assert lib.ref_allocate_bandwidth(n, w.ctypes.data, c.ctypes.data, cap, int(wf), g.ctypes.data,
                                      ctypes.byref(res)) == 0
    return list(g), res.value


@pytest.mark.parametrize("flows,cap,wf,expect,residual", [
    ([(1.0, None), (1.0, None)], 16e9, False, [8e9, 8e9], 0.0),
    ([(2.0, None), (1.0, None), (1.0, None)], 16e9, False, [8e9, 4e9, 4e9], 0.0),
    ([(1.0, 2e9), (1.0, None)], 16e9, False, [2e9, 8e9], 6e9),
    ([(1.0, 2e9), (1.0, None)], 16e9, True, [2e9, 14e9], 0.0),
    ([(1.0, 3e9), (1.0, 5e9)], 16e9, True, [3e9, 5e9], 8e9),
])
def test_fabric_kats(flows, cap, wf, expect, residual):
    g, r = restate.allocate_bandwidth(flows, cap, wf)
    for a, b in zip(g, expect):
        assert a == pytest.approx(b, rel=1e-9)
    assert r == pytest.approx(residual, abs=1e-9 * cap)
    assert (g, r) == _ref_alloc(flows, cap, wf)  # bit-exact vs the compiled reference


def test_fabric_property_vs_reference():
    # test_fabric.cpp:86-140 style: 10^3 random epochs, restatement == reference bit for bit,
    # conservation and caps hold
    rng = np.random.default_rng(0xFAB51C)
    for _ in range(1000):
        n = int(rng.integers(1, 9))
        flows = [(float(rng.uniform(0.1, 5.0)), None if rng.random() < 0.4 else float(rng.uniform(1e8, 1e10)))
                 for _ in range(n)]
        cap = float(rng.uniform(1e9, 3e10))
        wf = bool(rng.random() < 0.7)
        g, r = restate.allocate_bandwidth(flows, cap, wf)
        assert (g, r) == _ref_alloc(flows, cap, wf)
        assert abs(sum(g) + r - cap) <= 1e-9 * cap
        for (w, c), x in zip(flows, g):
            if c is not None:
                assert x <= c * (1 + 1e-12)


# ---- telemetry (test_telemetry.cpp:41-131) --------------------------------------------------


def test_quantile_kats():
    v = [30.0, 10.0, 40.0, 20.0]
    assert restate.nearest_rank(v, 0.25) == 10.0
    assert restate.nearest_rank(v, 0.5) == 20.0
    assert restate.nearest_rank(v, 0.75) == 30.0
    assert restate.nearest_rank(v, 0.99) == 40.0
    assert restate.nearest_rank(v, 1.0) == 40.0
    assert restate.nearest_rank(v, 0.0) == 10.0
    assert restate.nearest_rank([7.5], 0.01) == 7.5


@pytest.mark.parametrize("cap", [64, 256, 512])
def test_sliding_window_vs_reference(cap):
    # test_telemetry.cpp:75-92 (W=64 oracle) and acceptance.cpp:176-208 (W=512, lognormal)
    rng = np.random.default_rng(cap)
    xs = np.ascontiguousarray(rng.lognormal(1.0, 0.7, 4000))
    out = np.zeros_like(xs)
    oracle().ref_tailwindow_run(cap, xs.ctypes.data, len(xs), 0.99, out.ctypes.data)
    for i in range(0, len(xs), 37):
        lo = max(0, i + 1 - cap)
        assert out[i] == restate.nearest_rank(xs[lo:i + 1].tolist(), 0.99)


def test_ema_kats_and_reference():
    seq = restate.ema_run(0.2, 15.0, 13.5, [10.0, 20.0, 20.0, 20.0, 20.0])
    assert seq[0][0] == 10.0 and seq[1][0] == pytest.approx(12.0, rel=1e-12)
    assert [s[1] for s in seq] == [False, False, False, False, True]
    assert seq[4][0] == pytest.approx(15.904, rel=1e-12)
    xs = np.ascontiguousarray(np.random.default_rng(3).uniform(0, 30, 500))
    ema = np.zeros_like(xs)
    st = np.zeros(len(xs), np.int32)
    oracle().ref_ema_run(0.2, 15.0, 13.5, xs.ctypes.data, len(xs), ema.ctypes.data, st.ctypes.data)
    mine = restate.ema_run(0.2, 15.0, 13.5, xs.tolist())
    assert [m[0] for m in mine] == ema.tolist()
    assert [int(m[1]) for m in mine] == st.tolist()


# ---- harness CI (test_harness.cpp:24-42) ----------------------------------------------------


def test_confidence_interval_kats():
    m, h = restate.confidence_interval([8.0, 12.0])
    assert m == pytest.approx(10.0, rel=1e-12)
    assert h == pytest.approx(1.96 * 2.0 / math.sqrt(2.0), rel=1e-12)
    assert restate.confidence_interval([5.0, 5.0, 5.0]) == (5.0, 0.0)
    assert restate.confidence_interval([7.0]) == (7.0, 0.0)
    v = np.ascontiguousarray(np.random.default_rng(1).uniform(0, 100, 37))
    mean, half = ctypes.c_double(), ctypes.c_double()
    oracle().ref_confidence_interval(v.ctypes.data, len(v), ctypes.byref(mean), ctypes.byref(half))
    assert restate.confidence_interval(v.tolist()) == (mean.value, half.value)


# ---- RNG substreams (workload.cpp:24-47) -----------------------------------------------------


@pytest.mark.parametrize("seed,name,purpose", [(1, "t1", 1), (42, "llm", 3), (7, "etl", 6), (2**63 + 5, "s2", 5)])
def test_substream_restatement(seed, name, purpose):
    out = np.zeros(700, np.uint64)
    oracle().ref_substream(seed, name.encode(), purpose, out.ctypes.data, len(out))
    g = restate.MT19937_64(restate.substream_seed(seed, name, purpose))
    assert [g() for _ in range(700)] == [int(x) for x in out]
