"""CPU tests of the engine's own logic (no GPU): glibc-exact math, the arrival generator, the
scenario loader, and the full replica simulator (compiled for the CPU as a test harness) against
the compiled reference."""
import ctypes
import json
import os

import numpy as np
import pytest

from tests._libs import (CONFIG_SCENARIOS, GOLDEN_SCENARIOS, PRODUCT_SO, build_product, diff_results, hostsim,
                         hostsim_run, oracle, ref_run, scenario_json)

LIBM = ctypes.CDLL("libm.so.6")
for _f in ("log", "exp"):
    getattr(LIBM, _f).restype = ctypes.c_double
    getattr(LIBM, _f).argtypes = [ctypes.c_double]
LIBM.pow.restype = ctypes.c_double
LIBM.pow.argtypes = [ctypes.c_double, ctypes.c_double]


def _math_inputs(n, rng):
    bits = rng.integers(0, 2**63, n, dtype=np.int64).astype(np.uint64) | (rng.integers(0, 2, n).astype(np.uint64) << 63)
    anyv = bits.view(np.float64)
    unit = rng.random(n)
    near1 = 1.0 + (rng.random(n) - 0.5) * 0.25
    wide = (rng.random(n) - 0.5) * 1400
    return np.concatenate([anyv, unit, near1, wide, [0.0, -0.0, 1.0, np.inf, -np.inf, np.nan, 5e-324, 1e-310]])


@pytest.mark.parametrize("fn", [0, 1, 2])
def test_glibc_math_bit_exact(fn):
    """glibc_math.h vs the host's libm (the FMA IFUNC variants the reference links)."""
    rng = np.random.default_rng(100 + fn)
    x = np.ascontiguousarray(_math_inputs(60000, rng))
    if fn == 2:
        x = np.abs(x)
        y = np.ascontiguousarray(np.concatenate([rng.uniform(0.5, 3.0, len(x) - 8), [0.5, 2.0, -1.5, 1e-70, 1e300,
                                                                                    np.nan, 0.0, -0.0]]))
    else:
        y = np.zeros_like(x)
    out = np.zeros_like(x)
    hostsim().hostsim_math(fn, x.ctypes.data, y.ctypes.data, out.ctypes.data, len(x))
    f = [LIBM.log, LIBM.exp, None][fn]
    ref = np.array([LIBM.pow(a, b) for a, b in zip(x, y)] if fn == 2 else [f(a) for a in x])
    same = (out.view(np.uint64) == ref.view(np.uint64)) | (np.isnan(out) & np.isnan(ref))
    assert same.all(), (x[~same][:5], out[~same][:5], ref[~same][:5])


@pytest.mark.parametrize("path", GOLDEN_SCENARIOS + CONFIG_SCENARIOS)
def test_arrival_streams_bit_exact(path):
    """generator (gen_times/gen_marks of arrivals.h) vs workload::generate_arrivals."""
    spec = json.loads(ctypes.string_at(oracle().ref_scenario_dump(scenario_json(path), b"x")).decode())
    ids = sorted(t["id"] for t in spec["tenants"])
    sj = scenario_json(path)
    for seed in (1, 17):
        for ti, tid in enumerate(ids):
            cap = 2_000_000
            ref = np.zeros((cap, 4))
            n = oracle().ref_generate_arrivals(sj, tid.encode(), seed, spec["duration_s"], ref.ctypes.data, cap)
            mine = np.zeros((cap, 4))
            m = hostsim().hostsim_arrivals(path.encode(), seed, ti, mine.ctypes.data, cap)
            assert n == m
            assert (ref[:n].view(np.uint64) == mine[:m].view(np.uint64)).all()


def _product():
    if not os.path.exists(PRODUCT_SO):
        build_product()
    lib = ctypes.CDLL(PRODUCT_SO)
    lib.migsim_scenario_dump.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p), ctypes.c_char_p,
                                         ctypes.c_size_t]
    lib.migsim_free.argtypes = [ctypes.c_void_p]
    return lib


def _dump(path):
    lib = _product()
    out = ctypes.c_void_p()
    err = ctypes.create_string_buffer(1024)
    rc = lib.migsim_scenario_dump(path.encode(), ctypes.byref(out), err, 1024)
    if rc != 0:
        return rc, err.value.decode()
    s = ctypes.string_at(out.value).decode()
    lib.migsim_free(out)
    return 0, json.loads(s)


@pytest.mark.parametrize("path", GOLDEN_SCENARIOS + CONFIG_SCENARIOS)
def test_scenario_loader_matches_reference(path):
    rc, mine = _dump(path)
    assert rc == 0, mine
    p = oracle().ref_scenario_dump(scenario_json(path), path.encode())
    ref = json.loads(ctypes.string_at(p).decode())
    oracle().ref_free(p)
    assert mine == ref


@pytest.mark.parametrize("mutation,expect", [
    (("version: scenario-v1", "version: scenario-v2"), ":7: unsupported scenario version 'scenario-v2'"),
    (("    arrival_rate_hz: 65", "    arrival_rate_hz: 65\n    arival_cv: 1.0"), ":31: unknown key 'arival_cv' in tenant"),
    (("duration_s: 1800", "duration_s: soon"), ":9: value of 'duration_s' is not a number"),
    (("profile: 2g.20gb, first_slice: 0 }", "profile: 9g.90gb, first_slice: 0 }"), "unknown MIG profile '9g.90gb'"),
    (("first_slice: 6 }", "first_slice: 1 }"), "overlap on GPU 0"),
    (("kind: square_wave, period_s: 120", "kind: sine, period_s: 120"), "unknown schedule kind 'sine'"),
])
def test_scenario_loader_errors(tmp_path, mutation, expect):
    """scenario.cpp error semantics: allowlists, version gate, typed values, cross-checks, file:line."""
    src = open(GOLDEN_SCENARIOS[0]).read()
    assert mutation[0] in src
    p = tmp_path / "bad.yaml"
    p.write_text(src.replace(mutation[0], mutation[1], 1))
    rc, msg = _dump(str(p))
    assert rc == 1 and expect in msg, msg


def test_yaml_numbers_follow_yaml_cpp(tmp_path):
    """12e9 is a double for yaml-cpp (YAML 1.1 would say string)."""
    rc, spec = _dump(GOLDEN_SCENARIOS[0])
    assert spec["hosts"][0]["pcie_roots"][0]["capacity_Bps"] == 12e9


FAST_CASES = [(GOLDEN_SCENARIOS[1], s) for s in (1, 2, 3)] + [(GOLDEN_SCENARIOS[0], 1), (GOLDEN_SCENARIOS[3], 1),
                                                              (CONFIG_SCENARIOS[2], 1), (CONFIG_SCENARIOS[0], 2)]
VARIANTS = [None, dict(enabled=True, enable_mig=True, enable_placement=False, enable_guardrails=False),
            dict(enabled=True, enable_mig=False, enable_placement=True, enable_guardrails=False),
            dict(enabled=True, enable_mig=False, enable_placement=False, enable_guardrails=True),
            dict(enabled=False, enable_mig=False, enable_placement=False, enable_guardrails=False)]


@pytest.mark.parametrize("path,seed", FAST_CASES)
@pytest.mark.parametrize("vi", range(len(VARIANTS)))
def test_replica_logic_vs_reference(path, seed, vi):
    """The replica simulator + controller (des_core.h) compiled for the CPU vs engine::run_scenario."""
    v = VARIANTS[vi]
    ref, _ = ref_run(path, seed, v)
    mine = hostsim_run(path, seed, v)
    assert diff_results(ref, mine) == []


def test_replica_logic_large_scenarios():
    for path, seed in ((CONFIG_SCENARIOS[1], 1), (GOLDEN_SCENARIOS[2], 1)):
        ref, _ = ref_run(path, seed)
        assert diff_results(ref, hostsim_run(path, seed)) == []


def test_capi_exports_every_declared_symbol():
    """The C-ABI library loads and exports every entry point include/migsim_b200.h declares."""
    import re

    hdr = open(os.path.join(os.path.dirname(PRODUCT_SO), "..", "..", "include", "migsim_b200.h")).read()
    declared = set(re.findall(r"MIGSIM_API\s+[\w\s\*]+?\b(migsim_\w+)\s*\(", hdr))
    assert len(declared) >= 20
    lib = _product()
    for name in declared:
        assert hasattr(lib, name), name
    from paper_2508_20274_b200.api import EXPORTED_SYMBOLS

    assert set(EXPORTED_SYMBOLS) <= declared


def test_latency_bins_monotone_and_exact_intervals():
    """lat_hist.h (DES-side histogram feeding the one-pass select): bins are monotone in the value,
    clamp at both ends, and an interior bin is exactly the key interval [lat_bin_lo(b), +2^46)."""
    from tests._libs import hostsim

    rng = np.random.default_rng(4)
    x = np.concatenate([rng.lognormal(2.0, 2.5, 200_000), [0.0, 1e-300, 2.0 ** -10, np.nextafter(2.0 ** -10, 0),
                                                           2.0 ** 22, np.nextafter(2.0 ** 22, 0), 1e300, 1.0, 2.0]])
    x = np.sort(x)
    n = len(x)
    b = np.zeros(n, np.uint32)
    k = np.zeros(n, np.uint64)
    lo = np.zeros(n, np.uint64)
    hostsim().hostsim_lat_bin(x.ctypes.data, b.ctypes.data, k.ctypes.data, lo.ctypes.data, n)
    assert (np.diff(b.astype(np.int64)) >= 0).all()
    assert b[0] == 0 and b[-1] == 2047
    assert b[np.searchsorted(x, 2.0 ** -10)] == 0 and b[np.searchsorted(x, 2.0 ** -10) + 0] == 0
    inner = (b > 0) & (b < 2047)
    assert inner.sum() > 150_000
    assert ((k[inner] >= lo[inner]) & (k[inner] - lo[inner] < np.uint64(1 << 46))).all()


def test_sweep_focus_is_reference_pick_focus_tenant():
    """sweep.default_focus == harness.cpp:80-87 pick_focus_tenant (smallest tail SLO after presets,
    first in file order on ties), via the engine's host-only scenario loader (no GPU)."""
    from paper_2508_20274_b200.sweep import default_focus

    expect = {"c2_cluster16.yaml": "ta", "c5_mc64.yaml": "h0g0a", "default.yaml": "t1", "llm.yaml": "llm"}
    for path in GOLDEN_SCENARIOS + CONFIG_SCENARIOS + [os.path.join(os.path.dirname(CONFIG_SCENARIOS[0]),
                                                                    "c5_mc64.yaml")]:
        name = os.path.basename(path)
        got = default_focus(path)
        spec = _dump(path)[1]
        best = min(spec["tenants"], key=lambda t: t["slo_tail_ms"])  # min() keeps the first of ties
        assert got == best["id"]
        if name in expect:
            assert got == expect[name]


def test_capi_error_codes_without_gpu():
    """C-ABI error behaviour on a host without a GPU (include/migsim_b200.h return codes): opening a
    device is a runtime error (2) with a message; a malformed experiment.json given to
    render_report is a runtime error too; no CPU fallback exists."""
    import ctypes

    import pytest as _pt

    from paper_2508_20274_b200 import ConfigError, Engine, load_library, render_report

    lib = load_library()
    h = ctypes.c_void_p()
    err = ctypes.create_string_buffer(256)
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        rc = lib.migsim_gpu_open(0, ctypes.byref(h), err, 256)
        assert rc == 2 and err.value
        with _pt.raises(RuntimeError):
            Engine(0)
    with _pt.raises(RuntimeError):
        render_report("{not json")
    from paper_2508_20274_b200.api import scenario_spec

    with _pt.raises(ConfigError):
        scenario_spec("/nonexistent/scenario.yaml")


def test_hist_bin_edges_match_restated_bins():
    """migsim_hist_bin_edges (host-only ABI) gives each bin's lower edge: the edge falls in its bin,
    the value just below it in the previous bin (restated binning, oracle/restate.lat_bins)."""
    from oracle import restate
    from paper_2508_20274_b200.api import HIST_BINS, hist_bin_edges

    lo = hist_bin_edges()
    assert len(lo) == HIST_BINS and lo[0] == 2.0 ** -10 and (np.diff(lo) > 0).all()
    assert (restate.lat_bins(lo) == np.arange(HIST_BINS)).all()
    below = np.nextafter(lo[1:], 0)
    assert (restate.lat_bins(below) == np.arange(HIST_BINS - 1)).all()
    # octave structure: 64 bins per doubling
    assert lo[64] == 2.0 ** -9 and lo[640] == 1.0


def test_shim_binaries_fail_loudly_without_gpu(tmp_path):
    """The reference linked against the B200 shim (oracle/_ref/shim_parity) has no CPU fallback:
    without a device the shim's engine::run_scenario raises, the binary reports it and exits 1."""
    import os
    import subprocess

    import pytest as _pt

    from oracle.json_scenarios import write_dir
    from tests._libs import GOLDEN_SCENARIOS, ROOT

    exe = os.path.join(ROOT, "oracle", "_ref", "shim_parity")
    if not os.path.exists(exe):
        _pt.skip("shim binaries are built only where /root/reference is mounted")
    try:
        import torch

        if torch.cuda.is_available():
            _pt.skip("a GPU is present")
    except ImportError:
        pass
    d = write_dir(str(tmp_path), GOLDEN_SCENARIOS[:1])
    p = subprocess.run([exe, "spec", os.path.join(d, "default.yaml")], capture_output=True, text=True, timeout=120)
    assert p.returncode == 1 and "ERROR migsim-b200" in p.stdout, p.stdout + p.stderr


@pytest.mark.parametrize("cap,q", [(256, 0.99), (2048, 0.99), (1024, 0.5), (600, 0.95), (64, 0.0), (3000, 0.999)])
def test_tailwin_any_rank_matches_reference(cap, q):
    """The engine's window (cached top-8 + linear bisection select past it) equals the reference's
    TailWindow (telemetry.cpp:30-56, copy + std::sort per query) for every push, including windows
    far longer than the cache reaches (ranks 20+ below the top) and mid quantiles, with ties."""
    import ctypes

    from tests._libs import hostsim, oracle

    rng = np.random.default_rng(cap)
    n = 3 * cap + 17
    xs = np.round(rng.lognormal(2.0, 0.8, n), 2)  # rounding creates ties
    want = np.zeros(n)
    got = np.zeros(n)
    oracle().ref_tailwindow_run(cap, xs.ctypes.data, n, q, want.ctypes.data)
    lib = hostsim()
    lib.hostsim_tailwin_run.argtypes = [ctypes.c_long, ctypes.c_void_p, ctypes.c_long, ctypes.c_double, ctypes.c_void_p]
    lib.hostsim_tailwin_run(cap, xs.ctypes.data, n, q, got.ctypes.data)
    assert (want.view(np.uint64) == got.view(np.uint64)).all()


def test_select_jth_largest_is_the_sorted_order_statistic():
    import ctypes

    from tests._libs import hostsim

    lib = hostsim()
    lib.hostsim_select_jth.argtypes = [ctypes.c_void_p, ctypes.c_long, ctypes.c_long]
    lib.hostsim_select_jth.restype = ctypes.c_double
    rng = np.random.default_rng(3)
    for n in (1, 2, 7, 64, 256, 1000):
        v = np.round(rng.exponential(5.0, n), 1)
        s = np.sort(v)[::-1]
        for j in {0, n // 3, n - 1}:
            assert lib.hostsim_select_jth(v.ctypes.data, n, j) == s[j]


def _fmod_inputs(n, rng):
    """schedule phases (t - offset over [0, 1800] s, periods 1..600 s) plus wide and edge cases"""
    t = rng.uniform(-700.0, 4000.0, n)
    p = rng.choice([60.0, 120.0, 0.1, 7.5, 1.0 / 3.0, 600.0], n) * rng.choice([1.0, 1.0 + 1e-12], n)
    wide_x = rng.standard_normal(n) * 10.0 ** rng.integers(-300, 300, n)
    wide_y = np.abs(rng.standard_normal(n)) * 10.0 ** rng.integers(-300, 300, n)
    k = rng.integers(0, 1 << 19, n).astype(np.float64)
    multiples = k * p  # exact and near-exact multiples: remainders 0 / tiny / y - tiny
    x = np.concatenate([t, wide_x, multiples, np.nextafter(multiples, np.inf), np.nextafter(multiples, -np.inf),
                        [0.0, -0.0, 5.0, -5.0, np.inf, np.nan, 1e-320, 7.0, 1e300]])
    y = np.concatenate([p, wide_y, p, p, p, [3.0, 3.0, 0.0, -3.0, 2.0, 2.0, 3.0, 1e-310, 1e-300]])
    return np.ascontiguousarray(x), np.ascontiguousarray(y)


def test_fmod_fast_exact():
    """glibc_math.h fmod_fast (schedule phase) vs C fmod: exact on every input (fast path + fallback)."""
    rng = np.random.default_rng(11)
    x, y = _fmod_inputs(200000, rng)
    out = np.zeros_like(x)
    hostsim().hostsim_math(3, x.ctypes.data, y.ctypes.data, out.ctypes.data, len(x))
    ref = np.fmod(x, y)
    same = (out.view(np.uint64) == ref.view(np.uint64)) | (np.isnan(out) & np.isnan(ref))
    assert same.all(), (x[~same][:5], y[~same][:5], out[~same][:5], ref[~same][:5])
