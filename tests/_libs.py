"""Test-side loaders/builders for the three native libraries the suite uses.

* product:  paper_2508_20274_b200/_lib/libmigsim_b200.so (the CUDA engine's C-ABI)
* oracle:   oracle/_ref/libmigsim_ref.so (the UNMODIFIED reference engine + restated loader)
* hostsim:  tests/native/_build/libhostsim.so (the engine's __host__ __device__ logic compiled for
            the CPU -- a test harness only; the product library has no CPU execution path)
"""
from __future__ import annotations

import ctypes
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

ORACLE_SO = os.path.join(ROOT, "oracle", "_ref", "libmigsim_ref.so")
HOSTSIM_SO = os.path.join(ROOT, "tests", "native", "_build", "libhostsim.so")
PRODUCT_SO = os.path.join(ROOT, "paper_2508_20274_b200", "_lib", "libmigsim_b200.so")
SCEN_DIR = os.path.join(ROOT, "tests", "golden", "scenarios")
CONFIG_DIR = os.path.join(ROOT, "scenarios")
NLOHMANN = os.path.join(ROOT, "paper_2508_20274_b200", "csrc", "third_party", "nlohmann")  # vendored 3.11.3

GOLDEN_SCENARIOS = [os.path.join(SCEN_DIR, f"{n}.yaml") for n in ("default", "llm", "stability", "unstable")]
CONFIG_SCENARIOS = [os.path.join(CONFIG_DIR, f) for f in ("c1_single_host.yaml", "c2_cluster16.yaml",
                                                          "c3_llm_bursty.yaml")]


def build_hostsim() -> str:
    src = os.path.join(ROOT, "tests", "native", "hostsim.cpp")
    host = os.path.join(ROOT, "paper_2508_20274_b200", "csrc", "host")
    deps = [src] + [os.path.join(host, f) for f in ("scenario.cpp", "packer.cpp", "result_json.cpp", "artifacts.cpp")]
    hdr_dir = os.path.join(ROOT, "paper_2508_20274_b200", "csrc", "common")
    hdrs = [os.path.join(hdr_dir, f) for f in os.listdir(hdr_dir)] + [
        os.path.join(host, f) for f in os.listdir(host) if f.endswith(".hpp")]
    newest = max(os.path.getmtime(p) for p in deps + hdrs)
    if os.path.exists(HOSTSIM_SO) and os.path.getmtime(HOSTSIM_SO) >= newest:
        return HOSTSIM_SO
    os.makedirs(os.path.dirname(HOSTSIM_SO), exist_ok=True)
    vmap = os.path.join(ROOT, "tests", "native", "exports.map")
    cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-static-libstdc++", f"-I{NLOHMANN}",
           "-static-libgcc", f"-Wl,--version-script={vmap}", "-o", HOSTSIM_SO] + deps
    subprocess.run(cmd, check=True)
    return HOSTSIM_SO


def build_oracle() -> str:
    if os.path.exists(ORACLE_SO):
        return ORACLE_SO
    if not os.path.isdir("/root/reference/proj"):
        raise RuntimeError("oracle/_ref missing and /root/reference not present to build it")
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "-j8"], check=True)
    return ORACLE_SO


def build_product() -> str:
    subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2508_20274_b200", "csrc"), "-j4"], check=True,
                   stdout=subprocess.DEVNULL)
    return PRODUCT_SO


_oracle = None
_hostsim = None


def oracle() -> ctypes.CDLL:
    global _oracle
    if _oracle is None:
        lib = ctypes.CDLL(build_oracle())
        vp, cp, sz = ctypes.c_void_p, ctypes.c_char_p, ctypes.c_size_t
        lib.ref_last_error.restype = cp
        lib.ref_scenario_dump.restype = vp
        lib.ref_scenario_dump.argtypes = [cp, cp]
        lib.ref_free.argtypes = [vp]
        lib.ref_run.restype = vp
        lib.ref_run.argtypes = [cp, cp, ctypes.c_uint64, ctypes.c_int]
        lib.ref_result_json.restype = cp
        lib.ref_result_json.argtypes = [vp]
        lib.ref_result_n_completions.restype = sz
        lib.ref_result_n_completions.argtypes = [vp]
        lib.ref_result_completions.argtypes = [vp] + [vp] * 9
        lib.ref_result_audit.argtypes = [vp, cp, cp, ctypes.POINTER(vp)]
        lib.ref_result_free.argtypes = [vp]
        lib.ref_run_artifacts.argtypes = [cp, cp, ctypes.c_uint64, cp, ctypes.c_int]
        lib.ref_run_plan.restype = vp
        lib.ref_run_plan.argtypes = [cp, cp, ctypes.c_int, ctypes.c_uint64, cp, cp, ctypes.c_int]
        lib.ref_render_report.restype = vp
        lib.ref_render_report.argtypes = [cp]
        lib.ref_admit.argtypes = [cp, ctypes.c_int] + [vp] * 12
        lib.ref_run_batch.restype = ctypes.c_double
        lib.ref_run_batch.argtypes = [cp, ctypes.POINTER(cp), ctypes.c_int, ctypes.c_uint64, ctypes.c_int,
                                      ctypes.c_int, cp, vp, vp, vp, vp]
        lib.ref_substream.argtypes = [ctypes.c_uint64, cp, ctypes.c_int, vp, sz]
        lib.ref_generate_arrivals.restype = ctypes.c_long
        lib.ref_generate_arrivals.argtypes = [cp, cp, ctypes.c_uint64, ctypes.c_double, vp, ctypes.c_long]
        lib.ref_allocate_bandwidth.argtypes = [ctypes.c_int, vp, vp, ctypes.c_double, ctypes.c_int, vp, vp]
        lib.ref_tailwindow_run.argtypes = [sz, vp, sz, ctypes.c_double, vp]
        lib.ref_ema_run.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double, vp, sz, vp, vp]
        lib.ref_truncated_normal.argtypes = [ctypes.c_uint64, cp, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                             ctypes.c_double, ctypes.c_double, vp, sz]
        lib.ref_confidence_interval.argtypes = [vp, sz, vp, vp]
        _oracle = lib
    return _oracle


def hostsim() -> ctypes.CDLL:
    global _hostsim
    if _hostsim is None:
        lib = ctypes.CDLL(build_hostsim())
        vp = ctypes.c_void_p
        lib.hostsim_last_error.restype = ctypes.c_char_p
        lib.hostsim_run.restype = vp
        lib.hostsim_run.argtypes = [ctypes.c_char_p, ctypes.c_uint64] + [ctypes.c_int] * 5 + [vp, vp]
        lib.hostsim_free.argtypes = [vp]
        lib.hostsim_run_artifacts.restype = vp
        lib.hostsim_run_artifacts.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_char_p]
        lib.hostsim_arrivals.restype = ctypes.c_long
        lib.hostsim_arrivals.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_int, vp, ctypes.c_long]
        lib.hostsim_math.argtypes = [ctypes.c_int, vp, vp, vp, ctypes.c_long]
        lib.hostsim_lat_bin.argtypes = [vp, vp, vp, vp, ctypes.c_long]
        _hostsim = lib
    return _hostsim


def scenario_json(path: str) -> bytes:
    from oracle.yaml_to_json import yaml_file_to_json
    return yaml_file_to_json(path).encode()


def ref_run(path: str, seed: int, overrides: dict | None = None, keep_completions: bool = False):
    """(result json, completions or None) from the reference engine."""
    import numpy as np

    lib = oracle()
    h = lib.ref_run(scenario_json(path), json.dumps(overrides).encode() if overrides else None, seed,
                    int(keep_completions))
    if not h:
        raise RuntimeError(lib.ref_last_error().decode())
    try:
        res = json.loads(lib.ref_result_json(h).decode())
        comps = None
        if keep_completions:
            n = lib.ref_result_n_completions(h)
            tenant = np.zeros(n, np.int32)
            seq = np.zeros(n, np.uint64)
            cols = [np.zeros(n, np.float64) for _ in range(7)]
            lib.ref_result_completions(h, tenant.ctypes.data, seq.ctypes.data, *[c.ctypes.data for c in cols])
            comps = dict(tenant=tenant, seq=seq, arrived=cols[0], done=cols[1], total=cols[2], compute=cols[3],
                         transfer=cols[4], noise=cols[5], bytes=cols[6])
        return res, comps
    finally:
        lib.ref_result_free(h)


def hostsim_run(path: str, seed: int, variant: dict | None = None):
    lib = hostsim()
    v = variant or {}
    flags = [int(v[k]) if k in v else -1 for k in ("enabled", "enable_mig", "enable_placement", "enable_guardrails")]
    p = lib.hostsim_run(path.encode(), seed, *flags, 0, None, None)
    if not p:
        raise RuntimeError(lib.hostsim_last_error().decode())
    try:
        return json.loads(ctypes.string_at(p).decode())
    finally:
        lib.hostsim_free(p)


SUMMARY_KEYS = ("completed_total", "completed_window", "mean_ms", "p50_ms", "p95_ms", "p99_ms", "miss_rate",
                "throughput_hz", "slo_tail_ms")
ACTION_KEYS = ("seq", "t_s", "tenant", "target", "kind", "diagnosis", "p99_pre_ms", "ema_p99_ms", "breach_windows",
               "obs_since_prev", "detail")


def diff_results(ref: dict, mine: dict) -> list:
    """Bit-exact comparison of a reference RunResult json with ours; returns mismatches."""
    bad = []
    rs = ref["summary"]
    for tid, s in rs["tenants"].items():
        m = mine["tenants"].get(tid)
        if m is None:
            bad.append(("missing tenant", tid))
            continue
        for k in SUMMARY_KEYS:
            if s[k] != m[k]:
                bad.append((tid, k, s[k], m[k]))
    for tid, e in rs["end_states"].items():
        m = mine["end_states"][tid]
        for k in ("host", "gpu", "first_slice", "profile", "claim_Bps", "status", "cpu_pinned"):
            if e[k] != m[k]:
                bad.append(("end", tid, k, e[k], m[k]))
    if len(ref["actions"]) != len(mine["actions"]):
        bad.append(("n_actions", len(ref["actions"]), len(mine["actions"])))
    for a, b in zip(ref["actions"], mine["actions"]):
        for k in ACTION_KEYS:
            if a[k] != b[k]:
                bad.append(("action", a["seq"], k, a[k], b[k]))
        if a["_pause_s"] != b["pause_s"] or a["_rolled_back_seq"] != b["rolled_back_seq"]:
            bad.append(("action", a["seq"], "pause/rollback", a["_pause_s"], b["pause_s"]))
        if a["_throttle_Bps"] != b["throttle_Bps"] or a["_quota_pct"] != b["quota_pct"]:
            bad.append(("action", a["seq"], "guardrail values"))
    if len(ref["pauses"]) != len(mine["pauses"]):
        bad.append(("n_pauses", len(ref["pauses"]), len(mine["pauses"])))
    for a, b in zip(ref["pauses"], mine["pauses"]):
        if a != b:
            bad.append(("pause", a, b))
    if rs["stability"] != mine["stability"]:
        bad.append(("stability", rs["stability"], mine["stability"]))
    # summary.json aggregates (trace.cpp:159-181)
    if rs["actions"]["total"] != len(mine["actions"]) or rs["pauses"]["count"] != len(mine["pauses"]):
        bad.append(("summary counts",))
    return bad


def ref_runs_parallel(jobs, threads: int | None = None):
    """ref_run over [(path, seed, overrides)] on every host core (ctypes releases the GIL while the
    reference engine runs), results in job order."""
    from concurrent.futures import ThreadPoolExecutor

    oracle()  # load once before the threads start
    with ThreadPoolExecutor(threads or os.cpu_count() or 1) as ex:
        return list(ex.map(lambda j: ref_run(j[0], j[1], j[2] if len(j) > 2 else None)[0], jobs))


def ref_audit_gpu(path: str, gpu_result: dict, overrides: dict | None = None):
    """The reference's audit::audit_run (audit.cpp:52-122) over a GPU RunResult; returns the issue list."""
    lib = oracle()
    lib.ref_audit_gpu_result.restype = ctypes.c_int
    lib.ref_audit_gpu_result.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p,
                                         ctypes.POINTER(ctypes.c_void_p)]
    out = ctypes.c_void_p()
    n = lib.ref_audit_gpu_result(scenario_json(path), json.dumps(overrides).encode() if overrides else None,
                                 json.dumps(gpu_result).encode(), ctypes.byref(out))
    if n < 0:
        raise RuntimeError(lib.ref_last_error().decode())
    try:
        return json.loads(ctypes.string_at(out.value).decode())
    finally:
        lib.ref_free(out)


def ref_audit_ref(path: str, seed: int, overrides: dict | None = None):
    """audit::audit_run over the reference's own run of (path, seed, overrides)."""
    lib = oracle()
    sj = scenario_json(path)
    ov = json.dumps(overrides).encode() if overrides else None
    h = lib.ref_run(sj, ov, seed, 0)
    if not h:
        raise RuntimeError(lib.ref_last_error().decode())
    out = ctypes.c_void_p()
    try:
        lib.ref_result_audit(h, sj, ov, ctypes.byref(out))
        return json.loads(ctypes.string_at(out.value).decode())
    finally:
        lib.ref_free(out)
        lib.ref_result_free(h)
