"""Python mirror of the reference's replica API, driving the B200 engine through its C-ABI.

Reference interfaces mirrored (same names, argument meaning and error behaviour):
  engine::run_scenario(spec, RunOptions)   /root/reference/proj/include/migsim/engine.hpp:117
  harness::run_plan(PlanOptions)           /root/reference/proj/include/migsim/harness.hpp:91
  scenario::load_scenario(path)            /root/reference/proj/include/migsim/scenario.hpp:68
Errors: ConfigError (scenario/config problems, message carries "file:line" like
model::ConfigError), RuntimeError (CUDA/runtime), ParityGuardError (a device buffer would have
truncated results).  There is no CPU fallback: if the CUDA library is missing or no GPU is
visible, every call raises.
"""
from __future__ import annotations

import ctypes
import json
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MIGSIM_LIB") or os.path.join(_HERE, "_lib", "libmigsim_b200.so")  # env: A/B builds


class ConfigError(ValueError):
    """model::ConfigError (model.hpp:29-37)."""


class ParityGuardError(RuntimeError):
    """A device-sized buffer would have truncated output (C-ABI code 3)."""


class _Variant(ctypes.Structure):
    _fields_ = [
        ("name", ctypes.c_char_p),
        ("enabled", ctypes.c_int32),
        ("enable_mig", ctypes.c_int32),
        ("enable_placement", ctypes.c_int32),
        ("enable_guardrails", ctypes.c_int32),
        ("sample_interval_s", ctypes.c_double),
        ("persistence_windows", ctypes.c_int32),
        ("dwell_obs", ctypes.c_int32),
        ("cooldown_obs", ctypes.c_int32),
        ("validation_obs", ctypes.c_int32),
    ]


class _RunOpts(ctypes.Structure):
    _fields_ = [
        ("keep_completions", ctypes.c_int32),
        ("max_wave_replicas", ctypes.c_int32),
        ("action_cap", ctypes.c_int32),
        ("pause_cap", ctypes.c_int32),
        ("write_traces", ctypes.c_int32),
    ]


class _Timing(ctypes.Structure):
    _fields_ = [
        ("gen_ms", ctypes.c_double),
        ("des_ms", ctypes.c_double),
        ("select_ms", ctypes.c_double),
        ("total_device_ms", ctypes.c_double),
        ("wall_ms", ctypes.c_double),
        ("replicas", ctypes.c_int64),
        ("tenant_ticks", ctypes.c_int64),
        ("completions", ctypes.c_int64),
        ("arrivals", ctypes.c_int64),
        ("events", ctypes.c_int64),
        ("waves", ctypes.c_int64),
        ("select_samples", ctypes.c_int64),
        ("des_form", ctypes.c_int64),
        ("des_blocks_per_sm", ctypes.c_int64),
        ("des_smem_bytes", ctypes.c_int64),
        ("kernel_launches", ctypes.c_int64),
        ("h2d_bytes", ctypes.c_int64),
        ("d2h_bytes", ctypes.c_int64),
        ("pipeline_slots", ctypes.c_int64),
    ]


TENANT_ROW_DTYPE = np.dtype(
    [
        ("completed_total", np.uint64),
        ("completed_window", np.uint64),
        ("window_misses", np.uint64),
        ("mean_ms", np.float64),
        ("p50_ms", np.float64),
        ("p95_ms", np.float64),
        ("p99_ms", np.float64),
        ("p999_ms", np.float64),
        ("miss_rate", np.float64),
        ("throughput_hz", np.float64),
    ]
)

EXPORTED_SYMBOLS = [
    "migsim_gpu_open",
    "migsim_gpu_close",
    "migsim_gpu_load_scenario",
    "migsim_gpu_load_scenario_file",
    "migsim_scenario_n_tenants",
    "migsim_scenario_tenant_id",
    "migsim_gpu_run_batch",
    "migsim_batch_n_runs",
    "migsim_batch_n_tenants",
    "migsim_batch_timing",
    "migsim_batch_tenant_rows",
    "migsim_batch_run_json",
    "migsim_batch_completions",
    "migsim_batch_result_free",
    "migsim_gpu_select",
    "migsim_run_plan",
    "migsim_free",
]

_lib_handle = None


def load_library() -> ctypes.CDLL:
    """Load the CUDA engine library; raises if it was not built (no CPU fallback)."""
    global _lib_handle
    if _lib_handle is not None:
        return _lib_handle
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"B200 engine library missing at {LIB_PATH}; build it with __graft_entry__.build() "
            "(make -C paper_2508_20274_b200/csrc)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    vp, cp, sz = ctypes.c_void_p, ctypes.c_char_p, ctypes.c_size_t
    lib.migsim_gpu_open.argtypes = [ctypes.c_int, ctypes.POINTER(vp), cp, sz]
    lib.migsim_gpu_close.argtypes = [vp]
    lib.migsim_gpu_load_scenario.argtypes = [vp, cp, cp, ctypes.POINTER(ctypes.c_int32), cp, sz]
    lib.migsim_gpu_load_scenario_file.argtypes = [vp, cp, ctypes.POINTER(ctypes.c_int32), cp, sz]
    lib.migsim_scenario_n_tenants.argtypes = [vp, ctypes.c_int32]
    lib.migsim_scenario_tenant_id.argtypes = [vp, ctypes.c_int32, ctypes.c_int32, cp, sz]
    lib.migsim_gpu_run_batch.argtypes = [
        vp, ctypes.c_int32, ctypes.POINTER(_Variant), sz, ctypes.POINTER(ctypes.c_uint64), sz,
        ctypes.POINTER(_RunOpts), ctypes.POINTER(vp), cp, sz,
    ]
    lib.migsim_batch_n_runs.argtypes = [vp]
    lib.migsim_batch_n_runs.restype = sz
    lib.migsim_batch_n_tenants.argtypes = [vp]
    lib.migsim_batch_timing.argtypes = [vp, ctypes.POINTER(_Timing)]
    lib.migsim_batch_tenant_rows.argtypes = [vp, ctypes.c_void_p, sz]
    lib.migsim_batch_run_json.argtypes = [vp, sz]
    lib.migsim_batch_run_json.restype = ctypes.c_char_p
    lib.migsim_batch_completions.argtypes = [vp, sz, ctypes.c_void_p, ctypes.c_int64]
    lib.migsim_batch_completions.restype = ctypes.c_int64
    lib.migsim_batch_result_free.argtypes = [vp]
    lib.migsim_gpu_select.argtypes = [
        vp, ctypes.c_void_p, ctypes.c_void_p, sz, ctypes.c_void_p, sz, ctypes.c_void_p,
        ctypes.POINTER(ctypes.c_double), cp, sz,
    ]
    lib.migsim_gpu_run_scenario.argtypes = [vp, ctypes.c_int32, ctypes.POINTER(_Variant), ctypes.c_uint64, cp,
                                            ctypes.c_int32, ctypes.POINTER(vp), cp, sz]
    lib.migsim_run_plan.argtypes = [vp, cp, cp, ctypes.c_int32, ctypes.c_uint64, cp, cp, ctypes.POINTER(vp), cp, sz]
    lib.migsim_render_report.argtypes = [cp, ctypes.POINTER(vp), cp, sz]
    lib.migsim_gpu_admit.argtypes = [vp, ctypes.c_int32, sz] + [vp] * 12 + [ctypes.POINTER(ctypes.c_double), cp, sz]
    lib.migsim_free.argtypes = [vp]
    lib.migsim_scenario_dump.argtypes = [cp, ctypes.POINTER(vp), cp, sz]
    lib.migsim_batch_n_variants.argtypes = [vp]
    lib.migsim_batch_n_variants.restype = sz
    lib.migsim_batch_latency_hist.argtypes = [vp, vp, sz]
    lib.migsim_batch_tenant_counts.argtypes = [vp, vp, sz]
    lib.migsim_hist_bin_edges.argtypes = [vp, sz]
    _lib_handle = lib
    return lib


def _check(code: int, err: ctypes.Array) -> None:
    if code == 0:
        return
    msg = err.value.decode(errors="replace")
    if code == 1:
        raise ConfigError(msg)
    if code == 3:
        raise ParityGuardError(msg)
    raise RuntimeError(msg)


KEEP_INT = -(2 ** 31)  # MIGSIM_KEEP_INT (include/migsim_b200.h)
HIST_BINS = 2048  # MIGSIM_HIST_BINS


def hist_bin_edges() -> np.ndarray:
    """Lower edge (ms) of each latency-histogram bin (64 bins per binary octave from 2^-10 ms)."""
    lo = np.zeros(HIST_BINS, dtype=np.float64)
    if load_library().migsim_hist_bin_edges(lo.ctypes.data, HIST_BINS) != 0:
        raise RuntimeError("migsim_hist_bin_edges failed")
    return lo


@dataclass
class Variant:
    """harness::Variant (harness.hpp:40-46); None (and only None) keeps the scenario's setting.
    Every other value is applied and validated like ControllerConfig::validate (model.cpp:184-206),
    so an invalid knob raises ConfigError instead of being dropped."""

    name: str = "as-is"
    enabled: Optional[bool] = None
    enable_mig: Optional[bool] = None
    enable_placement: Optional[bool] = None
    enable_guardrails: Optional[bool] = None
    sample_interval_s: Optional[float] = None
    persistence_windows: Optional[int] = None
    dwell_obs: Optional[int] = None
    cooldown_obs: Optional[int] = None
    validation_obs: Optional[int] = None

    def _c(self) -> _Variant:
        def b(x):
            return -1 if x is None else int(bool(x))

        return _Variant(
            self.name.encode(), b(self.enabled), b(self.enable_mig), b(self.enable_placement),
            b(self.enable_guardrails),
            float("nan") if self.sample_interval_s is None else float(self.sample_interval_s),
            *[KEEP_INT if x is None else int(x)
              for x in (self.persistence_windows, self.dwell_obs, self.cooldown_obs, self.validation_obs)],
        )


# harness.cpp:45-60
def ablation_variants() -> List[Variant]:
    return [
        Variant("full", True, True, True, True),
        Variant("mig-only", True, True, False, False),
        Variant("placement-only", True, False, True, False),
        Variant("guards-only", True, False, False, True),
        Variant("static", False, False, False, False),
    ]


def main_variants() -> List[Variant]:
    return [Variant("full", True, True, True, True), Variant("static", False, False, False, False)]


@dataclass
class BatchResult:
    n_runs: int
    n_tenants: int
    tenant_ids: List[str]
    variants: List[Variant]
    seeds: List[int]
    rows: np.ndarray  # [n_runs, n_tenants] TENANT_ROW_DTYPE
    timing: Dict[str, float]
    _handle: int = 0
    _engine: "Engine" = None
    _json_cache: Dict[int, dict] = field(default_factory=dict)

    def run(self, i: int) -> dict:
        """Full RunResult of run i (variant-major, seed-minor)."""
        if i not in self._json_cache:
            s = self._engine._lib.migsim_batch_run_json(self._handle, i)
            self._json_cache[i] = json.loads(s.decode())
        return self._json_cache[i]

    def latency_hist(self) -> np.ndarray:
        """int64 [n_variants, n_tenants, HIST_BINS]: every measurement-window latency of every seed,
        binned (hist_bin_edges()) and summed per (variant, tenant) on the device."""
        lib = self._engine._lib
        nv = lib.migsim_batch_n_variants(self._handle)
        out = np.zeros((nv, self.n_tenants, HIST_BINS), dtype=np.uint64)
        if lib.migsim_batch_latency_hist(self._handle, out.ctypes.data, out.size) != 0:
            raise RuntimeError("migsim_batch_latency_hist failed")
        return out.astype(np.int64)

    def tenant_counts(self) -> np.ndarray:
        """int64 [n_variants, n_tenants, 3]: completed_total, completed_window, window_misses summed
        over the batch's seeds (engine.cpp:497-501)."""
        lib = self._engine._lib
        nv = lib.migsim_batch_n_variants(self._handle)
        out = np.zeros((nv, self.n_tenants, 3), dtype=np.uint64)
        if lib.migsim_batch_tenant_counts(self._handle, out.ctypes.data, out.size) != 0:
            raise RuntimeError("migsim_batch_tenant_counts failed")
        return out.astype(np.int64)

    def completions(self, i: int) -> np.ndarray:
        """Per-completion records [n, 7] = tenant, seq, done_s, total, compute, transfer, noise."""
        lib = self._engine._lib
        n = lib.migsim_batch_completions(self._handle, i, None, 0)
        if n < 0:
            raise RuntimeError("batch was run without keep_completions")
        out = np.zeros((n, 7), dtype=np.float64)
        lib.migsim_batch_completions(self._handle, i, out.ctypes.data, n)
        return out

    def close(self) -> None:
        if self._handle:
            self._engine._lib.migsim_batch_result_free(self._handle)
            self._handle = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


ADMIT_DTYPE = np.dtype([("outcome", np.int32), ("host", np.int32), ("gpu", np.int32), ("first", np.int32),
                        ("count", np.int32), ("profile", np.int32), ("reason", np.int32), ("pad", np.int32),
                        ("score", np.float64)])


class Engine:
    """One B200 device (C-ABI handle)."""

    def __init__(self, device: int = 0):
        self._lib = load_library()
        self._h = ctypes.c_void_p()
        err = ctypes.create_string_buffer(1024)
        _check(self._lib.migsim_gpu_open(device, ctypes.byref(self._h), err, 1024), err)
        self.device = device

    def close(self) -> None:
        if self._h:
            self._lib.migsim_gpu_close(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load_scenario(self, path: str) -> int:
        sid = ctypes.c_int32()
        err = ctypes.create_string_buffer(1024)
        _check(self._lib.migsim_gpu_load_scenario_file(self._h, path.encode(), ctypes.byref(sid), err, 1024), err)
        return sid.value

    def parse_scenario(self, yaml_text: str, source_name: str = "<scenario>") -> int:
        sid = ctypes.c_int32()
        err = ctypes.create_string_buffer(1024)
        _check(self._lib.migsim_gpu_load_scenario(self._h, yaml_text.encode(), source_name.encode(),
                                                  ctypes.byref(sid), err, 1024), err)
        return sid.value

    def tenant_ids(self, sid: int) -> List[str]:
        n = self._lib.migsim_scenario_n_tenants(self._h, sid)
        buf = ctypes.create_string_buffer(256)
        out = []
        for i in range(n):
            self._lib.migsim_scenario_tenant_id(self._h, sid, i, buf, 256)
            out.append(buf.value.decode())
        return out

    def run_batch(self, sid: int, seeds: Sequence[int], variants: Optional[Sequence[Variant]] = None,
                  keep_completions: bool = False, max_wave_replicas: int = 0) -> BatchResult:
        variants = list(variants) if variants else [Variant()]
        cv = (_Variant * len(variants))(*[v._c() for v in variants])
        cs = (ctypes.c_uint64 * len(seeds))(*[int(s) for s in seeds])
        opts = _RunOpts(int(keep_completions), int(max_wave_replicas), 0, 0, 0)
        out = ctypes.c_void_p()
        err = ctypes.create_string_buffer(2048)
        _check(self._lib.migsim_gpu_run_batch(self._h, sid, cv, len(variants), cs, len(seeds), ctypes.byref(opts),
                                              ctypes.byref(out), err, 2048), err)
        n_runs = self._lib.migsim_batch_n_runs(out)
        T = self._lib.migsim_batch_n_tenants(out)
        rows = np.zeros(n_runs * T, dtype=TENANT_ROW_DTYPE)
        self._lib.migsim_batch_tenant_rows(out, rows.ctypes.data, n_runs * T)
        t = _Timing()
        self._lib.migsim_batch_timing(out, ctypes.byref(t))
        timing = {k: getattr(t, k) for k, _ in _Timing._fields_}
        return BatchResult(n_runs, T, self.tenant_ids(sid), variants, [int(s) for s in seeds],
                           rows.reshape(n_runs, T), timing, out.value, self)

    def run_scenario(self, sid: int, seed: int = 1, variant: Optional[Variant] = None, out_dir: str = "",
                     write_traces: bool = True) -> dict:
        """engine::run_scenario(spec, RunOptions{seed, out_dir, write_traces}) (engine.hpp:94-99,117):
        one replica on the GPU; with out_dir the reference's artifacts are written there byte-for-byte
        (summary.json, actions.jsonl, and requests/counters/fabric.csv when write_traces)."""
        cv = variant._c() if variant else None
        out = ctypes.c_void_p()
        err = ctypes.create_string_buffer(2048)
        _check(self._lib.migsim_gpu_run_scenario(self._h, sid, ctypes.byref(cv) if cv else None, int(seed),
                                                 out_dir.encode() if out_dir else None, int(write_traces),
                                                 ctypes.byref(out), err, 2048), err)
        try:
            return json.loads(ctypes.string_at(out.value).decode())
        finally:
            self._lib.migsim_free(out)

    def admit(self, sid: int, tenant, profile, admitted, host, gpu, first, count, tenant_pcie_Bps,
              tenant_host_io_Bps, irq_recent, queue_epochs: Optional[np.ndarray] = None) -> (np.ndarray, float):
        """Controller::admit (controller.cpp:637-692) for n independent cases on the GPU.

        tenant/profile: [n] canonical tenant index / MIG lattice index of each request;
        admitted/host/gpu/first/count and tenant_pcie_Bps/tenant_host_io_Bps: [n, T] TenantStates and
        snapshot fields (tenants in canonical order); irq_recent: [n, n_hosts] core-group bitmasks.
        Returns (decisions, device_ms); decisions has fields outcome (0 admitted, 1 queued,
        2 rejected), host, gpu, first, count, profile, reason, score.

        queue_epochs: optional int32 [n], each case's controller queue_epochs_[tenant] (0 = none),
        updated IN PLACE (controller.cpp:671-691) -- pass the same array again to retry; None =
        fresh controllers."""
        i32 = lambda a: np.ascontiguousarray(np.asarray(a, np.int32))  # noqa: E731
        f64 = lambda a: np.ascontiguousarray(np.asarray(a, np.float64))  # noqa: E731
        args = [i32(tenant), i32(profile), i32(admitted), i32(host), i32(gpu), i32(first), i32(count),
                f64(tenant_pcie_Bps), f64(tenant_host_io_Bps), np.ascontiguousarray(np.asarray(irq_recent, np.uint32))]
        n = len(args[0])
        out = np.zeros(n, dtype=ADMIT_DTYPE)
        ms = ctypes.c_double()
        err = ctypes.create_string_buffer(1024)
        if queue_epochs is not None:
            if not (isinstance(queue_epochs, np.ndarray) and queue_epochs.dtype == np.int32
                    and queue_epochs.flags.c_contiguous and queue_epochs.shape == (n,)):
                raise ValueError("queue_epochs must be a contiguous int32 array of shape (n,)")
        qe = queue_epochs.ctypes.data if queue_epochs is not None else None
        _check(self._lib.migsim_gpu_admit(self._h, sid, n, *[a.ctypes.data for a in args], qe, out.ctypes.data,
                                          ctypes.byref(ms), err, 1024), err)
        return out, ms.value

    def select(self, segments: Sequence[np.ndarray], qs: Sequence[float]) -> (np.ndarray, float):
        """Nearest-rank quantiles of each segment on the GPU; returns (out[n_seg, n_q], device_ms)."""
        vals = np.ascontiguousarray(np.concatenate([np.asarray(s, np.float64) for s in segments])
                                    if len(segments) else np.zeros(0))
        off = np.zeros(len(segments) + 1, dtype=np.int64)
        off[1:] = np.cumsum([len(s) for s in segments])
        q = np.ascontiguousarray(np.asarray(qs, np.float64))
        out = np.zeros((len(segments), len(q)), dtype=np.float64)
        ms = ctypes.c_double()
        err = ctypes.create_string_buffer(1024)
        _check(self._lib.migsim_gpu_select(self._h, vals.ctypes.data, off.ctypes.data, len(segments), q.ctypes.data,
                                           len(q), out.ctypes.data, ctypes.byref(ms), err, 1024), err)
        return out, ms.value

    def run_plan(self, plan: str, scenario_path: str, seeds: int = 7, seed_base: int = 1,
                 focus_tenant: str = "", out_dir: str = "") -> dict:
        """harness::run_plan(PlanOptions{plan, scenario_path, seeds, seed_base, out_dir, focus_tenant})
        (harness.hpp:84-94) with the replica fan-out as one GPU batch."""
        out = ctypes.c_void_p()
        err = ctypes.create_string_buffer(2048)
        _check(self._lib.migsim_run_plan(self._h, plan.encode(), scenario_path.encode(), seeds, seed_base,
                                         focus_tenant.encode(), out_dir.encode() if out_dir else None,
                                         ctypes.byref(out), err, 2048), err)
        try:
            return json.loads(ctypes.string_at(out.value).decode())
        finally:
            self._lib.migsim_free(out)


_default_engine: Optional[Engine] = None


def default_engine() -> Engine:
    global _default_engine
    if _default_engine is None:
        _default_engine = Engine(int(os.environ.get("LOCAL_RANK", "0")))
    return _default_engine


def run_scenario(scenario_path: str, seed: int = 1, variant: Optional[Variant] = None,
                 keep_completions: bool = False, out_dir: str = "", write_traces: bool = True) -> dict:
    """engine::run_scenario as a 1x1 batch on the GPU (engine.hpp:117).  With out_dir, the run's
    artifacts are written like RunOptions{seed, out_dir, write_traces} (engine.cpp:279-288,889-892)."""
    eng = default_engine()
    sid = eng.load_scenario(scenario_path)
    if out_dir:
        return eng.run_scenario(sid, seed, variant, out_dir, write_traces)
    res = eng.run_batch(sid, [seed], [variant] if variant else None, keep_completions=keep_completions)
    out = res.run(0)
    if keep_completions:
        out["completions"] = res.completions(0)
    res.close()
    return out


def run_plan(plan: str, scenario_path: str, seeds: int = 7, seed_base: int = 1, focus_tenant: str = "",
             out_dir: str = "") -> dict:
    """harness::run_plan (harness.cpp:114-216) with the replica fan-out as one GPU batch."""
    return default_engine().run_plan(plan, scenario_path, seeds, seed_base, focus_tenant, out_dir)


def scenario_spec(path: str) -> dict:
    """The scenario-v1 file as the engine's loader normalises it (presets applied, file order of
    tenants kept): scenario::load_scenario (scenario.cpp:376-384)."""
    lib = load_library()
    out = ctypes.c_void_p()
    err = ctypes.create_string_buffer(1024)
    _check(lib.migsim_scenario_dump(path.encode(), ctypes.byref(out), err, 1024), err)
    try:
        return json.loads(ctypes.string_at(out.value).decode())
    finally:
        lib.migsim_free(out)


def render_report(experiment: "dict | str") -> str:
    """harness::render_report (harness.cpp:285-313): the comparison table of an experiment.json."""
    lib = load_library()
    text = experiment if isinstance(experiment, str) else json.dumps(experiment)
    out = ctypes.c_void_p()
    err = ctypes.create_string_buffer(1024)
    _check(lib.migsim_render_report(text.encode(), ctypes.byref(out), err, 1024), err)
    try:
        return ctypes.string_at(out.value).decode()
    finally:
        lib.migsim_free(out)
