"""Reference CPU throughput sample (oracle/_ref: the unmodified reference engine + its std::async
fan-out) on this host's cores, for the sweep configs: tenant-ticks/s over a contiguous block of
REF_PER_CORE (default 8) replicas per core, seeds 1.. (>= 8 x nproc, extrapolated
linearly)."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests._libs import oracle, scenario_json  # noqa: E402

cores = os.cpu_count() or 1
per_core = int(os.environ.get("REF_PER_CORE", "8"))
out = {}
for path in sys.argv[1:]:
    spec = json.loads(scenario_json(path))
    T = len(spec["tenants"])
    duration = float(spec["duration_s"])
    lib = oracle()
    n = per_core * cores
    w = lib.ref_run_batch(scenario_json(path), (ctypes.c_char_p * 1)(None), 1, 1, n, cores, b"", None, None,
                          None, None)
    out[path] = {"replicas": n, "seeds": f"1..{n}", "cores": cores, "wall_s": w,
                 "tenant_ticks_per_s": n * T * int(duration) / w, "kind": "reference (oracle/_ref), extrapolated"}
print(json.dumps(out))
