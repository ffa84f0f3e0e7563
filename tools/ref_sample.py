"""Reference CPU throughput sample (oracle/_ref: the unmodified reference engine + its std::async
fan-out) on this host's cores, for the sweep configs: tenant-ticks/s over one batch of one replica
per core."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests._libs import oracle, scenario_json  # noqa: E402

cores = os.cpu_count() or 1
out = {}
for path in sys.argv[1:]:
    spec = json.loads(scenario_json(path))
    T = len(spec["tenants"])
    duration = float(spec["duration_s"])
    lib = oracle()
    w = lib.ref_run_batch(scenario_json(path), (ctypes.c_char_p * 1)(None), 1, 70001, cores, cores, b"", None, None,
                          None, None)
    out[path] = {"replicas": cores, "cores": cores, "wall_s": w,
                 "tenant_ticks_per_s": cores * T * int(duration) / w}
print(json.dumps(out))
