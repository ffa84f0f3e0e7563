"""Debug: per-tenant quantiles of one run vs the sorted completion records (GPU)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_20274_b200 import Engine  # noqa: E402

path = sys.argv[1]
seeds = [int(x) for x in sys.argv[2].split(",")]
eng = Engine(0)
sid = eng.load_scenario(path)
res = eng.run_batch(sid, seeds, keep_completions=True)
ms = res.run(0)["measure_start_s"]
bad = 0
for i, seed in enumerate(seeds):
    comp = res.completions(i)
    for t, tid in enumerate(res.tenant_ids):
        sel = (comp[:, 0] == t) & (comp[:, 2] >= ms)
        v = np.sort(comp[sel, 3])
        n = len(v)
        row = res.rows[i, t]
        for q, k in ((0.5, "p50_ms"), (0.95, "p95_ms"), (0.99, "p99_ms"), (0.999, "p999_ms")):
            r = min(max(int(np.ceil(q * n)), 1), n) - 1
            if n and v[r] != row[k]:
                bad += 1
                print("MISMATCH seed", seed, tid, n, k, row[k], v[r])
print("done, mismatches:", bad, "n_window:", [int(x) for x in res.rows[0]["completed_window"]])
