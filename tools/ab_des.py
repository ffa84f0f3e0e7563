"""A/B of the DES forms (MIGSIM_DES=warp|simt) on one batch: per-kernel device ms, tenant-ticks/s and
a byte-level identity check of every tenant row + a sample of full RunResults between the forms.

  python tools/ab_des.py [scenario] [seeds] [variants: c4|full|asis] [modes: warp,simt] [reps]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_20274_b200 import Engine, Variant  # noqa: E402

path = sys.argv[1] if len(sys.argv) > 1 else "tests/golden/scenarios/default.yaml"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
vset = sys.argv[3] if len(sys.argv) > 3 else "c4"
modes = (sys.argv[4] if len(sys.argv) > 4 else "warp,simt").split(",")
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
vs = {"c4": [Variant("static", False, False, False, False), Variant("mig-only", True, True, False, False),
             Variant("placement-only", True, False, True, False), Variant("full", True, True, True, True)],
      "full": [Variant("full", True, True, True, True)], "asis": None}[vset]
eng = Engine(0)
sid = eng.load_scenario(path)
seeds = list(range(1, n + 1))
out = {}
for mode in modes:
    os.environ["MIGSIM_DES"] = mode
    best = None
    for _ in range(reps):
        res = eng.run_batch(sid, seeds, vs)
        t = res.timing
        if best is None or t["des_ms"] < best["des_ms"]:
            best = dict(t)
        rows = res.rows.copy()
        sample = [res.run(k) for k in range(0, res.n_runs, max(1, res.n_runs // 16))]
        res.close()
    out[mode] = (rows, sample)
    tt = best["tenant_ticks"] / (best["total_device_ms"] / 1e3)
    print(json.dumps({"mode": mode, "form": int(best["des_form"]), "regs": os.environ.get("MIGSIM_DES_REGS", "auto"), "replicas": int(best["replicas"]),
                      "waves": int(best["waves"]), "blocks_per_sm": int(best["des_blocks_per_sm"]),
                      "smem": int(best["des_smem_bytes"]), "lib": os.environ.get("MIGSIM_LIB", "default"),
                      "rings": os.environ.get("MIGSIM_RINGS", "auto"), "gen_ms": round(best["gen_ms"], 1), "des_ms": round(best["des_ms"], 1),
                      "select_ms": round(best["select_ms"], 2), "completions": int(best["completions"]), "tenant_ticks_per_s": tt,
                      "events_per_s": best["events"] / (best["des_ms"] / 1e3)}), flush=True)
if len(out) > 1:
    ms = list(out)
    a = out[ms[0]]
    for m in ms[1:]:
        b = out[m]
        same_rows = bool((a[0].view(np.uint8) == b[0].view(np.uint8)).all())
        print(json.dumps({"identical_rows": same_rows, "identical_sample_runs": a[1] == b[1], "modes": [ms[0], m]}))
