"""A/B timing of an alternative build (MIGSIM_LIB=<so>): C2 batch, 256 seeds, per-kernel device ms;
prints the quantile checksum so variants can be compared for identical results."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_20274_b200 import Engine  # noqa: E402

path = sys.argv[1] if len(sys.argv) > 1 else "scenarios/c2_cluster16.yaml"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
eng = Engine(0)
sid = eng.load_scenario(path)
sel, des, gen = [], [], []
chk = None
for it in range(4):
    res = eng.run_batch(sid, list(range(1, n + 1)))
    t = res.timing
    if it:
        sel.append(t["select_ms"])
        des.append(t["des_ms"])
        gen.append(t["gen_ms"])
    q = np.stack([res.rows[k] for k in ("p50_ms", "p95_ms", "p99_ms", "p999_ms")]).view(np.uint64)
    chk = int(np.bitwise_xor.reduce(q.ravel()))
    res.close()
print(f"{os.environ.get('MIGSIM_LIB', 'default')}: select {np.median(sel):.4f} ms  des {np.median(des):.1f} ms  "
      f"gen {np.median(gen):.1f} ms  quant-xor {chk:#x}", flush=True)
