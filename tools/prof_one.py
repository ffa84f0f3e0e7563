"""One C2 batch (256 seeds, full controller) through the C-ABI -- the unit profiled by ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_20274_b200 import Engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
path = sys.argv[2] if len(sys.argv) > 2 else "scenarios/c2_cluster16.yaml"
eng = Engine(0)
sid = eng.load_scenario(path)
res = eng.run_batch(sid, list(range(1, n + 1)))
print({k: v for k, v in res.timing.items()})
res.close()
