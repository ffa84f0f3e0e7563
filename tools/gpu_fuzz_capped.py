"""Differential fuzz of the saturated-regime DES (des_kernel_reg_occ, forced with MIGSIM_DES_REGS=capped)
against the compiled reference: random scenarios (tests/fuzz_scenarios.py) x 4 seeds x the 5 ablation
variants per batch, every run diffed field by field; reference runs on every host core.
  python tools/gpu_fuzz_capped.py LO HI [wide]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["MIGSIM_DES_REGS"] = "capped"
from paper_2508_20274_b200 import Engine, Variant  # noqa: E402
from tests._libs import diff_results, ref_runs_parallel  # noqa: E402
from tests.fuzz_scenarios import make_scenario  # noqa: E402
from tests.test_gpu_parity_wide import ABLATION  # noqa: E402

lo, hi = int(sys.argv[1]), int(sys.argv[2])
wide = len(sys.argv) > 3 and sys.argv[3] == "wide"
eng = Engine(0)
vs = [Variant(n, **ov) for n, ov in ABLATION]
n_runs = n_fail = 0
for seed in range(lo, hi):
    path = f"/tmp/fc{seed}.yaml"
    with open(path, "w") as f:
        f.write(make_scenario(seed, wide=wide))
    sid = eng.load_scenario(path)
    seeds = [seed % 7 + 1 + k for k in range(4)]
    res = eng.run_batch(sid, seeds, vs)
    assert res.timing["des_form"] == 2 or res.T > 10
    jobs = [(path, s, ov) for _, ov in ABLATION for s in seeds]
    refs = ref_runs_parallel(jobs)
    for k, ref in enumerate(refs):
        d = diff_results(ref, res.run(k))
        n_runs += 1
        if d:
            n_fail += 1
            print("FAIL", seed, jobs[k][1], jobs[k][2], d[:6], flush=True)
    res.close()
print(f"capped-DES fuzz scenarios {lo}..{hi - 1}{' (wide)' if wide else ''}: {n_runs} runs, {n_fail} mismatches", flush=True)
