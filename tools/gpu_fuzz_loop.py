import sys
sys.path.insert(0, '.')
from tests.fuzz_scenarios import make_scenario
from tests._libs import ref_run, diff_results
from paper_2508_20274_b200 import Engine
lo, hi = int(sys.argv[1]), int(sys.argv[2])
wide = len(sys.argv) > 3 and sys.argv[3] == 'wide'
eng = Engine(0)
for seed in range(lo, hi):
    path = f'/tmp/f{seed}.yaml'
    open(path, 'w').write(make_scenario(seed, wide=wide))
    sid = eng.load_scenario(path)
    seeds = [seed % 5 + 1, seed % 5 + 2]
    res = eng.run_batch(sid, seeds)
    for i, s in enumerate(seeds):
        ref, _ = ref_run(path, s)
        d = diff_results(ref, res.run(i))
        if d:
            print('FAIL', seed, s, d[:8], flush=True)
            e2 = Engine(0); sid2 = e2.load_scenario(path)
            r2 = e2.run_batch(sid2, seeds)
            print('  fresh engine:', diff_results(ref, r2.run(i))[:4], flush=True)
            r3 = eng.run_batch(sid, seeds)
            print('  same engine rerun:', diff_results(ref, r3.run(i))[:4], flush=True)
    res.close()
print('done')
