import sys
sys.path.insert(0, '.')
from tests.fuzz_scenarios import make_scenario
from tests._libs import ref_run, diff_results
from paper_2508_20274_b200 import Engine
seed = int(sys.argv[1]); seeds = [int(x) for x in sys.argv[2].split(',')]
open('/tmp/f.yaml', 'w').write(make_scenario(seed))
eng = Engine(0)
sid = eng.load_scenario('/tmp/f.yaml')
res = eng.run_batch(sid, seeds)
for i, s in enumerate(seeds):
    ref, _ = ref_run('/tmp/f.yaml', s)
    print(s, diff_results(ref, res.run(i))[:6])
res2 = eng.run_batch(sid, [seeds[-1]])
ref, _ = ref_run('/tmp/f.yaml', seeds[-1])
print('alone', seeds[-1], diff_results(ref, res2.run(0))[:6])
