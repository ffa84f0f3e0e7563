#!/bin/bash
# Generator A/B: arrival parity of the in-tree build, then the in-tree build against side-by-side
# builds (VARS, build/var<NAME>) on the C4 shapes, and a short C4 headline bench of the in-tree build.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "arrivals or c4_headline or capped_scenarios or all_variants or fuzz" > gpurun_out/gen_pytest.txt 2>&1; tail -1 gpurun_out/gen_pytest.txt
VARS="${VARS:-head default}" bash tools/gpu_ab_libs.sh > /dev/null 2>&1; cat gpurun_out/ab_libs.txt | python -c "
import sys, json
for l in sys.stdin:
    tag, js = l.split(' ', 1); d = json.loads(js); print(tag, d['replicas'], 'gen_ms', d['gen_ms'], 'des_ms', d['des_ms'])"
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --c2-seeds 0 > gpurun_out/gen_bench.json 2> gpurun_out/gen_bench.err
python -c "
import json; d=json.load(open('gpurun_out/gen_bench.json')); k=d['kernels']; print('bench', d['value'], d['e2e']['value'], k['gen_ms_per_step'], k['des_ms_per_step'])"
