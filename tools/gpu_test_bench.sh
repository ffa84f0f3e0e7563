cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_K} > gpurun_out/pytest_gpu.txt 2>&1; tail -15 gpurun_out/pytest_gpu.txt
timeout 900 python bench.py --steps 3 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('VALUE', d['value'], 'e2e', d['e2e']['value']); print(d['kernels'])"
