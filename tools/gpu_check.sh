#!/bin/bash
# one GPU-box pass: A/B of the wave pipeline on the C4 shape, the GPU test suite, a short bench
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for p in 0 1; do
  MIGSIM_PIPELINE=$p timeout 600 python tools/ab_des.py tests/golden/scenarios/default.yaml 4096 c4 warp 1 2>&1 | tail -1
done > gpurun_out/ab_pipeline.txt
timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest_gpu.txt 2>&1
timeout 900 python bench.py --steps 2 --warmup 3 --seeds 4096 > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
cat gpurun_out/ab_pipeline.txt; tail -25 gpurun_out/pytest_gpu.txt; cat gpurun_out/bench_quick.json; tail -5 gpurun_out/bench_quick.err
