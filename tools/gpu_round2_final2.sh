#!/bin/bash
# Round-2 closing pass (after the generator work): full GPU suite, smoke, bench line (C4 headline + C2
# secondary + CPU baseline), the reference arm and the ncu launch list of a bench run (the DES kernel is
# unchanged since profiles/r2_ncu_des_c4_wave_final.txt, which stays the roofline.traffic source).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; head -c 400 gpurun_out/bench.json; echo
timeout 900 python bench.py --impl reference --steps 3 > gpurun_out/bench_reference.json 2>&1; tail -c 300 gpurun_out/bench_reference.json
timeout 1200 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --c2-seeds 0 > gpurun_out/bench_under_ncu.txt 2>&1; tail -2 gpurun_out/launches.csv


