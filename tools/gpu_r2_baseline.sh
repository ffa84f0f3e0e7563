#!/bin/bash
# Session baseline: default bench line (C4 headline) + ncu --set full of the DES in the saturated C4 regime
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
tail -c 3000 gpurun_out/bench_default.json; tail -3 gpurun_out/bench_default.err
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:des_kernel_reg -c 1 -o gpurun_out/ncu_des_c4 \
  python tools/ab_des.py tests/golden/scenarios/default.yaml 2048 c4 warp 1 > gpurun_out/ncu_des_c4.log 2>&1
tail -3 gpurun_out/ncu_des_c4.log
