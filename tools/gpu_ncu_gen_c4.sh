#!/bin/bash
# ncu --set full of the arrival generator (gen_times_kernel + gen_marks_kernel) on the C4 shape
# (default.yaml, 1800 s, 4 variants x NSEEDS (1024) seeds)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 1200 $NCU --set full --import-source on --clock-control none -k regex:"gen_times_kernel|gen_marks_kernel" -c 2 -o gpurun_out/ncu_gen_c4 \
  python tools/ab_des.py tests/golden/scenarios/default.yaml ${NSEEDS:-1024} c4 warp 1 > gpurun_out/ncu_gen_c4.log 2>&1
tail -2 gpurun_out/ncu_gen_c4.log
