#!/bin/bash
# ncu --set full of the DES in the saturated C4 regime (default.yaml cut to 300 s, 4 variants x 592 seeds
# = 2368 replicas = 16 warps/SM on 148 SMs, one wave) + the SIMT-vs-warp probe at many replicas
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 1200 $NCU --set full --import-source on --clock-control none -k regex:${KREGEX:-des_kernel_reg} -c 1 -o gpurun_out/ncu_des_c4 \
  python tools/ab_des.py scenarios/exp/default_300s.yaml ${NSEEDS:-592} c4 warp 1 > gpurun_out/ncu_des_c4.log 2>&1
tail -3 gpurun_out/ncu_des_c4.log
${EXTRA:-true}
