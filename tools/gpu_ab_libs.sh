#!/bin/bash
# A/B of side-by-side builds (build/var<NAME>/libmigsim_b200.so; "default" = the in-tree library) on the
# saturated C4 shape: default.yaml cut to 300 s x 4 variants x 4096 seeds, and the 1800 s default.yaml x 4 x 1024
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for v in ${VARS:-default}; do
  if [ "$v" = default ]; then L=""; else L=$PWD/build/var$v/libmigsim_b200.so; fi
  for a in "scenarios/exp/default_300s.yaml 4096" "tests/golden/scenarios/default.yaml 1024"; do
    MIGSIM_LIB=$L timeout 600 python tools/ab_des.py $a c4 warp 2 2>&1 | tail -1 | sed "s/^/$v /"
  done
done | tee gpurun_out/ab_libs.txt
