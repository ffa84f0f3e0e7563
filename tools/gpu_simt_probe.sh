#!/bin/bash
# SIMT vs warp DES when the wave holds many more replicas (short horizon => small per-replica memory)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for n in 8192 16384; do
  timeout 900 python tools/ab_des.py scenarios/exp/default_300s.yaml $n c4 warp,simt 1 2>&1 | tail -3
done > gpurun_out/simt_probe.txt
cat gpurun_out/simt_probe.txt
