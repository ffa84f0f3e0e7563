#!/bin/bash
# Rare-path check of the generator's call walk: a build whose long-call threshold is 6 positions
# (-DMG_GEN_LONG_CALL=6; production: 255, never reached) sends every call with a rejection through
# lane 0's serial fallback and leaves many 4-call lengths unknown; the arrival parity tests must
# still pass bit-exact.  Build first: tools/build_var.sh long6 "-DMG_GEN_LONG_CALL=6"
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
MIGSIM_LIB=$PWD/build/varlong6/libmigsim_b200.so timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k arrivals \
  > gpurun_out/long6_pytest.txt 2>&1; tail -2 gpurun_out/long6_pytest.txt
