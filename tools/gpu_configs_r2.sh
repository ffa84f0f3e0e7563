#!/bin/bash
# Round-2 BASELINE config sweep on one B200 (C1, C3, C5; C4 is bench.py's headline, C2 its secondary)
# plus the reference fan-out (oracle/_ref) on this box's cores over 8 x nproc contiguous seeds each.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m paper_2508_20274_b200.sweep --scenario scenarios/c1_single_host.yaml --variants full --seeds 4096 --out gpurun_out/sweep_c1.json > gpurun_out/sweep_c1.log 2>&1; tail -c 300 gpurun_out/sweep_c1.json; echo
timeout 900 python -m paper_2508_20274_b200.sweep --scenario scenarios/c3_llm_bursty.yaml --variants full --seeds 4096 --out gpurun_out/sweep_c3.json > gpurun_out/sweep_c3.log 2>&1; tail -c 300 gpurun_out/sweep_c3.json; echo
timeout 1500 python -m paper_2508_20274_b200.sweep --scenario scenarios/c5_mc64.yaml --variants full --seeds 2048 --out gpurun_out/sweep_c5.json > gpurun_out/sweep_c5.log 2>&1; tail -c 300 gpurun_out/sweep_c5.json; echo
timeout 1500 python tools/ref_sample.py scenarios/c1_single_host.yaml scenarios/c3_llm_bursty.yaml scenarios/c5_mc64.yaml > gpurun_out/ref_sample.json 2>&1; cat gpurun_out/ref_sample.json
