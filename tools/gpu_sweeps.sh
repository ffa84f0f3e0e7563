# C4 / C5 sweep measurements on one GPU (BASELINE configs[3] / configs[4] shapes) + sweep tests.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_sweep.py -x -q > gpurun_out/pytest_sweep.txt 2>&1; tail -3 gpurun_out/pytest_sweep.txt
timeout 900 python -m paper_2508_20274_b200.sweep --scenario tests/golden/scenarios/default.yaml --variants ablation --seeds ${C4_SEEDS:-4096} --out gpurun_out/sweep_c4.json > gpurun_out/sweep_c4.log 2>&1; tail -c 600 gpurun_out/sweep_c4.json
timeout 900 python -m paper_2508_20274_b200.sweep --scenario scenarios/c5_mc64.yaml --variants full --seeds ${C5_SEEDS:-2048} --out gpurun_out/sweep_c5.json > gpurun_out/sweep_c5.log 2>&1; tail -c 600 gpurun_out/sweep_c5.json
tail -3 gpurun_out/sweep_c5.log
