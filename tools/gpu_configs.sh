# Full-size BASELINE configs on one GPU: C3 (4096 seeds), C4 (16384 seeds x 4 variants), plus fuzz.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m paper_2508_20274_b200.sweep --scenario scenarios/c3_llm_bursty.yaml --variants full --seeds 4096 --out gpurun_out/sweep_c3.json > gpurun_out/sweep_c3.log 2>&1; tail -c 300 gpurun_out/sweep_c3.json
timeout 1200 python -m paper_2508_20274_b200.sweep --scenario tests/golden/scenarios/default.yaml --variants c4 --seeds 16384 --out gpurun_out/sweep_c4_full.json > gpurun_out/sweep_c4_full.log 2>&1; tail -c 300 gpurun_out/sweep_c4_full.json
timeout 900 python tools/gpu_fuzz_loop.py 20000 24000 > gpurun_out/fuzz_20000.txt 2>&1; echo "fuzz fails: $(grep -c FAIL gpurun_out/fuzz_20000.txt)"
timeout 900 python tools/ref_sample.py scenarios/c3_llm_bursty.yaml tests/golden/scenarios/default.yaml scenarios/c5_mc64.yaml > gpurun_out/ref_sample.json 2>&1; cat gpurun_out/ref_sample.json
