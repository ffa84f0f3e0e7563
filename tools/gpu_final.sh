# Round-end measurement pass: full GPU suite, smoke, bench (+CPU baseline, C4 secondary), reference
# arm, 2-rank bench (both ranks on this GPU, gloo collectives), ncu launch list + full captures.
cd $GRAFT_REPO_ROOT
bash tools/gpu_round.sh
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference.json 2>&1; tail -c 400 gpurun_out/bench_reference.json
bash tools/gpu_multirank.sh
