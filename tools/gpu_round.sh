# One GPU pass: parity tests, smoke, bench (N=1), launch list, ncu --set full of select + DES.
# Inner timeouts sum below the gpurun limit given by the caller (see each line).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout ${T_TEST:-900} python -m pytest tests -m gpu -x -q ${PYTEST_K} > gpurun_out/pytest_gpu.txt 2>&1; tail -4 gpurun_out/pytest_gpu.txt
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
if [ -z "$NO_BENCH" ]; then
timeout 600 python bench.py --steps 3 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('VALUE', d['value'], 'e2e', d['e2e']['value']); print(d['kernels']); print(d['cpu_baseline']); print(d['clocks'])"
fi
NCU=/usr/local/cuda/bin/ncu
[ -z "$NO_LAUNCHES" ] && timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --c4-seeds 0 > gpurun_out/bench_under_ncu.txt 2>&1
[ -z "$NO_SEL_NCU" ] && timeout 300 $NCU --set full --clock-control none --import-source on -k regex:"select" -c 1 -o gpurun_out/prof_select python tools/prof_one.py 256 > gpurun_out/prof_select.txt 2>&1
[ -z "$NO_DES_NCU" ] && timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"des_kernel" -c 1 -o gpurun_out/prof_des python tools/prof_one.py 256 > gpurun_out/prof_des.txt 2>&1
ls gpurun_out
