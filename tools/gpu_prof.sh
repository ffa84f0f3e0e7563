cd $GRAFT_REPO_ROOT
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.txt 2>&1
tail -3 gpurun_out/launches.csv
timeout 1200 $NCU --set full --clock-control none --import-source on -k regex:"des_kernel|gen_times_kernel|gen_marks_kernel|select_kernel" -c 4 -o gpurun_out/prof_full python tools/prof_one.py 256 > gpurun_out/prof_full.txt 2>&1
tail -5 gpurun_out/prof_full.txt
ls -la gpurun_out
