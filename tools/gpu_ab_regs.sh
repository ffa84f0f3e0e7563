cd $GRAFT_REPO_ROOT
for lib in default 64 80 96; do
  for rings in auto global; do
    if [ $lib = default ]; then L=""; else L=$PWD/build/var$lib/libmigsim_b200.so; fi
    MIGSIM_LIB=$L MIGSIM_RINGS=$rings timeout 300 python tools/ab_des.py tests/golden/scenarios/default.yaml 4096 c4 warp 1 2>&1 | tail -1
  done
done > gpurun_out/ab_regs_c4.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:des_kernel_reg -c 1 -o gpurun_out/ncu_des_c4 python tools/ab_des.py tests/golden/scenarios/default.yaml 2048 c4 warp 1 > gpurun_out/ncu_des_c4.log 2>&1
cat gpurun_out/ab_regs_c4.txt; tail -3 gpurun_out/ncu_des_c4.log
