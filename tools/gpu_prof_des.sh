cd $GRAFT_REPO_ROOT
NCU=/usr/local/cuda/bin/ncu
timeout 1500 $NCU --set full --clock-control none --import-source on -k regex:"${KERNEL:-des_kernel}" -c 1 -o gpurun_out/prof_${TAG:-des} python tools/prof_one.py ${NSEEDS:-64} > gpurun_out/prof_${TAG:-des}.txt 2>&1
tail -3 gpurun_out/prof_${TAG:-des}.txt
