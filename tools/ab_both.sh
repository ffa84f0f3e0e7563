cd $GRAFT_REPO_ROOT
for v in ${VARS}; do MIGSIM_LIB=$PWD/build/var$v/libmigsim_b200.so timeout 300 python tools/ab_variant.py 2>&1 | tail -1; MIGSIM_LIB=$PWD/build/var$v/libmigsim_b200.so timeout 300 python tools/ab_variant.py scenarios/c5_mc64.yaml 512 2>&1 | tail -1; done
