#!/bin/bash
# Side-by-side builds for A/B timing: tools/build_var.sh NAME "EXTRA_NVFLAGS" -> build/varNAME/libmigsim_b200.so
set -e
cd "$(dirname "$0")/.."
make -s -C paper_2508_20274_b200/csrc OUT=$PWD/build/var$1 OBJ=$PWD/build/var$1/obj EXTRA_NVFLAGS="$2" -j8
grep -A2 "des_kernel_reg" build/var$1/obj/engine_kernels.ptxas.txt | grep -E "Used|spill" | head -2
