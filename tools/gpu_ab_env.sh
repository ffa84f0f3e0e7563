#!/bin/bash
# A/B of environment settings / side-by-side builds on the saturated C4 shapes.
# ARMS="name|ENV=val ENV2=val|libvar" entries separated by ';' (libvar empty = in-tree library)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
IFS=';' read -ra A <<< "$ARMS"
for arm in "${A[@]}"; do
  name=$(echo "$arm" | cut -d'|' -f1); envs=$(echo "$arm" | cut -d'|' -f2); lv=$(echo "$arm" | cut -d'|' -f3)
  if [ -n "$lv" ]; then L=$PWD/build/var$lv/libmigsim_b200.so; else L=""; fi
  for a in ${SHAPES:-"scenarios/exp/default_300s.yaml:4736" "tests/golden/scenarios/default.yaml:2368"}; do
    sc=${a%%:*}; n=${a##*:}
    env $envs MIGSIM_LIB=$L timeout 600 python tools/ab_des.py $sc $n ${VSET:-c4} warp 2 2>&1 | tail -1 | sed "s/^/$name /"
  done
done | tee gpurun_out/ab_env.txt
