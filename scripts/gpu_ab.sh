#!/bin/bash
# A/B the in-tree library against variant builds (lib/variants/libtwb200_<v>.so).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
{
for v in default ${VARIANTS}; do
  if [ "$v" != default ]; then export TWB_LIBRARY=$PWD/paper_2007_16135_b200/lib/variants/libtwb200_$v.so; else unset TWB_LIBRARY; fi
  for spec in ${SPECS:-"pair 1000000 3 f64 0" "pair 1000000 1 f64 0"}; do
    timeout 100 python scripts/tune.py $spec | sed "s/\$/ variant=$v/"
  done
  for c in ${CFGS}; do
    TWB_WAVE_CFG=$c timeout 100 python scripts/tune.py pair 1000000 3 f64 0 | sed "s/\$/ variant=$v $c/"
  done
done
} > gpurun_out/${TAG:-ab}_ab.log 2>&1
cat gpurun_out/${TAG:-ab}_ab.log
