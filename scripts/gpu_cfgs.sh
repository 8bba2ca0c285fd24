#!/bin/bash
# Wave configurations per variant build at n=1M d=3 fp64 (and d=1).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
{
for vc in ${VCS}; do
  v=${vc%%:*}; c=${vc#*:}
  if [ "$v" != default ]; then export TWB_LIBRARY=$PWD/paper_2007_16135_b200/lib/variants/libtwb200_$v.so; else unset TWB_LIBRARY; fi
  if [ "$c" != "-" ]; then export TWB_WAVE_CFG=$c; else unset TWB_WAVE_CFG; fi
  for spec in ${SPECS:-"1000000 3 f64 0"}; do
    timeout 100 python scripts/tune.py pair $(echo $spec | tr , " ") 2>&1 | tail -1 | sed "s/\$/ variant=$v cfg=$c/"
  done
done
} > gpurun_out/${TAG:-cfgs}.log 2>&1
cat gpurun_out/${TAG:-cfgs}.log
