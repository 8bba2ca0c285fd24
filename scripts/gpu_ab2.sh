#!/bin/bash
# A/B variant builds: 1M d=3 fp64 pair and one pinned 12-warp CTA.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
{
for v in default ${VARIANTS}; do
  if [ "$v" != default ]; then export TWB_LIBRARY=$PWD/paper_2007_16135_b200/lib/variants/libtwb200_$v.so; else unset TWB_LIBRARY; fi
  timeout 100 python scripts/tune.py pair 1000000 3 f64 0 | sed "s/\$/ variant=$v/"
  TWB_WAVE_WS=12 TWB_WAVE_CFG=k6w12 timeout 100 python scripts/tune.py pair2 2304 400000 3 f64 | sed "s/\$/ variant=$v/"
  for s in ${SPECS}; do timeout 100 python scripts/tune.py pair $(echo $s | tr , ' ') | sed "s/\$/ variant=$v/"; done
done
} > gpurun_out/${TAG:-ab2}.log 2>&1
cat gpurun_out/${TAG:-ab2}.log
