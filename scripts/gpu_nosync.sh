#!/bin/bash
# Coupling headroom: the wave kernel with its CTA (1) / CTA+warp (2) waits removed.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
{
for v in default nosync1 nosync2; do
  if [ "$v" != default ]; then export TWB_LIBRARY=$PWD/paper_2007_16135_b200/lib/variants/libtwb200_$v.so; else unset TWB_LIBRARY; fi
  timeout 100 python scripts/tune.py pair 1000000 3 f64 0 | sed "s/\$/ variant=$v/"
  TWB_WAVE_CFG=k6w12 timeout 100 python scripts/tune.py pair2 2304 400000 3 f64 | sed "s/\$/ variant=$v/"
  TWB_WAVE_CFG=k6w12 timeout 100 python scripts/tune.py pair2 36864 400000 3 f64 | sed "s/\$/ variant=$v/"
done
unset TWB_LIBRARY
timeout 300 python scripts/diag/gap.py > gpurun_out/gap2.log 2>&1
} > gpurun_out/nosync.log 2>&1
cat gpurun_out/nosync.log gpurun_out/gap2.log
