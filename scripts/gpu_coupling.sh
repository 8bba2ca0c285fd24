#!/bin/bash
# Inter-CTA coupling: single CTA (pinned 12 warps) with and without waits, chg sweep at 1M.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
{
for v in default nosync1; do
  if [ "$v" != default ]; then export TWB_LIBRARY=$PWD/paper_2007_16135_b200/lib/variants/libtwb200_$v.so; else unset TWB_LIBRARY; fi
  for na in 2304 4608 36864; do
    TWB_WAVE_WS=12 TWB_WAVE_CFG=k6w12 timeout 100 python scripts/tune.py pair2 $na 400000 3 f64 | sed "s/\$/ variant=$v ws=12/"
  done
done
unset TWB_LIBRARY
for chg in 32 64 128 512 2048; do
  TWB_WAVE_CHG=$chg timeout 100 python scripts/tune.py pair 1000000 3 f64 0 | sed "s/\$/ chg=$chg/"
done
} > gpurun_out/coupling.log 2>&1
cat gpurun_out/coupling.log
