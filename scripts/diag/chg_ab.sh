#!/bin/bash
# Headline sweep: CTA publish granularity (TWB_WAVE_CHG) and the umin0 variant.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
TAG=${TAG:-r02G}
{
for rep in 1 2; do
  for chg in ${CHGS:-256 1024 4096}; do
    echo "== chg $chg rep $rep"; TWB_WAVE_CHG=$chg timeout 300 python scripts/tune.py pair 1000000 3 f64
  done
  [ -n "$NO_UMIN" ] || { echo "== umin0 rep $rep"; TWB_LIBRARY=$PWD/paper_2007_16135_b200/lib/variants/libtwb200_umin0.so timeout 300 python scripts/tune.py pair 1000000 3 f64; }
done
} > gpurun_out/${TAG}_chg.log 2>&1
cat gpurun_out/${TAG}_chg.log
