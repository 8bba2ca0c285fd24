#!/bin/bash
# Sweep wave-kernel variants over sizes (tuning; not bench numbers).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-sw}
{
for n_d in "1000000 3" "1000000 1" "300000 3" "100000 1" "100000 3"; do
  set -- $n_d
  for c in ${CFGS:-k8w8 k6w12 k8w12 k4w16 k4w12 k2w8 k2w16}; do
    TWB_WAVE_CFG=$c timeout 100 python scripts/tune.py pair $1 $2 f64 0 | sed "s/\$/ $c/"
  done
done
timeout 100 python scripts/tune.py pair 1000000 3 f32 0 | sed 's/$/ default/'
for c in k8w8 k6w12 k8w12; do TWB_WAVE_CFG=$c timeout 100 python scripts/tune.py pair 1000000 3 f32 0 | sed "s/\$/ $c/"; done
} > gpurun_out/${TAG}_sweep.log 2>&1
cat gpurun_out/${TAG}_sweep.log
