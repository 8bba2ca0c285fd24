#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
{
for nd in "100000 1" "100000 3" "300000 3"; do
set -- $nd
for c in k8w8 k4w12 k2w8; do
TWB_WAVE_CFG=$c timeout 120 python scripts/tune.py pair $1 $2 f64 1 2 3 4 6 8 12 | sed "s/\$/ $c/"
done; done
} > gpurun_out/mid_sweep.log 2>&1
cat gpurun_out/mid_sweep.log
