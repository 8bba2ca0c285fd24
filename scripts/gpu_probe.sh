#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-p}
{
for cfg in k8w8 k4w8x2; do
for na in 256 1024 2048 16384 303104; do
TWB_WAVE_CFG=$cfg timeout 100 python scripts/tune.py pair2 $na 400000 3 f64
done; done
TWB_WAVE_CFG=k8w8 timeout 100 python scripts/tune.py pair2 2048 400000 1 f64
TWB_WAVE_CFG=k8w8 timeout 100 python scripts/tune.py pair2 256 400000 1 f64
} > gpurun_out/${TAG}_probe.log 2>&1
cat gpurun_out/${TAG}_probe.log
