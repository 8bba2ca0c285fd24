#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
{
for cfg in ${CFGS:-k6w12}; do
for na in 192 2304 340992 1000000; do
TWB_WAVE_CFG=$cfg timeout 100 python scripts/tune.py pair2 $na 400000 3 f64
done; done
} > gpurun_out/${TAG:-p2}_probe.log 2>&1
cat gpurun_out/${TAG:-p2}_probe.log
