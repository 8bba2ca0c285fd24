#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
{
for na in 2048 4096 8192 32768 131072 303104; do
TWB_WAVE_CFG=k8w8 timeout 100 python scripts/tune.py pair2 $na 400000 3 f64
done
for chg in 32 1024; do
TWB_WAVE_CHG=$chg TWB_WAVE_CFG=k8w8 timeout 100 python scripts/tune.py pair2 32768 400000 3 f64 | sed "s/\$/ chg=$chg/"
done
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv -lms 100 > gpurun_out/p3_clocks.csv &
CP=$!
TWB_WAVE_CFG=k8w8 timeout 100 python scripts/tune.py pair2 303104 1000000 3 f64
kill $CP
} > gpurun_out/${TAG:-p3}_probe.log 2>&1
cat gpurun_out/${TAG:-p3}_probe.log; sort gpurun_out/p3_clocks.csv | uniq -c | sort -rn | head -8
