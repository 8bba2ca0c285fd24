#!/bin/bash
# Inbox ring length vs the headline sweep (kernel-only timings).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r02f}
{
for rb in 8192 32768 131072 1048576; do
  echo "== TWB_WAVE_RB=$rb"
  TWB_WAVE_RB=$rb timeout 300 python scripts/tune.py pair 1000000 3 f64
  TWB_WAVE_RB=$rb timeout 300 python scripts/tune.py pair 1000000 1 f64
done
echo "== per-stripe timestamps, rb default"
TWB_DBG_TIMES=gpurun_out/${TAG}_dbg_times.txt timeout 300 python scripts/tune.py pair 1000000 3 f64
} > gpurun_out/${TAG}_rb.log 2>&1
cat gpurun_out/${TAG}_rb.log
