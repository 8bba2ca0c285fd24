#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{
for chg in 16 32 64 0; do
  if [ $chg = 0 ]; then unset TWB_WAVE_CHG; else export TWB_WAVE_CHG=$chg; fi
  echo "== chg $chg (0 = default rule)"
  timeout 300 python scripts/tune.py pair 1000000 3 f64
  timeout 300 python scripts/tune.py pair 1000000 1 f64
  timeout 300 python scripts/tune.py pair 100000 1 f64
  timeout 300 python scripts/tune.py pair 300000 3 f64
  timeout 300 python scripts/tune.py pair 1000000 3 f32
done
} > gpurun_out/r02I_chg.log 2>&1
cat gpurun_out/r02I_chg.log
