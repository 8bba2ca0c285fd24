cd ${GRAFT_REPO_ROOT:-/root/repo}; mkdir -p gpurun_out
{ echo "== race hunt k8w8 ws8 (K=8 rows in registers)"; timeout 900 python scripts/diag/race_hunt2.py;
  echo "== mid sizes by config"
  for cfg in "" k8w8 k6w12 k4w12; do
    if [ -n "$cfg" ]; then export TWB_WAVE_CFG=$cfg; else unset TWB_WAVE_CFG; fi
    echo "-- ${cfg:-default}"
    for n in 100000 300000 600000; do timeout 300 python scripts/tune.py pair $n 3 f64; done
    timeout 300 python scripts/tune.py pair 300000 1 f64
  done; } > gpurun_out/r02O.log 2>&1
cat gpurun_out/r02O.log
