cd ${GRAFT_REPO_ROOT:-/root/repo}; mkdir -p gpurun_out
{ echo "== main k6w12 stress"; CFG=k6w12 timeout 900 python scripts/diag/race_hunt3.py;
  echo "== perf k8w8 ws8 300k d3: main / pfill0 / sa0";
  for v in main pfill0 sa0; do
    if [ $v = main ]; then unset TWB_LIBRARY; else export TWB_LIBRARY=$PWD/paper_2007_16135_b200/lib/variants/libtwb200_$v.so; fi
    echo "-- $v"; TWB_WAVE_CFG=k8w8 timeout 300 python scripts/tune.py pair 300000 3 f64 8; timeout 300 python scripts/tune.py pair 300000 3 f64; timeout 300 python scripts/tune.py pair 100000 3 f64; timeout 300 python scripts/tune.py pair 1000000 3 f64;
  done; } > gpurun_out/r02M_race.log 2>&1
cat gpurun_out/r02M_race.log
