#!/bin/bash
# Round-2 tuning sweep: headline pair on the main build, then mid-size pair
# configurations on variant builds (TWB_LIBRARY) -- kernel-only event timings.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r02t}
{
echo "== main"
timeout 300 python scripts/tune.py pair 1000000 3 f64
timeout 300 python scripts/tune.py pair 1000000 1 f64
timeout 300 python scripts/tune.py pair 100000 1 f64
timeout 300 python scripts/tune.py pair 100000 3 f64
for v in cfgx chs8; do
  export TWB_LIBRARY=$PWD/paper_2007_16135_b200/lib/variants/libtwb200_$v.so
  for cfg in k6w12 k4w12 k3w12 k2w12 k3w16 k2w16 k4w8 k2w8x2 k3w8x2; do
    echo "== $v $cfg (cfg2 n=100k d=1; n=300k d=3)"
    TWB_WAVE_CFG=$cfg timeout 120 python scripts/tune.py pair 100000 1 f64 0 4 8 12 16
    TWB_WAVE_CFG=$cfg timeout 120 python scripts/tune.py pair 300000 3 f64 0
  done
done
unset TWB_LIBRARY
} > gpurun_out/${TAG}_tune.log 2>&1
cat gpurun_out/${TAG}_tune.log | grep -v "^$" | tail -120
