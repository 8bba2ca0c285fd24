#!/bin/bash
# A/B of batch-kernel variants on short series (kernel-only timings).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
TAG=${TAG:-r02u}
{
for v in ${VARIANTS:-main lw16}; do
  if [ "$v" = main ]; then unset TWB_LIBRARY; else export TWB_LIBRARY=$PWD/paper_2007_16135_b200/lib/variants/libtwb200_$v.so; fi
  echo "== $v"
  IFS=';' read -ra cases <<< "${CASES:-2000 28 28 f64 1;2000 32 2 f64 1;4000 20 1 f32 1;3000 16 5 f64 0;10000 128 2 f32 1;2000 28 8 f64 1}"
  for c in "${cases[@]}"; do
    timeout 300 python scripts/tune.py batch $c
  done
done
unset TWB_LIBRARY
} > gpurun_out/${TAG}_batch_ab.log 2>&1
cat gpurun_out/${TAG}_batch_ab.log
