#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
{
for v in "" dsetp nomin; do
  if [ -n "$v" ]; then export TWB_LIBRARY=$PWD/paper_2007_16135_b200/lib/variants/libtwb200_$v.so; else unset TWB_LIBRARY; fi
  timeout 100 python scripts/tune.py pair 1000000 3 f64 0 | sed "s/\$/ variant=${v:-default}/"
  TWB_WAVE_CFG=k8w8 timeout 100 python scripts/tune.py pair 1000000 3 f64 0 | sed "s/\$/ variant=${v:-default} k8w8/"
  timeout 100 python scripts/tune.py pair 1000000 1 f64 0 | sed "s/\$/ variant=${v:-default}/"
done
} > gpurun_out/m1_variants.log 2>&1
unset TWB_LIBRARY
bash scripts/run_reference_suite.sh > gpurun_out/m1_refsuite.log 2>&1
cat gpurun_out/m1_variants.log; tail -25 gpurun_out/m1_refsuite.log
