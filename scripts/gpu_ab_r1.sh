#!/bin/bash
# A/B of library variants on one box, alternating; kernel-only event timings.
#   VARIANTS="main r1 nobp"  (main = the in-tree build; others lib/variants/libtwb200_<v>.so)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r02h}
{
for rep in 1 2; do
  for v in ${VARIANTS:-main r1}; do
    unset TWB_WAVE_SCRATCH_MB
    case $v in
      main) unset TWB_LIBRARY;;
      rings) unset TWB_LIBRARY; export TWB_WAVE_SCRATCH_MB=0;;  # bounded rings forced
      *) export TWB_LIBRARY=$PWD/paper_2007_16135_b200/lib/variants/libtwb200_$v.so;;
    esac
    echo "== $v rep $rep"
    timeout 300 python scripts/tune.py pair 1000000 3 f64
    timeout 300 python scripts/tune.py pair 1000000 1 f64
    timeout 300 python scripts/tune.py pair 100000 1 f64
  done
done
unset TWB_LIBRARY TWB_WAVE_SCRATCH_MB
} > gpurun_out/${TAG}_ab.log 2>&1
cat gpurun_out/${TAG}_ab.log
