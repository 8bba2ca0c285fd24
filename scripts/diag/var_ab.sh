#!/bin/bash
# A/B of library variants (lib/variants/libtwb200_<v>.so) on the pair shapes; kernel-only.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
TAG=${TAG:-r02J}
{
for rep in 1 2; do
  for v in ${VARIANTS:-main}; do
    if [ "$v" = main ]; then unset TWB_LIBRARY; else export TWB_LIBRARY=$PWD/paper_2007_16135_b200/lib/variants/libtwb200_$v.so; fi
    echo "== $v rep $rep"
    timeout 300 python scripts/tune.py pair 1000000 3 f64
    timeout 300 python scripts/tune.py pair 1000000 1 f64
    timeout 300 python scripts/tune.py pair 300000 3 f64
    timeout 300 python scripts/tune.py pair 100000 1 f64
  done
done
unset TWB_LIBRARY
} > gpurun_out/${TAG}_var.log 2>&1
cat gpurun_out/${TAG}_var.log
