cd ${GRAFT_REPO_ROOT:-/root/repo}; mkdir -p gpurun_out
TAG=${TAG:-r02p}
{ echo "== main"; timeout 900 python scripts/diag/ring_debug.py;
  echo "== r1"; TWB_LIBRARY=$PWD/paper_2007_16135_b200/lib/variants/libtwb200_r1.so timeout 900 python scripts/diag/ring_debug.py; } > gpurun_out/${TAG}_debug.log 2>&1
cat gpurun_out/${TAG}_debug.log
