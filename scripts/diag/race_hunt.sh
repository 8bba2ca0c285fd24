cd ${GRAFT_REPO_ROOT:-/root/repo}; mkdir -p gpurun_out
{ echo "== main"; timeout 900 python scripts/diag/race_hunt.py;
  echo "== spin512"; TWB_LIBRARY=$PWD/paper_2007_16135_b200/lib/variants/libtwb200_spin512.so timeout 900 python scripts/diag/race_hunt.py; } > gpurun_out/r02K_race.log 2>&1
cat gpurun_out/r02K_race.log
