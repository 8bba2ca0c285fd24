cd ${GRAFT_REPO_ROOT:-/root/repo}; mkdir -p gpurun_out
{ for v in ${VS:-main pfill0 sa0}; do
    if [ $v = main ]; then unset TWB_LIBRARY; else export TWB_LIBRARY=$PWD/paper_2007_16135_b200/lib/variants/libtwb200_$v.so; fi
    echo "== $v"; timeout 600 python scripts/diag/race_hunt2.py; done; } > gpurun_out/r02L_race.log 2>&1
cat gpurun_out/r02L_race.log
