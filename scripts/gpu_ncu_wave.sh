#!/bin/bash
# ncu captures of the main (proven-safe) wave sweep: the gated NaN-exact launch
# that precedes it in twed_dev returns at once and is skipped by the name filter.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r01j}
K='regex:wave_kernel<.*\(bool\)0, \(bool\)[01], \(int\)'
TWB_WAVE_CFG=k6w12 TWB_WAVE_WS=12 timeout 900 ncu --set full --clock-control none --import-source on \
  --kernel-name-base demangled -k "$K" -c 1 -o gpurun_out/${TAG}_wave_k6w12_n400k -f \
  python scripts/prof_one.py cfg3 --n 400000 > gpurun_out/${TAG}_ncu_wave.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  --kernel-name-base demangled -k "$K" -c 1 --csv --log-file gpurun_out/${TAG}_wave_cfg3_dram.csv \
  python scripts/prof_one.py cfg3 > gpurun_out/${TAG}_ncu_wave_dram.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:lcs_kernel -c 1 \
  -o gpurun_out/${TAG}_lcs_1m -f python scripts/lcs_prof.py 1000000 4 > gpurun_out/${TAG}_ncu_lcs.log 2>&1
tail -n 2 gpurun_out/${TAG}_ncu_wave.log gpurun_out/${TAG}_ncu_lcs.log; tail -1 gpurun_out/${TAG}_wave_cfg3_dram.csv | cut -c1-200
