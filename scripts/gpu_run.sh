#!/bin/bash
# One gpurun call of the round's measurement loop. Steps are chosen by env:
#   TAG=r02c  STEPS="smoke tests bench ref launches ncu_wave ncu_batch ncu_prep refsuite"
#   BENCH_ARGS="..."  PYTEST_ARGS="..."
# Everything lands in gpurun_out/${TAG}_*.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r02}
STEPS=${STEPS:-"smoke tests bench"}
has() { [[ " $STEPS " == *" $1 "* ]]; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
K_WAVE='regex:wave_kernel<.*\(bool\)0, \(bool\)[01], \(int\)'
if has smoke; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
  echo "smoke exit $?" >> gpurun_out/${TAG}_smoke.log
fi
if has tests; then
  timeout 1500 python -m pytest tests -m gpu -q --durations=10 ${PYTEST_ARGS:-} > gpurun_out/${TAG}_pytest_gpu.log 2>&1
  echo "pytest exit $?" >> gpurun_out/${TAG}_pytest_gpu.log
fi
if has bench; then
  timeout 1200 python bench.py ${BENCH_ARGS:-} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
  echo "bench exit $?" >> gpurun_out/${TAG}_bench.err
fi
if has ref; then
  timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
  echo "ref exit $?" >> gpurun_out/${TAG}_bench_ref.err
fi
if has refsuite; then
  bash scripts/run_reference_suite.sh > gpurun_out/${TAG}_refsuite.log 2>&1
fi
if has launches; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-extra \
    > gpurun_out/${TAG}_ncu_launch_bench.log 2>&1
  echo "ncu launches exit $?" >> gpurun_out/${TAG}_ncu_launch_bench.log
fi
# every section of --set full except SourceCounters (its SASS instrumentation
# slows a 2 s launch past any timeout; the source view comes from ncu_wave_src)
FULL_NO_SRC="--section SpeedOfLight --section ComputeWorkloadAnalysis --section InstructionStats \
  --section LaunchStats --section Occupancy --section SchedulerStats --section WarpStateStats \
  --section MemoryWorkloadAnalysis --section MemoryWorkloadAnalysis_Chart \
  --section MemoryWorkloadAnalysis_Tables --section SpeedOfLight_RooflineChart --section WorkloadDistribution"
if has ncu_wave; then
  # the benchmarked cfg3 launch itself: no configuration overrides
  timeout 1500 ncu $FULL_NO_SRC --metrics dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --kernel-name-base demangled \
    -k "$K_WAVE" -c 1 -o gpurun_out/${TAG}_wave_cfg3 -f python scripts/prof_one.py cfg3 \
    > gpurun_out/${TAG}_ncu_wave.log 2>&1
  echo "ncu wave exit $?" >> gpurun_out/${TAG}_ncu_wave.log
fi
if has ncu_dram; then
  # DRAM bytes + duration of the benchmarked cfg3 sweep and of the fused precompute (one launch each)
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    --kernel-name-base demangled -k "$K_WAVE" -c 1 --csv --log-file gpurun_out/${TAG}_wave_cfg3_dram.csv \
    python scripts/prof_one.py cfg3 > gpurun_out/${TAG}_ncu_dram.log 2>&1
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    --kernel-name-base demangled -k regex:prepare_kernel -c 1 --csv --log-file gpurun_out/${TAG}_prepare_cfg3_dram.csv \
    python scripts/prof_one.py cfg3 >> gpurun_out/${TAG}_ncu_dram.log 2>&1
  echo "ncu dram exit $?" >> gpurun_out/${TAG}_ncu_dram.log
fi
if has ncu_wave_src; then
  # source-level counters on the same kernel configuration at n = 400k (one round of stripes)
  TWB_WAVE_CFG=k6w12 TWB_WAVE_WS=12 timeout 1200 ncu --set full --clock-control none --import-source on \
    --kernel-name-base demangled -k "$K_WAVE" -c 1 -o gpurun_out/${TAG}_wave_k6w12_n400k -f \
    python scripts/prof_one.py cfg3 --n 400000 > gpurun_out/${TAG}_ncu_wave_src.log 2>&1
  echo "ncu wave src exit $?" >> gpurun_out/${TAG}_ncu_wave_src.log
fi
if has ncu_batch; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:batch_kernel -c 1 \
    -o gpurun_out/${TAG}_batch_cfg5 -f python scripts/prof_one.py cfg5 > gpurun_out/${TAG}_ncu_batch.log 2>&1
  echo "ncu batch exit $?" >> gpurun_out/${TAG}_ncu_batch.log
fi
if has ncu_prep; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:prepare_kernel -c 1 \
    -o gpurun_out/${TAG}_prepare_cfg3 -f python scripts/prof_one.py cfg3 > gpurun_out/${TAG}_ncu_prep.log 2>&1
  echo "ncu prep exit $?" >> gpurun_out/${TAG}_ncu_prep.log
fi
if [ -n "$EXTRA_CMD" ]; then
  bash -c "$EXTRA_CMD" > gpurun_out/${TAG}_extra.log 2>&1
  echo "extra exit $?" >> gpurun_out/${TAG}_extra.log
fi
for f in gpurun_out/${TAG}_smoke.log gpurun_out/${TAG}_pytest_gpu.log gpurun_out/${TAG}_refsuite.log; do
  [ -f $f ] && tail -6 $f
done
[ -f gpurun_out/${TAG}_bench.json ] && cat gpurun_out/${TAG}_bench.json && tail -4 gpurun_out/${TAG}_bench.err
[ -f gpurun_out/${TAG}_bench_ref.json ] && cat gpurun_out/${TAG}_bench_ref.json
[ -f gpurun_out/${TAG}_extra.log ] && tail -40 gpurun_out/${TAG}_extra.log
tail -n 2 gpurun_out/${TAG}_ncu_*.log 2>/dev/null
exit 0
