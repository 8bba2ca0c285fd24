#!/bin/bash
# One gpurun call: parity tests, smoke, bench (with CPU baseline), reference
# arm, ncu launch list of the bench command, ncu --set full of the hot kernels.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/${TAG}_smoke.log
if [ -z "$SKIP_TESTS" ]; then
timeout 900 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/${TAG}_pytest_gpu.log
fi
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench exit $?" >> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
echo "ref exit $?" >> gpurun_out/${TAG}_bench_ref.err
if [ -z "$SKIP_REFSUITE" ]; then
bash scripts/run_reference_suite.sh > gpurun_out/${TAG}_refsuite.log 2>&1
fi
if [ -z "$SKIP_NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu \
  > gpurun_out/${TAG}_ncu_launch_bench.log 2>&1
echo "ncu launches exit $?" >> gpurun_out/${TAG}_ncu_launch_bench.log
TWB_WAVE_CFG=k6w12 TWB_WAVE_WS=12 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:wave_kernel<.*\(bool\)0, \(bool\)[01], \(int\)' -c 1 \
  -o gpurun_out/${TAG}_wave_k6w12_n400k -f python scripts/prof_one.py cfg3 --n 400000 > gpurun_out/${TAG}_ncu_wave.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k 'regex:wave_kernel<.*\(bool\)0, \(bool\)[01], \(int\)' -c 1 \
  --csv --log-file gpurun_out/${TAG}_wave_cfg3_dram.csv python scripts/prof_one.py cfg3 > gpurun_out/${TAG}_ncu_wave_dram.log 2>&1
echo "ncu wave exit $?" >> gpurun_out/${TAG}_ncu_wave.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:batch_kernel -c 1 \
  -o gpurun_out/${TAG}_batch_cfg5 -f python scripts/prof_one.py cfg5 > gpurun_out/${TAG}_ncu_batch.log 2>&1
echo "ncu batch exit $?" >> gpurun_out/${TAG}_ncu_batch.log
fi
tail -3 gpurun_out/${TAG}_smoke.log; tail -3 gpurun_out/${TAG}_refsuite.log; tail -15 gpurun_out/${TAG}_pytest_gpu.log; cat gpurun_out/${TAG}_bench.json gpurun_out/${TAG}_bench_ref.json; tail -n 3 gpurun_out/${TAG}_bench.err gpurun_out/${TAG}_bench_ref.err gpurun_out/${TAG}_ncu_*.log
