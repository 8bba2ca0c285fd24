#!/bin/bash
# Parity tests + kernel timings + small ncu captures (one gpurun call).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r01b}
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/${TAG}_pytest.log
{
timeout 300 python scripts/tune.py pair 1000000 3 f64 8 7 6
timeout 120 python scripts/tune.py pair 1000000 3 f32 8 7
timeout 120 python scripts/tune.py pair 100000 1 f64 0
timeout 120 python scripts/tune.py pair 1000 1 f64 0
timeout 120 python scripts/tune.py batch 10000 128 2 f32 1
timeout 120 python scripts/tune.py batch 1000 256 1 f64 0
} > gpurun_out/${TAG}_tune.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:wave_kernel -c 1 \
  -o gpurun_out/${TAG}_wave_n131k -f python scripts/prof_one.py cfg3 --n 131072 > gpurun_out/${TAG}_ncu_wave.log 2>&1
echo "ncu wave exit $?" >> gpurun_out/${TAG}_ncu_wave.log
tail -3 gpurun_out/${TAG}_pytest.log; cat gpurun_out/${TAG}_tune.log; tail -4 gpurun_out/${TAG}_ncu_wave.log
