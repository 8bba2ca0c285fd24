#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r01c}
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/${TAG}_pytest.log
{
for c in k8w8 k4w8x2 k4w16 k8w4x2; do TWB_WAVE_CFG=$c timeout 200 python scripts/tune.py pair 1000000 3 f64 0 7; echo "^ $c"; done
TWB_WAVE_CFG=k2w8 timeout 200 python scripts/tune.py pair 300000 3 f64 0; echo "^ k2w8 300k"
TWB_WAVE_CFG=k4w8x2 timeout 200 python scripts/tune.py pair 300000 3 f64 0; echo "^ k4w8x2 300k"
timeout 120 python scripts/tune.py batch 10000 128 2 f32 1
timeout 120 python scripts/tune.py batch 1000 256 1 f64 0
timeout 120 python scripts/tune.py batch 2000 64 3 f32 0
} > gpurun_out/${TAG}_tune.log 2>&1
TWB_WAVE_CFG=k8w8 timeout 400 ncu --set full --clock-control none --import-source on -k regex:wave_kernel -c 1 \
  -o gpurun_out/${TAG}_wave_k8_n300k -f python scripts/prof_one.py cfg3 --n 300000 > gpurun_out/${TAG}_ncu_wave.log 2>&1
echo "ncu wave exit $?" >> gpurun_out/${TAG}_ncu_wave.log
timeout 400 ncu --set full --clock-control none --import-source on -k regex:batch_kernel -c 1 \
  -o gpurun_out/${TAG}_batch_cfg5 -f python scripts/prof_one.py cfg5 > gpurun_out/${TAG}_ncu_batch.log 2>&1
echo "ncu batch exit $?" >> gpurun_out/${TAG}_ncu_batch.log
tail -15 gpurun_out/${TAG}_pytest.log; cat gpurun_out/${TAG}_tune.log; tail -2 gpurun_out/${TAG}_ncu_*.log
