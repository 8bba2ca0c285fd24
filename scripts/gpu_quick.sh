#!/bin/bash
# Quick: GPU parity tests + wave/batch timings.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-q}
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/${TAG}_pytest.log
{
timeout 200 python scripts/tune.py pair 1000000 3 f64 0
for c in ${CFGS:-k4w16}; do TWB_WAVE_CFG=$c timeout 200 python scripts/tune.py pair 1000000 3 f64 0; echo "^ $c"; done
timeout 200 python scripts/tune.py pair 300000 3 f64 0
timeout 200 python scripts/tune.py pair 100000 1 f64 0
timeout 120 python scripts/tune.py batch 10000 128 2 f32 1
${EXTRA:-true}
} > gpurun_out/${TAG}_tune.log 2>&1
tail -5 gpurun_out/${TAG}_pytest.log; cat gpurun_out/${TAG}_tune.log
