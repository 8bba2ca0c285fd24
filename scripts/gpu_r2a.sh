#!/bin/bash
# Round 2: GPU tests (all, no -x) + runtime-d timings.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r02a}
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/${TAG}_pytest.log
{
timeout 120 python scripts/tune.py batch 2000 28 28 f64 1
timeout 120 python scripts/tune.py batch 2000 28 28 f32 1
timeout 120 python scripts/tune.py batch 1000 128 8 f64 0
timeout 200 python scripts/tune.py pair 100000 8 f64 0
timeout 200 python scripts/tune.py pair 100000 28 f64 0
timeout 200 python scripts/tune.py pair 300000 3 f64 0
TWB_FORCE_DYN=1 timeout 200 python scripts/tune.py pair 300000 3 f64 0
TWB_FORCE_DYN=1 timeout 120 python scripts/tune.py batch 10000 128 2 f32 1
${EXTRA:-true}
} > gpurun_out/${TAG}_tune.log 2>&1
tail -30 gpurun_out/${TAG}_pytest.log; cat gpurun_out/${TAG}_tune.log
