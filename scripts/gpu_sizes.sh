#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG:-sz}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG:-sz}_pytest.log
{
for nd in "1000 1" "10000 1" "100000 1" "100000 3" "300000 3" "300000 1" "1000000 3" "1000000 1"; do
  set -- $nd; timeout 120 python scripts/tune.py pair $1 $2 f64 0
done
timeout 120 python scripts/tune.py pair 1000000 3 f32 0
} > gpurun_out/${TAG:-sz}_sizes.log 2>&1
tail -2 gpurun_out/${TAG:-sz}_pytest.log; cat gpurun_out/${TAG:-sz}_sizes.log
