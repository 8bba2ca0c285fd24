#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/c2_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/c2_pytest.log
{
for c in k6w12 k6w12c2 k4w12c2 k8w8c2; do
  TWB_WAVE_CFG=$c timeout 100 python scripts/tune.py pair 1000000 3 f64 0 | sed "s/\$/ $c/"
  TWB_WAVE_CFG=$c timeout 100 python scripts/tune.py pair 1000000 1 f64 0 | sed "s/\$/ $c/"
  TWB_WAVE_CFG=$c timeout 100 python scripts/tune.py pair 1000000 3 f32 0 | sed "s/\$/ $c/"
done
# correctness of the C=2 path against the fp64 1M golden and small sizes
for c in k6w12c2 k4w12c2; do
  TWB_WAVE_CFG=$c timeout 300 python -m pytest tests -m gpu -q -x -k "random_pairs or config_goldens or cfg2 or extreme or band_solve" 2>&1 | tail -1 | sed "s/\$/ pytest $c/"
done
} > gpurun_out/c2_tune.log 2>&1
tail -2 gpurun_out/c2_pytest.log; cat gpurun_out/c2_tune.log
