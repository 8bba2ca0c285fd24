#!/bin/bash
# Round 2: GPU tests (all, no -x) + timings per library variant.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r02b}
if [ -z "$SKIP_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -q --durations=5 ${PYTEST_ARGS:-} > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/${TAG}_pytest.log
fi
{
for v in "" ${VARIANTS:-}; do
  if [ -n "$v" ]; then export TWB_LIBRARY=$PWD/paper_2007_16135_b200/lib/variants/libtwb200_$v.so; else unset TWB_LIBRARY; fi
  echo "== variant ${v:-main}"
  ${TUNE:-true}
done
} > gpurun_out/${TAG}_tune.log 2>&1
tail -30 gpurun_out/${TAG}_pytest.log 2>/dev/null; cat gpurun_out/${TAG}_tune.log
