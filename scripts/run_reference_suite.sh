#!/bin/bash
# The reference's own tests (staged by scripts/stage_reference.sh) with the
# band solvers on the B200 kernels. Needs a GPU (gpurun).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
export NUMBA_CACHE_DIR=/tmp/twb_numba_cache
PYTHONPATH=$PWD/scripts:$PWD/baseline/_ref:$PWD timeout 1500 python -m pytest -q -p ref_seam_plugin \
  -p no:cacheprovider baseline/_ref_suite/tests baseline/_ref_suite/bindings/tests \
  -k "not test_plot_renders_heatmap and not test_out_writes_csv_and_figures" ${REF_ARGS:-} 2>&1 | tail -40
