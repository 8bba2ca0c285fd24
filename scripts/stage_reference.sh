#!/bin/bash
# Stage the reference package and its test-suite in the git-ignored baseline/
# (it travels to the GPU box with the gpurun snapshot; /root/reference does not).
# Run in the build container only.
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/twb_refcopy && cp -r /root/reference/pkg /tmp/twb_refcopy
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target baseline/_ref --upgrade /tmp/twb_refcopy /tmp/twb_refcopy/bindings
rm -rf baseline/_ref_suite && mkdir -p baseline/_ref_suite
cp -r /root/reference/pkg/tests baseline/_ref_suite/tests
mkdir -p baseline/_ref_suite/bindings && cp -r /root/reference/pkg/bindings/tests baseline/_ref_suite/bindings/tests
echo staged
