#!/bin/bash
# Stage the reference package and its own test files under baseline/_ref
# (git-ignored; travels to the GPU box with gpurun).  Run in the build
# container, where /root/reference exists.  tests/test_reference_own_suite_gpu.py
# then runs those files against the drop-in (tests/refsuite/dropin_plugin.py).
set -e
cd "$(dirname "$0")/../.."
rm -rf /tmp/bak_refpkg baseline/_ref
cp -r /root/reference/pkg /tmp/bak_refpkg          # the build writes into the source tree
python -m pip install -q --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref /tmp/bak_refpkg
mkdir -p baseline/_ref/tests
cp /root/reference/pkg/tests/*.py baseline/_ref/tests/
echo "staged: $(ls baseline/_ref) ; tests: $(ls baseline/_ref/tests | tr '\n' ' ')"
