#!/bin/bash
# Stage the REFERENCE's own test suite (/root/reference/pkg/tests, read-only,
# present only in the build container) into the git-ignored
# baseline/_ref_tests/, so a gpurun call can run it against this package
# imported under the name `batchode` (tools/batchode_alias.py is loaded as a
# pytest plugin before the reference's conftest imports batchode).
#   bash tools/stage_reference_tests.sh
#   gpurun -- 'PYTHONPATH=$PWD:$PWD/tools python -m pytest -p batchode_alias baseline/_ref_tests'
set -e
cd "$(dirname "$0")/.."
rm -rf baseline/_ref_tests
mkdir -p baseline/_ref_tests
cp /root/reference/pkg/tests/*.py baseline/_ref_tests/
echo "staged $(ls baseline/_ref_tests | wc -l) files"
