#!/bin/bash
# Run the staged reference tests (ref_tests/, see stage_ref_tests.sh) against the
# `dehaze` import name (dehaze/__init__.py -> paper_2512_16609_b200) on the GPU box.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
ROOT=$(pwd)
cd ref_tests
PYTHONPATH=$ROOT PYTHONDONTWRITEBYTECODE=1 timeout 3000 python -m pytest -q -p no:cacheprovider -rA \
  --continue-on-collection-errors -o addopts="" --junitxml=$ROOT/gpurun_out/ref_tests.xml . \
  > $ROOT/gpurun_out/ref_tests.log 2>&1
echo "pytest exit $?"
tail -5 $ROOT/gpurun_out/ref_tests.log
