#!/bin/bash
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
echo "== fit tests"; timeout 900 python -m pytest tests/test_gpu_fit.py -x -q -m gpu > gpurun_out/pytest_fit.log 2>&1; echo "rc=$?"; tail -30 gpurun_out/pytest_fit.log
