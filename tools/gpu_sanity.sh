#!/bin/bash
# gpurun session: GPU tests of the f1-f3 rows (program, sanity/samples),
# then the full GPU suite.  Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
echo "== pytest sanity+program"; timeout 1200 python -m pytest tests/test_gpu_sanity.py tests/test_gpu_program.py -q -m gpu > gpurun_out/pytest_sanity.log 2>&1; echo "rc=$?"; tail -40 gpurun_out/pytest_sanity.log
echo "== pytest gpu (all)"; timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_all.log 2>&1; echo "rc=$?"; tail -5 gpurun_out/pytest_gpu_all.log
