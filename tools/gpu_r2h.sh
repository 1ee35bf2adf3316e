#!/bin/bash
set -u
TAG=${1:-r02h}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
echo "== fit trace"; RPG_FIT_TRACE=1 timeout 900 python tools/bench_fit.py --reps 1 --noise 0.01 > $O/fit_trace.log 2>&1; echo "rc=$?"; grep -E 'minimizer|Newton tail|safeguard' $O/fit_trace.log | head -16
echo "== fit bench"; timeout 900 python tools/bench_fit.py --noise 0.01 > $O/fit_noisy.log 2>&1; echo "rc=$?"; tail -1 $O/fit_noisy.log | cut -c1-1200
echo "== pytest"
timeout 2400 python -m pytest tests/test_gpu_fit.py tests/test_gpu_fit_c4.py -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?"; tail -5 $O/pytest_gpu.log
