#!/bin/bash
# Round-2 GPU pass g: fit tests, the fit trace/timing, C4 bench line.
set -u
TAG=${1:-r02g}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
echo "== pytest"
timeout 2400 python -m pytest tests/test_gpu_fit.py tests/test_gpu_fit_c4.py tests/test_gpu_group.py tests/test_gpu_dist.py -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?"; tail -5 $O/pytest_gpu.log
echo "== fit trace"; RPG_FIT_TRACE=1 timeout 900 python tools/bench_fit.py --reps 1 --noise 0.01 > $O/fit_trace.log 2>&1; echo "rc=$?"; grep minimizer $O/fit_trace.log | head -8
echo "== fit bench"; timeout 900 python tools/bench_fit.py --noise 0.01 > $O/fit_noisy.log 2>&1; echo "rc=$?"; tail -1 $O/fit_noisy.log | cut -c1-1200
echo "== fit bench clean"; timeout 900 python tools/bench_fit.py > $O/fit_clean.log 2>&1; echo "rc=$?"; tail -1 $O/fit_clean.log | cut -c1-1200
echo "== bench c4"; timeout 900 python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu > $O/bench_c4.log 2>&1; echo "rc=$?"; tail -1 $O/bench_c4.log | cut -c1-2500
echo "== ncu fit launches"; timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/fit_launches.csv python tools/bench_fit.py --reps 1 --noise 0.01 > $O/ncu_fit_launch.log 2>&1; echo "rc=$?"
