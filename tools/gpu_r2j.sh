#!/bin/bash
set -u
TAG=${1:-r02j}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
echo "== bench c2"; timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > $O/bench_c2.log 2>&1; echo "rc=$?"; tail -1 $O/bench_c2.log | cut -c1-200; tail -1 $O/bench_c2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('frac', d['roofline']['frac'], 'kernel_ms', d['roofline']['kernel_ms'])"
echo "== bench dump"; timeout 900 python bench.py --workload dump --steps 5 --warmup 3 --no-cpu > $O/bench_dump.log 2>&1; echo "rc=$?"; tail -1 $O/bench_dump.log | cut -c1-300
echo "== fit trace"; RPG_FIT_TRACE=1 timeout 900 python tools/bench_fit.py --reps 1 --noise 0.01 > $O/fit_trace.log 2>&1; echo "rc=$?"; grep -E 'wall|Newton tail|minimizer:' $O/fit_trace.log | head -20
echo "== fit bench"; timeout 900 python tools/bench_fit.py --noise 0.01 > $O/fit_noisy.log 2>&1; echo "rc=$?"; tail -1 $O/fit_noisy.log | cut -c1-900
echo "== pytest"; timeout 2400 python -m pytest tests/test_gpu_fastcm.py tests/test_gpu_parity.py tests/test_gpu_fit.py tests/test_gpu_fit_c4.py -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?"; tail -3 $O/pytest_gpu.log
