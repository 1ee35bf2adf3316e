#!/bin/bash
# Fit: TSQR leaf tiles of 256 rows (default now); C4 stage agreement, timings.
set -u
O=gpurun_out/${1:-r02ab}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
RPG_FIT_TRACE=1 timeout 900 python tools/bench_fit.py --reps 1 --noise 0.01 --no-warmup > $O/trace.log 2>&1
grep -E '\] tsqr|host setup' $O/trace.log | head -8 | tr '\n' ' '; echo
timeout 900 python tools/bench_fit.py --reps 3 --noise 0.01 > $O/bench_noisy.log 2>&1
timeout 900 python tools/bench_fit.py --reps 3 > $O/bench_clean.log 2>&1
for f in bench_noisy bench_clean; do tail -1 $O/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f seq %.1f ms multi %.1f ms' % (1e3*d['gpu_seconds'], 1e3*d['multi_seconds']), d['safeguard'])"; done
echo "== pytest"; timeout 1800 python -m pytest tests/test_gpu_fit.py tests/test_gpu_fit_c4.py tests/test_gpu_dist.py tests/test_gpu_sanity.py -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?"; tail -3 $O/pytest_gpu.log; grep -E "^E  " $O/pytest_gpu.log | head -5 | cut -c1-300
