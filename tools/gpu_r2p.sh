#!/bin/bash
# Fit: lattice monomials + unsplit mid-range products.  Bit A/B vs the
# previous build, step anatomy, timings, fit tests, one full ncu capture.
set -u
TAG=${1:-r02p}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
echo "== bits vs old"; timeout 1200 python tools/fit_ab_bits.py build/old_librpgpu.so > $O/ab_bits.log 2>&1; tail -1 $O/ab_bits.log
RPG_FIT_TRACE=1 timeout 900 python tools/bench_fit.py --reps 1 --noise 0.01 > $O/trace.log 2>&1
grep -E 'wall|per step' $O/trace.log | head -10
timeout 900 python tools/bench_fit.py --reps 3 --noise 0.01 > $O/bench_noisy.log 2>&1
timeout 900 python tools/bench_fit.py --reps 3 > $O/bench_clean.log 2>&1
for f in bench_noisy bench_clean; do tail -1 $O/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f seq %.1f ms multi %.1f ms' % (1e3*d['gpu_seconds'], 1e3*d['multi_seconds']))"; done
echo "== pytest"; timeout 1800 python -m pytest tests/test_gpu_fit.py tests/test_gpu_fit_c4.py -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?"; tail -3 $O/pytest_gpu.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:min_step -s 30 -c 2 -o $O/minstep_full python tools/bench_fit.py --reps 1 --noise 0.01 --no-warmup > $O/ncu.log 2>&1; echo "ncu rc=$?"
