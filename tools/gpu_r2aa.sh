#!/bin/bash
# Fit: start vector from the main R (no second TSQR); TSQR tile height A/B.
set -u
O=gpurun_out/${1:-r02aa}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
echo "== bits vs old"; timeout 1200 python tools/fit_ab_bits.py build/old_librpgpu.so > $O/ab_old.log 2>&1; tail -1 $O/ab_old.log
for v in default kt256 kt512; do
  if [ $v = default ]; then L=""; else L="RPG_LIBRARY=build/$v/librpgpu.so"; fi
  echo "== $v"
  env $L RPG_FIT_TRACE=1 timeout 900 python tools/bench_fit.py --reps 1 --noise 0.01 --no-warmup > $O/trace_$v.log 2>&1
  grep -E '\] tsqr|host setup' $O/trace_$v.log | head -8 | tr '\n' ' '; echo
  env $L timeout 900 python tools/bench_fit.py --reps 3 --noise 0.01 > $O/bench_noisy_$v.log 2>&1
  env $L timeout 900 python tools/bench_fit.py --reps 3 > $O/bench_clean_$v.log 2>&1
  for f in bench_noisy_$v bench_clean_$v; do tail -1 $O/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f seq %.1f ms multi %.1f ms' % (1e3*d['gpu_seconds'], 1e3*d['multi_seconds']), d['safeguard'])"; done
done
echo "== pytest"; timeout 1800 python -m pytest tests/test_gpu_fit.py tests/test_gpu_fit_c4.py -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?"; tail -3 $O/pytest_gpu.log
