#!/bin/bash
# Fit: min_step launch bounds 2 (default) vs 3 CTAs/SM (build/minb3), bits,
# timings, fit tests (incl. the FMA-Gram path).
set -u
TAG=${1:-r02t}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
echo "== bits minb3 vs default"; timeout 1200 python tools/fit_ab_bits.py build/minb3/librpgpu.so > $O/ab_bits.log 2>&1; tail -1 $O/ab_bits.log
for v in default minb3; do
  if [ $v = default ]; then L=""; else L="RPG_LIBRARY=build/$v/librpgpu.so"; fi
  echo "== $v"
  env $L RPG_FIT_TRACE=1 timeout 900 python tools/bench_fit.py --reps 1 --noise 0.01 --no-warmup > $O/trace_$v.log 2>&1
  grep -E 'wall|per step|tail' $O/trace_$v.log | head -4
  env $L timeout 900 python tools/bench_fit.py --reps 3 --noise 0.01 > $O/bench_noisy_$v.log 2>&1
  env $L timeout 900 python tools/bench_fit.py --reps 3 > $O/bench_clean_$v.log 2>&1
  for f in bench_noisy_$v bench_clean_$v; do tail -1 $O/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f seq %.1f ms multi %.1f ms' % (1e3*d['gpu_seconds'], 1e3*d['multi_seconds']))"; done
done
echo "== pytest"; timeout 1800 python -m pytest tests/test_gpu_fit.py tests/test_gpu_fit_c4.py -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?"; tail -3 $O/pytest_gpu.log
