#!/bin/bash
# Fit: the specialized nd<=8 sample pass (row source templates, straight-line
# rows, one-barrier epilogue).  Bit A/B vs the round's earlier build, source
# A/B (RPG_FIT_DM), step anatomy, timings, fit tests, one ncu capture.
set -u
TAG=${1:-r02s}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
echo "== bits vs old"; timeout 1200 python tools/fit_ab_bits.py build/old_librpgpu.so > $O/ab_bits.log 2>&1; tail -1 $O/ab_bits.log
for dm in 0 1; do
  echo "== dm=$dm"
  RPG_FIT_DM=$dm RPG_FIT_TRACE=1 timeout 900 python tools/bench_fit.py --reps 1 --noise 0.01 --no-warmup > $O/trace_dm$dm.log 2>&1
  grep -E 'wall|per step|tail' $O/trace_dm$dm.log | head -6
  RPG_FIT_DM=$dm timeout 900 python tools/bench_fit.py --reps 3 --noise 0.01 > $O/bench_noisy_dm$dm.log 2>&1
  RPG_FIT_DM=$dm timeout 900 python tools/bench_fit.py --reps 3 > $O/bench_clean_dm$dm.log 2>&1
  for f in bench_noisy_dm$dm bench_clean_dm$dm; do tail -1 $O/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f seq %.1f ms multi %.1f ms' % (1e3*d['gpu_seconds'], 1e3*d['multi_seconds']))"; done
done
echo "== pytest"; timeout 1800 python -m pytest tests/test_gpu_fit.py tests/test_gpu_fit_c4.py -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?"; tail -3 $O/pytest_gpu.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:min_step -s 30 -c 2 -o $O/minstep_full python tools/bench_fit.py --reps 1 --noise 0.01 --no-warmup > $O/ncu.log 2>&1; echo "ncu rc=$?"
