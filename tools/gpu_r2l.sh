#!/bin/bash
# Fit A/B: denominator monomials recomputed from x by bit masks (default for
# 0/1 exponents) vs the precomputed m x 8 array (RPG_FIT_DM=1); fit tests.
set -u
TAG=${1:-r02l}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
run() {  # name env...
  local name=$1; shift
  env "$@" RPG_FIT_TRACE=1 timeout 900 python tools/bench_fit.py --reps 1 --noise 0.01 > $O/trace_$name.log 2>&1
  env "$@" timeout 900 python tools/bench_fit.py --reps 3 --noise 0.01 > $O/bench_$name.log 2>&1
  env "$@" timeout 900 python tools/bench_fit.py --reps 3 > $O/bench_clean_$name.log 2>&1
  echo "== $name"; grep -E 'wall' $O/trace_$name.log | head -4
  for f in bench bench_clean; do tail -1 $O/${f}_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f seq %.1f ms multi %.1f ms' % (1e3*d['gpu_seconds'], 1e3*d['multi_seconds']))"; done
}
run x01
run dm RPG_FIT_DM=1
echo "== bench c4"; timeout 900 python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu > $O/bench_c4.log 2>&1; tail -1 $O/bench_c4.log | cut -c1-300
echo "== pytest"; timeout 1800 python -m pytest tests/test_gpu_fit.py tests/test_gpu_fit_c4.py -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?"; tail -3 $O/pytest_gpu.log
