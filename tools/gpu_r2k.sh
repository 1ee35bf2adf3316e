#!/bin/bash
# Fit A/B: FP64 tensor-core Gram (default) vs FMA Gram (RPG_FIT_NO_DMMA=1), and
# sample-pass CTAs per SM; per-step wall times from the minimizer trace.
set -u
TAG=${1:-r02k}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
run() {  # name env...
  local name=$1; shift
  env "$@" RPG_FIT_TRACE=1 timeout 900 python tools/bench_fit.py --reps 1 --noise 0.01 > $O/trace_$name.log 2>&1
  env "$@" timeout 900 python tools/bench_fit.py --reps 3 --noise 0.01 > $O/bench_$name.log 2>&1
  echo "== $name"; grep -E 'wall' $O/trace_$name.log | head -8; tail -1 $O/bench_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('seq %.1f ms multi %.1f ms' % (1e3*d['gpu_seconds'], 1e3*d['multi_seconds']))"
}
run dmma3
run dmma2 RPG_FIT_PASS_CTAS=2
run fma2 RPG_FIT_NO_DMMA=1 RPG_FIT_PASS_CTAS=2
echo "== pytest"; timeout 1200 python -m pytest tests/test_gpu_fit.py tests/test_gpu_fit_c4.py -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?"; tail -2 $O/pytest_gpu.log
