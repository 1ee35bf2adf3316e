#!/bin/bash
# Round-2 GPU pass b: full GPU suite, smoke, the per-call latency line, an
# extended FAST_CM variant sweep (tuples per thread x threads per CTA) and
# the fit's launch list (noisy C4).
#   gpurun -- 'bash tools/gpu_r2b.sh TAG'
set -u
TAG=${1:-r02b}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
echo "== smoke"; timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?"; tail -1 $O/smoke.log
echo "== pytest gpu (full)"
timeout 3000 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?"; tail -3 $O/pytest_gpu.log
echo "== cli per-call"; timeout 900 python tools/bench_cli.py > $O/bench_cli.log 2>&1; echo "rc=$?"; tail -1 $O/bench_cli.log
run() {  # name env...
  local name=$1; shift
  env "$@" timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu > $O/bench_$name.log 2>&1
  echo -n "$name: "; tail -1 $O/bench_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.3f G evals/s frac %.4f kernel_ms %.3f e2e %.3f G' % (d['value']/1e9, d['roofline']['frac'], d['roofline']['kernel_ms'], d['e2e']['value']/1e9))" 2>/dev/null || echo failed
}
run j2_512 RPG_CM_J=2
run j3_512 RPG_CM_J=3 RPG_CM_THREADS=512
run j4_512 RPG_CM_J=4 RPG_CM_THREADS=512
run j2_640 RPG_CM_J=2 RPG_CM_THREADS=640
run j2_768 RPG_CM_J=2 RPG_CM_THREADS=768
run j1_512x2 RPG_CM_J=1 RPG_CM_THREADS=512 RPG_JIT_MIN_BLOCKS=2
run j2_384 RPG_CM_J=2 RPG_CM_THREADS=384
echo "== fit bench noisy"; timeout 900 python tools/bench_fit.py --noise 0.01 > $O/fit_noisy.log 2>&1; echo "rc=$?"; tail -1 $O/fit_noisy.log | cut -c1-600
echo "== ncu fit launches"; timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/fit_launches.csv python tools/bench_fit.py --reps 1 --noise 0.01 > $O/ncu_fit_launch.log 2>&1; echo "rc=$?"
