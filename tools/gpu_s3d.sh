#!/bin/bash
# Session-3 sweep: tuples per thread J (proven-case bodies inline, 512 threads, 1 CTA/SM).
set -u
O=gpurun_out/${1:-s3d}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
run() {  # name workload env...
  local name=$1 wl=$2; shift 2
  env "$@" timeout 600 python bench.py --workload $wl --steps 8 --warmup 3 --no-cpu > $O/bench_$name.log 2>&1
  echo -n "$name: "; tail -1 $O/bench_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.3f G evals/s' % (d['value']/1e9), 'frac %.4f' % d['roofline']['frac'], 'kernel_ms %.3f' % d['roofline']['kernel_ms'], 'e2e %.3f G' % (d['e2e']['value']/1e9))" 2>/dev/null || echo failed
}
for wl in c2 c3 c6; do
  run ${wl}_j2 $wl RPG_CM_J=2
  run ${wl}_j3 $wl RPG_CM_J=3 RPG_JIT_MIN_BLOCKS=1
  run ${wl}_j4 $wl RPG_CM_J=4 RPG_JIT_MIN_BLOCKS=1
done
run c2_j3_384 c2 RPG_CM_J=3 RPG_CM_THREADS=384 RPG_JIT_MIN_BLOCKS=1
run c2_j1_1024 c2 RPG_CM_J=1 RPG_CM_THREADS=1024 RPG_JIT_MIN_BLOCKS=1
