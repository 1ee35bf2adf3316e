#!/bin/bash
# Session-3 sweep: proven-case bodies inline (all) vs cwp only, CTA size.
set -u
O=gpurun_out/${1:-s3b}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
run() {  # name workload env...
  local name=$1 wl=$2; shift 2
  env "$@" timeout 600 python bench.py --workload $wl --steps 8 --warmup 3 --no-cpu > $O/bench_$name.log 2>&1
  echo -n "$name: "; tail -1 $O/bench_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.3f G evals/s' % (d['value']/1e9), 'frac %.4f' % d['roofline']['frac'], 'kernel_ms %.3f' % d['roofline']['kernel_ms'], 'e2e %.3f G' % (d['e2e']['value']/1e9))" 2>/dev/null || echo failed
}
for wl in c2 c3 c6; do
  run ${wl}_inl_all_512 $wl RPG_CM_INLINE_ALL=1
  run ${wl}_cwp_only_512 $wl RPG_CM_INLINE_ALL=0
done
run c2_cwp_only_640 c2 RPG_CM_INLINE_ALL=0 RPG_CM_THREADS=640
run c2_inl_all_640 c2 RPG_CM_INLINE_ALL=1 RPG_CM_THREADS=640
run c2_cwp_only_j3 c2 RPG_CM_INLINE_ALL=0 RPG_CM_J=3 RPG_JIT_MIN_BLOCKS=1
