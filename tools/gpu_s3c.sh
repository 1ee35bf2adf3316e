#!/bin/bash
# Session-3 sweep: L1 prefetch distance of the FAST_CM rows; J = 3.
set -u
O=gpurun_out/${1:-s3c}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
run() {  # name workload env...
  local name=$1 wl=$2; shift 2
  env "$@" timeout 600 python bench.py --workload $wl --steps 8 --warmup 3 --no-cpu > $O/bench_$name.log 2>&1
  echo -n "$name: "; tail -1 $O/bench_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.3f G evals/s' % (d['value']/1e9), 'frac %.4f' % d['roofline']['frac'], 'kernel_ms %.3f' % d['roofline']['kernel_ms'], 'e2e %.3f G' % (d['e2e']['value']/1e9))" 2>/dev/null || echo failed
}
run c2_pf0 c2 RPG_CM_PF=0
run c2_pf1 c2 RPG_CM_PF=1
run c2_pf2 c2 RPG_CM_PF=2
run c2_pf4 c2 RPG_CM_PF=4
run c2_pf8 c2 RPG_CM_PF=8
run c2_pf2_j3 c2 RPG_CM_PF=2 RPG_CM_J=3 RPG_JIT_MIN_BLOCKS=1
run c3_pf0 c3 RPG_CM_PF=0
run c3_pf2 c3 RPG_CM_PF=2
run c3_pf4 c3 RPG_CM_PF=4
run c6_pf2 c6 RPG_CM_PF=2
run c6_pf2_j3 c6 RPG_CM_PF=2 RPG_CM_J=3 RPG_JIT_MIN_BLOCKS=1
run c3_pf2_j3 c3 RPG_CM_PF=2 RPG_CM_J=3 RPG_JIT_MIN_BLOCKS=1
