#!/bin/bash
# FAST_CM kernel variants: pass-1 body (legacy branchy cm2 vs branch-free
# cmj), tuples per thread J, threads per CTA.  C2 bench value + roofline per
# variant, then bit-exactness of the variants against O1's FAST_CM twin.
#   gpurun -- 'bash tools/gpu_cmj_sweep.sh TAG'
set -u
TAG=${1:-cmj}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
run() {  # name env...
  local name=$1; shift
  env "$@" timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu > $O/bench_$name.log 2>&1
  echo -n "$name: "; tail -1 $O/bench_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.3f G evals/s' % (d['value']/1e9), 'frac %.4f' % d['roofline']['frac'], 'kernel_ms %.3f' % d['roofline']['kernel_ms'], 'e2e %.3f G' % (d['e2e']['value']/1e9))" 2>/dev/null || echo failed
}
run legacy_j2_512 RPG_CM_SCAN=0 RPG_CM_J=2
run scan_j2_512 RPG_CM_J=2
run scan_j1_768 RPG_CM_J=1 RPG_CM_THREADS=768
run scan_j1_1024 RPG_CM_J=1 RPG_CM_THREADS=1024 RPG_JIT_MIN_BLOCKS=1
run scan_j3_384 RPG_CM_J=3 RPG_CM_THREADS=384
run scan_j4_256 RPG_CM_J=4 RPG_CM_THREADS=256
run scan_j2_256 RPG_CM_J=2 RPG_CM_THREADS=256
run scan_j2_256x2 RPG_CM_J=2 RPG_CM_THREADS=256 RPG_JIT_MIN_BLOCKS=2
run scan_j2_512_l16 RPG_CM_J=2 RPG_CM_TUPLES=16
run scan_j3_384_l16 RPG_CM_J=3 RPG_CM_THREADS=384 RPG_CM_TUPLES=16
for v in "1 768" "3 384" "4 256"; do
  set -- $v
  echo "== fastcm parity J=$1 threads=$2"
  RPG_CM_J=$1 RPG_CM_THREADS=$2 timeout 900 python -m pytest tests/test_gpu_fastcm.py -x -q -k "not bench_workload_full" > $O/pytest_j$1.log 2>&1; echo "rc=$?"; tail -1 $O/pytest_j$1.log
done
echo "== fastcm parity default"
timeout 1200 python -m pytest tests/test_gpu_fastcm.py tests/test_gpu_parity.py -x -q > $O/pytest_default.log 2>&1; echo "rc=$?"; tail -1 $O/pytest_default.log
