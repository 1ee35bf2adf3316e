#!/bin/bash
# FAST_CM pass-1 variants with the per-warp SMEM row ring (search_body_cmr):
# ring slots, configurations per step U, tuples per thread J, threads.  C2
# bench value + roofline per variant, then FAST_CM parity for the ring body.
#   gpurun -- 'bash tools/gpu_ring_sweep.sh TAG'
set -u
TAG=${1:-ring}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
run() {  # name env...
  local name=$1; shift
  env "$@" timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu > $O/bench_$name.log 2>&1
  echo -n "$name: "; tail -1 $O/bench_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.3f G evals/s' % (d['value']/1e9), 'frac %.4f' % d['roofline']['frac'], 'kernel_ms %.3f' % d['roofline']['kernel_ms'], 'e2e %.3f G' % (d['e2e']['value']/1e9))" 2>/dev/null || echo failed
}
run base_j2 RPG_CM_J=2
run unchecked_j2 RPG_CM_J=2 RPG_CM_UNCHECKED=1
run unchecked_ring4_u1_j2 RPG_CM_RING=4 RPG_CM_U=1 RPG_CM_J=2 RPG_CM_UNCHECKED=1
run unchecked_j2_640 RPG_CM_J=2 RPG_CM_UNCHECKED=1 RPG_CM_THREADS=640
run unchecked_j3_512 RPG_CM_J=3 RPG_CM_UNCHECKED=1 RPG_JIT_MIN_BLOCKS=1
run ring4_u1_j2 RPG_CM_RING=4 RPG_CM_U=1 RPG_CM_J=2
run ring8_u1_j2 RPG_CM_RING=8 RPG_CM_U=1 RPG_CM_J=2
run ring2_u1_j2 RPG_CM_RING=2 RPG_CM_U=1 RPG_CM_J=2
run ring4_u2_j1 RPG_CM_RING=4 RPG_CM_U=2 RPG_CM_J=1
run ring4_u2_j1_768 RPG_CM_RING=4 RPG_CM_U=2 RPG_CM_J=1 RPG_CM_THREADS=768
run ring4_u1_j1_1024 RPG_CM_RING=4 RPG_CM_U=1 RPG_CM_J=1 RPG_CM_THREADS=1024 RPG_JIT_MIN_BLOCKS=1
run ring8_u2_j2 RPG_CM_RING=8 RPG_CM_U=2 RPG_CM_J=2
run ring8_u4_j1 RPG_CM_RING=8 RPG_CM_U=4 RPG_CM_J=1
run ring4_u1_j3_384 RPG_CM_RING=4 RPG_CM_U=1 RPG_CM_J=3 RPG_CM_THREADS=384
run base_j2_again RPG_CM_J=2
echo "== fastcm parity ring4_u1_j2"
RPG_CM_RING=4 RPG_CM_U=1 RPG_CM_J=2 timeout 900 python -m pytest tests/test_gpu_fastcm.py -x -q > $O/pytest_ring.log 2>&1; echo "rc=$?"; tail -1 $O/pytest_ring.log
echo "== fastcm parity ring4_u2_j1"
RPG_CM_RING=4 RPG_CM_U=2 RPG_CM_J=1 timeout 900 python -m pytest tests/test_gpu_fastcm.py -x -q -k "not bench_workload_full" > $O/pytest_ring_u2.log 2>&1; echo "rc=$?"; tail -1 $O/pytest_ring_u2.log
