#!/bin/bash
# fast_cm sweep: CTA size x tuples per CTA (x resident CTAs) on a workload;
# optional parity run of tests/test_gpu_fastcm.py under given RPG_CM_TUPLES.
#   gpurun -- 'COMBOS="128:16:6 ..." bash tools/gpu_cmsweep.sh TAG'   (T:L:blocks per SM)
set -u
O=gpurun_out/${1:-cmsweep}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/fp64_peak tools/fp64_peak.cu > /dev/null 2>&1
for L in ${TEST_TUPLES:-}; do
  echo "== pytest fastcm (RPG_CM_TUPLES=$L)"
  RPG_CM_TUPLES=$L timeout 900 python -m pytest tests/test_gpu_fastcm.py -x -q > $O/pytest_l$L.log 2>&1; echo "rc=$?"; tail -1 $O/pytest_l$L.log
done
for combo in ${COMBOS:-64:32:12}; do
  IFS=: read T L MB <<< "$combo"
  for w in ${WORKLOADS:-c2}; do
    RPG_CM_THREADS=$T RPG_CM_TUPLES=$L RPG_JIT_MIN_BLOCKS=$MB timeout 600 python bench.py --workload $w --arith fastcm --steps 5 --warmup 3 --no-cpu > $O/bench_${w}_t${T}_l${L}_mb$MB.log 2>&1
    tail -1 $O/bench_${w}_t${T}_l${L}_mb$MB.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('T=$T L=$L mb=$MB', d['config']['id'], '%.3f G evals/s' % (d['value']/1e9), 'frac %.4f' % d['roofline']['frac'], 'e2e %.3f G' % (d['e2e']['value']/1e9))" 2>&1 | tail -1
  done
done
