#!/bin/bash
# Occupancy sweep of the specialized search kernel: RPG_JIT_MIN_BLOCKS x workload.
set -u
O=gpurun_out/${1:-mbsweep}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/fp64_peak tools/fp64_peak.cu > /dev/null 2>&1
for mb in ${MBS:-3 4}; do for w in ${WORKLOADS:-c2}; do
  RPG_JIT_MIN_BLOCKS=$mb timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu > $O/bench_${w}_mb$mb.log 2>&1
  tail -1 $O/bench_${w}_mb$mb.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mb=$mb', d['config']['id'], '%.3f G evals/s' % (d['value']/1e9), 'frac %.4f' % d['roofline']['frac'], 'kernel_ms %.3f' % d['roofline']['kernel_ms'])"
done; done
