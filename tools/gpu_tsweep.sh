#!/bin/bash
# Sweep of the specialized kernels' CTA size / occupancy: "T:MB" pairs in $COMBOS.
set -u
O=gpurun_out/${1:-tsweep}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/fp64_peak tools/fp64_peak.cu > /dev/null 2>&1
if [ -n "${TEST_THREADS:-}" ]; then
  echo "== pytest gpu (RPG_JIT_THREADS=$TEST_THREADS)"
  RPG_JIT_THREADS=$TEST_THREADS timeout 1200 python -m pytest tests -x -q -m gpu > $O/pytest_t$TEST_THREADS.log 2>&1; echo "rc=$?"; tail -2 $O/pytest_t$TEST_THREADS.log
fi
for combo in ${COMBOS:-256:3}; do T=${combo%%:*}; MB=${combo##*:}
for w in ${WORKLOADS:-c2}; do
  RPG_JIT_THREADS=$T RPG_JIT_MIN_BLOCKS=$MB timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu > $O/bench_${w}_t${T}_mb$MB.log 2>&1
  tail -1 $O/bench_${w}_t${T}_mb$MB.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('T=$T mb=$MB', d['config']['id'], '%.3f G evals/s' % (d['value']/1e9), 'frac %.4f' % d['roofline']['frac'], 'kernel_ms %.3f' % d['roofline']['kernel_ms'])" 2>&1 | tail -1
done; done
if [ -n "${NCU_COMBO:-}" ]; then T=${NCU_COMBO%%:*}; MB=${NCU_COMBO##*:}
  RPG_JIT_THREADS=$T RPG_JIT_MIN_BLOCKS=$MB timeout 900 ncu --set full --clock-control none --import-source on -k regex:rpg_jit_search -s 3 -c 1 -o $O/search_t${T}_mb$MB python bench.py --steps 1 --warmup 3 --no-cpu > $O/ncu.log 2>&1; echo "ncu rc=$?"
fi
