#!/bin/bash
# Quick perf check: build, GPU tests (optional), bench C2, one ncu --set full capture.
#   gpurun -- 'bash tools/gpu_quick.sh TAG [tests]'
set -u
TAG=${1:-quick}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/fp64_peak tools/fp64_peak.cu > /dev/null 2>&1
if [ "${2:-}" = "tests" ]; then
  echo "== pytest gpu"; timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?"; tail -2 $O/pytest_gpu.log
fi
for w in ${WORKLOADS:-c2}; do
  echo "== bench $w"; timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu > $O/bench_$w.log 2>&1; echo "rc=$?"
  tail -1 $O/bench_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['id'], '%.3f G evals/s' % (d['value']/1e9), 'frac %.4f' % d['roofline']['frac'], 'kernel_ms %.3f' % d['roofline']['kernel_ms'], 'e2e %.3f G' % (d['e2e']['value']/1e9))"
done
if [ "${NCU:-1}" = "1" ]; then
  echo "== ncu full"; timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rpg_jit_search -s 3 -c 1 -o $O/search_full python bench.py --steps 1 --warmup 3 --no-cpu > $O/ncu_full.log 2>&1; echo "rc=$?"
fi
