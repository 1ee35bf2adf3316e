#!/bin/bash
# Quick perf iteration on the GPU box: build, a parity subset, benches and one
# full ncu capture of the specialized search kernel.  Outputs in gpurun_out/.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
echo "== parity subset"; timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "specialized" > gpurun_out/pytest_sub.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/pytest_sub.log
for a in fast exact; do
  echo "== bench $a"; timeout 600 python bench.py --steps 5 --warmup 3 --arith $a --no-cpu > gpurun_out/bench_$a.log 2>&1; echo "rc=$?"
  tail -1 gpurun_out/bench_$a.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,3), 'G evals/s  frac', round(d['roofline']['frac'],4), 'kernel_ms', round(d['roofline']['kernel_ms'],3), 'e2e', round(d['e2e']['value']/1e9,3))"
done
echo "== ncu full"; timeout 900 ncu --set full --clock-control none --import-source on -k regex:rpg_jit_search -s 3 -c 1 -o gpurun_out/search_full python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_full.log 2>&1; echo "rc=$?"
