#!/bin/bash
# Tuning sweep of the specialized kernel (ILP x launch-bound occupancy).
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
echo "== parity subset (ILP=2, mb=2)"; RPG_JIT_ILP=2 RPG_JIT_MIN_BLOCKS=2 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "specialized and search" > gpurun_out/pytest_ilp2.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/pytest_ilp2.log
for cfg in "1 3" "2 2" "2 3" "1 2"; do set -- $cfg
  echo "== ILP=$1 MB=$2"
  for a in fast exact; do
    RPG_JIT_ILP=$1 RPG_JIT_MIN_BLOCKS=$2 timeout 600 python bench.py --steps 5 --warmup 3 --arith $a --no-cpu > gpurun_out/sweep_$1_$2_$a.log 2>&1
    tail -1 gpurun_out/sweep_$1_$2_$a.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  $a', round(d['value']/1e9,3), 'G evals/s  kernel_ms', round(d['roofline']['kernel_ms'],3))"
  done
done
