#!/bin/bash
# One gpurun session: GPU tests, smoke, short benches (incl. a tuning sweep),
# the ncu launch list and one full ncu capture.  Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
echo "== pytest gpu" ; timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/pytest_gpu.log
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/smoke.log
for mb in 2 3 4; do
  echo "== bench fast minblocks=$mb"; RPG_JIT_MIN_BLOCKS=$mb timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_mb$mb.log 2>&1; echo "rc=$?"; tail -1 gpurun_out/bench_mb$mb.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['roofline']['frac'], d['roofline']['kernel_ms'])"
done
echo "== bench exact"; timeout 900 python bench.py --steps 5 --warmup 3 --arith exact --no-cpu > gpurun_out/bench_exact.log 2>&1; echo "rc=$?"; tail -1 gpurun_out/bench_exact.log | cut -c1-300
echo "== bench default"; timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "rc=$?"; tail -1 gpurun_out/bench.log
echo "== ncu launches"; timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch_bench.log 2>&1; echo "rc=$?"
echo "== ncu full"; timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rpg_jit_search -s 3 -c 1 -o gpurun_out/search_full python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_full.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/ncu_full.log
