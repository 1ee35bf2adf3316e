#!/bin/bash
# Session-3 check after J = 3 + alternate: full GPU suite, smoke, benches, ncu.
set -u
O=gpurun_out/${1:-s3e}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
echo "== pytest gpu"; timeout 3000 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?"; tail -3 $O/pytest_gpu.log
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?"; tail -1 $O/smoke.log
echo "== bench default"; timeout 900 python bench.py > $O/bench.log 2>&1; echo "rc=$?"; tail -1 $O/bench.log | cut -c1-300
for w in c3 c6 c5 dump; do timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu > $O/bench_$w.log 2>&1; tail -1 $O/bench_$w.log | cut -c1-200; done
python tools/cert_report.py c2 c3 c6 > $O/cert_report.log 2>&1; grep "mean coverage" $O/cert_report.log
echo "== ncu launches"; timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > $O/ncu_launch_bench.log 2>&1; echo "rc=$?"
echo "== ncu full"; timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rpg_jit_search -s 3 -c 1 -o $O/search_full python bench.py --steps 1 --warmup 3 --no-cpu > $O/ncu_full.log 2>&1; echo "rc=$?"
