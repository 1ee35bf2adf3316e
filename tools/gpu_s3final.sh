#!/bin/bash
# Session-3 round-end artifacts: build, full GPU suite, smoke, default bench
# (cpu_baseline), reference arm, C3/C5/C6/dump/C4 lines, ncu launch list +
# full capture of the search kernel, compute-sanitizer racecheck/synccheck.
#   gpurun -- 'bash tools/gpu_s3final.sh TAG'
set -u
O=gpurun_out/${1:-s3final}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
echo "== pytest gpu"; timeout 3000 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?"; tail -2 $O/pytest_gpu.log
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?"; tail -1 $O/smoke.log
echo "== bench default"; timeout 900 python bench.py > $O/bench.log 2>&1; echo "rc=$?"; tail -1 $O/bench.log | cut -c1-200
echo "== bench reference"; timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.log 2>&1; echo "rc=$?"; tail -1 $O/bench_ref.log | cut -c1-200
for w in c3 c5 c6 dump c4; do timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu > $O/bench_$w.log 2>&1; tail -1 $O/bench_$w.log | cut -c1-160; done
echo "== ncu launches"; timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > $O/ncu_launch_bench.log 2>&1; echo "rc=$?"
echo "== ncu full"; timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rpg_jit_search -s 6 -c 2 -o $O/search_full python bench.py --steps 1 --warmup 3 --no-cpu > $O/ncu_full.log 2>&1; echo "rc=$?"
for tool in racecheck synccheck; do
  echo "== sanitizer $tool"
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_search.py > $O/sanitize_$tool.log 2>&1; echo "rc=$?"; tail -3 $O/sanitize_$tool.log
done
