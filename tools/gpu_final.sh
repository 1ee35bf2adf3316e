#!/bin/bash
# Round-end artifact run: build, full GPU tests, smoke, default bench (with the
# CPU baseline), reference arm, C3/C5/dump lines, ncu launch list + full
# capture of the search kernel, C4 fit timings.  gpurun -- 'bash tools/gpu_final.sh TAG'
set -u
TAG=${1:-final}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
echo "== pytest gpu"; timeout 1800 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?"; tail -2 $O/pytest_gpu.log
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?"; tail -1 $O/smoke.log
echo "== bench default"; timeout 900 python bench.py > $O/bench.log 2>&1; echo "rc=$?"; tail -1 $O/bench.log | cut -c1-400
echo "== bench reference"; timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.log 2>&1; echo "rc=$?"
for w in c3 c5 dump c4; do timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu > $O/bench_$w.log 2>&1; tail -1 $O/bench_$w.log | cut -c1-200; done
echo "== ncu launches"; timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > $O/ncu_launch_bench.log 2>&1; echo "rc=$?"
echo "== ncu full"; timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rpg_jit_search -s 3 -c 1 -o $O/search_full python bench.py --steps 1 --warmup 3 --no-cpu > $O/ncu_full.log 2>&1; echo "rc=$?"
echo "== fit"; python tools/bench_fit.py --reps 5 --cpu > $O/fit_clean.log 2>&1; python tools/bench_fit.py --reps 5 --noise 0.01 --cpu > $O/fit_noisy.log 2>&1; tail -1 $O/fit_noisy.log | cut -c1-300
