#!/bin/bash
# One gpurun session: build, GPU tests, smoke, default bench (with the CPU
# baseline), the reference arm, the ncu launch list and one full ncu capture
# of the search kernel.  Everything lands under gpurun_out/.
#   gpurun --timeout 3000 -- 'bash tools/gpu_round.sh TAG'
set -u
TAG=${1:-run}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/fp64_peak tools/fp64_peak.cu > /dev/null 2>&1
echo "== pytest gpu"; timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?"; tail -3 $O/pytest_gpu.log
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?"; tail -2 $O/smoke.log
echo "== bench default"; timeout 900 python bench.py > $O/bench.log 2>&1; echo "rc=$?"; tail -1 $O/bench.log
echo "== bench reference"; timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.log 2>&1; echo "rc=$?"; tail -1 $O/bench_ref.log | cut -c1-400
echo "== ncu launches"; timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > $O/ncu_launch_bench.log 2>&1; echo "rc=$?"
echo "== ncu full"; timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rpg_jit_search -s 3 -c 1 -o $O/search_full python bench.py --steps 1 --warmup 3 --no-cpu > $O/ncu_full.log 2>&1; echo "rc=$?"; tail -3 $O/ncu_full.log
