#!/bin/bash
# Round-end artifact run: build, full GPU tests, smoke, default bench (with the
# CPU baseline), reference arm, C3/C5/C6/dump/C4 lines, ncu launch list + full
# capture of the search kernel, instruction mix, fit timings, per-call and
# CSV numbers.  gpurun -- 'bash tools/gpu_final.sh TAG [notests]'
set -u
TAG=${1:-final}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
if [ "${2:-tests}" = "tests" ]; then
  echo "== pytest gpu"; timeout 3600 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?"; tail -2 $O/pytest_gpu.log
fi
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?"; tail -1 $O/smoke.log
echo "== bench default"; timeout 900 python bench.py > $O/bench.log 2>&1; echo "rc=$?"; tail -1 $O/bench.log | cut -c1-400
echo "== bench reference"; timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.log 2>&1; echo "rc=$?"
for w in c3 c5 c6 dump c4; do timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu > $O/bench_$w.log 2>&1; tail -1 $O/bench_$w.log | cut -c1-200; done
echo "== ncu launches"; timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > $O/ncu_launch_bench.log 2>&1; echo "rc=$?"
echo "== ncu full"; timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rpg_jit_search -s 3 -c 1 -o $O/search_full python bench.py --steps 1 --warmup 3 --no-cpu > $O/ncu_full.log 2>&1; echo "rc=$?"
echo "== ncu mix"
timeout 1200 ncu --clock-control none -k regex:rpg_jit_search -s 3 -c 1 --metrics \
gpu__time_duration.sum,smsp__inst_executed.sum,smsp__inst_executed_pipe_fp64.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__inst_executed_pipe_xu.sum,smsp__inst_executed_pipe_fma.sum,smsp__inst_executed_pipe_alu.sum,smsp__inst_executed_pipe_lsu.sum,sm__warps_active.avg.pct_of_peak_sustained_active \
  --csv python bench.py --steps 1 --warmup 3 --no-cpu > $O/ncu_mix.csv 2>&1; echo "rc=$?"
echo "== fit"; timeout 1200 python tools/bench_fit.py --reps 5 --cpu > $O/fit_clean.log 2>&1; timeout 1200 python tools/bench_fit.py --reps 5 --noise 0.01 --cpu > $O/fit_noisy.log 2>&1; tail -1 $O/fit_noisy.log | cut -c1-300
echo "== ncu fit launches"; timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/fit_launches.csv python tools/bench_fit.py --reps 1 --noise 0.01 > $O/ncu_fit_launch.log 2>&1; echo "rc=$?"
echo "== per-call"; timeout 900 python tools/bench_cli.py > $O/bench_cli.log 2>&1; echo "rc=$?"
echo "== csv"; timeout 600 python tools/bench_csv.py 1000000 > $O/bench_csv.log 2>&1; echo "rc=$?"; tail -1 $O/bench_csv.log
