#!/bin/bash
# Round-2 GPU pass e: C6 (non-degenerate landscape) parity + bench + ncu
# (instruction mix and a --set full capture), the multi-metric fit, the C4
# stage test, the group / cpp tests.
#   gpurun -- 'bash tools/gpu_r2e.sh TAG'
set -u
TAG=${1:-r02e}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
echo "== pytest"
timeout 3000 python -m pytest tests/test_gpu_c6.py tests/test_gpu_fit.py tests/test_gpu_fit_c4.py tests/test_gpu_group.py tests/test_cpp_host.py -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?"; tail -5 $O/pytest_gpu.log
echo "== bench c6"; timeout 900 python bench.py --workload c6 --steps 10 --warmup 3 --no-cpu > $O/bench_c6.log 2>&1; echo "rc=$?"; tail -1 $O/bench_c6.log | cut -c1-400
echo "== bench c4"; timeout 900 python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu > $O/bench_c4.log 2>&1; echo "rc=$?"; tail -1 $O/bench_c4.log | cut -c1-800
echo "== fit bench"; timeout 900 python tools/bench_fit.py --noise 0.01 > $O/fit_noisy.log 2>&1; echo "rc=$?"; tail -1 $O/fit_noisy.log | cut -c1-900
echo "== fit compare clean"; timeout 900 python tools/fit_c4_compare.py --noise 0 > $O/fit_c4_clean.log 2>&1; echo "rc=$?"; grep -v '^{' $O/fit_c4_clean.log | cut -c1-400
echo "== ncu mix c6"
timeout 1200 ncu --clock-control none -k regex:rpg_jit_search -s 3 -c 1 --metrics \
gpu__time_duration.sum,smsp__inst_executed.sum,smsp__inst_executed_pipe_fp64.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum \
  --csv python bench.py --workload c6 --steps 1 --warmup 3 --no-cpu > $O/ncu_mix_c6.csv 2>&1; echo "rc=$?"
echo "== ncu full c6"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rpg_jit_search -s 3 -c 1 -o $O/c6_search_full python bench.py --workload c6 --steps 1 --warmup 3 --no-cpu > $O/ncu_full_c6.log 2>&1; echo "rc=$?"
