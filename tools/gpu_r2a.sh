#!/bin/bash
# Round-2 measurement run: build, targeted GPU tests, C2 bench, the search
# kernel's instruction mix (ncu, explicit metrics), compute-sanitizer
# racecheck/synccheck over the search kernels, and the C4 fit outcomes.
#   gpurun -- 'bash tools/gpu_r2a.sh TAG [tests|notests] [sanitize]'
set -u
TAG=${1:-r02a}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
if [ "${2:-tests}" = "tests" ]; then
  echo "== pytest gpu (${TESTS:-targeted})"
  timeout 2400 python -m pytest ${TESTS:-tests/test_gpu_reference_order.py tests/test_gpu_o2_agreement.py tests/test_gpu_fastcm.py tests/test_gpu_parity.py} -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?"; tail -3 $O/pytest_gpu.log
fi
echo "== bench c2"; timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > $O/bench_c2.log 2>&1; echo "rc=$?"; tail -1 $O/bench_c2.log | cut -c1-600
echo "== ncu mix"
timeout 1200 ncu --clock-control none -k regex:rpg_jit_search -s 3 -c 1 --metrics \
gpu__time_duration.sum,smsp__inst_executed.sum,smsp__inst_executed_pipe_fp64.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__inst_executed_pipe_xu.sum,smsp__inst_executed_pipe_fma.sum,smsp__inst_executed_pipe_alu.sum,smsp__inst_executed_pipe_lsu.sum,smsp__inst_executed_op_branch.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio \
  --csv python bench.py --steps 1 --warmup 3 --no-cpu > $O/ncu_mix.csv 2>&1; echo "rc=$?"
if [ "${3:-}" = "sanitize" ]; then
  for tool in racecheck synccheck; do
    echo "== sanitizer $tool"
    timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_search.py > $O/sanitize_$tool.log 2>&1; echo "rc=$?"; tail -3 $O/sanitize_$tool.log
  done
  echo "== sanitizer racecheck (one tuple per thread)"
  RPG_CM_PAIR=0 timeout 900 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_search.py > $O/sanitize_racecheck_cm1.log 2>&1; echo "rc=$?"; tail -2 $O/sanitize_racecheck_cm1.log
fi
if [ -f tools/fit_c4_compare.py ]; then
  echo "== fit c4 compare"; timeout 1800 python tools/fit_c4_compare.py --noise 0.01 > $O/fit_c4_noisy.log 2>&1; echo "rc=$?"; tail -8 $O/fit_c4_noisy.log
fi
