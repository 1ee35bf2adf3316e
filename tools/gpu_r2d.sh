#!/bin/bash
# Round-2 GPU pass d: FAST_CM parity after the integer-compare pass-1
# change, the C2 bench + instruction mix, the C4 stage-by-stage test, and
# the CUDA context-creation cost of a bare process.
#   gpurun -- 'bash tools/gpu_r2d.sh TAG'
set -u
TAG=${1:-r02d}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
echo "== pytest fastcm/parity/c4"
timeout 2400 python -m pytest tests/test_gpu_fastcm.py tests/test_gpu_reference_order.py tests/test_gpu_parity.py tests/test_gpu_fit_c4.py -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?"; tail -5 $O/pytest_gpu.log
echo "== bench c2"; timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > $O/bench_c2.log 2>&1; echo "rc=$?"; tail -1 $O/bench_c2.log | cut -c1-300
echo "== ncu mix"
timeout 1200 ncu --clock-control none -k regex:rpg_jit_search -s 3 -c 1 --metrics \
gpu__time_duration.sum,smsp__inst_executed.sum,smsp__inst_executed_pipe_fp64.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__inst_executed_pipe_xu.sum,smsp__inst_executed_pipe_fma.sum,smsp__inst_executed_pipe_alu.sum,smsp__inst_executed_pipe_lsu.sum,smsp__inst_executed_op_branch.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__sass_thread_inst_executed_op_dsetp_pred_on.sum \
  --csv python bench.py --steps 1 --warmup 3 --no-cpu > $O/ncu_mix.csv 2>&1; echo "rc=$?"
echo "== context probe"
cat > /tmp/ctx.cu <<'CU'
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
int main() { auto t0 = std::chrono::steady_clock::now(); cudaFree(0); auto t1 = std::chrono::steady_clock::now();
  printf("{\"bare_context_ms\": %.3f}\n", std::chrono::duration<double, std::milli>(t1 - t0).count()); return 0; }
CU
nvcc -o /tmp/ctx /tmp/ctx.cu > /dev/null 2>&1 && for i in 1 2 3; do /tmp/ctx; done > $O/ctx.log 2>&1; cat $O/ctx.log
for i in 1 2 3; do ./tools/percall_probe data/polybench/gemm.models.json data/b200.profile generic; done > $O/percall.log 2>&1; cat $O/percall.log
