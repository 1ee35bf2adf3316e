#!/bin/bash
# Round-2 GPU pass c: the GPU tests after the group test, the C4 stage-by-
# stage parity test, the fit's phase/tail trace, an ncu capture of the
# minimizer step kernel, and the per-call latency phases.
#   gpurun -- 'bash tools/gpu_r2c.sh TAG'
set -u
TAG=${1:-r02c}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
echo "== pytest gpu (rest)"
timeout 2400 python -m pytest tests/test_gpu_group.py tests/test_gpu_fit_c4.py tests/test_gpu_o2_agreement.py tests/test_gpu_parity.py tests/test_gpu_program.py tests/test_gpu_reference_order.py tests/test_gpu_sanity.py tests/test_gpu_threads.py tests/test_cpp_host.py -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?"; tail -5 $O/pytest_gpu.log
echo "== fit trace"; RPG_FIT_TRACE=1 timeout 900 python tools/bench_fit.py --reps 1 --noise 0.01 > $O/fit_trace.log 2>&1; echo "rc=$?"; grep -c rpg_fit $O/fit_trace.log
echo "== ncu min_step"; timeout 900 ncu --set full --clock-control none --import-source on -k regex:min_step -s 40 -c 1 -o $O/min_step_full python tools/bench_fit.py --reps 1 --noise 0.01 --no-warmup > $O/ncu_min_step.log 2>&1; echo "rc=$?"
echo "== cli per-call"; timeout 900 python tools/bench_cli.py > $O/bench_cli.log 2>&1; echo "rc=$?"; tail -1 $O/bench_cli.log | cut -c1-2000
