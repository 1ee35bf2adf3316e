#!/bin/bash
# Session-3: J = 3 full waves + J = 2 remainder split; benches, FAST_CM suites, instruction mix.
set -u
O=gpurun_out/${1:-s3f}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
for w in c2 c3 c6; do timeout 900 python bench.py --workload $w --steps 8 --warmup 3 --no-cpu > $O/bench_$w.log 2>&1; tail -1 $O/bench_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '%.3f G evals/s' % (d['value']/1e9), 'frac %.4f' % d['roofline']['frac'], 'kernel_ms %.3f' % d['roofline']['kernel_ms'], 'e2e %.3f G' % (d['e2e']['value']/1e9), 'launches', d['gpu_launches'])"; done
echo "== ncu mix"
timeout 1200 ncu --clock-control none -k regex:rpg_jit_search -s 6 -c 2 --metrics \
gpu__time_duration.sum,smsp__inst_executed.sum,smsp__inst_executed_pipe_fp64.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__inst_executed_pipe_xu.sum,smsp__inst_executed_pipe_fma.sum,smsp__inst_executed_pipe_alu.sum,smsp__inst_executed_pipe_lsu.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size \
  --csv python bench.py --steps 1 --warmup 3 --no-cpu > $O/ncu_mix.csv 2>&1; echo "rc=$?"
echo "== FAST_CM suites"
timeout 2400 python -m pytest tests/test_gpu_fastcm.py tests/test_gpu_cert.py tests/test_gpu_c6.py tests/test_gpu_reference_order.py tests/test_gpu_configs.py -x -q > $O/pytest_cm.log 2>&1; echo "rc=$?"; tail -2 $O/pytest_cm.log
