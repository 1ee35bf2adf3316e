#!/bin/bash
# Per-launch instruction count / DRAM bytes / duration of every min_step
# launch in one sequential C4 fit run (why do later metrics' passes take 3x?).
set -u
TAG=${1:-r02n}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
timeout 1500 ncu --clock-control none -k regex:min_step --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,lts__t_bytes.sum,smsp__sass_inst_executed_op_global_ld.sum,sm__warps_active.avg.pct_of_peak_sustained_active --csv --log-file $O/minstep.csv python tools/bench_fit.py --reps 1 --noise 0.01 --no-warmup > $O/run.log 2>&1; echo "rc=$?"
