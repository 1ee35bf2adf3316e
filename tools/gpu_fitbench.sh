#!/bin/bash
# C4 fit benchmark + fit kernel profiles.  gpurun -- 'bash tools/gpu_fitbench.sh TAG'
set -u
O=gpurun_out/${1:-fit}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
echo "== fit bench clean"; timeout 900 python tools/bench_fit.py --cpu > $O/fit_clean.log 2>&1; echo "rc=$?"; tail -1 $O/fit_clean.log
echo "== fit bench noisy"; timeout 900 python tools/bench_fit.py --noise 0.01 --cpu > $O/fit_noisy.log 2>&1; echo "rc=$?"; tail -1 $O/fit_noisy.log
echo "== ncu fit launches"; timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/fit_launches.csv python tools/bench_fit.py --reps 1 --noise 0.01 > $O/ncu_fit_launch.log 2>&1; echo "rc=$?"
echo "== ncu full tsqr"; timeout 900 ncu --set full --clock-control none --import-source on -k regex:tsqr_tiles -s 2 -c 1 -o $O/tsqr_full python tools/bench_fit.py --reps 1 > $O/ncu_tsqr.log 2>&1; echo "rc=$?"
