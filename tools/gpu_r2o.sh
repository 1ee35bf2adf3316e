#!/bin/bash
# Full ncu capture (source-level) of two min_step launches (a Newton and a line
# step) in the middle of the first C4 metric's minimizer.
set -u
TAG=${1:-r02o}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:min_step -s 30 -c 2 -o $O/minstep_full python tools/bench_fit.py --reps 1 --noise 0.01 --no-warmup > $O/run.log 2>&1; echo "rc=$?"
