#!/bin/bash
set -u
O=gpurun_out/${1:-r02z}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
RPG_FIT_TRACE=1 timeout 900 python tools/bench_fit.py --reps 1 --noise 0.01 > $O/trace.log 2>&1
grep -vE "minimizer:|Newton tail" $O/trace.log | head -60
