#!/bin/bash
set -u
O=gpurun_out/${1:-r02q}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
run() { echo "### $*"; RPG_FIT_TRACE=1 timeout 600 python tools/fit_order_probe.py "$@" 2>&1 | grep -E '==|wall|per step' ; }
run comp_insts_per_thread:4096 comp_insts_per_thread comp_insts_per_thread
run comp_insts_per_thread:4096 coal_mem_insts_per_thread
RPG_FIT_TRACE=1 timeout 900 python tools/bench_fit.py --reps 1 --noise 0.01 2>&1 | grep -E 'wall|per step' | head -4
RPG_FIT_TRACE=1 timeout 900 python tools/bench_fit.py --reps 1 --noise 0.01 --no-warmup 2>&1 | grep -E 'wall|per step' | head -4
