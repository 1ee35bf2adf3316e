#!/bin/bash
# Fit minimizer step anatomy: sample-pass span and inter-step gap per step
# (%globaltimer), x-mask monomials vs the precomputed array.
set -u
TAG=${1:-r02m}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
for mode in 0 1; do
  RPG_FIT_DM=$mode RPG_FIT_TRACE=1 timeout 900 python tools/bench_fit.py --reps 1 --noise 0.01 > $O/trace_dm$mode.log 2>&1
  echo "== dm=$mode"; grep -E 'wall|per step|tail' $O/trace_dm$mode.log | head -12
done
RPG_FIT_PASS_CTAS=1 RPG_FIT_TRACE=1 timeout 900 python tools/bench_fit.py --reps 1 --noise 0.01 > $O/trace_ctas1.log 2>&1
echo "== ctas=1"; grep -E 'wall|per step' $O/trace_ctas1.log | head -6
RPG_FIT_PASS_CTAS=4 RPG_FIT_TRACE=1 timeout 900 python tools/bench_fit.py --reps 1 --noise 0.01 > $O/trace_ctas4.log 2>&1
echo "== ctas=4"; grep -E 'wall|per step' $O/trace_ctas4.log | head -6
