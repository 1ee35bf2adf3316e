#!/bin/bash
# Fit: TSQR leaf fold variants — bit A/B vs build/head_librpgpu.so, timings, tsqr ncu.
set -u
O=gpurun_out/${1:-r02ac}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
echo "== bits vs head"; timeout 1200 python tools/fit_ab_bits.py build/head_librpgpu.so > $O/ab_head.log 2>&1; tail -1 $O/ab_head.log
RPG_FIT_TRACE=1 timeout 900 python tools/bench_fit.py --reps 1 --noise 0.01 --no-warmup > $O/trace.log 2>&1
grep -E '\] tsqr|host setup' $O/trace.log | head -8 | tr '\n' ' '; echo
timeout 900 python tools/bench_fit.py --reps 3 --noise 0.01 > $O/bench_noisy.log 2>&1
timeout 900 python tools/bench_fit.py --reps 3 > $O/bench_clean.log 2>&1
for f in bench_noisy bench_clean; do tail -1 $O/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f seq %.1f ms multi %.1f ms' % (1e3*d['gpu_seconds'], 1e3*d['multi_seconds']), d['safeguard'])"; done
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active -k regex:tsqr_tiles -c 3 --csv python tools/bench_fit.py --reps 1 --noise 0.01 --no-warmup > $O/ncu_tsqr.csv 2>&1; grep -E "tsqr_tiles" $O/ncu_tsqr.csv | awk -F'","' '{print $(NF-2), $NF}' | head -9
