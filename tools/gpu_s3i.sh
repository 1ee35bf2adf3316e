#!/bin/bash
# Session-3: unproven-case (kScanFree) body inline vs out of line.
set -u
O=gpurun_out/${1:-s3i}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
for wl in c2 c3 c6; do for fi in 0 1; do
  RPG_CM_FREE_INLINE=$fi timeout 600 python bench.py --workload $wl --steps 8 --warmup 3 --no-cpu > $O/bench_${wl}_$fi.log 2>&1
  echo -n "${wl} free_inline=$fi: "; tail -1 $O/bench_${wl}_$fi.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.3f G evals/s' % (d['value']/1e9), 'frac %.4f' % d['roofline']['frac'])" 2>/dev/null || echo failed
done; done
