#!/bin/bash
# Session-3 check: build, full GPU suite, smoke, default bench at HEAD.
set -u
O=gpurun_out/${1:-s3a}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
echo "== pytest gpu"; timeout 3000 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo "rc=$?"; tail -3 $O/pytest_gpu.log
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?"; tail -1 $O/smoke.log
echo "== bench default"; timeout 900 python bench.py > $O/bench.log 2>&1; echo "rc=$?"; tail -1 $O/bench.log | cut -c1-600
