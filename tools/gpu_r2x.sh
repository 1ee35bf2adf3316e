#!/bin/bash
set -u
O=gpurun_out/${1:-r02x}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
echo "== dmma"; timeout 300 python tools/fit_probe_xy.py 2>&1 | tail -2
echo "== fma"; RPG_FIT_NO_DMMA=1 timeout 300 python tools/fit_probe_xy.py 2>&1 | tail -2
