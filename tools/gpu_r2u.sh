#!/bin/bash
set -u
O=gpurun_out/${1:-r02u}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
echo "== new dmma"; timeout 300 python tools/fit_probe_xy.py 2>&1 | cut -c1-400
echo "== new fma"; RPG_FIT_NO_DMMA=1 timeout 300 python tools/fit_probe_xy.py 2>&1 | cut -c1-400
echo "== old fma"; RPG_LIBRARY=build/old_librpgpu.so RPG_FIT_NO_DMMA=1 timeout 300 python tools/fit_probe_xy.py 2>&1 | cut -c1-400
echo "== old dmma"; RPG_LIBRARY=build/old_librpgpu.so timeout 300 python tools/fit_probe_xy.py 2>&1 | cut -c1-400
echo "== initcheck"; timeout 900 compute-sanitizer --tool initcheck --print-limit 20 python tools/fit_probe_xy.py > $O/initcheck.log 2>&1; echo rc=$?; grep -E "ERROR SUMMARY|Uninitialized|at 0x" $O/initcheck.log | head -20
