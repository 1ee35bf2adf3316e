#!/bin/bash
set -u
O=gpurun_out/${1:-r02y}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
echo "== bits vs old"; timeout 1200 python tools/fit_ab_bits.py build/old_librpgpu.so > $O/ab_old.log 2>&1; tail -1 $O/ab_old.log
echo "== bits minb3"; timeout 1200 python tools/fit_ab_bits.py build/minb3/librpgpu.so > $O/ab_minb3.log 2>&1; tail -1 $O/ab_minb3.log
echo "== xy probe"; timeout 300 python tools/fit_probe_xy.py 2>&1 | tail -2 | cut -c1-300
echo "== pytest"; timeout 1800 python -m pytest tests/test_gpu_fit.py tests/test_gpu_fit_c4.py -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?"; tail -3 $O/pytest_gpu.log
