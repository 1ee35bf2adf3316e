#!/bin/bash
set -u
O=gpurun_out/${1:-r02w}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
echo "== determinism (same build twice)"; timeout 1200 python tools/fit_ab_bits.py paper_1906_00142_b200/librpgpu.so > $O/ab_self.log 2>&1; tail -1 $O/ab_self.log
echo "== pytest"; timeout 1800 python -m pytest tests/test_gpu_fit.py -q -m gpu -k sample_pass > $O/pytest_gpu.log 2>&1; echo "rc=$?"; grep -E "^E  " $O/pytest_gpu.log | head -30
echo "== initcheck first errors"; timeout 900 compute-sanitizer --tool initcheck --print-limit 30 python tools/fit_small_probe.py 5000 > /tmp/ic.log 2>&1; grep -B2 -A12 "Uninitialized" /tmp/ic.log | head -120 > $O/initcheck_head.txt; grep "ERROR SUMMARY" /tmp/ic.log
