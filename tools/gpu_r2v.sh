#!/bin/bash
set -u
O=gpurun_out/${1:-r02v}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
echo "== determinism (same build twice)"; timeout 1200 python tools/fit_ab_bits.py paper_1906_00142_b200/librpgpu.so > $O/ab_self.log 2>&1; tail -1 $O/ab_self.log
echo "== minb3 vs default"; timeout 1200 python tools/fit_ab_bits.py build/minb3/librpgpu.so > $O/ab_minb3.log 2>&1; tail -1 $O/ab_minb3.log
echo "== racecheck"; timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 100 python tools/fit_small_probe.py 20000 > $O/racecheck.log 2>&1; echo rc=$?; grep -E "ERROR SUMMARY|RACECHECK SUMMARY" $O/racecheck.log
echo "== initcheck"; timeout 1500 compute-sanitizer --tool initcheck --print-limit 100000 python tools/fit_small_probe.py 20000 > $O/initcheck.log 2>&1; echo rc=$?; grep -E "ERROR SUMMARY" $O/initcheck.log; grep -E "^=========     at " $O/initcheck.log | sort | uniq -c | sort -rn | head -20
echo "== synccheck"; timeout 1500 compute-sanitizer --tool synccheck python tools/fit_small_probe.py 20000 > $O/synccheck.log 2>&1; echo rc=$?; grep -E "ERROR SUMMARY" $O/synccheck.log
echo "== pytest"; timeout 1800 python -m pytest tests/test_gpu_fit.py -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?"; tail -3 $O/pytest_gpu.log
