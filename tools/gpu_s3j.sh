#!/bin/bash
# Session-3: defaults with the unproven-case body inline — benches and the FAST_CM suites.
set -u
O=gpurun_out/${1:-s3j}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
for w in c2 c3 c6; do timeout 900 python bench.py --workload $w --steps 8 --warmup 3 --no-cpu > $O/bench_$w.log 2>&1; tail -1 $O/bench_$w.log | cut -c1-120; done
timeout 2400 python -m pytest tests/test_gpu_fastcm.py tests/test_gpu_cert.py tests/test_gpu_c6.py tests/test_gpu_reference_order.py tests/test_gpu_configs.py tests/test_gpu_fuzz.py -q > $O/pytest.log 2>&1; echo "rc=$?"; tail -2 $O/pytest.log
