#!/bin/bash
# Session-3: certified Ec dump — dump bench with/without the certificate, dump parity suites.
set -u
O=gpurun_out/${1:-s3g}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
timeout 900 python bench.py --workload dump --steps 5 --warmup 3 --no-cpu > $O/bench_dump.log 2>&1; tail -1 $O/bench_dump.log | cut -c1-200
RPG_CM_CERT=0 timeout 900 python bench.py --workload dump --steps 5 --warmup 3 --no-cpu > $O/bench_dump_nocert.log 2>&1; tail -1 $O/bench_dump_nocert.log | cut -c1-200
timeout 900 python bench.py --workload c2 --steps 8 --warmup 3 --no-cpu > $O/bench_c2.log 2>&1; tail -1 $O/bench_c2.log | cut -c1-200
timeout 900 python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu > $O/bench_c4.log 2>&1; tail -1 $O/bench_c4.log | cut -c1-200
echo "== suites"
timeout 2400 python -m pytest tests/test_gpu_fastcm.py tests/test_gpu_cert.py tests/test_gpu_c6.py -q > $O/pytest.log 2>&1; echo "rc=$?"; tail -2 $O/pytest.log
