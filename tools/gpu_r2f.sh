#!/bin/bash
# Round-2 GPU pass f: fit tests + C4 parity after the warp-parallel minimizer
# tail, fit timing (with and without the precomputed denominator monomials),
# the tie-group rescan skip on C6 / C2 parity + bench.
set -u
TAG=${1:-r02f}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
echo "== pytest"
timeout 3000 python -m pytest tests/test_gpu_fit.py tests/test_gpu_fit_c4.py tests/test_gpu_c6.py tests/test_gpu_fastcm.py tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_dist.py -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?"; tail -5 $O/pytest_gpu.log
echo "== fit trace"; RPG_FIT_TRACE=1 timeout 900 python tools/bench_fit.py --reps 1 --noise 0.01 > $O/fit_trace.log 2>&1; echo "rc=$?"; grep -c rpg_fit $O/fit_trace.log
echo "== fit bench"; timeout 900 python tools/bench_fit.py --noise 0.01 > $O/fit_noisy.log 2>&1; echo "rc=$?"; tail -1 $O/fit_noisy.log | cut -c1-900
echo "== fit bench no-dm"; RPG_FIT_NO_DM=1 timeout 900 python tools/bench_fit.py --noise 0.01 > $O/fit_noisy_nodm.log 2>&1; echo "rc=$?"; tail -1 $O/fit_noisy_nodm.log | cut -c1-900
echo "== bench c6"; timeout 900 python bench.py --workload c6 --steps 10 --warmup 3 --no-cpu > $O/bench_c6.log 2>&1; echo "rc=$?"; tail -1 $O/bench_c6.log | cut -c1-300
echo "== bench c2"; timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > $O/bench_c2.log 2>&1; echo "rc=$?"; tail -1 $O/bench_c2.log | cut -c1-300
echo "== bench c4"; timeout 900 python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu > $O/bench_c4.log 2>&1; echo "rc=$?"; tail -1 $O/bench_c4.log | cut -c1-300
