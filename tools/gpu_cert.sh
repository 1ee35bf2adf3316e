#!/bin/bash
# FAST_CM range certificate: C2/C6 bench with and without it, then the
# FAST_CM parity suites (byte-identity vs O1's twin) with it on.
#   gpurun -- 'bash tools/gpu_cert.sh TAG'
set -u
TAG=${1:-cert}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
run() {  # name workload env...
  local name=$1 wl=$2; shift 2
  env "$@" timeout 600 python bench.py --workload $wl --steps 8 --warmup 3 --no-cpu > $O/bench_$name.log 2>&1
  echo -n "$name: "; tail -1 $O/bench_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.3f G evals/s' % (d['value']/1e9), 'frac %.4f' % d['roofline']['frac'], 'kernel_ms %.3f' % d['roofline']['kernel_ms'], 'e2e %.3f G' % (d['e2e']['value']/1e9))" 2>/dev/null || echo failed
}
timeout 600 python tools/cert_report.py c2 c3 c6 > $O/cert_report.log 2>&1; echo "cert_report rc=$?"; grep "mean coverage" $O/cert_report.log
run c2_cert c2
run c2_nocert c2 RPG_CM_CERT=0
run c6_cert c6
run c6_nocert c6 RPG_CM_CERT=0
run c3_cert c3
if [ "${NCU:-0}" = "1" ]; then
  echo "== ncu full (C2 search kernel)"
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rpg_jit_search -s 3 -c 1 -o $O/search_full python bench.py --steps 1 --warmup 3 --no-cpu > $O/ncu_full.log 2>&1; echo "rc=$?"
fi
echo "== fastcm parity"
timeout 1800 python -m pytest tests/test_gpu_fastcm.py tests/test_gpu_c6.py tests/test_gpu_parity.py tests/test_gpu_reference_order.py -x -q > $O/pytest_cm.log 2>&1; echo "rc=$?"; tail -3 $O/pytest_cm.log
