#!/bin/bash
# gpurun session: bare-program GPU tests, the 2-rank bench path (gloo, same
# device), smoke.  Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
echo "== pytest program"; timeout 900 python -m pytest tests/test_gpu_program.py -q -m gpu > gpurun_out/pytest_prog.log 2>&1; echo "rc=$?"; tail -25 gpurun_out/pytest_prog.log
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/smoke.log
echo "== torchrun 2 ranks (gloo, same device)"; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --same-device --no-cpu > gpurun_out/bench_2rank.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/bench_2rank.log | cut -c1-600
echo "== reference arm 2 ranks"; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > gpurun_out/bench_ref2.log 2>&1; echo "rc=$?"; tail -1 gpurun_out/bench_ref2.log | cut -c1-400
