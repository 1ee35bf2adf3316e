"""Multi-rank GPU coverage of the data-tuple sharding, on the
one B200 a gpurun box has: two ranks (gloo for the winner all-gather, both
on cuda:0) each search their contiguous block of tuples with the CUDA plan;
the gathered winners must be byte-identical to a single-rank search and to
oracle O1 (the reference's --jobs invariance, acceptance.cpp:464-482, lifted
to ranks).  Also runs bench.py's multi-rank path (C5 stress workload shape,
strong scaling, padding of uneven blocks) under torch.distributed.run."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1906_00142_b200 import dist as D

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case():
    from . import zoo
    c = [x for x in zoo.cases() if x.name == "five_vars_3d"][0]
    rng = np.random.default_rng(7)
    data = rng.integers(16, 2049, size=(37, 2)).astype(np.int64)
    return c, data


def _plan(c, arith):
    from paper_1906_00142_b200 import search as S
    return S.Plan(c.spec, c.hw, c.space, S.SearchOptions(arith=arith, rep_mode=c.rep_mode))


def _worker(rank, world, port, outdir, arith):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c, data = _case()
        with _plan(c, arith) as plan:
            got = D.sharded_search(data, plan.search_batch)
        np.save(os.path.join(outdir, f"rank{rank}.npy"), got.view(np.uint8))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_two_rank_sharded_gpu_search_is_rank_invariant(tmp_path, arith):
    from oracle import o1
    from paper_1906_00142_b200 import abi as A
    from paper_1906_00142_b200 import search as S
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, str(tmp_path), arith), nprocs=2, join=True,
                       start_method="spawn")
    c, data = _case()
    with _plan(c, arith) as plan:
        single = plan.search_batch(data).view(np.uint8)
    opts = S.SearchOptions(arith=arith, rep_mode=c.rep_mode).struct()
    want = o1.search_batch(A.PackedModel(c.spec, drop_zero_terms=False), A.profile_struct(c.hw), opts,
                           A.config_array(c.space), data, 4)
    assert np.array_equal(single, want.view(np.uint8))
    for r in range(2):
        assert np.array_equal(np.load(tmp_path / f"rank{r}.npy"), single)


def test_bench_two_rank_strong_scaling_line():
    """bench.py under torch.distributed.run with 2 ranks on cuda:0 (gloo
    test mode): rank 0 prints one JSON line counting the whole job's
    evaluations; the device-API and host-API winners agree."""
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "1", "--warmup", "3", "--workload", "c5", "--no-cpu",
           "--dist-backend", "gloo", "--same-device"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["evals_job_step"] == 182 * 182 * 30343
    assert d["agreement_device_vs_host_api"] is True


def _fit_worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist

    from .test_dist_gloo import _fit_case, _model_set_bytes
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec, pts, values, bounds, consts = _fit_case()
        values.pop("zz_failing")
        ms = D.sharded_fit_all_metrics(pts, values, spec.variables, bounds, consts)
        with open(os.path.join(outdir, f"fit{rank}.txt"), "wb") as f:
            f.write(_model_set_bytes(ms))
    finally:
        dist.destroy_process_group()


def test_two_rank_metric_sharded_gpu_fit_equals_single_process(tmp_path):
    """dist.sharded_fit_all_metrics with the GPU fit (2 ranks on cuda:0):
    every rank assembles the MetricModelSet a single-process GPU
    fit_all_metrics returns, bit for bit (the K3 fit is deterministic)."""
    from paper_1906_00142_b200 import fit as G

    from .test_dist_gloo import _fit_case, _model_set_bytes
    port = _free_port()
    mp.start_processes(_fit_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    spec, pts, values, bounds, consts = _fit_case()
    values.pop("zz_failing")
    want = _model_set_bytes(G.fit_all_metrics(pts, values, spec.variables, bounds, consts))
    for r in range(2):
        assert (tmp_path / f"fit{r}.txt").read_bytes() == want


def test_bench_c4_two_rank_line():
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "1", "--warmup", "3", "--workload", "c4", "--no-cpu",
           "--dist-backend", "gloo", "--same-device"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["unit"] == "samples/s"
    assert len(d["config"]["fitted"]) + len(d["config"]["failed"]) == 5 and d["config"]["fitted"]


def _cm_worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist

    from paper_1906_00142_b200 import formats as F
    from paper_1906_00142_b200 import search as S
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec = F.models_to_metric_spec(F.read_models(os.path.join(ROOT, "data", "polybench", "gemm.models.json")))
        hw = F.load_profile(os.path.join(ROOT, "data", "b200.profile"))
        data = np.arange(64, 64 + 1001, dtype=np.int64).reshape(-1, 1) * 37
        with S.Plan(spec, hw, F.integer_configs(), S.SearchOptions(arith="fastcm")) as plan:
            got = D.sharded_search(data, plan.search_batch)
        np.save(os.path.join(outdir, f"rank{rank}.npy"), got.view(np.uint8))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_fastcm_search_is_rank_invariant(tmp_path):
    """The headline arithmetic (FAST_CM) over two ranks: byte-identical to
    one rank."""
    from paper_1906_00142_b200 import formats as F
    from paper_1906_00142_b200 import search as S
    port = _free_port()
    mp.start_processes(_cm_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    spec = F.models_to_metric_spec(F.read_models(os.path.join(ROOT, "data", "polybench", "gemm.models.json")))
    hw = F.load_profile(os.path.join(ROOT, "data", "b200.profile"))
    data = np.arange(64, 64 + 1001, dtype=np.int64).reshape(-1, 1) * 37
    with S.Plan(spec, hw, F.integer_configs(), S.SearchOptions(arith="fastcm")) as plan:
        single = plan.search_batch(data).view(np.uint8)
    for r in range(2):
        assert np.array_equal(np.load(tmp_path / f"rank{r}.npy"), single)


def test_bench_c2_two_rank_strong_scaling_line():
    """The headline workload (C2, FAST_CM) under torch.distributed.run with
    2 ranks on cuda:0 (gloo test mode): N = 64..65536 split over the ranks
    (strong scaling), whole-job evaluations counted once."""
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "1", "--warmup", "3", "--no-cpu",
           "--dist-backend", "gloo", "--same-device"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["config"]["arith"] == "fastcm"
    assert d["config"]["evals_job_step"] == 3 * 65473 * 7262
    assert d["config"]["tuples_rank0"] == [[64], [64 + 32736]]
    assert d["agreement_device_vs_host_api"] is True


@pytest.mark.skipif(__import__("torch").cuda.device_count() < 2, reason="needs 2 GPUs (NCCL)")
def test_bench_c2_two_rank_nccl():
    """The production multi-GPU path: one rank per GPU, NCCL all-gather of
    the winner records inside the timed region."""
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--no-cpu"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    assert d["n_gpus"] == 2 and d["agreement_device_vs_host_api"] is True
