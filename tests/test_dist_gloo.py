"""Multi-process (world_size 2, gloo, CPU) coverage of the N-axis sharding:
the gathered winners of a 2-rank sharded search are byte-identical to a
single-process search (the reference's --jobs invariance,
acceptance.cpp:464-482, lifted to ranks).  Each rank evaluates its shard
with oracle O1 here (no GPU in this container); on GPUs the same
sharded_search drives Plan.search_batch over NCCL (bench.py)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1906_00142_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case():
    from . import zoo
    c = [x for x in zoo.cases() if x.name == "random3_1"][0]
    data = np.arange(64, 64 + 37, dtype=np.int64).reshape(-1, 1) * 37
    return c, data


def _o1_search(c, data):
    from oracle import o1
    from paper_1906_00142_b200 import abi as A
    pk = A.PackedModel(c.spec, drop_zero_terms=False)
    return o1.search_batch(pk, A.profile_struct(c.hw), A.options_struct(),
                           A.config_array(c.space), data, 2)


def _worker(rank, world, port, outdir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c, data = _case()
        got = D.sharded_search(data, lambda shard: _o1_search(c, shard))
        np.save(os.path.join(outdir, f"rank{rank}.npy"), got.view(np.uint8))
    finally:
        dist.destroy_process_group()


def test_shard_range_partition():
    for n in (0, 1, 7, 65473):
        for world in (1, 2, 3, 8):
            spans = [D.shard_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


def test_two_rank_gloo_sharded_search_matches_single_process(tmp_path):
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    c, data = _case()
    want = _o1_search(c, data).view(np.uint8)
    for r in range(2):
        got = np.load(tmp_path / f"rank{r}.npy")
        assert np.array_equal(got, want)


# --- metric-sharded fit (pipeline.hpp:145-184 over ranks) -------------------

SENTINEL = -1234.5  # y[0] == SENTINEL makes the test fit_fn fail that metric


def _fit_case():
    from paper_1906_00142_b200 import formats as F

    from .test_oracle_fit import stencil_samples
    from oracle import o3_fit as O3
    spec, pts = stencil_samples([64, 128, 256])
    bounds = {F.METRIC_COMP: ([1, 1, 0], [0, 1, 0]), F.METRIC_UNCOAL: ([0, 1, 0], [0, 1, 0]),
              F.METRIC_COAL: ([0, 0, 0], [0, 0, 0]), F.METRIC_SYNCH: ([1, 0, 0], [0, 1, 0]),
              F.METRIC_TOTAL_BLOCKS: ([2, 0, 0], [0, 1, 1])}
    values = {name: O3.eval_ratfunc(spec.ground_truth[name], pts) for name in bounds}
    values["zz_failing"] = np.full(len(pts), SENTINEL)
    return spec, pts, values, bounds, {F.METRIC_REGS: 20.0, F.METRIC_SHARED: 0.0}


def _o3_fit(X, y, variables, nb, db, tol):
    from oracle import o3_fit as O3
    from paper_1906_00142_b200 import fit as G
    if y[0] == SENTINEL:
        raise G.DegenerateFit("test: forced failure")
    return O3.fit_rational(X, y, variables, nb, db, tol)


def _canon(x):
    """Plain, bit-exact form (floats as hex) of a model set's contents."""
    if isinstance(x, (float, np.floating)):
        return float(x).hex()
    if isinstance(x, (bool, int, str, np.integer)) or x is None:
        return repr(x)
    if isinstance(x, dict):
        return "{" + ",".join(f"{k!r}:{_canon(v)}" for k, v in sorted(x.items())) + "}"
    if isinstance(x, (list, tuple, np.ndarray)):
        return "[" + ",".join(_canon(v) for v in x) + "]"
    return type(x).__name__ + _canon(vars(x))


def _model_set_bytes(ms):
    return _canon(ms).encode()


def _fit_worker(rank, world, port, outdir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec, pts, values, bounds, consts = _fit_case()
        ms = D.sharded_fit_all_metrics(pts, values, spec.variables, bounds, consts, fit_fn=_o3_fit)
        with open(os.path.join(outdir, f"fit{rank}.pkl"), "wb") as f:
            f.write(_model_set_bytes(ms))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_metric_sharded_fit_matches_single_process(tmp_path, world):
    from paper_1906_00142_b200 import fit as G
    port = _free_port()
    mp.start_processes(_fit_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    spec, pts, values, bounds, consts = _fit_case()
    order = G.check_metric_inputs(pts, values, spec.variables, bounds, consts)
    single = G.assemble_model_set(spec.variables, consts,
                                  G.fit_metrics(pts, values, spec.variables, bounds, order, fit_fn=_o3_fit))
    assert len(single.models) == 5 and list(single.failures) == ["zz_failing"]
    want = _model_set_bytes(single)
    for r in range(world):
        assert (tmp_path / f"fit{r}.pkl").read_bytes() == want


def test_fit_input_checks_run_before_any_fit():
    from paper_1906_00142_b200 import fit as G
    from paper_1906_00142_b200 import formats as F
    spec, pts, values, bounds, consts = _fit_case()
    with pytest.raises(F.PipelineError):
        G.check_metric_inputs(pts, values, spec.variables, bounds, {**consts, "zz_failing": 1.0})
    with pytest.raises(F.PipelineError):
        G.check_metric_inputs(pts, values, spec.variables, {**bounds, "zz_failing": ([1], [1])}, consts)
    with pytest.raises(ValueError):
        G.check_metric_inputs(pts[:0], values, spec.variables, bounds, consts)
    with pytest.raises(G.AllMetricsFailed):
        G.assemble_model_set(spec.variables, consts, {"a": "x", "b": "y"})


def _boom_fit(X, y, variables, nb, db, tol):
    raise MemoryError("out of memory (simulated)")


def _fit_error_worker(rank, world, port, outdir):
    import torch.distributed as dist
    from paper_1906_00142_b200 import dist as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec, pts, values, bounds, consts = _fit_case()
        fn = _boom_fit if rank == 1 else _o3_fit
        try:
            D.sharded_fit_all_metrics(pts, values, spec.variables, bounds, consts, fit_fn=fn)
            msg = "no error"
        except Exception as e:  # noqa: BLE001
            msg = f"{type(e).__name__}: {e}"
        with open(os.path.join(outdir, f"err{rank}.txt"), "w") as f:
            f.write(msg)
    finally:
        dist.destroy_process_group()


def test_sharded_fit_error_on_one_rank_raises_on_every_rank(tmp_path):
    """A non-numerical failure of one rank's local fit (here a simulated
    out-of-memory) must not leave the other ranks blocked in the gather:
    every rank raises (dist.py exception safety)."""
    port = _free_port()
    mp.start_processes(_fit_error_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    assert (tmp_path / "err1.txt").read_text() == "MemoryError: out of memory (simulated)"
    assert (tmp_path / "err0.txt").read_text().startswith(
        "RuntimeError: sharded fit failed on rank 1: MemoryError")


def test_fit_column_limit_checked_before_any_fit():
    from paper_1906_00142_b200 import fit as G
    spec, pts, values, bounds, consts = _fit_case()
    big = {k: ([2, 2, 3], [1, 1, 1]) for k in values}  # 3*3*4 + 8 = 44: fine
    G.check_metric_inputs(pts, values, spec.variables, big, consts)
    big = {k: ([3, 3, 3], [1, 1, 1]) for k in values}  # 64 + 8 = 72 > 64
    with pytest.raises(ValueError, match="exceed the GPU fit's limit of 64"):
        G.check_metric_inputs(pts, values, spec.variables, big, consts)
