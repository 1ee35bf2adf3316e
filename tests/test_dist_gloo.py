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
