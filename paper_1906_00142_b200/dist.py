"""Multi-GPU sharding of a batched search along the data-parameter axis.

Every (data tuple, config) point is independent and the argmin is per tuple
(SURVEY.md 8e), so a sweep shards by contiguous blocks of data tuples — the
same static partition the reference uses for its worker threads
(``lo = n*j/jobs``, pipeline.hpp:602) — with no cross-rank tie merging.  The
only exchange is one all-gather of the fixed-size 48-byte winner records.

One process per GPU (``torch.distributed``; NCCL on GPUs, gloo for CPU
tests).  ``search_fn`` evaluates one shard and returns its winner records
(``abi.WINNER_DTYPE``); on a GPU it is ``Plan.search_batch`` (host buffers)
or a device-buffer variant.

The fit (``fit_all_metrics``, pipeline.hpp:145-184) shards by metric: every
metric column is an independent least-squares problem over the same samples,
so each rank fits a contiguous block of the name-sorted metrics and one
all-gather of the (small) fitted models assembles the same MetricModelSet on
every rank.  Row-sharding one metric's samples would need a
collective inside every positivity-minimizer iteration (its line search and
barrier sums run over all samples), for a fit that already takes ~20 ms per
10^6-sample metric on one B200; see DESIGN.md §7.
"""
from __future__ import annotations

from typing import Callable, Dict, List, Sequence, Tuple

import numpy as np

from . import abi as A


def shard_range(n: int, world: int, rank: int) -> Tuple[int, int]:
    """[lo, hi) of rank's contiguous block (pipeline.hpp:602 partition)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return n * rank // world, n * (rank + 1) // world


def sharded_search(data: np.ndarray, search_fn: Callable[[np.ndarray], np.ndarray],
                   group=None) -> np.ndarray:
    """Runs ``search_fn`` on this rank's block of ``data`` rows and
    all-gathers the winners of every rank, in tuple order.  Returns the full
    winner array on every rank (byte-identical to a single-process search)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = len(data)
    lo, hi = shard_range(n, world, rank)
    local = search_fn(np.ascontiguousarray(data[lo:hi]))
    if local.dtype != A.WINNER_DTYPE or len(local) != hi - lo:
        raise ValueError("search_fn must return one winner record per tuple")
    # Fixed-size records; pad every block to the largest shard.
    max_rows = max(shard_range(n, world, r)[1] - shard_range(n, world, r)[0] for r in range(world))
    rec = A.WINNER_DTYPE.itemsize
    backend = dist.get_backend(group)
    device = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    buf = torch.zeros(max_rows * rec, dtype=torch.uint8, device=device)
    if hi > lo:
        buf[: (hi - lo) * rec] = torch.from_numpy(local.view(np.uint8).copy()).to(device)
    out = torch.empty(world * max_rows * rec, dtype=torch.uint8, device=device)
    dist.all_gather_into_tensor(out, buf, group=group)
    allrec = out.cpu().numpy().reshape(world, max_rows * rec)
    parts = []
    for r in range(world):
        a, b = shard_range(n, world, r)
        parts.append(allrec[r, : (b - a) * rec])
    return np.concatenate(parts).view(A.WINNER_DTYPE)


def sharded_fit_all_metrics(X, metric_values: Dict[str, np.ndarray], variables: Sequence[str],
                            bounds: Dict[str, Tuple[List[int], List[int]]], constants: Dict[str, float],
                            rank_tol: float = None, device: int = 0, fit_fn=None, group=None):
    """pipe::fit_all_metrics (pipeline.hpp:145-184) over the ranks of
    ``group``: rank r fits the metrics in block shard_range(#metrics, world,
    r) of the name-sorted list (``fit_fn``: fit.fit_rational on the GPU by
    default; tests pass oracle O3), then the per-metric outcomes are
    all-gathered.  Every rank returns the MetricModelSet a single-process
    fit_all_metrics returns (same models, reports and failures; a total
    wipeout raises AllMetricsFailed on every rank)."""
    import torch.distributed as dist

    from . import fit as G

    if rank_tol is None:
        rank_tol = G.K_DEFAULT_RANK_TOL
    order = G.check_metric_inputs(X, metric_values, variables, bounds, constants)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = shard_range(len(order), world, rank)
    # Any exception of the local fit (a CUDA error, an RpgError, OOM) is
    # carried through the collective and re-raised on every rank, so no rank
    # is left blocked in all_gather_object.
    mine = None
    try:
        local = ("ok", G.fit_metrics(X, metric_values, variables, bounds, order[lo:hi], rank_tol,
                                     device, fit_fn))
    except Exception as e:  # noqa: BLE001 - re-raised below on every rank
        mine = e
        local = ("error", (rank, type(e).__name__, str(e)))
    gathered: List[tuple] = [None] * world
    dist.all_gather_object(gathered, local, group=group)
    for kind, payload in gathered:
        if kind == "error":
            r, name, msg = payload
            if r == rank:
                raise mine
            raise RuntimeError(f"sharded fit failed on rank {r}: {name}: {msg}")
    outcomes: Dict[str, object] = {}
    for _, part in gathered:
        outcomes.update(part)
    return G.assemble_model_set(variables, constants, outcomes)
