"""Concurrent host callers (SURVEY.md 8b "Threading": the replacement must be
thread-safe for concurrent callers and its output independent of how the
work is split): several Python threads (ctypes releases the GIL during the
C-ABI calls) search through their own plans and through one shared plan at
the same time; every result equals the single-threaded one byte for byte."""
import os
import threading

import numpy as np
import pytest

from paper_1906_00142_b200 import formats as F
from paper_1906_00142_b200 import search as S

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _setup(kernel):
    spec = F.models_to_metric_spec(F.read_models(os.path.join(ROOT, "data", "polybench", f"{kernel}.models.json")))
    hw = F.load_profile(os.path.join(ROOT, "data", "b200.profile"))
    return spec, hw, F.integer_configs(1024, dims=2)


def _run_threads(fn, n):
    errs, outs = [], [None] * n

    def work(i):
        try:
            outs[i] = fn(i)
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    return outs


def test_concurrent_private_plans():
    kernels = ["2dconv", "gemm", "atax1", "gemm"]
    data = [np.arange(64 + 11 * i, 40000, 13, dtype=np.int64).reshape(-1, 1) for i in range(len(kernels))]
    want = []
    for k, d in zip(kernels, data):
        spec, hw, space = _setup(k)
        with S.Plan(spec, hw, space, S.SearchOptions()) as plan:
            want.append(plan.search_batch(d))

    def one(i):
        spec, hw, space = _setup(kernels[i])
        with S.Plan(spec, hw, space, S.SearchOptions()) as plan:
            return [plan.search_batch(data[i]) for _ in range(3)]

    for i, res in enumerate(_run_threads(one, len(kernels))):
        for r in res:
            assert np.array_equal(r.view(np.uint8), want[i].view(np.uint8))


def test_concurrent_shared_plan():
    spec, hw, space = _setup("gemm")
    with S.Plan(spec, hw, space, S.SearchOptions()) as plan:
        data = [np.arange(64 + i, 30000 + 997 * i, 7, dtype=np.int64).reshape(-1, 1) for i in range(6)]
        want = [plan.search_batch(d) for d in data]
        got = _run_threads(lambda i: plan.search_batch(data[i]), len(data))
    for g, w in zip(got, want):
        assert np.array_equal(g.view(np.uint8), w.view(np.uint8))
