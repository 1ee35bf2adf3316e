"""FAST_CM range certificate (cm_certify / cm_cert_kernel): pass 1 skips the
per-point fast-path range checks — and, where the MWP-CWP case is proven,
evaluates only that case — on (configuration, binade of N) cells the
certificate covers.  The certificate changes no result: the search with it
is byte-identical to the search without it (RPG_CM_CERT=0, a subprocess:
the switch is read once per process), on the bench landscapes (C2, C6: all
three case modes) and on the zoo's singular / guarded models, where it must
decline cells.  Coverage is reported by rpg_plan_cert_counts."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1906_00142_b200 import formats as F
from paper_1906_00142_b200 import search as S

from . import zoo

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _hw():
    return F.load_profile(os.path.join(ROOT, "data", "b200.profile"))


def _spec(path):
    return F.models_to_metric_spec(F.read_models(os.path.join(ROOT, "data", path)))


CASES = {
    "gemm": "polybench/gemm.models.json",
    "2dconv": "polybench/2dconv.models.json",
    "atax1": "polybench/atax1.models.json",
    "c6_stencil": "stressed/c6_stencil.models.json",
    "c6_kloop": "stressed/c6_kloop.models.json",
    "c6_reduce": "stressed/c6_reduce.models.json",
}

# N sample: every binade 2^0 .. 2^17 with dense runs (one 64-tuple group
# inside one binade) and sparse strides (groups spanning binades), plus N <= 0
# (no binade: never certified).
DATA = np.unique(np.concatenate([np.arange(1, 300), np.arange(300, 140000, 97), np.arange(65000, 65537),
                                 np.array([0, -5, 2**40, 2**40 + 12345])])).astype(np.int64).reshape(-1, 1)


def _winners_bytes(name, data):
    spec, hw, space = _spec(CASES[name]), _hw(), F.integer_configs(1024, dims=2)
    with S.Plan(spec, hw, space, S.SearchOptions(arith="fastcm")) as plan:
        return plan.search_batch(data).tobytes()


def _without_cert(names, data):
    code = ("import sys, json, numpy as np; sys.path.insert(0, %r); "
            "from tests.test_gpu_cert import _winners_bytes; "
            "d = np.load(sys.argv[1]); "
            "print(json.dumps({n: _winners_bytes(n, d).hex() for n in sys.argv[2:]}))" % ROOT)
    path = os.path.join("/tmp", f"rpg_cert_data_{os.getpid()}.npy")
    np.save(path, data)
    env = dict(os.environ, RPG_CM_CERT="0")
    out = subprocess.run([sys.executable, "-c", code, path, *names], env=env, capture_output=True,
                         text=True, check=True, cwd=ROOT).stdout
    os.unlink(path)
    return {k: bytes.fromhex(v) for k, v in json.loads(out.splitlines()[-1]).items()}


def test_cert_changes_no_result_bench_landscapes():
    names = list(CASES)
    ref = _without_cert(names, DATA)
    for n in names:
        assert _winners_bytes(n, DATA) == ref[n], n


ZOO_DATA = np.concatenate([np.arange(1, 200), np.arange(200, 70000, 331)]).astype(np.int64).reshape(-1, 1)


def _zoo_bytes(data):
    """FAST_CM winners of every one-data-parameter zoo case (singular and
    near-singular denominators, negative dips, the three hand-oracle cases,
    compute-only, flat ties, random profiles) over a broad N range."""
    out = {}
    for case in zoo.cases(small=True):
        if case.data.shape[1] != 1:
            continue
        opts = S.SearchOptions(arith="fastcm", rep_mode=case.rep_mode, regs_per_thread=case.regs_fallback,
                               shared_words_per_block=case.shared_fallback)
        try:
            plan = S.Plan(case.spec, case.hw, case.space, opts)
        except Exception:  # FAST_CM not applicable to this model
            continue
        with plan:
            out[case.name] = plan.search_batch(data).tobytes()
    return out


def test_cert_changes_no_result_zoo():
    got = _zoo_bytes(ZOO_DATA)
    code = ("import sys, json, numpy as np; sys.path.insert(0, %r); "
            "from tests.test_gpu_cert import _zoo_bytes; "
            "print(json.dumps({k: v.hex() for k, v in _zoo_bytes(np.load(sys.argv[1])).items()}))" % ROOT)
    path = os.path.join("/tmp", f"rpg_cert_zoo_{os.getpid()}.npy")
    np.save(path, ZOO_DATA)
    out = subprocess.run([sys.executable, "-c", code, path], env=dict(os.environ, RPG_CM_CERT="0"),
                         capture_output=True, text=True, check=True, cwd=ROOT).stdout
    os.unlink(path)
    ref = {k: bytes.fromhex(v) for k, v in json.loads(out.splitlines()[-1]).items()}
    assert len(got) >= 10 and set(ref) == set(got)
    for n in got:
        assert got[n] == ref[n], n


def test_cert_counts():
    hw, space = _hw(), F.integer_configs(1024, dims=2)
    with S.Plan(_spec(CASES["gemm"]), hw, space, S.SearchOptions(arith="fastcm")) as plan:
        c = plan.cert_counts()
    n = len(space)
    for k in range(6, 17):  # the C2 range: every cell free of checks, the case proven (cwp_bound)
        assert c["free"][k] == n
        assert c["cwp"][k] + c["mwp"][k] + c["both"][k] >= 0.99 * n
    assert all(c[m][62] == 0 and c[m][63] == 0 for m in c)
    for m in ("cwp", "mwp", "both"):  # case modes imply the free mode
        assert all(c[m][k] <= c["free"][k] for k in range(64))
    with S.Plan(_spec(CASES["gemm"]), hw, space, S.SearchOptions(arith="fast")) as plan:
        assert all(v == 0 for m in plan.cert_counts().values() for v in m)


@pytest.mark.parametrize("kernel", ["c6_stencil", "c6_kloop", "c6_reduce"])
def test_cert_dump_table_c6(kernel):
    """The Ec dump (rpg_evaluate, FAST_CM) takes the certificate's proven case
    as the point's tag (finish_point_cert): the whole table — Ec, tag,
    occupancy — bit-identical to O1's FAST_CM twin on the landscape with all
    three cases, infeasible configurations and exact ties."""
    from oracle import o1
    from paper_1906_00142_b200 import abi as A
    spec, hw, space = _spec(CASES[kernel]), _hw(), F.integer_configs(1024, dims=2)
    data = np.arange(64, 65537, 3637, dtype=np.int64).reshape(-1, 1)
    opts = S.SearchOptions(arith="fastcm")
    with S.Plan(spec, hw, space, opts) as plan:
        ec, tag, wocc = plan.evaluate(data)
    oec, otag, owocc = o1.evaluate_batch(A.PackedModel(spec, drop_zero_terms=False), A.profile_struct(hw),
                                         opts.struct(), A.config_array(space), data, os.cpu_count() or 1)
    assert np.array_equal(ec.view(np.int64), oec.view(np.int64))
    assert np.array_equal(tag, otag) and np.array_equal(wocc, owocc)
    assert len(np.unique(tag)) >= 3  # the three cases (plus infeasible points) are in the table
