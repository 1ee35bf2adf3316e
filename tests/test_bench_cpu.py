"""bench.py host logic on CPU: the workloads' data-tuple partitions (strong
C2/C3/C5 — every tuple exactly once, contiguous, equal blocks but the last) and the reference arm's JSON line (O1 on the host, tiny sample)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_c2_is_configs1():
    w = bench.Workload("c2")
    assert w.scaling == "strong" and len(w.space) == 7262 and w.kernels == ("2dconv", "gemm", "atax1")
    t = w.tuples(0, 1)
    assert len(t) == 65473 and t[0, 0] == 64 and t[-1, 0] == 65536 and np.all(np.diff(t[:, 0]) == 1)


@pytest.mark.parametrize("name,count", [("c2", 65473), ("c3", 65473), ("c5", 182 * 182), ("c6", 65473)])
def test_strong_partitions_cover_every_tuple_once(name, count):
    w = bench.Workload(name)
    assert w.scaling == "strong"
    allt = w.all_tuples()
    assert len(allt) == count
    for world in (1, 2, 3, 8):
        parts = [w.tuples(r, world) for r in range(world)]
        assert np.array_equal(np.concatenate(parts), allt)
        per = -(-count // world)
        assert all(len(p) == per for p in parts[:-1]) and 0 < len(parts[-1]) <= per


def test_c3_has_the_27_suite_kernels():
    w = bench.Workload("c3")
    assert len(w.kernels) == 27 and len(set(w.kernels)) == 27
    assert all(len(w.specs[k].variables) == 3 for k in w.kernels)


def test_c5_space_and_model():
    w = bench.Workload("c5")
    assert len(w.space) == 30343
    assert w.specs["stencil3d_nm"].variables == ["D1", "D2", "bx", "by", "bz"]
    assert bench.official_flops(w.specs["stencil3d_nm"]) == 390


def test_official_flops_c2():
    w = bench.Workload("c2")
    assert [bench.official_flops(w.specs[k]) for k in w.kernels] == [170, 170, 170]


def test_reference_arm_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "1", "--cpu-seconds", "0.5"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["unit"] == "evals/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_c4_data_shapes_and_reference_arm():
    X, ys, var = bench.c4_data(1000)
    assert X.shape == (1000, 3) and var == ["D1", "bx", "by"] and len(ys) == 5
    assert all(np.isfinite(y).all() and y.shape == (1000,) for y in ys.values())
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "c4",
                        "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["unit"] == "samples/s" and d["value"] > 0


def test_default_arith_per_workload():
    assert bench.default_arith("c2", "specialized") == "fastcm"
    assert bench.default_arith("c3", "specialized") == "fastcm"
    assert bench.default_arith("c5", "specialized") == "fast"
    assert bench.default_arith("dump", "specialized") == "fastcm"
    assert bench.default_arith("c2", "generic") == "fast"


def test_c6_is_the_non_degenerate_landscape():
    w = bench.Workload("c6")
    assert w.kernels == ("c6_stencil", "c6_kloop", "c6_reduce") and len(w.space) == 7262
    assert bench.default_arith("c6", "specialized") == "fastcm"
    for spec in w.specs.values():
        assert spec.constants["regs_per_thread"] == 80.0
