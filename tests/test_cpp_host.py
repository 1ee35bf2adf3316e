"""The C++ drop-in API (include/ratprog_b200/ratprog.hpp) and its CLI."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TEST = os.path.join(ROOT, "tests", "cpp", "test_host")
CLI = os.path.join(ROOT, "paper_1906_00142_b200", "ratprog-b200")


def _built():
    if not (os.path.exists(TEST) and os.path.exists(CLI)):
        import __graft_entry__ as g
        g.build()


def test_cpp_host_logic():
    _built()
    r = subprocess.run([TEST, "cpu", ROOT], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr


def test_cli_usage_errors():
    _built()
    r = subprocess.run([CLI, "search", "--profile", os.path.join(ROOT, "data", "b200.profile")],
                       capture_output=True, text=True, timeout=60)
    assert r.returncode == 1 and "usage error" in r.stderr
    r = subprocess.run([CLI, "frobnicate"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 1


@pytest.mark.gpu
def test_cpp_host_gpu_parity():
    _built()
    r = subprocess.run([TEST, "gpu", ROOT], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_cli_search_and_sweep(tmp_path):
    _built()
    models = os.path.join(ROOT, "data", "polybench", "gemm.models.json")
    prof = os.path.join(ROOT, "data", "b200.profile")
    out = tmp_path / "s.csv"
    r = subprocess.run([CLI, "search", "--models", models, "--profile", prof, "--size", "1024",
                        "--format", "csv", "-o", str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert r.stderr.startswith("chosen ")
    lines = out.read_text().splitlines()
    assert lines[0] == "bx,by,bz,Ec,occupancy,case" and len(lines) > 10
    # jobs never changes the output (acceptance.cpp:464-482)
    out8 = tmp_path / "s8.csv"
    subprocess.run([CLI, "search", "--models", models, "--profile", prof, "--size", "1024",
                    "--format", "csv", "--jobs", "8", "-o", str(out8)], check=True, timeout=300)
    assert out8.read_text() == out.read_text()
    sw = tmp_path / "sweep.csv"
    r = subprocess.run([CLI, "sweep", "--models", models, "--profile", prof, "--from", "1000",
                        "--to", "1100", "-o", str(sw)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    rows = sw.read_text().splitlines()
    assert len(rows) == 102
    # the sweep's N=1024 winner is the single search's chosen config
    row = [x for x in rows if x.startswith("1024,")][0].split(",")
    chosen = lines[1].split(",")
    assert row[1:4] == chosen[0:3]


@pytest.mark.gpu
@pytest.mark.parametrize("regs", [0.0, 32.0])
def test_cli_bare_program_search_matches_c_lowering(tmp_path, regs):
    """`ratprog-b200 search --rp` (ratprog_cli.cpp:305-307): the reference's
    emitted program, serialized to the .rp text form, parsed by the C++
    header, lowered and evaluated on the GPU — ranking, values and ties as
    O4's restatement of the C lowering; occupancy from --regs-per-thread, tag
    "-" (pipeline.hpp:648-650)."""
    _built()
    import numpy as np  # noqa: F401
    from oracle import o4_program as O4
    from paper_1906_00142_b200 import formats as F
    from paper_1906_00142_b200 import program as P
    models = os.path.join(ROOT, "data", "polybench", "gemm.models.json")
    prof = os.path.join(ROOT, "data", "b200.profile")
    spec = F.models_to_metric_spec(F.read_models(models))
    hw = F.load_profile(prof)
    prog = O4.generate_rp(spec, hw)
    rp = tmp_path / "gemm.rp"
    rp.write_text(P.serialize(prog))
    out = tmp_path / "r.csv"
    r = subprocess.run([CLI, "search", "--rp", str(rp), "--profile", prof, "--size", "1536",
                        "--regs-per-thread", str(regs), "--format", "csv", "-o", str(out)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    space = F.enumerate_configs()
    vals, order, ties, wocc = O4.search(prog, [1536], hw, space, regs, 0.0)
    rows = out.read_text().splitlines()[1:]
    assert len(rows) == len(order)
    for row, i in zip(rows, order):
        bx, by, bz, ec, occ, tag = row.split(",")
        assert (int(bx), int(by), int(bz)) == tuple(space[i])
        assert float(ec) == vals[i]
        assert float(occ) == wocc[i] / hw.W_max
        assert tag == "-"
    assert f"ties={ties}" in r.stderr
    # a malformed program is a runtime error naming the file (exit 2)
    bad = tmp_path / "bad.rp"
    bad.write_text("inputs: D1\noutput: y\n0: frob y D1\n")
    r = subprocess.run([CLI, "search", "--rp", str(bad), "--profile", prof, "--size", "8"],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 2 and "bad.rp: line 3" in r.stderr
    r = subprocess.run([CLI, "search", "--rp", str(rp), "--models", models, "--profile", prof,
                        "--size", "8"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 1 and "exactly one of --models or --rp" in r.stderr
