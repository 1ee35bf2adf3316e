"""The data kit on the CPU: shortest-round-trip formatting and the
mt19937_64 noise stream pinned against the C++ standard library
(tests/golden/std_vectors.json), the sample CSV (test_datakit.cpp:239-319),
design points, and the sanity-report formatters."""
import json
import math
import os

import numpy as np
import pytest

from oracle import o5_data as O5
from paper_1906_00142_b200 import formats as F
from paper_1906_00142_b200 import samples as SM
from paper_1906_00142_b200 import sanity as SN

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "std_vectors.json")))


def test_format_double_matches_std_to_chars():
    for hexv, want in GOLD["to_chars"]:
        assert SM.format_double(float.fromhex(hexv)) == want, hexv


def test_mt19937_64_restatement_and_library_stream():
    g = O5.MT19937_64()
    for _ in range(9999):
        g()
    assert str(g()) == GOLD["mt19937_64_default_10000th"]  # the standard's check value
    for seed, want in GOLD["uniform_real"].items():
        want = [float.fromhex(h) for h in want]
        g = O5.MT19937_64(int(seed))
        assert [O5.uniform_real(g, -0.03, 0.03) for _ in range(64)] == want
        assert SM.uniform_stream(int(seed), 64, -0.03, 0.03).tolist() == want


GOOD = "D1,bx,by,bz,m1,m2\n64,32,1,1,1.5,2\n128,32,1,1,0.25,7\n"


def test_csv_parse_and_provenance():
    ok = SM.parse_samples(GOOD)
    assert len(ok) == 2 and ok.provenance.kind == "measured" and ok.metric_names == ["m1", "m2"]
    assert ok.values.tolist() == [[1.5, 2.0], [0.25, 7.0]]
    prov = SM.parse_samples("# provenance: synthetic seed=9 noise_rel=0.25\n# extra note\n" + GOOD)
    assert prov.provenance.kind == "synthetic" and prov.provenance.seed == 9
    assert prov.provenance.noise_rel == 0.25


@pytest.mark.parametrize("text,needle", [
    ("bx,by,bz,m\n32,1,1,2\n", "D1"),
    ("D1,bx,by,bz\n64,32,1,1\n", "metric"),
    ("D1,bx,bz,by,m\n64,32,1,1,2\n", "bx,by,bz"),
    ("D1,bx,by,bz,m,m\n64,32,1,1,2,3\n", "duplicate metric"),
    ("D1,bx,by,bz,m\n64,32,1,1,2\n128,32,1\n", "line 3"),
    ("D1,bx,by,bz,m\nx4,32,1,1,2\n", "bad integer D1"),
    ("D1,bx,by,bz,m\n64,32,1,1,abc\n", "bad value"),
    ("D1,bx,by,bz,m\n64,32,1,1,inf\n", "line 2"),
    ("D1,bx,by,bz,m\n64,0,1,1,2\n", "positive"),
    ("D1,bx,by,bz,m\n64,32,1,1,2\n64,32,1,1,3\n", "line 3"),
    ("D1,bx,by,bz,m\n64,32,1,1,2\n# late comment\n", "before the header"),
    ("# provenance: alien x\nD1,bx,by,bz,m\n", "provenance"),
    ("", "no header"),
])
def test_csv_errors_name_the_line_and_cause(text, needle):
    with pytest.raises(SM.CsvError) as e:
        SM.parse_samples(text)
    assert needle in str(e.value)


def test_csv_round_trip_is_a_fixed_point(tmp_path):
    rng = np.random.default_rng(3)
    n = 200
    s = SM.SampleSet(["coal_mem_insts_per_thread", "comp_insts_per_thread"],
                     rng.integers(1, 10 ** 6, (n, 2)), rng.integers(1, 1025, (n, 3)),
                     rng.uniform(-1e6, 1e6, (n, 2)) * 10.0 ** rng.integers(-12, 12, (n, 2)),
                     SM.Provenance("synthetic", 99, 0.03))
    s.data[:, 0] = np.arange(n)  # distinct points
    text = SM.format_samples(s)
    back = SM.parse_samples(text)
    assert back.metric_names == s.metric_names and back.provenance == s.provenance
    assert np.array_equal(back.data, s.data) and np.array_equal(back.configs, s.configs)
    assert np.array_equal(back.values, s.values)
    assert SM.format_samples(back) == text
    p = tmp_path / "s.csv"
    SM.write_samples(s, str(p))
    assert SM.format_samples(SM.read_samples(str(p))) == text
    with pytest.raises(SM.CsvError):
        SM.format_samples(SM.SampleSet())
    with pytest.raises(SM.CsvError):
        SM.read_samples("/nonexistent/samples.csv")


def test_design_points_data_major():
    cfg = [(32, 1, 1), (64, 1, 1)]
    data, configs = SM.design_points([64, 128], cfg)
    assert data[:, 0].tolist() == [64, 64, 128, 128]
    assert [tuple(c) for c in configs] == cfg * 2
    data, _ = SM.design_points([1, 2, 3, 4], F.enumerate_configs())
    assert len(data) == 4 * 51
    with pytest.raises(ValueError):
        SM.design_points([], cfg)
    with pytest.raises(ValueError):
        SM.design_points([64], [])


def test_sanity_formatters():
    r = SN.SanityReport(["D1"], [
        SN.SanityRow([64], (32, 1, 1), 1234.5, (64, 1, 1), 1200.25, math.nan),
        SN.SanityRow([128], (64, 2, 1), 1e17, (64, 2, 1), 1e17, 1e17)],
        ["D=(256): no sampled configuration is feasible; skipped"])
    csv = SN.format_sanity_csv(r)
    assert csv.startswith("D1,ci_bx,ci_by,ci_bz,Ec_i,cr_bx,cr_by,cr_bz,Ec_r,collected_Ec\n")
    assert "64,32,1,1,1234.5,64,1,1,1200.25,nan\n" in csv and csv.count("\n") == 3
    text = SN.format_sanity_text(r)
    assert "collected Ec" in text and "x1" in text and text.endswith(
        "note: D=(256): no sampled configuration is feasible; skipped\n")
    lines = SN.format_sanity_jsonl(r).splitlines()
    assert json.loads(lines[0])["collected_Ec"] is None
    assert json.loads(lines[1])["predicted_best"] == [64, 2, 1]
