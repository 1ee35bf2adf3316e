"""The RcpDiv identity behind the specialized kernels' repetition quotient
(rpg_device.cuh rcp_div): with y = RN(1/d) the Markstein tail
q = fma(y, fma(-d, RN(a*y), a), RN(a*y)) is the correctly rounded a/d for
every repetition denominator d = b * num_SM a plan can build.  Checked
here in C on the host FPU (same IEEE binary64 + fused multiply-add)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))


def test_rcp_div_matches_ieee_division(tmp_path):
    exe = str(tmp_path / "rcp_div_check")
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-o", exe,
                    os.path.join(HERE, "c", "rcp_div_check.c"), "-lm"], check=True)
    r = subprocess.run([exe, "400"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout
    assert r.stdout.strip().startswith("0 mismatches"), r.stdout
