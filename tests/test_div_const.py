"""The device K1 series divides by the loop constant (j+1)(j+2) through its correctly
rounded reciprocal and one FMA correction (kernel_math.cuh).  This CPU test checks
that identity bit for bit against IEEE division on random significands and binade
edges for every divisor the series uses (tests/cpp/div_const_check.c)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))


def test_division_by_series_constants_is_correctly_rounded(tmp_path):
    exe = str(tmp_path / "div_const_check")
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-o", exe, os.path.join(HERE, "cpp", "div_const_check.c"),
                    "-lm"], check=True)
    out = subprocess.run([exe, "400000"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert '"mismatches": 0' in out.stdout
