"""The stencil kernels divide by their constant weights (STENCIL9 /20 in fp64, R12;
STENCIL7_3D /6 in fp32, R13) with a Markstein-corrected reciprocal product instead of
the IEEE division sequence.  Bit-parity with the oracle's plain `x / d` rests on the
identity RN(q0 + r*y) == RN(x/d); this checks it with the standalone C program
(strided fp32 sweep, 2e7 fp64 samples; the exhaustive fp32 run is committed in
profiles/r01/markstein_check.txt)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_markstein_quotient_equals_ieee_division(tmp_path):
    exe = str(tmp_path / "mc")
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-o", exe, os.path.join(ROOT, "tools", "markstein_check.c"),
                    "-lm"], check=True)
    r = subprocess.run([exe, "20000000", "61"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 mismatches" in r.stdout
