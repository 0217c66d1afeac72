"""Host-side checks of arithmetic shortcuts the CUDA kernels rely on (no GPU)."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_div25_sequence_is_correctly_rounded(tmp_path):
    """The box smoothing divides by 25 with q = RN(x RN(1/25)), r = fma(-q, 25, x),
    q1 = fma(r, RN(1/25), q).  tools/check_div25.c checks it against IEEE x / 25; here every
    61st non-negative finite float32 (35 M values, all binades incl. subnormals); run the tool
    with stride 1 for the exhaustive check."""
    exe = tmp_path / "div25"
    subprocess.run(["gcc", "-O2", "-mfma", "-ffp-contract=off", os.path.join(ROOT, "tools", "check_div25.c"), "-o",
                    str(exe), "-lm"], check=True)
    r = subprocess.run([str(exe), "61"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout
    assert "mismatches 0" in r.stdout
