"""Host logic of the tree executor's Pauli frames (program.cu: Diag::shift / inverse, frame_through,
frame_compose / frame_inverse, LinFrame), checked against dense 2^5 x 2^5 matrices: for random sweeps
G = post . gates . pre (factored gates I - iX / I - iY, T / CZ diagonals) and random frames
F = phi . X^m, whenever frame_through moves F it holds that G F = F' G exactly; compose and inverse
are the operator product and inverse; the bit-plane LinFrame agrees with the Diag form.  DESIGN.md §5.
"""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_frames_dense(tmp_path):
    exe = tmp_path / "frames_test"
    src = os.path.join(ROOT, "tests", "native", "frames_test.cpp")
    prog = os.path.join(ROOT, "paper_1802_06952_b200", "csrc", "program.cu")
    subprocess.run(["g++", "-O1", "-std=c++17", "-I", os.path.join(ROOT, "paper_1802_06952_b200", "csrc"),
                    "-I", os.path.join(ROOT, "include"), "-x", "c++", src, "-x", "c++", prog, "-o", str(exe)],
                   check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "bad 0" in r.stdout
