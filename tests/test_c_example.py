"""The C ABI from plain C (examples/encode_c.c, no PyTorch): compiles and links against
libgpufv.so here; runs on the GPU (unit-norm FV, synchronous error status)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1604_03498_b200")


def _build(tmp_path):
    import __graft_entry__
    __graft_entry__.build()
    exe = str(tmp_path / "encode_c")
    subprocess.check_call(["nvcc", "-o", exe, os.path.join(ROOT, "examples", "encode_c.c"), "-I",
                           os.path.join(ROOT, "include"), "-L", PKG, "-lgpufv", "-Xlinker", f"-rpath={PKG}"])
    return exe


def test_c_example_compiles_and_links(tmp_path):
    exe = _build(tmp_path)
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_c_example_runs(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "||fv|| = 1.0000" in r.stdout and "FV_ERR_UNSUPPORTED" in r.stdout
