"""The C ABI from plain C (examples/encode_c.c, no PyTorch): compiles and links against
libgpufv.so here; runs on the GPU (unit-norm FV, synchronous error status)."""
import os
import subprocess
import sys

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


# compute-sanitizer runs are opt-in (GPUFV_RUN_SANITIZER=1): the GPU pool this repo is measured on has
# closed the tool (runs under it left GPUs needing a reset), and its wrapper refuses every run there.
# The clean reports of the earlier runs are recorded in DESIGN.md §14.
_SANITIZER_OPT_IN = os.environ.get("GPUFV_RUN_SANITIZER") == "1"


def _run_sanitizer(cmd, timeout):
    if not _SANITIZER_OPT_IN:
        pytest.skip("compute-sanitizer runs are opt-in (GPUFV_RUN_SANITIZER=1)")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
    out = r.stdout + r.stderr
    if "closed on this pool" in out:
        pytest.skip("compute-sanitizer is closed on this GPU pool")
    return r, out


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


@pytest.mark.gpu
@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
@pytest.mark.parametrize("shape", [("256", "64", "5000"), ("512", "128", "3000"), ("16", "36", "1000")])
def test_compute_sanitizer_clean(tmp_path, tool, shape):
    """compute-sanitizer memcheck / racecheck / synccheck / initcheck over the whole encode
    (prep, schedule, persistent tcgen05 stats kernel, finalize) for the narrow, wide and masked-D
    families report no error."""
    exe = _build(tmp_path)
    r, out = _run_sanitizer(["compute-sanitizer", "--tool", tool, exe, *shape], timeout=900)
    print(out[-2000:])
    assert r.returncode == 0, out[-2000:]
    assert ("ERROR SUMMARY: 0 errors" in out) or ("0 hazards displayed (0 errors, 0 warnings)" in out)


@pytest.mark.gpu
@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer_all_entry_points(tool):
    """Every entry point (encode, host pipeline, stats/finalize, posteriors, scoring, EM, embedding) on
    narrow, wide and masked-D shapes under compute-sanitizer (PyTorch's own kernels included)."""
    import __graft_entry__
    __graft_entry__.build()
    r, out = _run_sanitizer(["compute-sanitizer", "--tool", tool, "--kernel-name", "kns=gpufv",
                             sys.executable, os.path.join(ROOT, "tools", "sanitize_entrypoints.py")], timeout=1500)
    print(out[-3000:])
    assert r.returncode == 0 and "entry points ok" in out, out[-3000:]
    assert ("ERROR SUMMARY: 0 errors" in out) or ("0 hazards displayed (0 errors, 0 warnings)" in out)
