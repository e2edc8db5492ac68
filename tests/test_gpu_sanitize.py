"""compute-sanitizer over small decodes of every kernel family
(tools/sanitize_smoke.py): memcheck (out-of-bounds / misaligned global and
shared accesses, leaks of device errors), racecheck (shared-memory hazards:
the persistent kernels' mbarrier rings, bulk copies, cluster DSMEM and the
row-reduction scratch), synccheck (barrier misuse).  SURVEY.md §5.

V = 64 (Vp = 256): every kernel and the CTA-wide exact row reduction; the
SMSP-balanced joiner tiling (Vp = 512 only) is left to the parity tests --
memcheck of a V >= 257 model (>= 66K decoder-table contexts) exceeds 10 min.
The V = 500 cluster kernels get racecheck and synccheck on two streams.
racecheck found (and this test now guards) a read of the FSA group's raw
candidate count racing its write (fsa.cu expand_arcs)."""
import os
import shutil
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


def _run(tool, *args, timeout=600):
    cmd = [SAN, "--tool", tool, "--error-exitcode", "97", "--print-limit", "20", "python",
           os.path.join(ROOT, "tools", "sanitize_smoke.py"), *args]
    if tool == "memcheck":
        cmd[3:3] = ["--leak-check", "no"]
    # own process group: a timeout kills the sanitizer AND its python child
    p = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True, start_new_session=True)
    try:
        out, _ = p.communicate(timeout=timeout)
    except subprocess.TimeoutExpired:
        os.killpg(p.pid, 9)
        p.communicate()
        raise
    r = p
    assert r.returncode == 0, out[-4000:]
    assert "sanitize smoke ok" in out
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-2000:]
    return out


def test_memcheck():
    _run("memcheck", "64", "3", "12")


def test_racecheck():
    _run("racecheck", "64", "3", "6")


def test_synccheck():
    _run("synccheck", "64", "3", "8")


def test_racecheck_cluster_kernels():
    """The V = 500 cluster kernels (beam: st.async h / logit slices on
    mbarrier phases; greedy: slice maxima and h rows the same way) on two
    streams.  ~5 min, most of it the instrumented decoder-table build."""
    _run("racecheck", "cluster", "4", timeout=900)


def test_synccheck_cluster_kernels():
    _run("synccheck", "cluster", "4")
