"""glibc 2.39 exp / log / log1p ports (paper_2211_00484_b200/csrc/glibc_f64.h)
vs this host's libm, and the device log-softmax normaliser vs the reference.

The reference's fp64 log-probabilities (log_softmax_row, model.hpp:115-125),
log_add (common.hpp:48-54) and lattice sampling (fsa.hpp:390-448) call libm;
the decoders reproduce them bit for bit.  CPU: the header compiled for the
host (tools/glibc_f64_check.cpp) against libm on random and edge inputs.
GPU: the device ports and the decoders' row log-softmax against the host
libm / the compiled reference, bit for bit."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

from tests import helpers as H

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_host_port_matches_libm(tmp_path):
    exe = tmp_path / "glibc_f64_check"
    subprocess.run(
        ["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-o", str(exe),
         os.path.join(ROOT, "tools", "glibc_f64_check.cpp")],
        check=True,
    )
    r = subprocess.run([str(exe), "1000000", "11"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


def _libm(op, x):
    f = getattr(C.CDLL("libm.so.6"), op)
    f.restype, f.argtypes = C.c_double, [C.c_double]
    return np.array([f(float(v)) for v in x])


def _inputs(rng, n):
    lo = rng.uniform(-30, 30, n).astype(np.float32).astype(np.float64)
    return {
        "exp": np.concatenate([lo - np.maximum(lo, rng.uniform(-30, 30, n).astype(np.float32)),
                               rng.uniform(-745.2, 709.8, n), [0.0, -0.0, 1e-17, -800.0, 710.0, -np.inf]]),
        "log": np.concatenate([rng.uniform(1.0, 600.0, n), rng.uniform(0.9, 1.1, n), [1.0, 2.0, 5e-324]]),
        "log1p": np.concatenate([np.exp(rng.uniform(-50, 0, n)), rng.uniform(-0.9, 1.0, n), [0.0, 1.0, 1e-20]]),
    }


@pytest.mark.gpu
def test_device_ports_match_libm():
    from paper_2211_00484_b200.api import f64_math

    xs = _inputs(np.random.default_rng(5), 60000)
    for op, x in xs.items():
        want = _libm(op, x)
        got = f64_math(op, x)
        assert np.array_equal(got.view(np.int64), want.view(np.int64)), op
    x = xs["exp"][np.isfinite(xs["exp"])]
    got = f64_math("exp_g", x)
    assert np.array_equal(got.view(np.int64), _libm("exp", x).view(np.int64))


@pytest.mark.gpu
def test_device_log_softmax_bit_exact():
    """Rows of real joiner logits plus ties, -0.0 / +0.0 maxima, V = 1, 31,
    33, 500, 512: lp = double(l) - lse bit-equal to the reference's
    log_softmax_row."""
    from paper_2211_00484_b200.api import log_softmax_lse

    rng = np.random.default_rng(3)
    m = H.model(V=500, seed=1, blank_bias=0.4)
    rows = H.ref_logits(m, 512, seed=9)  # [512][500] real joiner rows
    cases = [rows]
    for V in (1, 2, 31, 32, 33, 500, 512):
        x = rng.normal(0, 4, (64, V)).astype(np.float32)
        x[0, :] = 0.0
        x[1, 0] = -0.0
        x[2, :] = x[2, 0]  # all tied
        cases.append(x)
    for L in cases:
        lse = log_softmax_lse(L)
        lp = L.astype(np.float64) - lse[:, None]
        want = H.ref().log_softmax(L)
        assert np.array_equal(lp.view(np.int64), np.asarray(want).reshape(lp.shape).view(np.int64)), L.shape
