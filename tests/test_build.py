"""Build-level checks that need no GPU: the library compiles for sm_100a,
loads, exports every symbol include/rnntg.h declares, and the exact kernels
contain no fused multiply-add outside the correctly rounded IEEE division
routine (an FFMA in a dot product would silently change logits)."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2211_00484_b200 import build as B


@pytest.fixture(scope="module")
def lib():
    return B.build()


def test_library_loads_and_exports(lib):
    from paper_2211_00484_b200.api import exported_symbols

    so = ctypes.CDLL(lib)
    syms = exported_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(so, s), s
    so.rnntg_version.restype = ctypes.c_char_p
    assert b"sm_100a" in so.rnntg_version()


def test_sass_is_sm100a_and_uses_bulk_copies(lib):
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in sass
    assert "UBLKCP" in sass  # cp.async.bulk staging of out_w chunks


def _functions(sass):
    cur, out = None, {}
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            out[cur] = []
        elif cur:
            m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
            if m:
                out[cur].append(m.group(2).strip())
    return out


def test_no_ffma_outside_division(lib):
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    funcs = _functions(sass)
    exact = [f for f in funcs if re.search(r"gemm_exact|beam_(dual_|ws_|multi_)?kernel|greedy_(cluster_)?kernel|fsa_kernel|joiner_rows", f)]
    assert len(exact) >= 6
    for f in exact:
        ins = funcs[f]
        # The division slow path is a subroutine placed after the last EXIT.
        last_exit = max(i for i, s in enumerate(ins) if s.endswith("EXIT") or " EXIT" in s or s == "EXIT")
        for i, s in enumerate(ins[: last_exit + 1]):
            if re.search(r"\bFFMA2?\b", s):
                # fp32 division (FCHK-guarded Newton steps, or the unchecked
                # reciprocal + Newton + residual sequence of
                # exact_math.h:fdiv_nochk after MUFU.RCP) and the fp64
                # division's range check (FFMA ..., RZ, ... after DFMA steps)
                # are correctly rounded sequences, not dot-product math.
                window = ins[max(0, i - 10) : i]
                rcp_window = ins[max(0, i - 32) : i]
                assert any("FCHK" in w or "DFMA" in w for w in window) or any(
                    "MUFU.RCP" in w for w in rcp_window
                ), f"{f}: FFMA outside division: {s}"
