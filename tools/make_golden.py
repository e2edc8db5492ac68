"""Generates tests/golden/decode_golden.json from the compiled reference.

Tokens come from the reference's own public functions (greedy_search_batch,
beam_search, fsa_beam_search + lattice_to_best_seq); beam scores (which the
reference does not return) come from the oracle restatement after asserting
its tokens equal the reference's.  Run in the dev container, where
/root/reference exists:  python tools/make_golden.py
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests import helpers as H  # noqa: E402

CASES = [
    dict(method="greedy", model=[500, 80, 512, 512, 512, 3, 0.4], T=[24, 0, 17, 24], seed0=100),
    dict(method="greedy", model=[6, 6, 16, 64, 16, 9, 0.0], T=[5, 9, 1], seed0=7),
    dict(method="beam", model=[500, 80, 512, 512, 512, 3, 0.4], T=[16, 0, 9, 16], seed0=200,
         params=dict(beam=4, merge_op=0, length_norm=0, max_total=0)),
    dict(method="beam", model=[500, 80, 512, 512, 512, 3, 0.0], T=[12, 12], seed0=300,
         params=dict(beam=4, merge_op=1, length_norm=1, max_total=0)),
    dict(method="beam", model=[6, 6, 16, 64, 16, 9, -1.0], T=[6, 7, 8], seed0=11,
         params=dict(beam=3, merge_op=0, length_norm=0, max_total=3)),
    dict(method="fsa", model=[500, 80, 512, 512, 512, 3, 0.4], T=[14, 0, 14], seed0=400,
         params=[4.0, 8, 4]),
    dict(method="fsa", model=[6, 6, 16, 64, 16, 9, -0.5], T=[4, 6, 1], seed0=12,
         params=[1e9, 64, 32]),
]


def main():
    out = []
    for c in CASES:
        m = H.ref().model(*c["model"])
        feats, enc, splits = H.frames(m, c["T"], seed0=c["seed0"])
        if c["method"] == "greedy":
            c["tokens"] = m.greedy(feats, splits)
        elif c["method"] == "beam":
            p = c["params"]
            toks = m.beam(feats, splits, beam=p["beam"], merge_op=p["merge_op"],
                          length_norm=p["length_norm"], max_total=p["max_total"])
            ot, sc = H.orc().beam(m.w, enc, splits, **p)
            assert ot == toks
            c["tokens"], c["scores"] = toks, sc.tolist()
        else:
            g = H.ref().graph_trivial(c["model"][0])
            toks, sc, _ = m.fsa(feats, splits, g, *c["params"])
            c["tokens"], c["scores"] = toks, sc.tolist()
        out.append(c)
    path = os.path.join(H.GOLDEN, "decode_golden.json")
    json.dump({"generator": "tools/make_golden.py (compiled reference, oracle/_ref)", "cases": out},
              open(path, "w"), indent=1)
    print(path)


if __name__ == "__main__":
    main()
