"""Beam-search timing on the bench workload (reference-encoder frames in HBM),
for A/B comparisons of builds / knobs and for ncu captures.  Usage: python tools/prof_beam.py [B] [T] [reps]"""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2211_00484_b200.api import BeamParams, Decoder, ModelWeights  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
T = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
w = bench.reference_weights()
dec = Decoder(ModelWeights.from_dict(w))
dec.set_encoder(w)
if os.environ.get("RNNTG_PROF_BF16") == "1":  # the tcgen05 bf16 joiner variant
    dec.set_joiner_mode("bf16")
d_enc, splits = bench.synthetic_frames(dec, 0, B, T, "cuda:0")
tok = torch.zeros(B * T, dtype=torch.int32, device="cuda")
sc = torch.zeros(B, dtype=torch.float64, device="cuda")
out = []
for r in range(reps):
    osp, otok, osc = dec.beam_search_batch(d_enc, splits, BeamParams(4), tok, sc)
    st = dec.stats()
    out.append(st["decode_ms"])
ph = st["phase_cycles"]
tot = sum(ph) or 1
print(json.dumps(dict(B=B, T=T, decode_ms=out, gpu_ms=st["gpu_ms"], fps_decode=B * T / (min(out) * 1e-3),
                      rows_per_sf=st["joiner_rows"] / st["stream_frames"], ties=st["tie_breaks"],
                      gather_share=round(st["gather_cycles"] / tot, 3),
                      gemm_wait_share=round(st["gemm_wait_cycles"] / tot, 4),
                      gemm_bar_share=round(st["lattice_arcs"] / tot, 4),
                      padded_per_row=st["joiner_rows_computed"] / max(1, st["joiner_rows"]),
                      gemm_mac_per_s_per_sm=st["joiner_rows_computed"] * 512 * 512 /
                      max(1e-9, st["phase_cycles"][1] / 1.965e9),
                      phase_share=[round(x / tot, 3) for x in ph],
                      tokens=int(osp[-1]), checksum=float(osc.sum()))))
