"""Beam cluster kernel (config 5 small batches, T=1000): per-frame phase
cycles of thread 0 of CTA 0 (h+GEMM+push, reduce, beam steps, cluster-barrier
waits) averaged over clusters and frames."""
import json, os, sys
import torch
sys.path.insert(0, ".")
import bench
from paper_2211_00484_b200.api import BeamParams, Decoder, ModelWeights
w = bench.reference_weights()
for B in [int(b) for b in (sys.argv[1:] or ["64", "128"])]:
    dec = Decoder(ModelWeights.from_dict(w)); dec.set_encoder(w)
    d_enc, splits = bench.synthetic_frames(dec, 0, B, 1000, "cuda:0")
    tok = torch.zeros(B * 1000, dtype=torch.int32, device="cuda"); sc = torch.zeros(B, dtype=torch.float64, device="cuda")
    for r in range(2):
        dec.beam_search_batch(d_enc, splits, BeamParams(4), tok, sc)
    st = dec.stats(); ph = st["phase_cycles"]
    ncl = min(15, B)  # resident clusters used (launcher: occupancy-bound)
    print(json.dumps(dict(B=B, decode_ms=st["decode_ms"], rows_per_sf=st["joiner_rows"] / st["stream_frames"],
                          per_frame_kcyc=[round(p / 1000 / 1000 / ncl, 2) for p in ph],
                          h_kcyc=round(st["gather_cycles"] / 1000 / 1000 / ncl, 2),
                          steps_kcyc=round(st["gemm_wait_cycles"] / 1000 / 1000 / ncl, 2))), flush=True)
    dec.close()
