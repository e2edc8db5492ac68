"""End-to-end timing of the beam search with pinned host frames (the bench's
e2e leg) for A/B comparisons of the host-frame paths (RNNTG_SLICED /
RNNTG_FUSED_PE / slice lengths).  Usage: python tools/prof_e2e.py [B] [T] [reps]"""
import json
import sys
import time

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
d_enc, splits = bench.synthetic_frames(dec, 0, B, T, "cuda:0")
pin = torch.from_numpy(d_enc.cpu().numpy()).pin_memory()
dec.beam_search_batch(pin, splits, BeamParams(4))
wall, gpu = [], []
for r in range(reps):
    t0 = time.perf_counter()
    toks, sc = dec.beam_search_batch(pin, splits, BeamParams(4))
    wall.append((time.perf_counter() - t0) * 1e3)
    gpu.append(dec.stats()["gpu_ms"])
print(json.dumps(dict(B=B, T=T, wall_ms=[round(x, 2) for x in wall], gpu_ms=[round(x, 2) for x in gpu],
                      e2e_fps=B * T / (min(wall) * 1e-3), launches=dec.stats()["kernel_launches"],
                      checksum=float(sum(sc)))))
