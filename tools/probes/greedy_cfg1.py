"""Config 1 (greedy, B=8, T=200) timing and the cluster kernel's phase split."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from tests import helpers as H
from paper_2211_00484_b200.api import Decoder
m = H.model(V=500, seed=0, blank_bias=0.4)
_, enc, splits = H.frames(m, [200] * 8, seed0=1000)
dec = Decoder(H.api_weights(m.w))
d_enc = torch.from_numpy(enc).cuda()
tok = torch.zeros(8 * 200, dtype=torch.int32, device="cuda")
for r in range(3):
    osp, _ = dec.greedy_search_batch(d_enc, splits, 1, tok)
st = dec.stats()
ph = st["phase_cycles"]
print(json.dumps(dict(decode_ms=st["decode_ms"], gpu_ms=st["gpu_ms"], per_frame_cycles=[p / 8 / 200 for p in ph], chain=st["gather_cycles"] / 8 / 200, spec=st["gemm_wait_cycles"] / 8 / 200, tokens_per_frame=int(osp[-1]) / 1600,
                      frames_per_s=8 * 200 / (st["gpu_ms"] * 1e-3))))
