"""Quick device timing of the decode paths (development aid)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle.py_oracle import Reference  # weights only (init_model)
from paper_2211_00484_b200.api import BeamParams, Decoder, ModelWeights

ref = Reference()
m = ref.model(500, 80, 512, 512, 512, 1, 0.4)
t0 = time.time()
dec = Decoder(ModelWeights.from_dict(m.w.p))
torch.cuda.synchronize()
print("model create s", time.time() - t0, flush=True)
rng = np.random.default_rng(0)
for B, T in [(1024, 100), (1024, 300)]:
    enc = np.tanh(rng.standard_normal((B * T, 512)).astype(np.float32) * 0.5)
    splits = (np.arange(B + 1) * T).astype(np.int32)
    d_enc = torch.from_numpy(enc).cuda()
    tok = torch.zeros(B * T, dtype=torch.int32, device="cuda")
    sc = torch.zeros(B, dtype=torch.float64, device="cuda")
    for name, fn in [
        ("greedy", lambda: dec.greedy_search_batch(d_enc, splits, 1, tok)),
        ("beam4", lambda: dec.beam_search_batch(d_enc, splits, BeamParams(4), tok, sc)),
    ]:
        fn()
        torch.cuda.synchronize()
        t = time.time()
        fn()
        torch.cuda.synchronize()
        wall = time.time() - t
        st = dec.stats()
        print(json.dumps(dict(name=name, B=B, T=T, wall_s=wall, fps_wall=B * T / wall, **st,
                              fps_gpu=B * T / (st["gpu_ms"] * 1e-3), rows_per_sf=st["joiner_rows"] / st["stream_frames"])), flush=True)
