import json, os, sys
import torch
sys.path.insert(0, ".")
import bench
from paper_2211_00484_b200.api import BeamParams, Decoder, ModelWeights
from paper_2211_00484_b200.api import _load
w = bench.reference_weights()
for B in (64, 128, 192, 240):
    for env in ("1", "0"):
        os.environ["RNNTG_BEAM_CLUSTER"] = env
        dec = Decoder(ModelWeights.from_dict(w)); dec.set_encoder(w)
        d_enc, splits = bench.synthetic_frames(dec, 0, B, 1000, "cuda:0")
        tok = torch.zeros(B * 1000, dtype=torch.int32, device="cuda"); sc = torch.zeros(B, dtype=torch.float64, device="cuda")
        for r in range(2):
            dec.beam_search_batch(d_enc, splits, BeamParams(4), tok, sc)
        st = dec.stats(); ph = st["phase_cycles"]
        print(json.dumps(dict(B=B, cluster=env, decode_ms=st["decode_ms"], rows=st["joiner_rows"]/st["stream_frames"], ph=[p/1e6 for p in ph], h=st["gather_cycles"]/1e6)), flush=True)
        dec.close()
