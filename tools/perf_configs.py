"""Device throughput of every BASELINE.json config (and the config-5 batch
sweep) on one GPU, with encoder frames resident in HBM, next to the compiled
reference on the host cores for a bounded sample.  Development/evidence tool:
writes gpurun_out/perf_configs.json (summarised in profiles/).

Inputs are the reference's own (init_model weights, DetRng features through
the reference encoder) so the emission statistics are the reference's."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.py_oracle import Reference, synthetic_arpa  # noqa: E402
from paper_2211_00484_b200.api import BeamParams, Decoder, FsaParams, Graph, ModelWeights  # noqa: E402

ref = Reference()
THREADS = os.cpu_count() or 1
out = {"host_threads": THREADS, "configs": []}


def enc_for(m, B, T, seed0, unique=64):
    """Reference encoder frames for `unique` distinct streams, tiled to B
    streams (keeps host encoder time bounded; streams are independent)."""
    U = min(unique, B)
    feats = np.concatenate([ref.features(seed0 + i, T, 80) for i in range(U)])
    splits_u = (np.arange(U + 1) * T).astype(np.int32)
    enc_u = m.encoder(feats, splits_u, threads=THREADS).reshape(U, T, -1)
    enc = np.ascontiguousarray(np.concatenate([enc_u] * ((B + U - 1) // U))[:B].reshape(B * T, -1))
    return feats, splits_u, enc, (np.arange(B + 1) * T).astype(np.int32)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts), r


def run(name, m, B, T, kind, params, graph=None, ref_graph=None, cpu_streams=None):
    feats, splits_u, enc, splits = enc_for(m, B, T, 1000)
    dec = Decoder(ModelWeights.from_dict(m.w.p))
    d_enc = torch.from_numpy(enc).cuda()
    tok = torch.zeros(B * T, dtype=torch.int32, device="cuda")
    sc = torch.zeros(B, dtype=torch.float64, device="cuda")
    g = None
    if kind == "fsa":
        g = Graph(dec, graph.num_states, graph.arc_splits, graph.dst, graph.label, graph.weight)

    def fn():
        if kind == "greedy":
            return dec.greedy_search_batch(d_enc, splits, 1, tok)
        if kind == "beam":
            return dec.beam_search_batch(d_enc, splits, BeamParams(**params), tok, sc)
        return dec.fsa_beam_search(d_enc, splits, g, FsaParams(*params), tok, sc)

    ms, _ = timed(fn)
    st = dec.stats()
    row = dict(name=name, B=B, T=T, kind=kind, params=params, gpu_ms=ms, frames_per_s=B * T / (ms * 1e-3),
               decode_ms=st["decode_ms"], rows_per_sf=st["joiner_rows"] / max(1, st["stream_frames"]),
               arcs_per_sf=st["arcs_expanded"] / max(1, st["stream_frames"]),
               lattice_arcs_per_sf=st["lattice_arcs"] / max(1, st["stream_frames"]),
               phase_cycles=st["phase_cycles"],
               note="frames resident in HBM")
    if cpu_streams:
        n = min(cpu_streams, len(splits_u) - 1)
        f = feats[: n * T]
        s = splits_u[: n + 1]
        t0 = time.perf_counter()
        if kind == "greedy":
            m.greedy(f, s, threads=THREADS)
        elif kind == "beam":
            m.beam(f, s, beam=params["beam_size"], threads=THREADS)
        else:
            m.fsa(f, s, ref_graph, *params, threads=THREADS)
        dt = time.perf_counter() - t0
        row["cpu_ref_frames_per_s"] = n * T / dt
        row["cpu_ref_sample"] = f"{n} streams x T={T}, {THREADS} threads, reference API incl. its encoder"
        row["speedup_vs_cpu_ref"] = row["frames_per_s"] / row["cpu_ref_frames_per_s"]
    out["configs"].append(row)
    print(json.dumps(row), flush=True)
    dec.close()


m4 = ref.model(500, 80, 512, 512, 512, 0, 0.4)
run("config1 greedy B=8 T=200", m4, 8, 200, "greedy", {}, cpu_streams=8)
run("config2 beam4 B=256 T=500", m4, 256, 500, "beam", {"beam_size": 4}, cpu_streams=2 * THREADS)
tg = ref.graph_trivial(500)
run("config3 fsa trivial (4,8,4) B=512 T=500", m4, 512, 500, "fsa", [4.0, 8, 4], graph=tg.g, ref_graph=tg,
    cpu_streams=2 * THREADS)
m14 = ref.model(500, 80, 512, 512, 512, 0, -1.4)
lg = ref.graph_from_arpa(synthetic_arpa(500), 500)
out["ngram_graph"] = {"states": lg.g.num_states, "arcs": lg.g.num_arcs}
run("config4 fsa ngram (8,64,8) B=256 T=500", m14, 256, 500, "fsa", [8.0, 64, 8], graph=lg.g, ref_graph=lg,
    cpu_streams=THREADS)
for B in (64, 128, 256, 512, 1024, 2048, 4096):
    run(f"config5 beam4 T=1000 B={B}", m4, B, 1000, "beam", {"beam_size": 4})
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "perf_configs.json"), "w"), indent=1)
