"""Stage timeline of one consumer step (BASELINE config 2) from the library's
trace events (ds_trace_begin/ds_trace_end): when each recompute layer's K/V
land, when each anchor layer finishes, where the copy stream waits.

    python tools/timeline.py [--n 8192] [--k 6] [--single]
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2411_02820_b200 as P  # noqa: E402
from paper_2411_02820_b200 import _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--k", type=int, default=6)
ap.add_argument("--single", action="store_true", help="one stream (no copy stream)")
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
cfg = P.ModelConfig(32, 4096, 32, 8, 128, 14336, 128256, max(args.n, 8192), 0)
Lh = cfg.n_layers
A = P.random_model(cfg, seed=1000)
B = P.random_model(cfg, seed=2000, base=A, perturb_layers=range(Lh - args.k, Lh))
rc = P.RecomputeConfig([(Lh - args.k, Lh - 1)])
ids = np.random.default_rng(7).integers(0, cfg.vocab_size, size=args.n, dtype=np.int64)
tok = torch.from_numpy(ids).cuda()
prod = P.full_prefill(A, ids, e_layers=rc.transition_layers, tokens_dev=tok)
cache = P.PagedKV.allocate(cfg, args.n)
side = None if args.single else torch.cuda.Stream()
lib = L.lib()


def step():
    P.partial_prefill(B, ids, rc, prod.kv, prod.e_map(), out=cache, copy_stream=side, tokens_dev=tok)


for _ in range(3):
    step()
torch.cuda.synchronize()
runs = []
for _ in range(args.reps):
    lib.ds_trace_begin()
    step()
    ms = (C.c_float * 4096)()
    tg = (C.c_int32 * 4096)()
    cnt = lib.ds_trace_end(ms, tg, 4096)
    runs.append({int(tg[i]): float(ms[i]) for i in range(cnt)})


def name(t):
    if t == 0:
        return "start"
    if t == 1:
        return "ingest"
    if t == 4000:
        return "logits"
    kind = {1: "qkv", 2: "layer", 3: "anchor"}[t // 1000]
    return f"{kind}{t % 1000}"


tags = sorted(runs[0], key=lambda t: runs[0][t])
med = {t: float(np.median([r[t] for r in runs])) for t in tags}
for t in sorted(tags, key=lambda t: med[t]):
    print(f"{med[t]:8.3f} ms  {name(t)}")
print(json.dumps({name(t): round(med[t], 3) for t in tags}))

# ---- anchor CTA placement (one per SM is the design) and CUDA-graph replay time
from paper_2411_02820_b200.engine import _workspace  # noqa: E402

ws = _workspace(B, args.n)
dims = B.desc().dims


def placement():
    out = (C.c_int32 * 1024)()
    cnt = lib.ds_anchor_placement(C.byref(dims), args.n, C.c_void_p(ws.data_ptr()), out, 1024)
    sms = [out[i] for i in range(max(cnt, 0))]
    return len(sms), len(set(sms))


torch.cuda.synchronize()
print("placement eager (ctas, distinct SMs):", placement())
cs = torch.cuda.Stream()
with torch.cuda.stream(cs):
    P.partial_prefill(B, ids, rc, prod.kv, prod.e_map(), out=cache, stream=cs, copy_stream=side, tokens_dev=tok)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=cs):
    P.partial_prefill(B, ids, rc, prod.kv, prod.e_map(), out=cache, stream=cs, copy_stream=side, tokens_dev=tok)
ts = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(cs)
    with torch.cuda.stream(cs):
        g.replay()
    b.record(cs)
    b.synchronize()
    ts.append(a.elapsed_time(b))
print("graph replay ms:", [round(t, 3) for t in ts], "placement graph:", placement())
