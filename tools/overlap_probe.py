"""Where does the consumer step's time go?  Times (CUDA events, median of 10,
CUDA graphs) the fused two-stream step, the single-stream step, and the stages
alone: ingest, recompute group, anchor pass.

    python tools/overlap_probe.py [--n 8192] [--k 6]
"""
import argparse
import ctypes as C
import json
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2411_02820_b200 as P  # noqa: E402
from paper_2411_02820_b200 import _lib as L, ops  # noqa: E402
from paper_2411_02820_b200.engine import _workspace  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--k", type=int, default=6)
args = ap.parse_args()
SHAPE = dict(n_layers=32, d_model=4096, n_heads=32, n_kv_heads=8, head_dim=128, d_ff=14336, vocab_size=128256)
cfg = P.ModelConfig(max_seq=max(args.n, 8192), base_seed=0, **SHAPE)
L_ = cfg.n_layers
n, k = args.n, args.k
A = P.random_model(cfg, seed=1000)
B = P.random_model(cfg, seed=2000, base=A, perturb_layers=range(L_ - k, L_))
rc = P.RecomputeConfig([(L_ - k, L_ - 1)])
ids = np.random.default_rng(7).integers(0, cfg.vocab_size, size=n, dtype=np.int64)
tok = torch.from_numpy(ids).cuda()
prod = P.full_prefill(A, ids, e_layers=rc.transition_layers, tokens_dev=tok)
cache = P.PagedKV.allocate(cfg, n)
s = torch.cuda.Stream()
side_hi = torch.cuda.Stream(priority=-1)   # high priority copy/anchor stream
side_lo = torch.cuda.Stream(priority=0)
side = side_lo
ws = _workspace(B, n)
lib = L.lib()


def graph_time(fn, reps=10, cs=None):
    cs = cs or s
    with torch.cuda.stream(cs):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cs):
        fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cs)
        with torch.cuda.stream(cs):
            g.replay()
        b.record(cs)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


out = {}
out["fused_two_stream_ms"] = graph_time(lambda: P.partial_prefill(B, ids, rc, prod.kv, prod.e_map(), out=cache, stream=s,
                                                                  copy_stream=side, tokens_dev=tok))
out["fused_two_stream_hiprio_ms"] = graph_time(lambda: P.partial_prefill(B, ids, rc, prod.kv, prod.e_map(), out=cache,
                                                                         stream=s, copy_stream=side_hi, tokens_dev=tok))
s_hi = torch.cuda.Stream(priority=-1)
out["fused_two_stream_compute_hiprio_ms"] = graph_time(
    lambda: P.partial_prefill(B, ids, rc, prod.kv, prod.e_map(), out=cache, stream=s_hi, copy_stream=side_lo,
                              tokens_dev=tok), cs=s_hi)
out["fused_single_stream_ms"] = graph_time(lambda: P.partial_prefill(B, ids, rc, prod.kv, prod.e_map(), out=cache,
                                                                     stream=s, tokens_dev=tok))
reused = list(range(L_ - k))
d = cache.desc()
sd = prod.kv.desc()
out["ingest_ms"] = graph_time(lambda: ops.kv_ingest(sd, d, reused, n - 1, cfg.n_kv_heads, cfg.head_dim, stream=s))
e = prod.e_map()[L_ - k].hidden


def recompute():
    L.check(lib.ds_recompute_group(C.byref(B.desc()), tok.data_ptr(), n, L_ - k, L_ - 1, e.data_ptr(), e.shape[0],
                                   C.byref(d), ws.data_ptr(), ws.numel(), s.cuda_stream))


logits = torch.empty(cfg.vocab_size, device="cuda")
t32 = torch.empty(1, dtype=torch.int32, device="cuda")


def anchor():
    L.check(lib.ds_anchor(C.byref(B.desc()), tok.data_ptr(), n, C.byref(d), logits.data_ptr(), t32.data_ptr(),
                          ws.data_ptr(), ws.numel(), s.cuda_stream))


out["recompute_ms"] = graph_time(recompute)
out["anchor_ms"] = graph_time(anchor)
out["full_prefill_ms"] = graph_time(lambda: P.full_prefill(B, ids, e_layers=(), stream=s, tokens_dev=tok), reps=3)
print(json.dumps({k2: round(v, 3) for k2, v in out.items()}))
