"""Persistent-anchor behaviour inside the two-stream consumer step (BASELINE
config 2): step time, CTA placement (distinct SMs) and the anchor's own phase
timeline (global-timer stamps written by CTA 0), for eager launches with
device tokens, eager with host tokens (the e2e path) and CUDA-graph replay.

    python tools/anchor_probe.py [--n 8192] [--k 6] [--reps 6]
"""
import argparse
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2411_02820_b200 as P  # noqa: E402
from paper_2411_02820_b200 import _lib as L  # noqa: E402
from paper_2411_02820_b200.engine import _workspace  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--k", type=int, default=6)
ap.add_argument("--reps", type=int, default=6)
args = ap.parse_args()
cfg = P.ModelConfig(32, 4096, 32, 8, 128, 14336, 128256, max(args.n, 8192), 0)
Lh = cfg.n_layers
A = P.random_model(cfg, seed=1000)
B = P.random_model(cfg, seed=2000, base=A, perturb_layers=range(Lh - args.k, Lh))
rc = P.RecomputeConfig([(Lh - args.k, Lh - 1)])
ids = np.random.default_rng(7).integers(0, cfg.vocab_size, size=args.n, dtype=np.int64)
tok = torch.from_numpy(ids).cuda()
pinned = torch.from_numpy(ids).pin_memory().numpy()
prod = P.full_prefill(A, ids, e_layers=rc.transition_layers, tokens_dev=tok)
cache = P.PagedKV.allocate(cfg, args.n)
cs, side = torch.cuda.Stream(), torch.cuda.Stream()
lib = L.lib()
ws = _workspace(B, args.n, cs)
dims = B.desc().dims


def anchor_info():
    sm = (C.c_int32 * 1024)()
    cnt = lib.ds_anchor_placement(C.byref(dims), args.n, C.c_void_p(ws.data_ptr()), sm, 1024)
    ns = (C.c_uint64 * 1024)()
    m = lib.ds_anchor_timeline(C.byref(dims), args.n, C.c_void_p(ws.data_ptr()), ns, 1024)
    t = np.array([ns[i] for i in range(m)], dtype=np.float64)
    rel = (t - t[0]) / 1e6
    layer_end = rel[5::5]  # after each layer's w2 phase
    per_layer = np.diff(np.concatenate([[0.0], layer_end]))
    phases = np.diff(rel).reshape(Lh, 5) if m == 1 + 5 * Lh else None
    return len(set(sm[i] for i in range(cnt))), rel[-1], per_layer, phases


def step(host=False):
    with torch.cuda.stream(cs):
        if host:
            return P.partial_prefill(B, pinned, rc, prod.kv, prod.e_map(), out=cache, stream=cs, copy_stream=side)
        return P.partial_prefill(B, ids, rc, prod.kv, prod.e_map(), out=cache, stream=cs, copy_stream=side,
                                 tokens_dev=tok)


for _ in range(3):
    step()
torch.cuda.synchronize()


def timed(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    a.record(cs)
    fn()
    b.record(cs)
    b.synchronize()
    return a.elapsed_time(b), (time.perf_counter() - w0) * 1e3


g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=cs):
    step()
torch.cuda.synchronize()
modes = {"eager_devtok": lambda: step(), "eager_hosttok": lambda: step(True), "graph": lambda: g.replay()}
for name, fn in modes.items():
    for r in range(args.reps):
        ms, wall = timed(fn)
        sms, anchor_ms, per_layer, phases = anchor_info()
        print(f"{name:14s} gpu {ms:7.3f} ms wall {wall:7.3f} ms  anchor SMs {sms}  anchor span {anchor_ms:7.3f} ms  "
              f"reused-layer avg {per_layer[:Lh - args.k].mean():.3f} ms  recomputed {np.round(per_layer[Lh - args.k:], 3)}")
    if phases is not None:
        print("  last run phase ms (qkv, attn, o, w1, w2) layer 0:", np.round(phases[0], 4), " layer 31:", np.round(phases[-1], 4))
