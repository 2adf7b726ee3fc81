"""The stand-alone anchor pass (per-launch kernels, `ds_anchor`) at the 8B
shape: CUDA-event time per pass, per-layer split from the stage trace, and an
optional profiled pass (cudaProfilerStart/Stop around one call) for ncu:

    python tools/anchor_alone.py [--n 8192] [--reps 20]
    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
        --cache-control none --csv --log-file gpurun_out/anchor.csv python tools/anchor_alone.py --profile
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
from paper_2411_02820_b200.engine import _workspace  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--profile", action="store_true")
ap.add_argument("--swiglu", action="store_true")
ap.add_argument("--batch", type=int, default=0, help="rows of a batched pass (ds_anchor_batch), 0 = ds_anchor")
args = ap.parse_args()
cfg = P.ModelConfig(32, 4096, 32, 8, 128, 14336, 128256, max(args.n, 8192), 0,
                    mlp_kind="swiglu" if args.swiglu else "ungated")
n = args.n
B = P.random_model(cfg, seed=2000)
cache = P.PagedKV.allocate(cfg, n)
cache.k.normal_()
cache.v.normal_()
s = torch.cuda.Stream()
ws = _workspace(B, n, s)
tok = torch.from_numpy(np.random.default_rng(7).integers(0, cfg.vocab_size, size=n, dtype=np.int64)).cuda()
lg = torch.empty(cfg.vocab_size, device="cuda")
t32 = torch.empty(1, dtype=torch.int32, device="cuda")
bdesc, desc = B.desc(), cache.desc()
lib = L.lib()


def run():
    L.check(lib.ds_anchor(C.byref(bdesc), tok.data_ptr(), n, C.byref(desc), lg.data_ptr(), t32.data_ptr(),
                          ws.data_ptr(), ws.numel(), s.cuda_stream))


if args.batch:
    nb = args.batch
    caches = [cache] + [P.PagedKV.allocate(cfg, n, zero=False) for _ in range(nb - 1)]
    for c in caches[1:]:
        c.k.normal_()
        c.v.normal_()
    descs = (L.KvCache * nb)(*[c.desc() for c in caches])
    pos = (C.c_int32 * nb)(*([n - 1] * nb))
    ids = tok[-nb:].clone()
    lgb = torch.empty(nb, cfg.vocab_size, device="cuda")
    tb = torch.empty(nb, dtype=torch.int32, device="cuda")
    with torch.cuda.stream(s):
        wsb = torch.empty(P.engine.batch_workspace_bytes(cfg, n, nb), dtype=torch.uint8, device="cuda")

    def run():  # noqa: F811
        L.check(lib.ds_anchor_batch(C.byref(bdesc), nb, ids.data_ptr(), pos, descs, lgb.data_ptr(), tb.data_ptr(),
                                    wsb.data_ptr(), wsb.numel(), s.cuda_stream))


with torch.cuda.stream(s):
    for _ in range(5):
        run()
torch.cuda.synchronize()
if args.profile:
    torch.cuda.profiler.start()
    with torch.cuda.stream(s):
        run()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("ok")
    sys.exit(0)

lw = B.layers[0]
w_bytes = sum(t.numel() * t.element_size() for t in (lw["wqkv"], lw["wo"], lw["w1"], lw["w2"]))
kv_bytes = 2 * cfg.n_kv_heads * cfg.head_dim * n * 2
nrows = max(1, args.batch)
total = cfg.n_layers * (w_bytes + nrows * kv_bytes) + cfg.vocab_size * cfg.d_model * 2
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.reps)]
with torch.cuda.stream(s):
    for a, b in ev:
        a.record(s)
        run()
        b.record(s)
torch.cuda.synchronize()
ms = sorted(a.elapsed_time(b) for a, b in ev)
med = ms[len(ms) // 2]
# per-layer split (events between layers break the PDL chain: indicative only)
lib.ds_trace_begin()
with torch.cuda.stream(s):
    run()
cap = 256
tm, tg = (C.c_float * cap)(), (C.c_int32 * cap)()
m = lib.ds_trace_end(tm, tg, cap)
marks = [(int(tg[i]), float(tm[i])) for i in range(max(m, 0))]
out = {"n": n, "rows": nrows, "ms_median": med, "ms_min": ms[0], "gbs": total / med / 1e6, "bytes": total,
       "per_layer_bytes": w_bytes + kv_bytes, "trace": marks}
print(json.dumps(out))
