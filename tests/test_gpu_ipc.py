"""P2P-pull transport through CUDA IPC, two processes on one GPU.

The producer process prefills and exports its buffers (ds_ipc_export); the
consumer process maps them (ds_ipc_open) and runs the layer-pipelined partial
prefill whose ingest and recompute kernels read the producer's memory in
place.  On one GPU this exercises the same handles and kernels as the
NVLink path between GPUs (where the mapped pointers are peer memory).  The
consumer's logits and cache must equal a local run bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

TINY = (4, 256, 4, 1, 64, 1024, 4096, 1024, 7)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE="2")
    import torch.distributed as dist

    import paper_2411_02820_b200 as P
    from oracle import crosskv_oracle as O
    from paper_2411_02820_b200.pipeline import ConsumerPipeline
    from paper_2411_02820_b200.transport import RemoteExport, export_prefill

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        cfg = P.ModelConfig(*TINY)
        toks = O.synthetic_tokens(31, 1, 400, 4096)[0]
        rc = P.RecomputeConfig([(2, 3)])
        if rank == 0:
            A = P.build_model(cfg)
            prod = P.full_prefill(A, toks, e_layers=rc.transition_layers)
            torch.cuda.synchronize()
            obj = [export_prefill(prod, A.ident, toks)]
            dist.broadcast_object_list(obj, src=0)
            dist.barrier()  # consumer done with our memory
            out_q.put((0, "ok"))
        else:
            obj = [None]
            dist.broadcast_object_list(obj, src=0)
            remote = RemoteExport(obj[0])
            B = P.build_model(cfg, P.PerturbationSpec.block(4, [2], 0.5, 1000))
            got = ConsumerPipeline(B).run(toks, rc, remote.kv, remote.e_map)
            fused = P.partial_prefill(B, toks, rc, remote.kv, remote.e_map)
            torch.cuda.synchronize()
            # local reference: the same producer computation in this process
            A = P.build_model(cfg)
            prod = P.full_prefill(A, toks, e_layers=rc.transition_layers)
            ref = P.partial_prefill(B, toks, rc, prod.kv, prod.e_map())
            torch.cuda.synchronize()
            ok = (torch.equal(got.logits, ref.logits) and torch.equal(fused.logits, ref.logits)
                  and torch.equal(got.kv.dense().k, ref.kv.dense().k))
            remote.close()
            dist.barrier()
            out_q.put((1, bool(ok)))
    finally:
        dist.destroy_process_group()


MIDP = dict(n_layers=8, d_model=1024, n_heads=8, n_kv_heads=2, head_dim=128, d_ff=2816, vocab_size=8192,
            max_seq=4096, base_seed=3)


def _worker_persistent(rank, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE="2")
    if rank == 1:
        os.environ["DS_FORCE_REMOTE"] = "1"  # read before the library's first use in this process
    import torch.distributed as dist

    import paper_2411_02820_b200 as P
    from paper_2411_02820_b200 import _lib
    from paper_2411_02820_b200.transport import RemoteExport, export_prefill

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        cfg = P.ModelConfig(**MIDP)
        n = 4096
        toks = np.random.default_rng(44).integers(0, cfg.vocab_size, size=n, dtype=np.int64)
        rc = P.RecomputeConfig([(5, 7)])
        A = P.random_model(cfg, seed=1)
        B = P.random_model(cfg, seed=2, base=A, perturb_layers=range(5, 8), eps=0.5)
        if rank == 0:
            prod = P.full_prefill(A, toks, e_layers=rc.transition_layers)
            with _lib.anchor_shape("persistent"):
                ref = P.partial_prefill(B, toks, rc, prod.kv, prod.e_map(), copy_stream=torch.cuda.Stream())
            torch.cuda.synchronize()
            d = ref.kv.dense()
            obj = [export_prefill(prod, A.ident, toks), ref.logits.cpu(), d.k.cpu(), d.v.cpu()]
            dist.broadcast_object_list(obj, src=0)
            dist.barrier()  # consumer done with our memory
            out_q.put((0, "ok"))
        else:
            obj = [None] * 4
            dist.broadcast_object_list(obj, src=0)
            handles, ref_logits, ref_k, ref_v = obj
            remote = RemoteExport(handles)
            with _lib.anchor_shape("persistent"):
                got = P.partial_prefill(B, toks, rc, remote.kv, remote.e_map, copy_stream=torch.cuda.Stream())
                # the captured serving form over the mapped export (context tag from the handles)
                cap = P.CapturedPartialPrefill(B, n, rc, remote.kv, remote.e_map)
                served = cap.run(toks).logits.clone()
            torch.cuda.synchronize()
            d = got.kv.dense()
            ok = (torch.equal(got.logits.cpu(), ref_logits) and torch.equal(d.k.cpu(), ref_k)
                  and torch.equal(d.v.cpu(), ref_v) and torch.equal(served.cpu(), ref_logits))
            remote.close()
            dist.barrier()
            out_q.put((1, bool(ok)))
    finally:
        dist.destroy_process_group()


def _spawn(target):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    return res


def test_ipc_persistent_two_stream_remote_path():
    res = _spawn(_worker_persistent)
    assert res[0] == "ok" and res[1] is True


def test_ipc_pull_two_processes():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res[0] == "ok" and res[1] is True
