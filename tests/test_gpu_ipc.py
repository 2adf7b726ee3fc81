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
