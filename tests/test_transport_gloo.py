"""Multi-process producer -> consumer transport logic on CPU (gloo, world size 2).

The NCCL transport's message sequence is the planner's link order
(sched.py:217-223): E of each transition layer first, then the reused
layers' K and V ascending.  Rank 0 serves a prefill; rank 1 receives every
job through NcclTransport's staging slots and must reassemble the producer's
window K/V and E bit-exactly.  Runs on gloo so it needs no GPU; the NCCL
path on B200s runs the same code with device tensors.
"""

import os
import socket

import pytest
import torch
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _prefill(n_layers, G, n, D, d):
    import paper_2411_02820_b200 as P
    g = torch.Generator().manual_seed(123)
    k = torch.randn(n_layers, G, n, D, generator=g).to(torch.bfloat16)
    v = torch.randn(n_layers, G, n, D, generator=g).to(torch.bfloat16)
    es = tuple(P.ECache(l, torch.randn(n - 1, d, generator=g)) for l in range(n_layers))
    return P.PrefillResult(P.LayerKV(k, v), es, torch.zeros(4), torch.zeros(1, dtype=torch.int32))


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist

    import paper_2411_02820_b200 as P
    from paper_2411_02820_b200.planner import ScheduledRequest, link_order
    from paper_2411_02820_b200.transport import NcclSender, NcclTransport

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        Ln, G, n, D, d = 6, 2, 130, 16, 64
        cfg = P.ModelConfig(Ln, d, 4, G, D, 128, 256, 512, 0)
        configs = {1: P.RecomputeConfig([(2, 3)]), 2: P.RecomputeConfig([(0, 1), (4, 4)])}
        pf = _prefill(Ln, G, n, D, d)
        if rank == 0:
            NcclSender().serve(pf, [(r, configs[r], n) for r in sorted(configs)], Ln)
            out_q.put((0, "ok"))
            return
        got = {}

        def capture(layer, k, v, dst_desc, window, cfg_, link):
            got[layer] = (k.clone(), v.clone())

        tr = NcclTransport(0, cfg, n, "cpu", ingest=capture)
        req = ScheduledRequest("r", 0.0, "m", configs[rank], Ln)
        order = []
        e_got = {}
        for job in link_order([req]):
            order.append((job.kind, job.layer))
            if job.kind == "e":
                e_got[job.layer] = tr.e_job(job.layer, None, None).clone()
            else:
                tr.kv_job(job.layer, None, None, n - 1, cfg, None)
        ok = set(got) == set(configs[rank].reused_layers(Ln))
        for l, (k, v) in got.items():
            ok &= torch.equal(k, pf.kv.k[l, :, :n - 1]) and torch.equal(v, pf.kv.v[l, :, :n - 1])
        for a, e in e_got.items():
            ok &= torch.equal(e, pf.e_map()[a].hidden)
        ok &= sorted(e_got) == list(configs[rank].transition_layers)
        out_q.put((rank, (bool(ok), order)))
    finally:
        dist.destroy_process_group()


def test_nccl_transport_sequence_over_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == "ok"
    ok1, order1 = res[1]
    ok2, order2 = res[2]
    assert ok1 and ok2
    # E first, then KV ascending (planner link order)
    assert order1 == [("e", 2), ("kv", 0), ("kv", 1), ("kv", 4), ("kv", 5)]
    assert order2 == [("e", 4), ("kv", 2), ("kv", 3), ("kv", 5)]


def _bcast_worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist

    import paper_2411_02820_b200 as P
    from paper_2411_02820_b200.transport import broadcast_export

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        Ln, G, n, D, d = 5, 2, 70, 16, 64
        cfg = P.ModelConfig(Ln, d, 4, G, D, 128, 256, 512, 0)
        pf = _prefill(Ln, G, n, D, d)
        pf.kv.context = "ctx-digest"
        rc = P.RecomputeConfig([(3, 4)])
        kv, e = broadcast_export(pf if rank == 0 else None, 0, cfg, n, rc.transition_layers, "cpu",
                                 layers=rc.reused_layers(Ln))
        ok = kv.context == "ctx-digest" and sorted(e) == list(rc.transition_layers)
        for l in rc.reused_layers(Ln):
            ok = ok and torch.equal(kv.k[l], pf.kv.k[l]) and torch.equal(kv.v[l], pf.kv.v[l])
        for l in rc.transition_layers:
            ok = ok and torch.equal(e[l].hidden, pf.e_map()[l].hidden)
        out_q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_broadcast_fanout_gloo():
    """broadcast_export (the collective fan-out): every consumer rank receives
    the producer's E and reused-layer K/V bit-exactly, with the context tag."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 3
    procs = [ctx.Process(target=_bcast_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(res[r] for r in range(world)), res
