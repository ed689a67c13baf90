"""Multi-rank host logic on CPU (world size 2, gloo): batch-aligned query shards, the
timing max over ranks and the gather of scores ciphertexts.

The per-rank evaluation here is the CPU oracle (no GPU in this tier); the point is that
sharding + per-rank evaluation + gather reproduces the single-process result exactly,
i.e. the path shards with no data-path exchange.
"""
import os
import socket

import numpy as np
import pytest

import ephdc_inputs as inp
from paper_2511_00737_b200 import dist as pdist

torch = pytest.importorskip("torch")


def test_shard_range_partitions_whole_batches():
    for nq, B, world in [(1300, 512, 2), (65536, 2340, 8), (16, 512, 4), (2340 * 29, 2340, 3), (1, 7, 2)]:
        spans = [pdist.shard_range(nq, r, world, B) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == nq
        for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
            assert a1 == b0
        for q0, q1 in spans:
            assert q0 <= q1 and (q0 % B == 0 or q0 == q1 == nq)   # empty trailing shards allowed
            assert q1 == nq or q1 % B == 0            # only the last shard ends ragged
        nb = [(q1 - q0 + B - 1) // B for q0, q1 in spans]
        assert max(nb) - min(nb) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, nq, q):
    import torch.distributed as dist
    from oracle import pipeline as opipe
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        cfg = inp.CONFIGS["c1q3"]
        Xtr, ytr, Xq, _ = inp.gen_features(cfg, nq)
        P = inp.gen_projection(cfg)
        om = opipe.build_model(cfg, P, Xtr, ytr)
        q0, q1 = pdist.shard_range(nq, rank, world, om.bfv.B)
        H = opipe.encode_queries(om, P, Xq[q0:q1])
        local = opipe.infer_all(om, H) if q1 > q0 else np.zeros((0, 2, om.bfv.L, om.bfv.N), np.uint64)
        t = pdist.max_over_ranks(float(rank + 1))
        got = pdist.gather_ciphertexts(local)
        if rank == 0:
            H_all = opipe.encode_queries(om, P, Xq)
            want = opipe.infer_all(om, H_all)
            q.put((t, np.concatenate(got).tobytes() == want.tobytes(), sum(g.shape[0] for g in got), want.shape[0]))
    finally:
        dist.destroy_process_group()


def test_two_rank_shard_and_gather_reproduces_single_process():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    nq = 512 * 2 + 300                      # 3 batches of B = 512, the last ragged
    procs = [ctx.Process(target=_worker, args=(r, 2, port, nq, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    tmax, same, n_got, n_want = q.get(timeout=10)
    assert tmax == 2.0
    assert n_got == n_want == 3
    assert same
