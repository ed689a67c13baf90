"""Multi-GPU host logic: one process per GPU, query batches sharded with no data-path
collective.

The client evaluation is independent per ciphertext batch (one scores
ciphertext per B queries), so ranks split the query stream into contiguous,
batch-aligned shards and run the whole hot path on their own shard against a
replicated encrypted model.  The only cross-rank operations are the timing max
(bench.py) and, when a caller wants all scores ciphertexts on one rank (e.g. to hand
them to the server), a gather -- both through torch.distributed (NCCL on GPUs, gloo in
the CPU tests).
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np


def shard_range(nq_total: int, rank: int, world: int, B: int) -> Tuple[int, int]:
    """[q0, q1) of rank's shard: whole batches of B queries, as even as possible; the
    ragged last batch (if any) goes to the last non-empty shard."""
    if world < 1 or not 0 <= rank < world or B < 1:
        raise ValueError("bad shard request")
    nb = (nq_total + B - 1) // B
    per, extra = divmod(nb, world)
    b0 = rank * per + min(rank, extra)
    b1 = b0 + per + (1 if rank < extra else 0)
    return min(nq_total, b0 * B), min(nq_total, b1 * B)


def max_over_ranks(value: float) -> float:
    """Max of a per-rank scalar (device time of the timed region) over all ranks."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_ciphertexts(local: np.ndarray, dst: int = 0) -> List[np.ndarray]:
    """Gather every rank's scores ciphertexts [nb_r][2][L][N] (uint64) on rank dst, in
    rank order (= query order for shard_range shards).  Returns [] on other ranks."""
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    # NCCL moves only CUDA tensors (over NVLink); gloo moves CPU tensors
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    shape = list(local.shape)
    n = torch.tensor([shape[0]], dtype=torch.int64, device=dev)
    sizes = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(sizes, n)
    counts = [int(s.item()) for s in sizes]
    nmax = max(counts)
    pad = np.zeros([nmax] + shape[1:], dtype=np.uint64)
    pad[: shape[0]] = local
    t = torch.from_numpy(pad.view(np.int64)).to(dev)
    bufs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(bufs, t)   # gloo/NCCL both implement all_gather; NCCL has no gather
    if rank != dst:
        return []
    return [b.cpu().numpy().view(np.uint64)[: counts[r]] for r, b in enumerate(bufs)]
