"""Sample-sharded multi-GPU runs (bench.py:123-153 of the
reference).

One process per GPU.  The graph is replicated (each rank regenerates the same
keyed graph or uploads the same arrays); sample ids are split by
``worker_ranges`` and each rank runs its contiguous range with the global ids,
so the concatenated rows are byte-identical to a single-GPU run.  The only
collective is the final gather of the compacted rows to rank 0:
``all_gather`` of the per-rank sizes, then a padded ``gather`` (NCCL over
NVLink on GPUs, gloo on CPU tensors in the tests).
"""

from __future__ import annotations

import numpy as np

from .sharding import shard_for_rank, worker_ranges  # noqa: F401


def gather_rows(off, ids, group=None, dst: int = 0):
    """Gather per-rank final-layout CSR pieces (off[n_r+1], ids) to `dst`.

    Works for any torch.distributed backend; tensors live on the backend's
    device (CUDA for NCCL, CPU for gloo).  `ids` may be int64 (F_FINAL_IDS) or
    int32 (F_FINAL_IDS32, half the NVLink bytes).  Returns (off, ids) concatenated in
    rank order on `dst` (None elsewhere)."""
    import torch
    import torch.distributed as dist
    ws = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if dist.get_backend(group) == "gloo" and ids.is_cuda:
        off, ids = off.cpu(), ids.cpu()  # gloo gathers host tensors
    dev = ids.device
    sizes = torch.tensor([off.numel() - 1, ids.numel()], dtype=torch.int64, device=dev)
    all_sizes = [torch.zeros_like(sizes) for _ in range(ws)]
    dist.all_gather(all_sizes, sizes, group=group)
    n_max = int(max(s[0].item() for s in all_sizes))
    e_max = int(max(s[1].item() for s in all_sizes))
    pad_off = torch.zeros(n_max + 1, dtype=torch.int64, device=dev)
    pad_off[:off.numel()] = off
    pad_ids = torch.full((max(e_max, 1),), -1, dtype=ids.dtype, device=dev)
    pad_ids[:ids.numel()] = ids
    offs = [torch.empty_like(pad_off) for _ in range(ws)] if rank == dst else None
    idss = [torch.empty_like(pad_ids) for _ in range(ws)] if rank == dst else None
    dist.gather(pad_off, offs, dst=dst, group=group)
    dist.gather(pad_ids, idss, dst=dst, group=group)
    if rank != dst:
        return None, None
    out_off, out_ids, base = [torch.zeros(1, dtype=torch.int64, device=dev)], [], 0
    for r in range(ws):
        n_r, e_r = int(all_sizes[r][0]), int(all_sizes[r][1])
        out_off.append(offs[r][1:n_r + 1] + base)
        out_ids.append(idss[r][:e_r])
        base += e_r
    return torch.cat(out_off), torch.cat(out_ids)


def run_sharded(app, graph, n_samples: int, seed: int, paradigm: str = "sp", group=None):
    """This rank's share of an N-sample job on its GPU, gathered to rank 0.
    Returns (final_off, final_ids int32) on rank 0, (None, None) elsewhere."""
    import torch.distributed as dist
    from . import _lib
    from .engine import run_device
    ws = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = shard_for_rank(n_samples, ws, rank)
    dr = run_device(app, graph, n_samples=hi - lo, sample_lo=lo, seed=seed, paradigm=paradigm)
    off, ids = gather_rows(dr.view(_lib.F_FINAL_OFF), dr.narrow_ids(), group)
    if off is not None:
        off, ids = off.clone(), ids.clone()
    dr.close()
    return off, ids
