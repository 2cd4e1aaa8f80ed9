"""Multi-GPU plumbing: utterances are independent, so a batch shards by
utterance across the ranks of one node with no collective inside decoding; the LM and boost
handles are replicated per device, and only the final fixed-size results are gathered.

Host logic only (no kernels): LPT assignment and the result gather over torch.distributed
(NCCL on GPUs; gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np


def lpt_assign(lengths, world_size: int):
    """Longest-processing-time-first: sort utterances by length (desc, index asc) and give each
    to the rank with the least total frames so far (ties -> lower rank). Returns a list of
    index arrays, one per rank, each in ascending utterance order."""
    L = np.asarray(lengths, dtype=np.int64)
    order = sorted(range(len(L)), key=lambda i: (-int(L[i]), i))
    load = [0] * world_size
    parts = [[] for _ in range(world_size)]
    for i in order:
        r = min(range(world_size), key=lambda k: (load[k], k))
        parts[r].append(i)
        load[r] += int(L[i])
    return [np.array(sorted(p), dtype=np.int64) for p in parts]


def gather_results(local: dict, index, B_total: int, T: int, group=None, device=None):
    """All-gather fixed-size padded per-rank results (tokens/timestamps [b, T], num_tokens,
    scores) and reassemble them in global utterance order on every rank.

    local: dict of tensors for this rank's utterances (in `index` order)."""
    import torch
    import torch.distributed as dist

    ws = dist.get_world_size(group)
    dev = device if device is not None else local["tokens"].device
    # ranks may hold different padded lengths (ragged batches): pad every row to the largest
    tm = torch.tensor([int(local["tokens"].shape[1])], dtype=torch.int64, device=dev)
    dist.all_reduce(tm, op=dist.ReduceOp.MAX, group=group)
    T = max(T, int(tm.item()))
    local = dict(local)
    for k in ("tokens", "timestamps"):
        x = local[k]
        if x.shape[1] < T:
            y = torch.full((x.shape[0], T), -1, dtype=x.dtype, device=x.device)
            y[:, : x.shape[1]] = x
            local[k] = y
    n = torch.tensor([len(index)], dtype=torch.int64, device=dev)
    ns = [torch.zeros_like(n) for _ in range(ws)]
    dist.all_gather(ns, n, group=group)
    cap = int(max(int(x.item()) for x in ns))

    def pad(x, fill):
        out = torch.full((cap,) + tuple(x.shape[1:]), fill, dtype=x.dtype, device=dev)
        out[: x.shape[0]] = x.to(dev)
        return out

    idx = pad(torch.as_tensor(np.asarray(index), dtype=torch.int64), -1)
    packs = {"tokens": pad(local["tokens"], -1), "timestamps": pad(local["timestamps"], -1),
             "num_tokens": pad(local["num_tokens"], 0), "scores": pad(local["scores"], float("-inf"))}
    all_idx = [torch.empty_like(idx) for _ in range(ws)]
    dist.all_gather(all_idx, idx, group=group)
    out = {
        "tokens": torch.full((B_total, T), -1, dtype=torch.int32, device=dev),
        "timestamps": torch.full((B_total, T), -1, dtype=torch.int32, device=dev),
        "num_tokens": torch.zeros(B_total, dtype=torch.int32, device=dev),
        "scores": torch.full((B_total,), float("-inf"), dtype=torch.float32, device=dev),
    }
    for k, v in packs.items():
        parts = [torch.empty_like(v) for _ in range(ws)]
        dist.all_gather(parts, v, group=group)
        for r in range(ws):
            m = all_idx[r] >= 0
            out[k][all_idx[r][m]] = parts[r][m]
    return out
