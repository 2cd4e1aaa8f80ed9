"""Multi-GPU host logic on CPU: LPT sharding and the final result gather, world_size 2 over
gloo (the GPU path uses the same code over NCCL)."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_07315_b200.shard import gather_results, lpt_assign


def test_lpt_assign_partitions_and_balances():
    rng = np.random.default_rng(0)
    L = rng.integers(30, 875, 512)
    for ws in (1, 2, 4, 8):
        parts = lpt_assign(L, ws)
        allidx = np.sort(np.concatenate(parts))
        assert np.array_equal(allidx, np.arange(512))
        loads = [int(L[p].sum()) for p in parts]
        assert max(loads) - min(loads) <= int(L.max())  # LPT bound
    # deterministic and ties -> lower rank
    assert [p.tolist() for p in lpt_assign([5, 5, 5], 2)] == [[0, 2], [1]]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, B, T, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    L = np.random.default_rng(1).integers(1, T, B)
    idx = lpt_assign(L, ws)[rank]
    # fake per-utterance results that encode the utterance id
    n = len(idx)
    tok = torch.full((n, T), -1, dtype=torch.int32)
    ts = torch.full((n, T), -1, dtype=torch.int32)
    num = torch.zeros(n, dtype=torch.int32)
    sc = torch.zeros(n, dtype=torch.float32)
    for j, b in enumerate(idx):
        k = int(b % 5)
        tok[j, :k] = int(b)
        ts[j, :k] = torch.arange(k, dtype=torch.int32)
        num[j] = k
        sc[j] = -float(b)
    out = gather_results({"tokens": tok, "timestamps": ts, "num_tokens": num, "scores": sc}, idx, B, T,
                         device=torch.device("cpu"))
    if rank == 0:
        q.put({k: v.numpy() for k, v in out.items()})
    dist.destroy_process_group()


def test_gather_results_world2_gloo():
    B, T = 23, 9
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, B, T, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for b in range(B):
        k = b % 5
        assert out["num_tokens"][b] == k
        assert (out["tokens"][b, :k] == b).all() and (out["tokens"][b, k:] == -1).all()
        assert out["scores"][b] == -b
