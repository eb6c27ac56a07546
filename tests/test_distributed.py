"""Multi-rank host logic on CPU (gloo, world_size 2): token sharding, the u64 SUM reduction of
partial counts (as int64 all-reduce), candidate slicing and the global argmin merge, checked
bit-exact against the single-process oracle.  The per-rank counts come from the oracle here; the
product's own run_distributed / stream_distributed run multi-rank on the GPU in
tests/test_gpu_distributed.py (gloo, world 2-3, and NCCL through the C ABI)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, ret):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2602_21626_b200.pipeline import merge_argmin, shard_range

    o = oracle.Oracle()
    L, ne, k, g, T, C = 6, 16, 3, 4, 5001, 37
    rng = np.random.default_rng(3)
    ids = rng.integers(0, ne, size=(T, L, k)).astype(np.uint8)  # same on both ranks
    cands = np.stack([np.random.default_rng(c).permutation(np.arange(L * ne) % g) for c in range(C)]).astype(np.uint8)
    lo, hi = shard_range(T, rank, world)
    A, E, _ = o.stats(L, ne, k, ids[lo:hi])
    buf = torch.from_numpy(E.astype(np.uint64).view(np.int64).ravel().copy())
    dist.all_reduce(buf, op=dist.ReduceOp.SUM)
    E_red = buf.numpy().view(np.uint64).reshape(L - 1, ne, ne)
    bufA = torch.from_numpy(A.view(np.int64).ravel().copy())
    dist.all_reduce(bufA, op=dist.ReduceOp.SUM)
    A_red = bufA.numpy().view(np.uint64).reshape(L, ne)
    c_lo, c_hi = shard_range(C, rank, world)
    _, _, obj, _ = o.eval_costs(L, ne, g, A_red, E_red, cands[c_lo:c_hi])
    full = torch.full((C,), float("inf"), dtype=torch.float64)
    full[c_lo:c_hi] = torch.from_numpy(obj)
    dist.all_reduce(full, op=dist.ReduceOp.MIN)
    am = merge_argmin(full.numpy())
    if rank == 0:
        A1, E1, _ = o.stats(L, ne, k, ids)
        _, _, obj1, am1 = o.eval_costs(L, ne, g, A1, E1, cands)
        ret["ok"] = bool(np.array_equal(E_red, E1) and np.array_equal(A_red, A1) and am == am1
                         and np.array_equal(full.numpy(), obj1))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_shard_reduce_argmin():
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), ret), nprocs=2, join=True)
    assert ret.get("ok") is True


def test_shard_range_partitions():
    from paper_2602_21626_b200.pipeline import merge_argmin, shard_range

    for n in (0, 1, 7, 4096, 67108864):
        for w in (1, 2, 4, 8):
            parts = [shard_range(n, r, w) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
    assert merge_argmin(np.array([3.0, 1.0, 1.0, 2.0])) == 1
    assert merge_argmin(np.array([])) == -1
