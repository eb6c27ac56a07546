"""The product's multi-rank code on the GPU, bit-exact against one GPU / the oracle.

* gloo, world 2 and 3, every rank on cuda:0: HotPath.run_distributed and stream_distributed with
  real token shards and candidate slices (uneven splits, C < world so some ranks hold no
  candidates) give the single-GPU HotPath.run / stream answers (argmin, objective, M, greedy,
  moved).  NCCL itself cannot put two ranks on one device, so the collective here is gloo's; the
  sharding, lead-row and merge logic is the product's.
* NCCL through the C ABI (world 1: this pool exposes one GPU per call): gimbal_dist_comm_init +
  gimbal_pass_distributed_async on a later candidate slice, and gimbal_stats_allreduce with the
  token count left on the device, against the oracle.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _shape(name):
    return {"qwen3": (48, 128, 8, 8), "dsv2lite": (26, 64, 6, 8), "mixtral": (32, 8, 2, 8)}[name]


def _worker(rank, world, port, name, T, Cn, ret):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import paper_2602_21626_b200 as G
    from paper_2602_21626_b200.pipeline import shard_range

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L, ne, k, g = _shape(name)
        topo = G.MoeTopology(L, ne, k, g)
        trace = G.generate_trace(topo, T, model_seed=5, stream_seed=6, device=0)  # same on every rank
        cands = torch.from_numpy(G.shuffled_candidates(L * ne, g, 40, Cn)).cuda()
        lo, hi = shard_range(T, rank, world)
        c_lo, c_hi = shard_range(Cn, rank, world)
        hp = G.HotPath(topo, 0)
        got = hp.run_distributed(trace[lo:hi], cands[c_lo:c_hi].clone(), c_lo, Cn)
        # streaming windows, each window's tokens sharded over the ranks
        wins = [G.generate_trace(topo, 3001, model_seed=5, stream_seed=7, first_token=w * 3001, drift=0.05,
                                 drift_epoch=w + 1, device=0) for w in range(3)]
        M = G.HotPath(topo, 0).calibrate(wins[0])
        shards = [w[shard_range(3001, rank, world)[0]:shard_range(3001, rank, world)[1]] for w in wins]
        sgot = G.HotPath(topo, 0).stream_distributed(shards, cands[c_lo:c_hi].clone(), c_lo, Cn, M)
        if rank == 0:
            ref = G.HotPath(topo, 0)
            want = ref.run(trace, cands.clone())
            objs = ref._out[2].cpu().numpy()
            swant = G.HotPath(topo, 0).stream(wins, cands.clone(), M)
            ret["ok"] = (got.argmin == want.argmin and got.greedy == want.greedy
                         and got.affinity.experts == want.affinity.experts
                         and got.objective == float(objs.min()))
            ret["stream_ok"] = all(a[0] == b[0] and a[1] == b[1] and np.array_equal(np.asarray(a[2]), np.asarray(b[2]))
                                   for a, b in zip(sgot, swant)) and len(sgot) == len(swant)
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world,name,T,Cn", [(2, "qwen3", 20011, 33), (3, "dsv2lite", 9001, 2), (2, "mixtral", 5001, 1)])
def test_multirank_gloo_matches_single_gpu(world, name, T, Cn):
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), name, T, Cn, ret), nprocs=world, join=True)
    assert ret.get("ok") is True
    assert ret.get("stream_ok") is True


def test_c_abi_nccl_pass_and_allreduce(G, orc):
    """gimbal_dist_comm_init (1 rank) + gimbal_pass_distributed_async on the slice [5, 20) of 20
    candidates (scored behind a scratch greedy row) and on the leading slice; the global argmin,
    objectives and the device-side token count match the oracle."""
    lib = G._native.lib()
    L, ne, k, g = _shape("qwen3")
    topo = G.MoeTopology(L, ne, k, g)
    trace = G.generate_trace(topo, 7001, model_seed=2, stream_seed=3, device=0)
    Cn, off = 20, 5
    cands_np = G.shuffled_candidates(L * ne, g, 9, Cn)
    oA, oE, _ = orc.stats(L, ne, k, trace.cpu().numpy())
    M = list(orc.affinity_set(L, ne, g, oE, 0.0, 4, L * ne // g, 0))
    greedy = orc.greedy_place(L, ne, g, oA, M, 0)
    full = cands_np.copy()
    full[0] = greedy
    _, _, obj, am = orc.eval_costs(L, ne, g, oA, oE, full)

    uid = (C.c_uint8 * 128)()
    G._native.check(lib.gimbal_dist_unique_id(uid), "uid")
    comm = C.c_void_p()
    G._native.check(lib.gimbal_dist_comm_init(1, 0, uid, 0, C.byref(comm)), "comm")
    n, r = C.c_int32(), C.c_int32()
    G._native.check(lib.gimbal_dist_comm_size(comm, C.byref(n), C.byref(r)), "size")
    assert (n.value, r.value) == (1, 0)
    try:
        m = L * ne
        for lo, hi in ((off, Cn), (0, Cn)):
            s = G.RoutingStats(topo, 0)
            s.add_tokens(trace)
            lead = 0 if lo == 0 else 1
            buf = torch.zeros((hi - lo + lead, m), dtype=torch.uint8, device="cuda")
            buf[lead:] = torch.from_numpy(cands_np[lo:hi]).cuda()
            rows = buf.shape[0]
            scores = torch.empty((3, rows), dtype=torch.float64, device="cuda")
            gobj = torch.empty(Cn, dtype=torch.float64, device="cuda")
            out = torch.zeros(8 + 2 * m, dtype=torch.int32, device="cuda")
            base = out.data_ptr()
            torch.cuda.synchronize()
            G._native.check(lib.gimbal_pass_distributed_async(
                s.handle, comm, 0.0, 4, m // g, 0, C.c_void_p(buf.data_ptr()), hi - lo, lo, Cn, 1.0, 1.0,
                C.c_void_p(scores.data_ptr()), C.c_void_p(gobj.data_ptr()), C.c_void_p(base),
                C.c_void_p(base + 32 + 4 * m), C.c_void_p(base + 32), C.c_void_p(base + 8), C.c_void_p(base + 16)),
                "pass_distributed")
            s.sync()
            h = out.cpu().numpy()
            want_obj = np.full(Cn, np.inf)
            want_obj[lo:hi] = obj[lo:hi]
            if lo == 0:
                want_obj[0] = obj[0]
            assert np.array_equal(gobj.cpu().numpy(), want_obj)
            assert int(h[0:2].view(np.int64)[0]) == int(np.flatnonzero(want_obj == want_obj.min())[0])
            assert list(h[8 + m:8 + 2 * m]) == list(greedy)
            assert s.tokens() == 7001  # left on the device by the all-reduce, read back as sum A0 / k
            A, E, _ = s.read()
            assert np.array_equal(A, oA) and np.array_equal(E, oE)
    finally:
        G._native.check(lib.gimbal_dist_comm_destroy(comm), "destroy")
