"""Multi-rank protocol of the N>1 path on the CPU (torch.distributed, gloo,
world_size 2 and 4): every rank builds its plan, the shards are disjoint and
cover the table, the rank-local layout maps consistently, and the per-child
best gathered from the ranks and merged equals the global best (bench.py does
the same with NCCL on GPUs, with the tables computed by the CUDA path)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import datagen
import oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, m, n, k, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1901_07643_b200 as bn
        opt = bn.options(free_vars=k, world=world, rank=rank)
        starts, lens = bn.bnreg_plan_shard_ranges(m, n, opt)
        gidx = np.concatenate([np.arange(s, s + l) for s, l in zip(starts, lens)])
        info = bn.bnreg_plan_query(m, n, opt)
        assert len(gidx) == info["local_families"]
        for qq in range(0, len(gidx), max(1, len(gidx) // 300)):
            assert bn.bnreg_plan_local_index(m, n, opt, int(gidx[qq])) == qq
        # "broadcast R": rank 0 factors, the others receive it
        X = datagen.dag_data(m, n, 0.3, 0.5, 2.0, seed=21)
        R = torch.zeros(m * m, dtype=torch.float64)
        if rank == 0:
            R = torch.from_numpy(oracle.qr_r(oracle.centre(X)).ravel().copy())
        dist.broadcast(R, 0)
        # this rank's families and their BIC (oracle O2 on the broadcast R stands in for the GPU)
        rss = oracle.rss_reduced_indices(R.numpy().reshape(m, m), gidx)
        v, S = oracle.masks_of(m, gidx)
        ks = np.array([bin(int(s)).count("1") for s in S])
        bic = -(n / 2) * np.log(rss / n) - (n / 2) * (1 + np.log(2 * np.pi)) - (ks / 2) * np.log(n)
        bm = np.full(m, 0xFFFFFFFF, dtype=np.int64)
        bb = np.full(m, -np.inf)
        for c in range(m):
            sel = np.nonzero(v == c)[0]
            if len(sel) == 0:
                continue
            order = sorted(sel, key=lambda j: (-bic[j], ks[j], S[j]))
            bm[c], bb[c] = S[order[0]], bic[order[0]]
        gm = [torch.zeros(m, dtype=torch.int64) for _ in range(world)]
        gb = [torch.zeros(m, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gm, torch.from_numpy(bm))
        dist.all_gather(gb, torch.from_numpy(bb))
        allidx = [torch.zeros(m << (m - 1), dtype=torch.int8) for _ in range(world)]
        mine = torch.zeros(m << (m - 1), dtype=torch.int8)
        mine[torch.from_numpy(gidx)] = 1
        dist.all_gather(allidx, mine)
        if rank == 0:
            cover = sum(t.numpy().astype(np.int32) for t in allidx)
            M = np.stack([t.numpy() for t in gm]).astype(np.uint32)
            B = np.stack([t.numpy() for t in gb])
            mm, mb = bn.bnreg_best_merge(m, M, B)
            q.put((bool((cover == 1).all()), mm.tolist(), mb.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_shard_protocol(world):
    m, n, k = 11, 60, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    cover_ok, mm, mb = q.get(timeout=10)
    assert cover_ok
    X = datagen.dag_data(m, n, 0.3, 0.5, 2.0, seed=21)
    Xc = oracle.centre(X)
    ref = oracle.rss_reduced_indices(oracle.qr_r(Xc))
    _, S = oracle.masks_of(m, np.arange(m << (m - 1)))
    ks = np.array([bin(int(s)).count("1") for s in S])
    bic = -(n / 2) * np.log(ref / n) - (n / 2) * (1 + np.log(2 * np.pi)) - (ks / 2) * np.log(n)
    om, ob = oracle.best(bic, m)
    assert mm == [int(x) for x in om]
    np.testing.assert_allclose(mb, ob, rtol=0, atol=1e-9)
