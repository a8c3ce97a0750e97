"""GPU tests of the multi-GPU path on one device.

* a3 root receive: rank 0 factors X (bnreg_load) and hands R out through
  bnreg_get_root_device; the other ranks never see X -- they install R with
  bnreg_set_root_device and walk their shards from it.  Every shard must be
  bit-identical to the same entries of a single-rank run, the shards must
  partition the table, and the device merge of the per-rank bests
  (bnreg_best_merge_async, the step after the NCCL all-gather) must equal the
  oracle's argmax (cfg2: the O1 table; cfg4 at full size with 8 logical ranks:
  the committed O2 golden, tests/golden/best_cfg4.json).
* bench.py's N>1 step functions (bench.Pipeline: load, broadcast of R, run,
  all-gather, device merge) in 2 processes sharing cuda:0, over gloo with the
  tensors staged through the host (NCCL refuses two ranks on one device).

The paper's p-processor scheme (§6) has every processor walk
from the root QRD; the north star broadcasts it from rank 0."""
import json
import os
import sys

import numpy as np
import pytest

import datagen
import oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _full_pairs(bn, X, opt=None):
    import torch
    h = bn.Bnreg.create(X, opt)
    F = h.num_families()
    t = torch.full((F, 2), float("nan"), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    bm, bb = h.run_pairs(t)
    torch.cuda.synchronize()
    h.close()
    return t, bm, bb


def _receive_run(bn, X, world, pairs_ranks=True):
    """Rank 0 loads X; ranks 1.. only receive R.  Returns the per-rank (shard index
    ranges, device table) and the device-merged best."""
    import torch
    n, m = X.shape
    h0 = bn.Bnreg(n, m, bn.options(world=world, rank=0))
    h0.load(X)
    Rt = torch.empty(m * m, dtype=torch.float64, device="cuda")
    h0.get_root_device(Rt)
    h0.sync()
    handles = [h0]
    for rank in range(1, world):
        h = bn.Bnreg(n, m, bn.options(world=world, rank=rank))
        h.set_root_device(Rt)               # never loads X
        handles.append(h)
    rec = torch.empty((world, 2 * m), dtype=torch.float64, device="cuda")
    shards = []
    for rank, h in enumerate(handles):
        F = h.num_families()
        t = torch.full((F, 2), float("nan"), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        base = rec[rank].data_ptr()
        if pairs_ranks or rank % 2 == 0:
            h.run_pairs_async(t, base + 8 * m, base)
        else:
            r = torch.full((F,), float("nan"), dtype=torch.float64, device="cuda")
            b = torch.full((F,), float("nan"), dtype=torch.float64, device="cuda")
            torch.cuda.synchronize()
            h.run_async(r, b, base + 8 * m, base)
            h.sync()
            t[:, 0] = r
            t[:, 1] = b
        h.sync()
        starts, lens = h.shard_ranges()
        shards.append((starts, lens, t))
    bm = torch.empty(m, dtype=torch.int32, device="cuda")
    bb = torch.empty(m, dtype=torch.float64, device="cuda")
    handles[0].best_merge_async(world, rec.data_ptr() + 8 * m, rec.data_ptr(), bm, bb, row_bytes=16 * m)
    handles[0].sync()
    # the host merge of the same records agrees bit for bit
    rc = rec.cpu().numpy()
    hm, hb = bn.bnreg_best_merge(m, rc[:, m:].copy().view(np.uint32)[:, :m], rc[:, :m].copy())
    dm, db = bm.cpu().numpy().view(np.uint32), bb.cpu().numpy()
    np.testing.assert_array_equal(dm, hm)
    np.testing.assert_array_equal(db, hb)
    for h in handles:
        h.close()
    return shards, dm, db


def _check_shards(full, shards, total):
    import torch
    seen = torch.zeros(total, dtype=torch.int32, device="cuda")
    for starts, lens, t in shards:
        gidx = torch.cat([torch.arange(s, s + l, device="cuda", dtype=torch.int64) for s, l in zip(starts, lens)])
        assert gidx.numel() == t.shape[0]
        assert not torch.isnan(t).any().item()
        assert torch.equal(t, full[gidx])            # bit-identical to the single-rank run
        seen[gidx] += 1
    assert bool((seen == 1).all().item())             # the shards partition the table


@pytest.mark.parametrize("world", [2, 4])
def test_root_receive_cfg2(world):
    import paper_1901_07643_b200 as bn
    X = datagen.config_data(2)
    n, m = X.shape
    full, fbm, fbb = _full_pairs(bn, X)
    shards, dm, db = _receive_run(bn, X, world, pairs_ranks=(world == 4))
    _check_shards(full, shards, m << (m - 1))
    _, refb = oracle.table(oracle.centre(X))
    om, ob = oracle.best(refb, m)
    np.testing.assert_array_equal(dm, om)
    np.testing.assert_array_equal(dm, fbm)
    np.testing.assert_array_equal(db, fbb)
    assert np.abs(db - ob).max() <= 1e-6


def test_root_receive_cfg4_eight_ranks():
    """cfg4 at full size (201 M families), 8 logical ranks; ranks 1-7 fed only by
    bnreg_set_root_device; merged best = the O2 golden argmax."""
    import torch
    import paper_1901_07643_b200 as bn
    X = datagen.config_data(4)
    n, m = X.shape
    full, fbm, fbb = _full_pairs(bn, X)
    shards, dm, db = _receive_run(bn, X, 8)
    _check_shards(full, shards, m << (m - 1))
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "best_cfg4.json")))
    gm = np.array([r["best_mask"] for r in g["children"]], dtype=np.uint32)
    gb = np.array([r["best_bic"] for r in g["children"]])
    np.testing.assert_array_equal(dm, gm)
    assert np.abs(db - gb).max() <= 1e-6
    np.testing.assert_array_equal(dm, fbm)
    del full, shards
    torch.cuda.empty_cache()


def _gloo_worker(rank, world, port, cfg, outdir):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import bench
    import paper_1901_07643_b200 as bn
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    X = datagen.config_data(cfg)
    n, m = X.shape
    h = bn.Bnreg(n, m, bn.options(world=world, rank=rank))
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    h.set_stream(stream.cuda_stream)
    # pipelined like the bench (the next dataset's load and R broadcast on a second stream)
    pipe = bench.Pipeline(bn, h, X, world, rank, dev, bench.HostStagedComm(dist), pairs=True,
                          load_stream=torch.cuda.Stream(dev))
    pipe.step_device()
    pipe.step_device()
    pipe.h.sync()
    bm1, bb1 = pipe.best_mask.cpu().numpy().view(np.uint32), pipe.best_bic.cpu().numpy()
    pipe.tab.fill_(float("nan"))
    r = pipe.step_e2e()                 # pipelined: returns the previous e2e step's result (none yet)
    assert r is None
    bm, bb = pipe.finish_e2e()
    h.sync()
    starts, lens = h.shard_ranges()
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), tab=pipe.tab.cpu().numpy(), bm=bm, bb=bb, bm1=bm1, bb1=bb1,
             starts=starts, lens=lens)
    h.close()
    dist.barrier()
    dist.destroy_process_group()


def test_bench_pipeline_two_processes_gloo(tmp_path):
    """bench.py's N>1 step (bench.Pipeline) in 2 processes on cuda:0 (gloo, host-staged
    exchanges): every rank's shard = the single-rank table's entries, both ranks hold
    the merged best = the oracle's argmax, for the device step and the e2e step."""
    import socket
    import torch
    import torch.multiprocessing as mp
    import paper_1901_07643_b200 as bn
    cfg, world = 2, 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.start_processes(_gloo_worker, args=(world, port, cfg, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    X = datagen.config_data(cfg)
    n, m = X.shape
    full, fbm, fbb = _full_pairs(bn, X)
    full = full.cpu().numpy()
    _, refb = oracle.table(oracle.centre(X))
    om, _ = oracle.best(refb, m)
    seen = np.zeros(m << (m - 1), dtype=np.int32)
    for rank in range(world):
        d = np.load(tmp_path / f"rank{rank}.npz")
        gidx = np.concatenate([np.arange(s, s + l) for s, l in zip(d["starts"], d["lens"])])
        np.testing.assert_array_equal(d["tab"], full[gidx])
        seen[gidx] += 1
        for key_m, key_b in (("bm", "bb"), ("bm1", "bb1")):
            np.testing.assert_array_equal(d[key_m], om)
            np.testing.assert_array_equal(d[key_b], fbb)
    assert (seen == 1).all()
    torch.cuda.empty_cache()


def test_pipelined_loads_bit_identical():
    """bnreg_set_load_stream: three datasets loaded on a second stream while the previous
    one is walked (load_async + run_pairs_async, no host synchronisation in between), on a
    rank-0 handle that loads X and a rank-1 handle fed by set_root_device: every table is
    bit-identical to the same dataset run without pipelining."""
    import torch
    import paper_1901_07643_b200 as bn
    datasets = [datagen.config_data(2, seed=2001 + i) for i in range(3)]
    n, m = datasets[0].shape
    ref = []
    for X in datasets:
        t, _, _ = _full_pairs(bn, X)
        ref.append(t)
    for world in (1, 2):
        hs = [bn.Bnreg(n, m, bn.options(world=world, rank=r)) for r in range(world)]
        run_st = torch.cuda.Stream()
        load_st = torch.cuda.Stream()
        for h in hs:
            h.set_stream(run_st.cuda_stream)
            h.set_load_stream(load_st.cuda_stream)
        Rt = torch.empty(m * m, dtype=torch.float64, device="cuda")
        Xd = [torch.from_numpy(np.ascontiguousarray(X.T)).cuda() for X in datasets]
        outs = [[torch.full((h.num_families(), 2), float("nan"), dtype=torch.float64, device="cuda") for h in hs]
                for _ in datasets]
        torch.cuda.synchronize()
        for i in range(len(datasets)):
            hs[0].load_async(Xd[i])
            if world > 1:
                hs[0].get_root_device(Rt)
                hs[1].set_root_device(Rt)      # both on the load stream, after the rank-0 load
            for h, o in zip(hs, outs[i]):
                h.run_pairs_async(o)
        for h in hs:
            h.sync()
        torch.cuda.synchronize()
        for i in range(len(datasets)):
            for h, o in zip(hs, outs[i]):
                starts, lens = h.shard_ranges()
                gidx = torch.cat([torch.arange(s0, s0 + l, device="cuda") for s0, l in zip(starts, lens)])
                assert torch.equal(o, ref[i][gidx]), (world, i)
        for h in hs:
            h.close()


def test_create_dist_in_library_nccl():
    """bnreg_create_dist / bnreg_run_pairs_dist: the library's own NCCL communicator
    (dlopen'd libnccl.so.2), R broadcast from rank 0, the per-rank bests all-gathered and
    merged on the device.  One process and one device here (NCCL refuses two ranks on one
    GPU), so world = 1: the table and the merged best must equal the plain handle's bit for
    bit, and the argmax the oracle's; a handle not made by create_dist is refused."""
    import torch
    import paper_1901_07643_b200 as bn
    X = datagen.config_data(2)
    n, m = X.shape
    full, fbm, fbb = _full_pairs(bn, X)
    uid = bn.nccl_unique_id()
    assert len(uid) == 128
    h = bn.Bnreg.create_dist(X, n, m, uid, 0, 1)
    t = torch.full((h.num_families(), 2), float("nan"), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    bm, bb = h.run_pairs_dist(t)
    torch.cuda.synchronize()
    assert torch.equal(t, full)
    np.testing.assert_array_equal(bm, fbm)
    np.testing.assert_array_equal(bb, fbb)
    # new data through the collective load: the same as a plain load of it
    X2 = datagen.dag_data(m, n, 0.2, 0.5, 2.0, seed=77)
    h.load_dist(X2)
    bm2, bb2 = h.run_pairs_dist(t)
    torch.cuda.synchronize()
    full2, fbm2, fbb2 = _full_pairs(bn, X2)
    assert torch.equal(t, full2)
    np.testing.assert_array_equal(bm2, fbm2)
    h.close()
    _, refb = oracle.table(oracle.centre(X))
    om, _ = oracle.best(refb, m)
    np.testing.assert_array_equal(bm, om)
    plain = bn.Bnreg.create(X)
    with pytest.raises(bn.BnregError, match="BNREG_E_STATE"):
        plain.run_pairs_dist(t)
    plain.close()
