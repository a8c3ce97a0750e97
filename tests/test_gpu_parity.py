"""GPU parity: the CUDA path (through the C-ABI) against the oracle, element by
element, on seeded inputs.  Tolerances (north_star):
RSS relative <= 1e-9, BIC absolute <= 1e-6, per-child argmax exact."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import datagen
import oracle

pytestmark = pytest.mark.gpu

RSS_RTOL = 1e-9
BIC_ATOL = 1e-6


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1901_07643_b200 as bn
    bn.lib()


def _bn():
    import paper_1901_07643_b200 as bn
    return bn


def _check_full(X, opt=None, o2=False, threads=0, pairs=False):
    from gpu_util import run_tables
    Xc = oracle.centre(X)
    n, m = X.shape
    rss, bic, bm, bb, h = run_tables(X, opt, pairs=pairs)
    assert not np.isnan(rss).any(), f"{np.isnan(rss).sum()} RSS entries never written"
    assert not np.isnan(bic).any(), f"{np.isnan(bic).sum()} BIC entries never written"
    if o2:
        R0 = oracle.qr_r(Xc)
        ref = oracle.rss_reduced_indices(R0, None, threads)
    else:
        ref, _ = oracle.table(Xc, want_bic=False, threads=threads)
    err = np.abs(rss - ref) / ref
    assert err.max() <= RSS_RTOL, f"max rel RSS err {err.max():.3e} at {int(err.argmax())}"
    # BIC from the oracle's RSS through the oracle's BIC (reading G5)
    _, S = oracle.masks_of(m, np.arange(m << (m - 1)))
    ks = np.array([bin(int(s)).count("1") for s in S])
    ref_bic = -(n / 2) * np.log(ref / n) - (n / 2) * (1 + np.log(2 * np.pi)) - (ks / 2) * np.log(n)
    berr = np.abs(bic - ref_bic)
    assert berr.max() <= BIC_ATOL, f"max abs BIC err {berr.max():.3e}"
    om, ob = oracle.best(ref_bic, m)
    assert np.array_equal(bm, om), f"argmax mismatch: {bm} vs {om}"
    np.testing.assert_allclose(bb, ob, atol=BIC_ATOL)
    h.close()
    _check_full.best = (bm, bb)
    return rss, bic


def test_golden_m3():
    from gpu_util import run_tables
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "m3_table.json")))
    X = np.asfortranarray(np.array(g["rows"], dtype=float))
    rss, bic, bm, bb, h = run_tables(X)
    for e in g["table"]:
        assert rss[e["idx"]] == pytest.approx(float(Fraction(e["rss"])), rel=1e-12)
        assert bic[e["idx"]] == pytest.approx(e["bic"], abs=1e-10)
    assert [int(x) for x in bm] == [g["best"][str(v)] for v in range(3)]
    h.close()


@pytest.mark.parametrize("k", [8, 6, 4, 3, 2])
def test_cfg1_full_all_k(k):
    """cfg1 (m=8, n=100): every free-block size, so packs, tree levels and the
    single-worker case (k = m) are all exercised."""
    bn = _bn()
    X = datagen.config_data(1)
    _check_full(X, bn.options(free_vars=k))


@pytest.mark.parametrize("k", [8, 3, 2])
def test_cfg1_pairs(k):
    """bnreg_run_pairs (one table of 16 B (RSS, BIC) records, the bench's layout)
    on cfg1: same parity bar."""
    bn = _bn()
    X = datagen.config_data(1)
    _check_full(X, bn.options(free_vars=k), pairs=True)


def test_cfg2_pairs():
    X = datagen.config_data(2)
    _check_full(X, pairs=True)


def test_pairs_rejects_misaligned():
    import torch
    bn = _bn()
    X = datagen.config_data(1)
    h = bn.Bnreg.create(X)
    t = torch.zeros(2 * h.num_families() + 1, dtype=torch.float64, device="cuda")
    with pytest.raises(bn.BnregError):
        h.run_pairs(t.data_ptr() + 8)
    with pytest.raises(bn.BnregError):
        h.run_pairs(None)
    h.close()


@pytest.mark.parametrize("lw", [0, 1, 2, 5])
def test_tree_split_levels(lw):
    """Same table whatever split of the seed tree between global levels and
    in-warp derivation."""
    bn = _bn()
    X = datagen.dag_data(11, 300, 0.3, 0.5, 2.0, seed=77)
    _check_full(X, bn.options(free_vars=4, levels_in_warp=lw))


@pytest.mark.parametrize("m,k,seed", [(5, 2, 1), (6, 3, 2), (9, 5, 3), (10, 7, 4), (12, 8, 5), (13, 6, 6)])
def test_small_random(m, k, seed):
    bn = _bn()
    X = datagen.gaussian(4 * m + 7, m, seed=seed, offset=3.0)
    _check_full(X, bn.options(free_vars=k))


@pytest.mark.parametrize("m,k", [(2, 2), (3, 2), (3, 3), (4, 2), (4, 3), (4, 4), (7, 2), (11, 8)])
@pytest.mark.parametrize("pairs", [False, True])
def test_edge_shapes(m, k, pairs):
    """Edge shapes: the smallest m (no pinned variable, one worker), k = m, k = 2 (the
    shortest schedule), no gang or warp variables (G < 4, fewer than 8 workers per warp),
    and the minimum n = m + 1, in both layouts."""
    bn = _bn()
    X = datagen.gaussian(m + 1, m, seed=40 + m * 10 + k, offset=-2.0)
    _check_full(X, bn.options(free_vars=k), pairs=pairs)


def test_cfg2_full_o1():
    X = datagen.config_data(2)
    _check_full(X)


def test_cfg3_collinear_full_o2_and_o1_sample():
    """m=20, n=5000 with a near-collinear pair: full table against O2 (O2 itself
    pinned to O1 in test_oracle_pins), plus an O1 sample touching the pair."""
    from gpu_util import run_tables
    meta = {}
    X = datagen.config_data(3, meta=meta)
    rss, bic = _check_full(X, o2=True)
    from test_gpu_fullsize import check_argmax_golden
    check_argmax_golden(3, *_check_full.best)     # the committed oracle-only golden (G14, gaps >= 3.2e-5)
    Xc = oracle.centre(X)
    m = 20
    i, j = meta["pair"]
    rng = np.random.default_rng(5)
    idx = []
    for _ in range(300):
        v = int(rng.integers(0, m))
        S = int(rng.integers(0, 1 << m)) & ~(1 << v)
        if v not in (i, j):
            S |= (1 << i) if rng.random() < 0.5 else (1 << j)
        idx.append(oracle.index(m, v, S))
    idx = np.array(sorted(set(idx)), dtype=np.int64)
    ref = oracle.rss_indices(Xc, idx)
    err = np.abs(rss[idx] - ref) / ref
    assert err.max() <= RSS_RTOL


def test_errors_nonfinite_and_rank():
    bn = _bn()
    X = datagen.gaussian(50, 5, seed=1)
    X[7, 2] = np.inf
    with pytest.raises(bn.BnregError) as e:
        bn.Bnreg.create(X)
    assert e.value.status == bn.E_NONFINITE
    X = datagen.gaussian(50, 5, seed=1)
    X[:, 3] = 2.0 * X[:, 1]
    with pytest.raises(bn.BnregError) as e:
        bn.Bnreg.create(X)
    assert e.value.status == bn.E_RANK
    with pytest.raises(bn.BnregError) as e:
        bn.Bnreg(3, 5)
    assert e.value.status == bn.E_INVAL


def test_deferred_load_errors_and_recovery():
    """bnreg_load_async defers the NaN/Inf and rank checks to the next synchronous call
    (bnreg_sync, bnreg_run): both report the error, the handle refuses to run on the
    rejected data until a good load, and a good load afterwards gives the oracle's table;
    the same with a load stream (pipelined mode)."""
    import torch
    bn = _bn()
    good = datagen.config_data(1)
    n, m = good.shape
    bad_nan = good.copy(); bad_nan[3, 2] = np.nan
    bad_rank = good.copy(); bad_rank[:, 5] = 3.0 * bad_rank[:, 1]
    ref, _ = oracle.table(oracle.centre(good), want_bic=False)
    for pipelined in (False, True):
        h = bn.Bnreg(n, m, bn.options(free_vars=4))
        if pipelined:
            st = torch.cuda.Stream()
            h.set_load_stream(st.cuda_stream)
        for bad, code in ((bad_nan, bn.E_NONFINITE), (bad_rank, bn.E_RANK)):
            xb = np.asfortranarray(bad)
            h.load_async(xb)
            with pytest.raises(bn.BnregError) as e:
                h.sync()
            assert e.value.status == code
            with pytest.raises(bn.BnregError) as e:
                h.run()
            assert e.value.status == bn.E_STATE
            h.load_async(np.asfortranarray(bad))
            r = torch.empty(h.num_families(), dtype=torch.float64, device="cuda")
            torch.cuda.synchronize()
            with pytest.raises(bn.BnregError) as e:
                h.run(r, None)                      # the run itself reports the deferred error
            assert e.value.status == code
        h.load_async(np.asfortranarray(good))
        r = torch.full((h.num_families(),), float("nan"), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        h.run(r, None)
        torch.cuda.synchronize()
        assert (np.abs(r.cpu().numpy() - ref) / ref).max() <= RSS_RTOL
        h.close()


def test_async_api_argument_errors():
    """The round-2 entry points reject bad arguments with BNREG_E_INVAL: the device merge
    (nparts < 1, NULL arrays, a row stride that is not a multiple of 8 or is shorter than
    m doubles), root export before a load (BNREG_E_STATE)."""
    import torch
    bn = _bn()
    X = datagen.config_data(1)
    n, m = X.shape
    h = bn.Bnreg(n, m)
    R = torch.empty(m * m, dtype=torch.float64, device="cuda")
    with pytest.raises(bn.BnregError) as e:
        h.get_root_device(R)
    assert e.value.status == bn.E_STATE
    rec = torch.empty((2, 2 * m), dtype=torch.float64, device="cuda")
    om = torch.empty(m, dtype=torch.int32, device="cuda")
    ob = torch.empty(m, dtype=torch.float64, device="cuda")
    base = rec.data_ptr()
    for args in ((0, base + 8 * m, base, om, ob, 16 * m), (2, 0, base, om, ob, 16 * m),
                 (2, base + 8 * m, base, om, ob, 12), (2, base + 8 * m, base, om, ob, 8 * m - 8)):
        with pytest.raises(bn.BnregError) as e:
            h.best_merge_async(args[0], args[1], args[2], args[3], args[4], row_bytes=args[5])
        assert e.value.status == bn.E_INVAL
    h.close()


def test_root_r_gram():
    bn = _bn()
    X = datagen.config_data(3)
    Xc = oracle.centre(X)
    h = bn.Bnreg.create(X)
    R, order = h.root_r()
    G = Xc[:, order].T @ Xc[:, order]
    assert np.linalg.norm(R.T @ R - G) <= 1e-10 * np.linalg.norm(G)
    assert np.all(np.diag(R) > 0) and np.allclose(np.tril(R, -1), 0)
    Ro = oracle.qr_r(np.asfortranarray(Xc[:, order]))
    np.testing.assert_allclose(np.abs(np.diag(R)), np.abs(np.diag(Ro)), rtol=1e-7)
    h.close()


def test_deterministic_and_device_load():
    from gpu_util import run_tables
    X = datagen.config_data(2)
    a = run_tables(X)
    b = run_tables(X, device_load=True)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert np.array_equal(a[2], b[2])
    a[4].close(); b[4].close()


def test_all_rss_and_bic_entry_points():
    import torch
    bn = _bn()
    X = datagen.config_data(1)
    h = bn.Bnreg.create(X, bn.options(free_vars=4))
    F = h.num_families()
    r = torch.full((F,), np.nan, dtype=torch.float64, device="cuda")
    b = torch.full((F,), np.nan, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()      # the fills run on torch's stream, the handle on its own
    h.all_rss(r)
    h.bic(b)
    r2 = torch.zeros(F, dtype=torch.float64, device="cuda")
    b2 = torch.zeros(F, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    h.run(r2, b2)
    assert torch.equal(r, r2) and torch.equal(b, b2)
    h.close()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_logical_ranks_union(world):
    """Multi-GPU partition run rank by rank on one GPU: shards are disjoint,
    their union is the whole table, and the merged best is the global best."""
    from gpu_util import run_tables
    bn = _bn()
    X = datagen.dag_data(12, 200, 0.25, 0.5, 2.0, seed=12)
    m = 12
    full, fullb, fbm, fbb, h0 = run_tables(X, bn.options(free_vars=3))
    h0.close()
    seen = np.zeros(m << (m - 1), dtype=np.int32)
    masks, bics = [], []
    for rank in range(world):
        # odd ranks through the record layout (bnreg_run_pairs), even ranks the two tables
        rss, bic, bm, bb, h = run_tables(X, bn.options(free_vars=3, world=world, rank=rank), pairs=bool(rank & 1))
        starts, lens = h.shard_ranges()
        gidx = np.concatenate([np.arange(s, s + l) for s, l in zip(starts, lens)])
        assert len(gidx) == h.num_families() == len(rss)
        step = max(1, len(gidx) // 500)
        assert all(h.local_index(int(gidx[q])) == q for q in range(0, len(gidx), step))
        seen[gidx] += 1
        assert not np.isnan(rss).any()
        np.testing.assert_array_equal(rss, full[gidx])
        np.testing.assert_array_equal(bic, fullb[gidx])
        masks.append(bm); bics.append(bb)
        h.close()
    assert (seen == 1).all()
    mm, mb = bn.bnreg_best_merge(m, np.array(masks), np.array(bics))
    assert np.array_equal(mm, fbm)


def test_fast_ln_accuracy():
    """The BIC epilogue's table+polynomial log against numpy's log (libm) over
    the whole normal range used by RSS values: |err| <= 4e-15 * max(1, |ln x|)."""
    import torch
    bn = _bn()
    rng = np.random.default_rng(0)
    x = np.concatenate([10.0 ** rng.uniform(-299, 300, 200000), rng.uniform(0.5, 2.0, 100000),
                        np.nextafter(1.0, 2.0) ** np.arange(1, 1000), [1.0, 2.0, 0.5, 1e-300 * 1.0001]])
    h = bn.Bnreg(10, 3)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    h.debug_ln(xd, yd, len(x))
    y = yd.cpu().numpy()
    ref = np.log(x)
    err = np.abs(y - ref) / np.maximum(1.0, np.abs(ref))
    assert err.max() <= 4e-15, err.max()
    h.close()


def test_tree_direct_matches_level_by_level():
    """The seed tree's depth-L1 nodes derived per node from the root in one launch
    equal the level-by-level tree (BNREG_TREE_LEVELS=1) bit for bit: same GRC
    sequence, same arithmetic."""
    import os
    from gpu_util import run_tables
    bn = _bn()
    X = datagen.config_data(2)
    opt = bn.options(free_vars=4, levels_in_warp=2)   # a deep global tree (L1 = 7)
    r1, b1, m1, _, h1 = run_tables(X, opt)
    h1.close()
    os.environ["BNREG_TREE_LEVELS"] = "1"
    try:
        r2, b2, m2, _, h2 = run_tables(X, opt)
        h2.close()
    finally:
        del os.environ["BNREG_TREE_LEVELS"]
    assert np.array_equal(r1, r2) and np.array_equal(b1, b2) and np.array_equal(m1, m2)


@pytest.mark.parametrize("pairs", [False, True])
def test_perfect_fit_scale_g13(pairs):
    """Reading G13: RSS <= 1e-300 -> BIC = +inf.  cfg1 scaled by 1e-152 passes the
    (relative) rank check while every RSS is ~1e-302, so every family takes the
    +inf path (the candidate threshold min(best, tiny_bic) of the walk); every
    child's best is then the empty set (G14: equal BIC -> smaller |S|)."""
    from gpu_util import run_tables
    X = datagen.config_data(1) * 1e-152
    n, m = X.shape
    rss, bic, bm, bb, h = run_tables(X, pairs=pairs)
    ref, _ = oracle.table(oracle.centre(X), want_bic=False)
    assert (ref <= 1e-300).all()
    assert (np.abs(rss - ref) / ref).max() <= RSS_RTOL
    assert np.isposinf(bic).all()
    assert bm.tolist() == [0] * m and np.isposinf(bb).all()
    h.close()


@pytest.mark.parametrize("score", [1, 2])
@pytest.mark.parametrize("pairs", [False, True])
def test_other_scores(score, pairs):
    """bnreg_set_score: AIC (loglik - |S|) and the log-likelihood
    as the score epilogue, element by element against oracle_score on cfg1 and cfg2
    (absolute 1e-6 as for BIC), per-child argmax exact (G14); the log-likelihood best
    is the full parent set."""
    import torch
    bn = _bn()
    for cfg in (1, 2):
        X = datagen.config_data(cfg)
        n, m = X.shape
        h = bn.Bnreg.create(X)
        h.set_score(score)
        F = h.num_families()
        if pairs:
            t = torch.full((F, 2), float("nan"), dtype=torch.float64, device="cuda")
            torch.cuda.synchronize()
            bm, bb = h.run_pairs(t)
            torch.cuda.synchronize()
            rss, sc = t[:, 0].cpu().numpy(), t[:, 1].cpu().numpy()
        else:
            r = torch.full((F,), float("nan"), dtype=torch.float64, device="cuda")
            b = torch.full((F,), float("nan"), dtype=torch.float64, device="cuda")
            torch.cuda.synchronize()
            bm, bb = h.run(r, b)
            torch.cuda.synchronize()
            rss, sc = r.cpu().numpy(), b.cpu().numpy()
        ref, _ = oracle.table(oracle.centre(X), want_bic=False)
        assert (np.abs(rss - ref) / ref).max() <= RSS_RTOL
        _, S = oracle.masks_of(m, np.arange(F))
        ks = np.array([bin(int(s)).count("1") for s in S])
        ref_sc = oracle.score_array(ref, n, ks, score)
        assert np.abs(sc - ref_sc).max() <= BIC_ATOL
        om, ob = oracle.best(ref_sc, m)
        assert np.array_equal(bm, om)
        np.testing.assert_allclose(bb, ob, atol=BIC_ATOL)
        if score == 2:
            assert [int(x) for x in bm] == [((1 << m) - 1) & ~(1 << v) for v in range(m)]
        with pytest.raises(bn.BnregError):
            h.set_score(3)
        h.close()


def test_coefficients_against_oracle():
    """bnreg_coefficients: the per-child best sets of the last run
    and random sets on cfg1, cfg2 and the near-collinear cfg3, against oracle.coefficients
    (lstsq on the centred data); relative 1e-8 of the coefficient scale (cfg3: 1e-5, its
    pair is ill-conditioned, kappa ~ 5e7)."""
    import torch
    bn = _bn()
    rng = np.random.default_rng(11)
    for cfg, tol in ((1, 1e-8), (2, 1e-8), (3, 1e-5)):
        X = datagen.config_data(cfg)
        n, m = X.shape
        Xc = oracle.centre(X)
        h = bn.Bnreg.create(X)
        with pytest.raises(bn.BnregError):
            h.coefficients()                      # no run yet
        bm, _ = h.run_pairs(torch.empty((h.num_families(), 2), dtype=torch.float64, device="cuda"))
        torch.cuda.synchronize()
        sets = [bm.astype(np.uint32), rng.integers(0, 1 << m, size=m, dtype=np.int64).astype(np.uint32)]
        for i, masks in enumerate(sets):
            beta = h.coefficients(None if i == 0 else masks)
            for v in range(m):
                ref = oracle.coefficients(Xc, v, int(masks[v]) & ~(1 << v))
                scale = max(1.0, np.abs(ref).max())
                assert np.abs(beta[v] - ref).max() <= tol * scale, (cfg, v)
        h.close()


def test_coefficients_batch_against_oracle():
    """bnreg_coefficients_batch (coefficients per family): every
    family of cfg1 (1024) and 3000 random families of cfg3 (near-collinear pair
    included) against oracle.coefficients (lstsq on the centred data), relative 1e-8
    of the coefficient scale (cfg3: 1e-5, kappa of its pair ~ 5e7); a child
    outside [0, m) gives a NaN row; bits >= m and the child's own bit are ignored;
    count 0 is a no-op, a negative count an error."""
    import torch
    bn = _bn()
    rng = np.random.default_rng(12)
    for cfg in (1, 3):
        X = datagen.config_data(cfg)
        n, m = X.shape
        Xc = oracle.centre(X)
        h = bn.Bnreg.create(X)
        if cfg == 1:
            fams = [(v, S) for v in range(m) for S in range(1 << m) if not (S >> v) & 1]
        else:
            fams = [(int(rng.integers(0, m)), int(rng.integers(0, 1 << m))) for _ in range(3000)]
            fams = [(v, S & ~(1 << v)) for v, S in fams]
        ch = np.array([v for v, _ in fams] + [-1, m, 0], dtype=np.int32)
        mk = np.array([S for _, S in fams] + [3, 3, 0xffffffff], dtype=np.uint32)
        F = len(ch)
        cd = torch.from_numpy(ch).cuda()
        md = torch.from_numpy(mk.view(np.int32)).cuda()
        beta = torch.full((F, m), 7.0, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        h.coefficients_batch(cd, md, F, beta)
        h.coefficients_batch(cd, md, 0, beta)
        with pytest.raises(bn.BnregError):
            h.coefficients_batch(cd, md, -1, beta)
        torch.cuda.synchronize()
        b = beta.cpu().numpy()
        h.close()
        for f, (v, S) in enumerate(fams):
            ref = oracle.coefficients(Xc, v, S)
            scale = max(1.0, np.abs(ref).max())
            tol = 1e-5 if cfg == 3 else 1e-8
            assert np.abs(b[f] - ref).max() <= tol * scale, (cfg, v, S)
        assert np.isnan(b[F - 3]).all() and np.isnan(b[F - 2]).all()
        ref = oracle.coefficients(Xc, 0, ((1 << m) - 1) & ~1)       # 0xffffffff: every other variable
        assert np.abs(b[F - 1] - ref).max() <= 1e-5 * max(1.0, np.abs(ref).max())


def _bps_run(cfg, layout):
    import torch
    bn = _bn()
    X = datagen.config_data(cfg)
    n, m = X.shape
    h = bn.Bnreg.create(X)
    F = h.num_families()
    bs = torch.full((F,), float("nan"), dtype=torch.float64, device="cuda")
    bmk = torch.zeros(F, dtype=torch.int32, device="cuda")
    if layout == "pairs":
        t = torch.empty((F, 2), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        best_m, best_b = h.run_pairs(t)
        h.best_subsets(t.data_ptr() + 8, 2, bs, bmk)
        sc = t[:, 1]
    else:
        sc = torch.empty(F, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        best_m, best_b = h.run(None, sc)
        scores = sc.clone()
        h.best_subsets(sc, 1, sc, bmk)                 # in place over the BIC table
        sc, bs = scores, sc
    torch.cuda.synchronize()
    out = (sc.cpu().numpy(), bs.cpu().numpy(), bmk.cpu().numpy().view(np.uint32), best_m, best_b, m)
    h.close()
    return out


@pytest.mark.parametrize("cfg,layout", [(1, "pairs"), (2, "pairs"), (2, "tables"), (3, "pairs")])
def test_best_subsets(cfg, layout):
    """bnreg_best_subsets on the GPU's own score column, exactly:
    cfg1 against the plain enumeration of every candidate set's subsets, cfg2 (15 mask
    bits: the low tile and a high group) against the subset-max recursion of the
    oracle, both layouts (the two-table one in place); the full candidate set gives the
    run's per-child best."""
    sc, bs, bmk, best_m, best_b, m = _bps_run(cfg, layout)
    ref = oracle.best_subsets_brute(sc, m) if cfg == 1 else oracle.best_subsets(sc, m)
    np.testing.assert_array_equal(bs, ref[0])
    np.testing.assert_array_equal(bmk, ref[1])
    for v in range(m):
        i = oracle.index(m, v, ((1 << m) - 1) & ~(1 << v))
        assert bmk[i] == best_m[v] and bs[i] == best_b[v]


@pytest.mark.parametrize("m", [9, 13, 16, 17, 20, 21])
def test_best_subsets_ties_pass_shapes(m):
    """bnreg_best_subsets on a score table full of ties (4 distinct values), so that the
    G14 tie-break (smaller |S|, then smaller mask) decides most entries, at every pass
    shape launch_bps uses: one shared-memory tile (m = 9), the register-tiled low pass
    alone (13) or followed by a small group (16: 3 bits) or by one register-tiled group
    of 4 / 7 / 8 bits (17, 20, 21; two groups: cfg4 in test_gpu_fullsize), exactly
    against the oracle's recursion (the scores are an input: any table is a valid one)."""
    import torch
    bn = _bn()
    h = bn.Bnreg.create(datagen.gaussian(4 * m, m, seed=m))
    F = h.num_families()
    rng = np.random.default_rng(100 + m)
    sc = rng.integers(0, 4, F).astype(np.float64) - 1.5
    sd = torch.from_numpy(sc).cuda()
    bs = torch.full((F,), float("nan"), dtype=torch.float64, device="cuda")
    bmk = torch.zeros(F, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    h.best_subsets(sd, 1, bs, bmk)
    torch.cuda.synchronize()
    h.close()
    ref = oracle.best_subsets(sc, m)
    np.testing.assert_array_equal(bs.cpu().numpy(), ref[0])
    np.testing.assert_array_equal(bmk.cpu().numpy().view(np.uint32), ref[1])


def test_best_subsets_errors():
    import torch
    bn = _bn()
    h = bn.Bnreg.create(datagen.config_data(1))
    t = torch.empty(h.num_families(), dtype=torch.float64, device="cuda")
    k = torch.empty(h.num_families(), dtype=torch.int32, device="cuda")
    with pytest.raises(bn.BnregError):
        h.best_subsets(t, 0, t, k)
    with pytest.raises(bn.BnregError):
        h.best_subsets(t, 2, t, k)                     # aliasing needs stride 1
    # the record table: best_score = the records themselves overlaps the BIC column (stride 2)
    F = h.num_families()
    rec = torch.empty((F, 2), dtype=torch.float64, device="cuda")
    with pytest.raises(bn.BnregError):
        h.best_subsets(rec.data_ptr() + 8, 2, rec, k)
    with pytest.raises(bn.BnregError):
        h.best_subsets(t, 1, torch.empty_like(t), t)   # best_mask over the scores
    with pytest.raises(bn.BnregError):
        h.best_subsets(t, 1, t.data_ptr() + 8 * (F // 2), k)   # partial alias
    h.close()


def test_coefficients_after_async_run():
    """bnreg_coefficients(masks=NULL) uses the per-child best of the last run even when
    that run wrote its best into a caller's device array (bnreg_run_async /
    bnreg_run_pairs_async), and refuses after new data is loaded (no stale sets)."""
    import torch
    bn = _bn()
    X = datagen.config_data(2)
    n, m = X.shape
    h = bn.Bnreg.create(X)
    F = h.num_families()
    bm_d = torch.zeros(m, dtype=torch.int32, device="cuda")
    bb_d = torch.zeros(m, dtype=torch.float64, device="cuda")
    rec = torch.empty((F, 2), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    h.run_pairs_async(rec, bm_d, bb_d)
    beta_none = h.coefficients(None)
    bm = bm_d.cpu().numpy().view(np.uint32)
    np.testing.assert_array_equal(beta_none, h.coefficients(bm))
    _, refb = oracle.table(oracle.centre(X))
    om, _ = oracle.best(refb, m)
    np.testing.assert_array_equal(bm, om)
    h.load(X)
    with pytest.raises(bn.BnregError):
        h.coefficients(None)
    h.close()


def test_cholesky_root_comparison():
    """SURVEY §8(f) NEXT 2, the paper's covariance alternative (it "comes at
    cost of numerical accuracy"): the root R by Cholesky of the Gram matrix.  On the
    well-conditioned cfg1 and cfg2 it meets the same parity bar as the QR root; on cfg3
    (near-collinear pair, kappa(X) ~ 5e7, kappa(G) ~ 1e15) the families that contain both
    members of the pair lose accuracy by orders of magnitude while the QR root does not."""
    from gpu_util import run_tables
    bn = _bn()
    for cfg in (1, 2):
        X = datagen.config_data(cfg)
        Xc = oracle.centre(X)
        h = bn.Bnreg(*X.shape)
        h.set_root_method(bn.ROOT_CHOLESKY)
        h.load(X)
        import torch
        t = torch.empty((h.num_families(), 2), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        h.run_pairs(t)
        torch.cuda.synchronize()
        rss = t[:, 0].cpu().numpy()
        ref, _ = oracle.table(Xc, want_bic=False)
        assert (np.abs(rss - ref) / ref).max() <= RSS_RTOL
        with pytest.raises(bn.BnregError):
            h.set_root_method(2)
        h.close()
    meta = {}
    X = datagen.config_data(3, meta=meta)
    Xc = oracle.centre(X)
    n, m = X.shape
    i, j = meta["pair"]
    rng = np.random.default_rng(9)
    idx = []
    for _ in range(200):
        v = int(rng.integers(0, m))
        if v in (i, j):
            continue
        S = (int(rng.integers(0, 1 << m)) | (1 << i) | (1 << j)) & ~(1 << v)
        idx.append(oracle.index(m, v, S))
    idx = np.array(sorted(set(idx)), dtype=np.int64)
    ref = oracle.rss_indices(Xc, idx)
    errs = {}
    for method in (bn.ROOT_TSQR, bn.ROOT_CHOLESKY):
        import torch
        h = bn.Bnreg(n, m)
        h.set_root_method(method)
        h.load(X)
        t = torch.empty((h.num_families(), 2), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        h.run_pairs(t)
        torch.cuda.synchronize()
        got = t[torch.from_numpy(idx).cuda(), 0].cpu().numpy()
        errs[method] = (np.abs(got - ref) / ref).max()
        h.close()
    assert errs[bn.ROOT_TSQR] <= RSS_RTOL
    assert errs[bn.ROOT_CHOLESKY] >= 1e3 * max(errs[bn.ROOT_TSQR], 1e-15), errs


@pytest.mark.parametrize("case", ["cfg1_k4", "cfg1_k8", "cfg2", "cfg2_pairs", "m12_k3", "m6_k2", "cfg3"])
def test_walk7_parity(case):
    """The alternative walk design (bnreg_options.pack_bits = 5: 32 lockstep workers per
    warp, one lane each; walk7_kernel.cu + seed7) against the oracle exactly like the
    default: every entry written, RSS relative 1e-9, BIC absolute 1e-6, exact argmax."""
    bn = _bn()
    if case.startswith("cfg1"):
        X, opt = datagen.config_data(1), bn.options(free_vars=int(case[-1]), pack_bits=5)
        _check_full(X, opt)
    elif case == "cfg2":
        _check_full(datagen.config_data(2), bn.options(pack_bits=5))
    elif case == "cfg2_pairs":
        _check_full(datagen.config_data(2), bn.options(pack_bits=5), pairs=True)
    elif case == "m12_k3":
        _check_full(datagen.dag_data(12, 200, 0.25, 0.5, 2.0, seed=12), bn.options(free_vars=3, pack_bits=5))
    elif case == "m6_k2":
        _check_full(datagen.dag_data(6, 40, 0.3, 0.5, 2.0, seed=6), bn.options(free_vars=2, pack_bits=5))
    else:
        _check_full(datagen.config_data(3), bn.options(pack_bits=5), o2=True, pairs=True)


def test_split_items_cfg3_k3():
    """Items with more than 16 back slots (the default walk's TMEM holds 4 back entries x 4
    lanes per warp) run as two passes (the second over back slots 16..): cfg3 with k = 3
    (m = 20, 17 pinned variables: up to 17 back slots per gang) against the full O2 table,
    both layouts, exact argmax; and the same with the split disabled (two launch classes)."""
    import os
    bn = _bn()
    X = datagen.config_data(3)
    info = bn.bnreg_plan_query(20, X.shape[0], bn.options(free_vars=3))
    assert info["p"] + info["g"] + (info["bh"] - info["g"]) > 16     # some items are split
    _check_full(X, bn.options(free_vars=3), o2=True, pairs=True)
    _check_full(X, bn.options(free_vars=3), o2=True, pairs=False)
    os.environ["BNREG_NO_SPLIT"] = "1"
    try:
        _check_full(X, bn.options(free_vars=3), o2=True, pairs=True)
    finally:
        del os.environ["BNREG_NO_SPLIT"]


@pytest.mark.parametrize("case", ["cfg1_k3", "cfg2_k5", "cfg2_k5_tables", "m12_k4", "cfg3_k3", "cfg3"])
def test_walk_slot_split_parity(case, monkeypatch):
    """The slot-split walk (design S, walks_kernel.cuh, BNREG_WALK_S=1: the gang's 4 warps
    run the same 32 workers one lane each and split the walk slots; step mbarriers and a
    staging buffer for the pivot rows instead of the gang barrier; plans with 3 warp and 2
    gang variables, m >= k + 5) against the oracle like the default design: every entry
    written, RSS relative 1e-9, BIC absolute 1e-6, exact argmax; cfg3 with k = 3 has split
    items (a second pass over back slots 16..)."""
    bn = _bn()
    monkeypatch.setenv("BNREG_WALK_S", "1")
    if case == "cfg1_k3":
        _check_full(datagen.config_data(1), bn.options(free_vars=3), pairs=True)
    elif case.startswith("cfg2_k5"):
        _check_full(datagen.config_data(2), bn.options(free_vars=5), pairs=not case.endswith("tables"))
    elif case == "m12_k4":
        _check_full(datagen.dag_data(12, 200, 0.25, 0.5, 2.0, seed=12), bn.options(free_vars=4), pairs=True)
    elif case == "cfg3_k3":
        _check_full(datagen.config_data(3), bn.options(free_vars=3), o2=True, pairs=True)
    else:
        _check_full(datagen.config_data(3), None, o2=True, pairs=True)
