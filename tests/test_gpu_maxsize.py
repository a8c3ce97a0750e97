"""GPU parity at the largest problem the library accepts (include/bnreg.h limits):
m = 30 (15.6 G families in all) as logical ranks of a 4-rank job -- each rank's shard is
30 2^29 / 4 = 4.03 G entries (64 GB of (RSS, BIC) records), just under the 2^32
entries one rank may write -- and the refusal of the same problem on 2 ranks.

Two of the four ranks (0 and 3: complementary selector patterns) are run one after the
other on one device.  Each shard is checked element by element on a sample (uniform
families of the shard, both ends of every index range) against O1, for every entry
written (NaN prefill), and the rank's per-child best against the maximum of the
child's entries in the shard.  Tolerances as everywhere: RSS relative 1e-9, BIC absolute
1e-6.  The oracle cannot compute m = 30 tables whole; O1 solves each sampled family
from the centred data independently (§1, the families of every child)."""
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


def _bic(rss, n, ks):
    return -(n / 2) * np.log(rss / n) - (n / 2) * (1 + np.log(2 * np.pi)) - (ks / 2) * np.log(n)


def test_max_size_m30_four_ranks():
    import torch
    import paper_1901_07643_b200 as bn
    m, n = 30, 600
    X = datagen.dag_data(m, n, 0.08, 0.5, 2.0, seed=3030)
    Xc = oracle.centre(X)
    # 2 ranks: 7.5 G entries per rank > 2^32, refused at create
    with pytest.raises(bn.BnregError):
        bn.Bnreg(n, m, bn.options(world=2, rank=0))
    rng = np.random.default_rng(30)
    for rank in (0, 3):
        h = bn.Bnreg(n, m, bn.options(world=4, rank=rank))
        h.load(X)
        F = h.num_families()
        assert F <= 1 << 32 and F == (m << (m - 1)) // 4
        t = torch.full((F, 2), float("nan"), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        bm, bb = h.run_pairs(t)
        torch.cuda.synchronize()
        starts, lens = h.shard_ranges()
        h.close()
        assert int(np.sum(lens)) == F
        assert not torch.isnan(t).any().item()
        assert (t[:, 0] > 0).all().item()
        # the sample: uniform over the shard, both ends of every range
        offs = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
        loc = rng.integers(0, F, size=4000, dtype=np.int64)
        loc = np.unique(np.concatenate([loc, offs, offs + np.asarray(lens, dtype=np.int64) - 1]))
        r_of = np.searchsorted(offs, loc, side="right") - 1
        gidx = np.asarray(starts, dtype=np.int64)[r_of] + (loc - offs[r_of])
        tl = t[torch.from_numpy(loc).cuda()].cpu().numpy()
        ref = oracle.rss_indices(Xc, gidx)
        err = np.abs(tl[:, 0] - ref) / ref
        assert err.max() <= RSS_RTOL, f"rank {rank}: max rel RSS err {err.max():.3e} at {int(gidx[err.argmax()])}"
        _, S = oracle.masks_of(m, gidx)
        ks = np.array([bin(int(s)).count("1") for s in S])
        assert np.abs(tl[:, 1] - _bic(ref, n, ks)).max() <= BIC_ATOL
        # the rank's per-child best = the maximum of the child's entries in its shard
        block = 1 << (m - 1)
        for v in range(m):
            mx = -np.inf
            for s, ln_, o in zip(starts, lens, offs):
                if s // block == v:
                    mx = max(mx, t[int(o):int(o + ln_), 1].max().item())
            assert mx == bb[v], f"rank {rank} child {v}"
            if np.isfinite(mx):
                i = oracle.index(m, v, int(bm[v]))
                r_ = np.searchsorted(np.asarray(starts, dtype=np.int64), i, side="right") - 1
                assert t[int(offs[r_] + i - starts[r_]), 1].item() == bb[v]
        del t
        torch.cuda.empty_cache()
