"""Helpers for the GPU parity tests: run the C-ABI path on torch device buffers."""
from __future__ import annotations

import numpy as np

import paper_1901_07643_b200 as bn


def run_tables(X, opt=None, want_rss=True, want_bic=True, fill=np.nan, device_load=False, pairs=False):
    """Create + load + run; returns (rss, bic, best_mask, best_bic, handle) with
    tables as numpy arrays in the handle's (rank-local) layout.  pairs=True runs
    bnreg_run_pairs (one table of (RSS, BIC) records) and splits it."""
    import torch
    X = np.asfortranarray(X, dtype=np.float64)
    n, m = X.shape
    h = bn.Bnreg(n, m, opt)
    if device_load:
        Xd = torch.from_numpy(X.T.copy()).cuda()  # (m, n) row-major == column-major (n, m)
        torch.cuda.synchronize()                  # the copy runs on torch's stream, the handle on its own
        h.load(Xd.data_ptr())
    else:
        h.load(X)
    F = h.num_families()
    if pairs:
        t = torch.full((F, 2), fill, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        bm, bb = h.run_pairs(t)
        torch.cuda.synchronize()
        tt = t.cpu().numpy()
        return tt[:, 0].copy(), tt[:, 1].copy(), bm, bb, h
    r = torch.full((F,), fill, dtype=torch.float64, device="cuda") if want_rss else None
    b = torch.full((F,), fill, dtype=torch.float64, device="cuda") if want_bic else None
    torch.cuda.synchronize()      # the fills run on torch's stream, the handle on its own
    bm, bb = h.run(r, b)
    torch.cuda.synchronize()
    rr = r.cpu().numpy() if r is not None else None
    bbt = b.cpu().numpy() if b is not None else None
    return rr, bbt, bm, bb, h


def rel_err(got, ref):
    got = np.asarray(got)
    ref = np.asarray(ref)
    return np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300)
