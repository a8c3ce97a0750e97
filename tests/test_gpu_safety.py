"""Safety nets of the CUDA path:

* K8 exactly-once: the debug library libbnreg_k8.so (built by __graft_entry__.build(),
  -DBNREG_K8) counts every table store per entry; every entry of every table must be
  written exactly once (reading G11: the Alg.2 workers partition the families, PAPER.md
  :299-324) -- for the three walk designs (default, walk7, design S), both output layouts,
  world 1, 2 and 4, m <= 20.
  (The NaN-prefilled parity tests show every entry is written at least once.)
* bounds checks (the same debug build): every walk-kernel table index, shared-memory
  state address and TMEM column range is checked in range; violations are counted in
  the counter array's extra slot and must be 0.  (compute-sanitizer is closed on this
  GPU pool -- runs under it left GPUs needing a reset -- so the checks are our own.)"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
K8_LIB = os.path.join(ROOT, "paper_1901_07643_b200", "libbnreg_k8.so")

K8_SCRIPT = r"""
import os, sys, numpy as np, torch
sys.path.insert(0, %r)
import datagen, paper_1901_07643_b200 as bn
cases = [("cfg1", datagen.config_data(1), dict(free_vars=4)),
         ("m12", datagen.dag_data(12, 200, 0.25, 0.5, 2.0, seed=12), dict(free_vars=3, levels_in_warp=1)),
         ("cfg2", datagen.config_data(2), {}),
         ("cfg3", datagen.config_data(3), {}),
         ("cfg3_k3", datagen.config_data(3), dict(free_vars=3))]   # split items (17 back slots)
checked = 0
for name, X, kw in cases:
    n, m = X.shape
    for pb, ws in ((3, False), (5, False), (3, True)):      # the default walk, walk7, design S
        if ws:
            os.environ["BNREG_WALK_S"] = "1"
        else:
            os.environ.pop("BNREG_WALK_S", None)
        for world in ((1, 2, 4) if m <= 16 else (1, 2)):
            try:
                bn.bnreg_plan_query(m, n, bn.options(pack_bits=pb, world=world, **kw))
            except bn.BnregError:
                continue                    # too few pinned variables to split this plan so many ways
            for rank in range(world):
                for pairs in (False, True):
                    if m == 20 and not pairs and rank > 0:
                        continue
                    h = bn.Bnreg(n, m, bn.options(pack_bits=pb, world=world, rank=rank, **kw))
                    h.load(X)
                    F = h.num_families()
                    cnt = torch.zeros(F + 1, dtype=torch.int32, device="cuda")
                    torch.cuda.synchronize()
                    h.debug_write_counts(cnt)
                    if pairs:
                        t = torch.empty((F, 2), dtype=torch.float64, device="cuda")
                        torch.cuda.synchronize()
                        h.run_pairs(t)
                    else:
                        r = torch.empty(F, dtype=torch.float64, device="cuda")
                        b = torch.empty(F, dtype=torch.float64, device="cuda")
                        torch.cuda.synchronize()
                        h.run(r, b)
                    torch.cuda.synchronize()
                    c = cnt.cpu().numpy()
                    assert c[F] == 0, (name, pb, ws, world, rank, pairs, "bounds violations", int(c[F]))
                    c = c[:F]
                    assert c.min() == 1 and c.max() == 1, (name, pb, ws, world, rank, pairs, int(c.min()), int(c.max()),
                                                           int((c != 1).sum()))
                    h.close()
                    checked += 1
assert checked >= 60, checked
print("K8 exactly-once:", checked, "runs")
""" % ROOT


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_k8_every_entry_written_exactly_once():
    if not os.path.exists(K8_LIB):
        from paper_1901_07643_b200 import build as b
        b.build_k8()
    env = dict(os.environ, BNREG_LIB=K8_LIB)
    p = subprocess.run([sys.executable, "-c", K8_SCRIPT], env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert "K8 exactly-once" in p.stdout


def test_k8_bounds_checks_fire():
    """Negative control of the bounds-check path: with BNREG_K8_SELFTEST, lane 0 of every
    walk warp reports one deliberate violation, which must arrive in the violation slot
    (one per warp of the launch), while the exactly-once counts stay intact."""
    env = dict(os.environ, BNREG_LIB=K8_LIB, BNREG_K8_SELFTEST="1")
    script = r"""
import sys, torch
sys.path.insert(0, %r)
import datagen, paper_1901_07643_b200 as bn
X = datagen.config_data(2)
for pb in (3, 5):
    h = bn.Bnreg.create(X, bn.options(pack_bits=pb))
    F = h.num_families()
    cnt = torch.zeros(F + 1, dtype=torch.int32, device="cuda")
    h.debug_write_counts(cnt)
    t = torch.empty((F, 2), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    h.run_pairs(t)
    torch.cuda.synchronize()
    c = cnt.cpu().numpy()
    assert (c[:F] == 1).all() and c[F] > 0, (pb, int(c[F]))
    print("selftest violations", pb, int(c[F]))
    h.close()
print("K8 selftest ok")
""" % ROOT
    p = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0 and "K8 selftest ok" in p.stdout, p.stdout[-2000:] + p.stderr[-2000:]
