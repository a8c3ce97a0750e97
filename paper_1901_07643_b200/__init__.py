"""bnreg -- B200-native exact all-family regressions (arXiv 1901.07643).

Thin ctypes binding of the C ABI in include/bnreg.h: argument marshalling only,
every step of the method runs in the sm_100a kernels of libbnreg.so.  There is
no CPU fallback: importing this package on a machine without the built library
raises, and calls that need a GPU fail with the CUDA error the library reports.

Device buffers are passed as raw pointers (ints) or any object with a
``data_ptr()`` method (e.g. a torch CUDA tensor); host arrays are numpy arrays.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# BNREG_LIB: load a variant build (e.g. tools/variants.sh A/B builds, the K8 debug build)
# from its own path; the in-tree libbnreg.so is never overwritten by a variant
LIB_PATH = os.environ.get("BNREG_LIB") or os.path.join(_HERE, "libbnreg.so")

OK, E_INVAL, E_NONFINITE, E_RANK, E_NOMEM, E_CUDA, E_STATE, E_NCCL = range(8)
SCORE_BIC, SCORE_AIC, SCORE_LOGLIK = 0, 1, 2
ROOT_TSQR, ROOT_CHOLESKY = 0, 1
_NAMES = {1: "BNREG_E_INVAL", 2: "BNREG_E_NONFINITE", 3: "BNREG_E_RANK", 4: "BNREG_E_NOMEM",
          5: "BNREG_E_CUDA", 6: "BNREG_E_STATE", 7: "BNREG_E_NCCL"}

# every symbol include/bnreg.h declares (checked by tests/test_abi.py)
SYMBOLS = ["bnreg_create", "bnreg_create_ex", "bnreg_load", "bnreg_load_async", "bnreg_sync", "bnreg_best_merge_async",
           "bnreg_set_load_stream", "bnreg_num_families", "bnreg_index",
           "bnreg_local_index", "bnreg_run", "bnreg_run_async", "bnreg_run_pairs", "bnreg_run_pairs_async", "bnreg_set_score", "bnreg_coefficients", "bnreg_coefficients_batch", "bnreg_best_subsets", "bnreg_set_root_method",
           "bnreg_all_rss", "bnreg_bic",
           "bnreg_set_stream", "bnreg_root_r", "bnreg_get_root_device", "bnreg_set_root_device",
           "bnreg_shard_ranges", "bnreg_plan_shard_ranges", "bnreg_plan_local_index", "bnreg_best_merge", "bnreg_timing", "bnreg_launches_per_run", "bnreg_plan_query",
           "bnreg_schedule", "bnreg_plan_packs", "bnreg_debug_ln", "bnreg_debug_write_counts", "bnreg_last_error",
           "bnreg_destroy", "bnreg_nccl_unique_id", "bnreg_create_dist", "bnreg_load_dist", "bnreg_run_pairs_dist"]


class BnregError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_NAMES.get(status, status)}: {msg}")
        self.status = status


class Options(ctypes.Structure):
    _fields_ = [("free_vars", ctypes.c_int32), ("levels_in_warp", ctypes.c_int32),
                ("world", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("pack_bits", ctypes.c_int32), ("ctas_per_sm", ctypes.c_int32)]


def options(free_vars=0, levels_in_warp=-1, world=1, rank=0, pack_bits=0, ctas_per_sm=0):
    """bnreg_options: pack_bits 0 = auto (3: 8 lockstep workers x 4 lanes per warp, gangs of
    4 warps), 5 = walk7 (32 workers per warp, one lane each)."""
    return Options(free_vars, levels_in_warp, world, rank, pack_bits, ctas_per_sm)


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, i32, i64, u32, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_double
    H = ctypes.c_void_p
    PH = ctypes.POINTER(ctypes.c_void_p)
    POPT = ctypes.POINTER(Options)
    sig = {
        "bnreg_create": ([P, i64, i32, PH], i32),
        "bnreg_create_ex": ([i64, i32, POPT, PH], i32),
        "bnreg_load": ([H, P, i32], i32),
        "bnreg_load_async": ([H, P, i32], i32),
        "bnreg_sync": ([H], i32),
        "bnreg_set_load_stream": ([H, P], i32),
        "bnreg_best_merge_async": ([H, i32, P, P, i64, P, P], i32),
        "bnreg_num_families": ([H], i64),
        "bnreg_index": ([i32, i32, u32], i64),
        "bnreg_local_index": ([H, i64], i64),
        "bnreg_run": ([H, P, P, P, P], i32),
        "bnreg_run_async": ([H, P, P, P, P], i32),
        "bnreg_run_pairs": ([H, P, P, P], i32),
        "bnreg_set_score": ([H, i32], i32),
        "bnreg_coefficients": ([H, P, P], i32),
        "bnreg_coefficients_batch": ([H, P, P, i64, P], i32),
        "bnreg_best_subsets": ([H, P, i64, P, P], i32),
        "bnreg_set_root_method": ([H, i32], i32),
        "bnreg_run_pairs_async": ([H, P, P, P], i32),
        "bnreg_all_rss": ([H, P], i32),
        "bnreg_bic": ([H, P], i32),
        "bnreg_set_stream": ([H, P], i32),
        "bnreg_root_r": ([H, P, P], i32),
        "bnreg_get_root_device": ([H, P], i32),
        "bnreg_set_root_device": ([H, P], i32),
        "bnreg_shard_ranges": ([H, P, P, P], i32),
        "bnreg_plan_shard_ranges": ([i32, i64, POPT, P, P, P], i32),
        "bnreg_plan_local_index": ([i32, i64, POPT, i64], i64),
        "bnreg_best_merge": ([i32, i32, P, P, P, P], i32),
        "bnreg_timing": ([H, i32, P, P], i32),
        "bnreg_launches_per_run": ([H], i64),
        "bnreg_plan_query": ([i32, i64, POPT, P], i32),
        "bnreg_schedule": ([i32, P, i64], i64),
        "bnreg_plan_packs": ([i32, i64, POPT, P, i64], i64),
        "bnreg_debug_ln": ([H, P, P, i64], i32),
        "bnreg_debug_write_counts": ([H, P], i32),
        "bnreg_last_error": ([], ctypes.c_char_p),
        "bnreg_destroy": ([H], None),
        "bnreg_nccl_unique_id": ([P], i32),
        "bnreg_create_dist": ([P, i64, i32, P, i32, i32, PH], i32),
        "bnreg_load_dist": ([H, P], i32),
        "bnreg_run_pairs_dist": ([H, P, P, P], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def _check(st):
    if st != OK:
        raise BnregError(st, lib().bnreg_last_error().decode())


def _dptr(x):
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return x.data_ptr()


def _hptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------- host-only calls
def bnreg_index(m: int, child: int, mask: int) -> int:
    return lib().bnreg_index(m, child, mask)


def bnreg_schedule(k: int) -> np.ndarray:
    n = lib().bnreg_schedule(k, None, 0)
    if n < 0:
        raise ValueError("k out of range")
    out = np.zeros(n, dtype=np.int8)
    lib().bnreg_schedule(k, _hptr(out), n)
    return out


def bnreg_plan_query(m: int, n: int, opt: Options | None = None) -> dict:
    info = np.zeros(16, dtype=np.int64)
    _check(lib().bnreg_plan_query(m, n, ctypes.byref(opt) if opt else None, _hptr(info)))
    keys = ["k", "b", "p", "bh", "L1", "LW", "npacks", "sched_len", "local_families", "total_families",
            "smem_per_warp", "r", "g"]
    return {k: int(v) for k, v in zip(keys, info)}


def bnreg_plan_packs(m: int, n: int, opt: Options | None = None) -> np.ndarray:
    o = ctypes.byref(opt) if opt else None
    cnt = lib().bnreg_plan_packs(m, n, o, None, 0)
    if cnt < 0:
        raise BnregError(E_INVAL, lib().bnreg_last_error().decode())
    out = np.zeros(cnt, dtype=np.uint32)
    lib().bnreg_plan_packs(m, n, o, _hptr(out), cnt)
    return out


def bnreg_plan_shard_ranges(m: int, n: int, opt: Options | None = None):
    cnt = ctypes.c_int64(0)
    starts = np.zeros(2 * m, dtype=np.int64)
    lens = np.zeros(2 * m, dtype=np.int64)
    _check(lib().bnreg_plan_shard_ranges(m, n, ctypes.byref(opt) if opt else None, ctypes.byref(cnt),
                                         _hptr(starts), _hptr(lens)))
    return starts[:cnt.value].copy(), lens[:cnt.value].copy()


def bnreg_plan_local_index(m: int, n: int, opt: Options | None, g: int) -> int:
    return lib().bnreg_plan_local_index(m, n, ctypes.byref(opt) if opt else None, g)


def nccl_unique_id() -> bytes:
    """bnreg_nccl_unique_id: a fresh NCCL communicator id (rank 0; hand it to the others)."""
    buf = ctypes.create_string_buffer(128)
    _check(lib().bnreg_nccl_unique_id(buf))
    return buf.raw


def bnreg_best_merge(m: int, masks: np.ndarray, bics: np.ndarray):
    masks = np.ascontiguousarray(masks, dtype=np.uint32).reshape(-1, m)
    bics = np.ascontiguousarray(bics, dtype=np.float64).reshape(-1, m)
    om = np.zeros(m, dtype=np.uint32)
    ob = np.zeros(m)
    _check(lib().bnreg_best_merge(m, masks.shape[0], _hptr(masks), _hptr(bics), _hptr(om), _hptr(ob)))
    return om, ob


# ---------------------------------------------------------------- handle
class Bnreg:
    """One handle = the device state for n x m data (bnreg_create_ex)."""

    def __init__(self, n: int, m: int, opt: Options | None = None):
        self.n, self.m = int(n), int(m)
        self.opt = opt
        h = ctypes.c_void_p()
        _check(lib().bnreg_create_ex(self.n, self.m, ctypes.byref(opt) if opt else None, ctypes.byref(h)))
        self._h = h

    @classmethod
    def create(cls, X: np.ndarray, opt: Options | None = None):
        """bnreg_create: host X (column-major n x m) -> loaded handle."""
        X = np.asfortranarray(X, dtype=np.float64)
        self = cls(X.shape[0], X.shape[1], opt)
        self.load(X)
        return self

    def load(self, X):
        """bnreg_load: host numpy X (copied H2D) or a device pointer / CUDA tensor."""
        if isinstance(X, np.ndarray):
            X = np.asfortranarray(X, dtype=np.float64)
            if X.shape != (self.n, self.m):
                raise ValueError("shape mismatch")
            _check(lib().bnreg_load(self._h, _hptr(X), 0))
        else:
            _check(lib().bnreg_load(self._h, _dptr(X), 1))

    def load_async(self, X):
        """bnreg_load_async: a device pointer / CUDA tensor, or a host numpy array that stays
        alive (pinned for an overlapped copy) until the stream passes the load; the NaN/rank
        checks surface on the next synchronous call."""
        if isinstance(X, np.ndarray):
            if X.shape != (self.n, self.m) or not X.flags.f_contiguous or X.dtype != np.float64:
                raise ValueError("load_async needs a Fortran-ordered float64 (n, m) array")
            self._keep = X
            _check(lib().bnreg_load_async(self._h, _hptr(X), 0))
        else:
            _check(lib().bnreg_load_async(self._h, _dptr(X), 1))

    def sync(self):
        """bnreg_sync: wait for the handle's stream; raises a deferred load error."""
        _check(lib().bnreg_sync(self._h))

    def best_merge_async(self, nparts: int, masks_dev, bics_dev, out_mask_dev, out_bic_dev, row_bytes: int = 0):
        """bnreg_best_merge_async: G14 merge of nparts rows of m device (mask, BIC) entries
        (row q at byte offset q * row_bytes; 0 = dense rows)."""
        _check(lib().bnreg_best_merge_async(self._h, nparts, _dptr(masks_dev), _dptr(bics_dev), row_bytes,
                                            _dptr(out_mask_dev), _dptr(out_bic_dev)))

    def num_families(self) -> int:
        return lib().bnreg_num_families(self._h)

    def local_index(self, g: int) -> int:
        return lib().bnreg_local_index(self._h, g)

    def run(self, out_rss=None, out_bic=None, best=True):
        """bnreg_run: device tables (pointers / tensors, None = skip) -> (best_mask, best_bic) host."""
        bm = np.zeros(self.m, dtype=np.uint32)
        bb = np.zeros(self.m)
        _check(lib().bnreg_run(self._h, _dptr(out_rss), _dptr(out_bic),
                               _hptr(bm) if best else None, _hptr(bb) if best else None))
        return bm, bb

    def set_root_method(self, method: int):
        """bnreg_set_root_method: ROOT_TSQR (default) or ROOT_CHOLESKY (Gram + Cholesky) for later loads."""
        _check(lib().bnreg_set_root_method(self._h, method))

    def best_subsets(self, scores, stride: int, best_score, best_mask):
        """bnreg_best_subsets: for every (child, candidate set) the best score over the set's
        subsets and that subset (DEVICE pointers / tensors; asynchronous)."""
        _check(lib().bnreg_best_subsets(self._h, _dptr(scores), stride, _dptr(best_score), _dptr(best_mask)))

    def coefficients_batch(self, children, masks, count: int, beta):
        """bnreg_coefficients_batch: coefficients of children[f] on masks[f] for count families
        into beta (count x m) -- DEVICE pointers / tensors; asynchronous."""
        _check(lib().bnreg_coefficients_batch(self._h, _dptr(children), _dptr(masks), count, _dptr(beta)))

    def coefficients(self, masks=None) -> np.ndarray:
        """bnreg_coefficients: least-squares coefficients of each child on masks[child] (None:
        the last run's per-child best sets) -> m x m array, beta[v, u] for parent u of child v."""
        beta = np.zeros((self.m, self.m))
        mk = None if masks is None else np.ascontiguousarray(masks, dtype=np.uint32)
        _check(lib().bnreg_coefficients(self._h, _hptr(mk) if mk is not None else None, _hptr(beta)))
        return beta

    def set_score(self, score: int):
        """bnreg_set_score: SCORE_BIC (default), SCORE_AIC or SCORE_LOGLIK for later runs."""
        _check(lib().bnreg_set_score(self._h, score))

    def run_pairs(self, out_pairs, best=True):
        """bnreg_run_pairs: one device table of (RSS, BIC) 16 B records -> (best_mask, best_bic) host."""
        bm = np.zeros(self.m, dtype=np.uint32)
        bb = np.zeros(self.m)
        _check(lib().bnreg_run_pairs(self._h, _dptr(out_pairs), _hptr(bm) if best else None,
                                     _hptr(bb) if best else None))
        return bm, bb

    def run_pairs_async(self, out_pairs, best_mask_dev=None, best_bic_dev=None):
        _check(lib().bnreg_run_pairs_async(self._h, _dptr(out_pairs), _dptr(best_mask_dev), _dptr(best_bic_dev)))

    def run_async(self, out_rss=None, out_bic=None, best_mask_dev=None, best_bic_dev=None):
        _check(lib().bnreg_run_async(self._h, _dptr(out_rss), _dptr(out_bic), _dptr(best_mask_dev),
                                     _dptr(best_bic_dev)))

    def all_rss(self, out):
        _check(lib().bnreg_all_rss(self._h, _dptr(out)))

    def bic(self, out):
        _check(lib().bnreg_bic(self._h, _dptr(out)))

    def set_stream(self, stream_handle: int | None):
        _check(lib().bnreg_set_stream(self._h, stream_handle))

    def set_load_stream(self, stream_handle: int | None):
        """bnreg_set_load_stream: prepare the next dataset (load + seed tree) on this stream
        while the current one is walked (None: loads on the handle's stream)."""
        _check(lib().bnreg_set_load_stream(self._h, stream_handle))

    def root_r(self):
        R = np.zeros((self.m, self.m))
        order = np.zeros(self.m, dtype=np.int32)
        _check(lib().bnreg_root_r(self._h, _hptr(R), _hptr(order)))
        return R, order

    @classmethod
    def create_dist(cls, X, n: int, m: int, nccl_id: bytes, rank: int, world: int):
        """bnreg_create_dist (collective): a rank of a world-rank job with the library's own
        NCCL communicator; X = rank 0's host data (None on the other ranks)."""
        self = cls.__new__(cls)
        self.n, self.m, self._keep = int(n), int(m), None
        self.opt = options(world=world, rank=rank)
        h = ctypes.c_void_p()
        Xp = None
        if X is not None:
            X = np.asfortranarray(X, dtype=np.float64)
            if X.shape != (n, m):
                raise ValueError("shape mismatch")
            Xp = _hptr(X)
        idb = ctypes.create_string_buffer(bytes(nccl_id), 128)
        _check(lib().bnreg_create_dist(Xp, n, m, idb, rank, world, ctypes.byref(h)))
        self._h = h
        return self

    def load_dist(self, X=None):
        """bnreg_load_dist (collective): new host data on rank 0 (None elsewhere)."""
        Xp = None
        if X is not None:
            X = np.asfortranarray(X, dtype=np.float64)
            Xp = _hptr(X)
        _check(lib().bnreg_load_dist(self._h, Xp))

    def run_pairs_dist(self, out_pairs):
        """bnreg_run_pairs_dist (collective): this rank's shard into out_pairs, returns the
        GLOBAL per-child best (mask, BIC) merged over the ranks."""
        bm = np.zeros(self.m, dtype=np.uint32)
        bb = np.zeros(self.m)
        _check(lib().bnreg_run_pairs_dist(self._h, _dptr(out_pairs), _hptr(bm), _hptr(bb)))
        return bm, bb

    def get_root_device(self, R_dev):
        """Copy the root R (m*m doubles) into a device buffer (for the broadcast)."""
        _check(lib().bnreg_get_root_device(self._h, _dptr(R_dev)))

    def set_root_device(self, R_dev):
        """Install a broadcast root R from a device buffer (instead of load)."""
        _check(lib().bnreg_set_root_device(self._h, _dptr(R_dev)))

    def shard_ranges(self):
        cnt = ctypes.c_int64(0)
        starts = np.zeros(2 * self.m, dtype=np.int64)
        lens = np.zeros(2 * self.m, dtype=np.int64)
        _check(lib().bnreg_shard_ranges(self._h, ctypes.byref(cnt), _hptr(starts), _hptr(lens)))
        c = cnt.value
        return starts[:c].copy(), lens[:c].copy()

    def launches_per_run(self) -> int:
        return lib().bnreg_launches_per_run(self._h)

    def timing(self, enable: int = -1):
        """bnreg_timing -> (ms[6]: run, seeds, walk, reduce, load total, load count; runs)."""
        ms = np.zeros(6)
        runs = ctypes.c_int64(0)
        _check(lib().bnreg_timing(self._h, enable, _hptr(ms), ctypes.byref(runs)))
        return ms, runs.value

    def debug_ln(self, x_dev, out_dev, count: int):
        """Test hook: the BIC epilogue's fp64 log on device buffers."""
        _check(lib().bnreg_debug_ln(self._h, _dptr(x_dev), _dptr(out_dev), count))

    def debug_write_counts(self, counts_dev):
        """K8 test hook (libbnreg_k8.so only): count every table store of later runs into
        counts_dev (zeroed device uint32[num_families]); None stops counting."""
        _check(lib().bnreg_debug_write_counts(self._h, _dptr(counts_dev)))

    def close(self):
        if getattr(self, "_h", None):
            lib().bnreg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
