"""numpy wrappers over the CPU checkers (TEST / BASELINE INFRASTRUCTURE ONLY).

  oracle()  -> oracle/_build/liboracle.so   C restatement (scout_oracle.c)
  ref()     -> oracle/_ref/libscout_ref.so   the unmodified reference headers
               behind ref_shim.cpp (None when not built / not shipped)

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "_build" / "liboracle.so"
REF_SO = HERE / "_ref" / "libscout_ref.so"
D = 128
B = 64

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_lp = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_c = {}


def _build():
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True, stdout=subprocess.DEVNULL)


def oracle() -> C.CDLL:
    if "o" not in _c:
        if not ORACLE_SO.exists():
            _build()
        L = C.CDLL(str(ORACLE_SO))
        dbl = C.c_double
        L.oracle_build_digest_minmax.argtypes = [_dp, C.c_int, C.c_int, _dp, _dp]
        L.oracle_build_digest_mean.argtypes = [_dp, C.c_int, C.c_int, _dp]
        L.oracle_digest_score_minmax.argtypes = [_dp, _dp, _dp, C.c_int]
        L.oracle_digest_score_minmax.restype = dbl
        L.oracle_digest_score_mean.argtypes = [_dp, _dp, C.c_int]
        L.oracle_digest_score_mean.restype = dbl
        L.oracle_select_topk.argtypes = [_dp, C.c_void_p, C.c_int, C.c_int, _lp]
        L.oracle_score_topk_split.argtypes = [C.c_int] * 6 + [_dp, _dp, _ip, C.c_void_p] + [_ip] * 7 + [C.c_void_p]
        L.oracle_partial_attention.argtypes = [_dp, C.c_int, _dp, _dp, C.c_int, dbl, _dp, C.POINTER(dbl),
                                               C.POINTER(dbl), C.POINTER(C.c_int64)]
        L.oracle_merge.argtypes = [C.c_int, _dp, dbl, dbl, C.c_int64, _dp, dbl, dbl, C.c_int64, _dp,
                                   C.POINTER(dbl), C.POINTER(dbl), C.POINTER(C.c_int64)]
        L.oracle_finalize.argtypes = [C.c_int, _dp, dbl, C.c_int64, _dp]
        _c["o"] = L
    return _c["o"]


def ref():
    if "r" not in _c:
        L = None
        if not REF_SO.exists() and Path("/root/reference/proj/include/scout").exists():
            _build()
        if REF_SO.exists():
            L = C.CDLL(str(REF_SO))
            dbl = C.c_double
            L.ref_build_digest.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _dp, _dp]
            L.ref_digest_score.argtypes = [_dp, _dp, _dp, C.c_int, C.c_int]
            L.ref_digest_score.restype = dbl
            L.ref_unit_topk.argtypes = [_dp, C.c_int, C.c_int, _dp, C.c_int, C.c_int, C.c_int, C.c_int, _ip,
                                        C.c_void_p]
            L.ref_select_topk.argtypes = [_dp, C.c_int, _dp, _dp, C.c_int, C.c_int, C.c_int, _ip]
            L.ref_partial_attention.argtypes = [_dp, C.c_int, _dp, _dp, _ip, C.c_int, dbl, _dp, C.POINTER(dbl),
                                                C.POINTER(dbl), C.POINTER(C.c_int64)]
            L.ref_merge.argtypes = [C.c_int, _dp, dbl, dbl, C.c_int64, _dp, dbl, dbl, C.c_int64, _dp,
                                    C.POINTER(dbl), C.POINTER(dbl), C.POINTER(C.c_int64)]
            L.ref_finalize.argtypes = [C.c_int, _dp, dbl, C.c_int64, _dp]
            L.ref_cpu_baseline.argtypes = [C.c_int] * 6 + [_dp, _dp, _ip, _dp, _ip, C.c_int, C.c_int, C.c_int,
                                                           C.POINTER(dbl)]
            L.ref_cpu_baseline.restype = dbl
            ll, vp = C.c_longlong, C.c_void_p
            L.ref_cache_new.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, ll]
            L.ref_cache_new.restype = vp
            L.ref_cache_free.argtypes = [vp]
            L.ref_cache_pin.argtypes = [vp, C.c_int]
            L.ref_cache_append.argtypes = [vp, C.c_int, _dp, _dp, C.c_int]
            L.ref_cache_append.restype = ll
            L.ref_cache_begin_layer.argtypes = [vp, ll, C.c_int]
            L.ref_cache_schedule_recall.argtypes = [vp, C.c_int, _ip, C.c_int, ll, C.c_int]
            L.ref_cache_mark_selected.argtypes = [vp, C.c_int, _ip, C.c_int, ll]
            L.ref_cache_residency.argtypes = [vp, C.c_int, _ip]
            L.ref_cache_state.argtypes = [vp, C.c_int, _ip, _lp, _ip]
            L.ref_cache_place.argtypes = [vp, C.c_int, _dp, C.c_int]
            L.ref_cache_digests.argtypes = [vp, C.c_int, C.c_int, C.c_int, _dp]
            L.ref_predict_query.argtypes = [_dp, C.c_int, _dp, C.c_int, _dp]
            if hasattr(L, "ref_recompute_layer_attention"):
                L.ref_recompute_layer_attention.argtypes = [C.c_int, C.c_int, _dp, _dp, C.c_int, C.c_int, C.c_int, _dp,
                                                            _dp, _ip, C.c_int, _ip, C.c_int, dbl, _dp]
            L.ref_recall_new.argtypes = [C.c_int, C.c_int, _ip, dbl]
            L.ref_recall_new.restype = vp
            L.ref_recall_free.argtypes = [vp]
            L.ref_maybe_schedule_recall.argtypes = [vp, C.c_int, C.c_int, ll, _ip, C.c_int, _ip, C.c_int, _ip]
            if hasattr(L, "ref_calibrate_intervals"):
                L.ref_calibrate_intervals.argtypes = [_lp, _lp, C.c_int, C.c_int, dbl, _ip]
        _c["r"] = L
    return _c["r"]


def f64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


# ------------------------------------------------------------------ oracle --
class Partial:
    """PartialAttention (attention.hpp:22-35)."""

    def __init__(self, o_acc, max_logit, denom, count):
        self.o_acc, self.max_logit, self.denom, self.count = o_acc, max_logit, denom, count

    @staticmethod
    def empty(d=D):
        return Partial(np.zeros(d), -np.inf, 0.0, 0)

    def finalize(self, lib=None):
        return finalize(self, lib)


def build_digest(keys, method=0, lib=None):
    keys = f64(keys)
    rows, d = keys.shape
    if lib is not None and lib is ref():
        lo, hi = np.zeros(d), np.zeros(d)
        if lib.ref_build_digest(keys, rows, d, method, lo, hi) != 0:
            raise ValueError("build_digest: empty block")
        return (lo, hi) if method == 0 else lo
    L = oracle()
    if rows == 0:
        raise ValueError("build_digest: empty block")
    if method == 0:
        lo, hi = np.zeros(d), np.zeros(d)
        L.oracle_build_digest_minmax(keys, rows, d, lo, hi)
        return lo, hi
    mean = np.zeros(d)
    L.oracle_build_digest_mean(keys, rows, d, mean)
    return mean


def select_topk_scores(scores, k):
    """select_topk given the scores (ids = positions)."""
    scores = f64(scores)
    out = np.zeros(max(k, 1), dtype=np.int64)
    m = oracle().oracle_select_topk(scores, None, len(scores), int(k), out)
    if m < 0:
        raise ValueError("select_topk: k must be >= 1")
    return out[:m].astype(np.int32)


def unit_topk(q, dig, nb, k, method=0, lib=None):
    """Stacked-GQA select_topk of one unit: q [G][d], dig [2|1][d][nb_stride]. Returns (ids, scores)."""
    q = f64(q)
    G = q.shape[0]
    dig = f64(dig)
    nbs = dig.shape[-1]
    if lib is not None and lib is ref():
        out = np.zeros(max(k, 1), dtype=np.int32)
        sc = np.zeros(max(nb, 1))
        m = lib.ref_unit_topk(q, G, D, dig.reshape(-1), nbs, nb, int(k), method, out,
                              sc.ctypes.data_as(C.c_void_p))
        if m < 0:
            raise ValueError("select_topk: k must be >= 1")
        return out[:m], sc[:nb]
    r = score_topk_split(q, dig[None], np.array([nb * B], dtype=np.int32), k, G, method=method)
    return r["sel_ids"][0, :r["n_sel"][0]], r["scores"][0, :nb]


def score_topk_split(q, digests, n_tokens, k, G, table=None, method=0, k_stride=None):
    """Batched K1 statement. q [U*G][d]; digests [U][2|1][d][nbs]; table [U][nbs] or None."""
    q = f64(q)
    digests = f64(digests)
    n_tokens = np.ascontiguousarray(n_tokens, dtype=np.int32)
    U = len(n_tokens)
    nbs = digests.shape[-1]
    ks = k_stride or max(k, 1)
    z = lambda *s: np.full(s, -7, dtype=np.int32)  # noqa: E731
    sel, nsel, rid, rsl, nres, cid, ncpu = z(U, ks), z(U), z(U, ks), z(U, ks), z(U), z(U, ks), z(U)
    scores = np.zeros((U, nbs))
    tb = None if table is None else np.ascontiguousarray(table, dtype=np.int32)
    rc = oracle().oracle_score_topk_split(U, G, method, int(k), ks, nbs, q.reshape(-1), digests.reshape(-1),
                                          n_tokens, None if tb is None else tb.ctypes.data_as(C.c_void_p),
                                          sel, nsel, rid, rsl, nres, cid, ncpu,
                                          scores.ctypes.data_as(C.c_void_p))
    if rc < 0:
        raise ValueError("select_topk: k must be >= 1")
    return dict(sel_ids=sel, n_sel=nsel, res_ids=rid, res_slots=rsl, n_res=nres, cpu_ids=cid, n_cpu=ncpu,
                scores=scores)


def partial_attention(q, keys, values, scale, lib=None, rows=None):
    """partial_attention over rows (blocks concatenated in visiting order)."""
    q, keys, values = f64(q), f64(keys).reshape(-1, len(q)), f64(values).reshape(-1, len(q))
    d = len(q)
    if not (scale > 0):
        raise ValueError("partial_attention: scale must be > 0")
    o = np.zeros(d)
    m, l, n = C.c_double(), C.c_double(), C.c_int64()
    if lib is not None and lib is ref():
        r = np.ascontiguousarray(rows if rows is not None else [keys.shape[0]], dtype=np.int32)
        lib.ref_partial_attention(q, d, keys, values, r, len(r), float(scale), o, C.byref(m), C.byref(l), C.byref(n))
    else:
        oracle().oracle_partial_attention(q, d, keys, values, keys.shape[0], float(scale), o, C.byref(m), C.byref(l),
                                          C.byref(n))
    return Partial(o, m.value, l.value, n.value)


def merge(a: Partial, b: Partial, lib=None) -> Partial:
    d = len(a.o_acc)
    o = np.zeros(d)
    m, l, n = C.c_double(), C.c_double(), C.c_int64()
    fn = lib.ref_merge if (lib is not None and lib is ref()) else oracle().oracle_merge
    fn(d, f64(a.o_acc), a.max_logit, a.denom, a.count, f64(b.o_acc), b.max_logit, b.denom, b.count, o, C.byref(m),
       C.byref(l), C.byref(n))
    return Partial(o, m.value, l.value, n.value)


def finalize(p: Partial, lib=None):
    d = len(p.o_acc)
    out = np.zeros(d)
    fn = lib.ref_finalize if (lib is not None and lib is ref()) else oracle().oracle_finalize
    if fn(d, f64(p.o_acc), p.denom, p.count, out) != 0:
        raise ValueError("finalize: empty partial")
    return out


class RefCache:
    """The reference TieredKvCache (kv_store.hpp) behind oracle/_ref (checker only)."""

    def __init__(self, layers, head_dim, capacity, block_size=64, method=0):
        self.L = ref()
        if self.L is None:
            raise RuntimeError("oracle/_ref/libscout_ref.so not built")
        self.h = self.L.ref_cache_new(layers, block_size, head_dim, method, capacity)
        self.d = head_dim

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_cache_free(self.h)

    def pin_layer(self, layer):
        self.L.ref_cache_pin(self.h, layer)

    def append_token(self, layer, k, v):
        r = self.L.ref_cache_append(self.h, layer, f64(k), f64(v), self.d)
        if r == -2:
            raise ValueError("append_token")
        return None if r < 0 else int(r)

    def begin_layer(self, step, layer):
        return self.L.ref_cache_begin_layer(self.h, step, layer)

    def schedule_recall(self, layer, ids, issue_step, issue_layer):
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        if self.L.ref_cache_schedule_recall(self.h, layer, ids, len(ids), issue_step, issue_layer) != 0:
            raise ValueError("schedule_recall")

    def mark_selected(self, layer, ids, step):
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        if self.L.ref_cache_mark_selected(self.h, layer, ids, len(ids), step) != 0:
            raise ValueError("mark_selected")

    def residency_set(self, layer, max_blocks=8192):
        out = np.zeros(max_blocks, np.int32)
        n = self.L.ref_cache_residency(self.h, layer, out)
        return out[:n]

    def state(self, layer, max_blocks=8192):
        t, ls, fl = np.zeros(max_blocks, np.int32), np.zeros(max_blocks, np.int64), np.zeros(max_blocks, np.int32)
        n = self.L.ref_cache_state(self.h, layer, t, ls, fl)
        return t[:n], ls[:n], fl[:n]

    def place_after_prefill(self, layer, q):
        if self.L.ref_cache_place(self.h, layer, f64(q), self.d) != 0:
            raise ValueError("place_after_prefill")

    def digests(self, layer, nb_stride):
        out = np.zeros((2, self.d, nb_stride))
        n = self.L.ref_cache_digests(self.h, layer, self.d, nb_stride, out)
        return out, n


def recompute_layer_attention(keys, values, tokens_at_attention, q_true, q_pred, res_ids, cpu_ids, scale,
                              block_size=64):
    """The reference's hybrid-query oracle (harness.hpp:318-329) for G heads of
    one unit: keys/values [n_rows][d] = the layer's whole K/V stream,
    q_true/q_pred [G][d]. Returns [G][d] (checker only)."""
    L = ref()
    if L is None or not hasattr(L, "ref_recompute_layer_attention"):
        raise RuntimeError("oracle/_ref built without harness.hpp (json.hpp missing)")
    keys, values = f64(keys), f64(values)
    qt, qp = f64(np.atleast_2d(q_true)), f64(np.atleast_2d(q_pred))
    G, d = qt.shape
    r = np.ascontiguousarray(res_ids, dtype=np.int32)
    c = np.ascontiguousarray(cpu_ids, dtype=np.int32)
    out = np.zeros((G, d))
    if L.ref_recompute_layer_attention(d, block_size, keys, values, keys.shape[0], int(tokens_at_attention), G, qt, qp,
                                       r, len(r), c, len(c), float(scale), out) != 0:
        raise ValueError("recompute_layer_attention")
    return out


class RefRecall:
    """The reference recall policy (recall.hpp:69-126: RecallSchedule +
    maybe_schedule_recall) for n_units independent engines behind oracle/_ref
    (checker only)."""

    def __init__(self, n_units, intervals, beta=0.12):
        self.L = ref()
        if self.L is None:
            raise RuntimeError("oracle/_ref/libscout_ref.so not built")
        iv = np.ascontiguousarray(intervals, dtype=np.int32)
        self.h = self.L.ref_recall_new(n_units, len(iv), iv, beta)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_recall_free(self.h)

    def maybe_schedule_recall(self, unit, layer, step, predicted, residency):
        """None when the layer is not due, else set_difference(predicted, residency)."""
        p = np.ascontiguousarray(predicted, dtype=np.int32)
        r = np.ascontiguousarray(residency, dtype=np.int32)
        out = np.zeros(max(len(p), 1), np.int32)
        n = self.L.ref_maybe_schedule_recall(self.h, unit, layer, step, p, len(p), r, len(r), out)
        return None if n < 0 else out[:n]


def predict_query(x, w):
    """The reference's predict_next_query(rms_normalize(x), w) (checker only)."""
    x, w = f64(x), f64(w)
    out = np.zeros(w.shape[1])
    if ref().ref_predict_query(x, x.shape[0], w, w.shape[1], out) != 0:
        raise ValueError("predict_next_query")
    return out


def ref_calibrate_intervals(cpu, budget, beta):
    """The reference's calibrate_intervals (recall.hpp:79-95) over a RatioTrace
    of [layers][steps] samples; None if it threw."""
    L_ = ref()
    cpu = np.ascontiguousarray(cpu, dtype=np.int64)
    bud = np.ascontiguousarray(budget, dtype=np.int64)
    out = np.zeros(cpu.shape[0], dtype=np.int32)
    rc = L_.ref_calibrate_intervals(cpu, bud, cpu.shape[0], cpu.shape[1], float(beta), out)
    return None if rc != 0 else out.tolist()
