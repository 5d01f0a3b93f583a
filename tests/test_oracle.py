"""The CPU oracle, pinned: golden vectors from the reference itself, the
reference tests' known answers, and (where the reference was built) randomized
cross-checks against the reference headers. No GPU needed."""
import numpy as np
import pytest

import py_oracle as P
from helpers import D, from_bf16, load_golden


# ------------------------------------------------------------- golden ----
@pytest.mark.parametrize("case", sorted(load_golden("topk")))
def test_oracle_topk_matches_reference_golden(case):
    c = load_golden("topk")[case]
    nb = (int(c["n_tokens"]) + 63) // 64
    dig = np.stack([from_bf16(c["lo"]), from_bf16(c["hi"])]).astype(np.float64)
    ids, scores = P.unit_topk(c["q"].astype(np.float64), dig, nb, int(c["k"]))
    assert np.array_equal(ids, c["ids"])
    assert np.array_equal(scores.view(np.uint64), c["scores"].view(np.uint64))  # bit-exact


@pytest.mark.parametrize("case", sorted(load_golden("attention")))
def test_oracle_attention_matches_reference_golden(case):
    c = load_golden("attention")[case]
    k, v = from_bf16(c["k"]), from_bf16(c["v"])
    p = P.partial_attention(c["q"].astype(np.float64), k, v, float(c["scale"]))
    assert p.count == int(c["count"])
    assert p.max_logit == float(c["max_logit"])
    np.testing.assert_allclose(p.denom, c["denom"], rtol=1e-13)
    np.testing.assert_allclose(p.o_acc, c["o_acc"], rtol=1e-12, atol=1e-13)
    p2 = P.partial_attention(c["q2"].astype(np.float64), from_bf16(c["k2"]), from_bf16(c["v2"]), float(c["scale"]))
    m = P.merge(p, p2)
    np.testing.assert_allclose(m.o_acc, c["merged_o"], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(P.finalize(m), c["final"], rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("case", sorted(load_golden("digest")))
def test_oracle_digest_matches_reference_golden(case):
    c = load_golden("digest")[case]
    k = from_bf16(c["k"]).astype(np.float64)
    lo, hi = P.build_digest(k, 0)
    assert np.array_equal(lo, c["lo"]) and np.array_equal(hi, c["hi"])
    assert np.array_equal(P.build_digest(k, 1), c["mean"])


# ------------------------------------------- reference known answers ----
def test_kat_minmax_digest():  # test_digest.cpp:35-44
    lo, hi = P.build_digest([[0.0, 1.0], [3.0, -2.0], [1.0, 0.5]], 0)
    assert list(lo) == [0.0, -2.0] and list(hi) == [3.0, 1.0]
    with pytest.raises(ValueError):
        P.build_digest(np.zeros((0, 2)), 0)


def test_kat_minmax_score():  # test_digest.cpp:46-55
    assert P.oracle().oracle_digest_score_minmax(P.f64([1, -1]), P.f64([0, -2]), P.f64([3, 1]), 2) == 5.0


def test_kat_mean_digest():  # test_digest.cpp:57-62
    mean = P.build_digest([[2.0, 4.0], [0.0, -2.0]], 1)
    assert list(mean) == [1.0, 1.0]
    assert P.oracle().oracle_digest_score_mean(P.f64([0.5, 2.0]), mean, 2) == 2.5


def test_kat_select_topk():  # test_digest.cpp:84-105
    assert list(P.select_topk_scores([5.0, 1.0, 3.0], 2)) == [0, 2]
    assert list(P.select_topk_scores([5.0, 1.0, 3.0], 10)) == [0, 1, 2]
    assert list(P.select_topk_scores([2.0, 2.0, 1.0], 1)) == [0]
    assert list(P.select_topk_scores([2.0, 2.0, 1.0], 2)) == [0, 1]
    with pytest.raises(ValueError):
        P.select_topk_scores([1.0], 0)


def test_kat_sub_kth_invariance():  # test_digest.cpp:129-139
    s = [10.0 - i for i in range(5)]
    before = P.select_topk_scores(s, 3)
    s[4] = 1.0
    assert np.array_equal(P.select_topk_scores(s, 3), before)


def test_merge_empty_identity_and_finalize_empty():  # test_attention.cpp:130-154
    rng = np.random.default_rng(43)
    p = P.partial_attention(rng.standard_normal(3), rng.standard_normal((4, 3)), rng.standard_normal((4, 3)), 1.0)
    e = P.Partial.empty(3)
    for m in (P.merge(p, e), P.merge(e, p)):
        assert np.array_equal(m.o_acc, p.o_acc) and m.denom == p.denom and m.max_logit == p.max_logit
    both = P.merge(e, P.Partial.empty(3))
    assert both.count == 0
    with pytest.raises(ValueError):
        P.finalize(both)
    assert P.partial_attention([1.0, 2.0], np.zeros((0, 2)), np.zeros((0, 2)), 1.0).count == 0


def test_partition_invariance():  # acceptance.cpp:99-137 (criterion 1)
    rng = np.random.default_rng(101)
    worst = 0.0
    for _ in range(25):
        rows = rng.integers(1, 10, size=6)
        keys = [rng.standard_normal((r, 8)) for r in rows]
        vals = [rng.standard_normal((r, 8)) for r in rows]
        q = rng.standard_normal(8)
        whole = P.finalize(P.partial_attention(q, np.vstack(keys), np.vstack(vals), 0.5))
        for _ in range(8):
            side = rng.integers(0, 2, size=6).astype(bool)
            parts = []
            for sel in (side, ~side):
                idx = np.nonzero(sel)[0]
                kk = np.vstack([keys[i] for i in idx]) if len(idx) else np.zeros((0, 8))
                vv = np.vstack([vals[i] for i in idx]) if len(idx) else np.zeros((0, 8))
                parts.append(P.partial_attention(q, kk, vv, 0.5))
            worst = max(worst, np.abs(P.finalize(P.merge(*parts)) - whole).max())
    assert worst <= 1e-10


# ---------------------------------------- randomized vs the reference ----
@pytest.mark.skipif(P.ref() is None, reason="reference not built here")
def test_topk_brute_force_vs_reference_ties_included():  # test_digest.cpp:107-127, acceptance crit 3
    rng = np.random.default_rng(23)
    ref = P.ref()
    for trial in range(300):
        tie = trial % 2 == 0
        nb = int(rng.integers(1, 40))
        G = int(rng.choice([1, 2, 4, 8]))
        q = rng.integers(-1, 2, size=(G, D)).astype(np.float64) if tie else rng.standard_normal((G, D))
        a = rng.integers(-2, 3, size=(D, 40)) if tie else rng.standard_normal((D, 40))
        b = rng.integers(-2, 3, size=(D, 40)) if tie else rng.standard_normal((D, 40))
        dig = np.stack([np.minimum(a, b), np.maximum(a, b)]).astype(np.float64)
        k = int(rng.integers(1, nb + 3))
        ids_o, sc_o = P.unit_topk(q, dig, nb, k)
        ids_r, sc_r = P.unit_topk(q, dig, nb, k, lib=ref)
        assert np.array_equal(ids_o, ids_r)
        assert np.array_equal(sc_o, sc_r)
