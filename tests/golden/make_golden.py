"""Generate the golden vectors under tests/golden/ from the REFERENCE itself.

Run in the build container (needs /root/reference): it builds
oracle/_ref/libscout_ref.so (the unmodified reference headers behind
oracle/ref_shim.cpp) and records, for seeded inputs, what the reference's
select_topk / digest_score / build_digest / partial_attention / merge /
finalize return. The inputs are stored exactly (bf16 bit patterns, f32), the
outputs in float64. The GPU box never runs this; tests read the .npz files.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT / "oracle"))
import py_oracle as P  # noqa: E402

OUT = Path(__file__).resolve().parent
D, B = 128, 64


def bf16(x: np.ndarray) -> np.ndarray:
    """Round to bf16; return the uint16 bit patterns."""
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16)
    return t.view(torch.int16).numpy().view(np.uint16)


def from_bf16(bits: np.ndarray) -> np.ndarray:
    return torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16).float().numpy()


def topk_cases(ref):
    rng = np.random.default_rng(2603)
    specs = [  # (G, n_tokens, k, kind)
        (1, 64 * 20, 5, "iid"), (4, 64 * 64, 32, "iid"), (8, 64 * 100 + 17, 64, "iid"),
        (8, 64 * 130, 64, "clustered"), (4, 64 * 40, 8, "tie"), (8, 64 * 33 + 1, 16, "tie"),
        (2, 64 * 7, 64, "iid"), (8, 64 * 1, 3, "iid"), (1, 64 * 24, 7, "tie"), (8, 64 * 520, 128, "iid"),
        (8, 64 * 96, 20, "perm"), (4, 64 * 64 + 9, 32, "perm"),
    ]
    cases = {}
    for i, (G, nt, k, kind) in enumerate(specs):
        nb = (nt + B - 1) // B
        nbs = ((nb + 7) // 8) * 8
        if kind == "tie":
            q = rng.integers(-1, 2, size=(G, D)).astype(np.float32)
            a = rng.integers(-2, 3, size=(D, nbs)).astype(np.float32)
            b = rng.integers(-2, 3, size=(D, nbs)).astype(np.float32)
            lo, hi = np.minimum(a, b), np.maximum(a, b)
        elif kind == "perm":  # channel permutations of 3 bases, q constant per head: ulp-level near-ties
            q = np.repeat(rng.standard_normal((G, 1)), D, axis=1).astype(np.float32)
            base = (rng.standard_normal((3, 2, D)) * 2.0 ** rng.integers(-20, 21, size=(3, 2, D))).astype(np.float32)
            lo = np.empty((D, nbs), np.float32)
            hi = np.empty((D, nbs), np.float32)
            for j in range(nbs):
                p_ = rng.permutation(D)
                w = rng.integers(0, 3)
                a_, b_ = base[w, 0, p_], base[w, 1, p_]
                lo[:, j], hi[:, j] = np.minimum(a_, b_), np.maximum(a_, b_)
        elif kind == "clustered":
            q = rng.standard_normal((G, D)).astype(np.float32)
            mu = rng.standard_normal((D, nbs)).astype(np.float32) * 0.7
            lo = mu - np.abs(rng.standard_normal((D, nbs))).astype(np.float32) * 0.5
            hi = mu + np.abs(rng.standard_normal((D, nbs))).astype(np.float32) * 0.5
        else:
            q = rng.standard_normal((G, D)).astype(np.float32)
            a = rng.standard_normal((D, nbs)).astype(np.float32)
            b = rng.standard_normal((D, nbs)).astype(np.float32)
            lo, hi = np.minimum(a, b), np.maximum(a, b)
        lo_b, hi_b = bf16(lo), bf16(hi)
        dig = np.stack([from_bf16(lo_b), from_bf16(hi_b)]).astype(np.float64)
        ids, scores = P.unit_topk(q.astype(np.float64), dig, nb, k, lib=ref)
        cases[f"topk{i}"] = dict(G=G, n_tokens=nt, k=k, q=q, lo=lo_b, hi=hi_b, ids=ids.astype(np.int32),
                                 scores=scores)
    return cases


def attention_cases(ref):
    rng = np.random.default_rng(27138)
    cases = {}
    for i, rows in enumerate([[64], [64, 64, 17], [1], [64] * 9 + [33], [5, 64, 64, 64]]):
        n = sum(rows)
        q = rng.standard_normal(D).astype(np.float32)
        k = bf16(rng.standard_normal((n, D)) * (1.0 + i))
        v = bf16(rng.standard_normal((n, D)))
        kd, vd = from_bf16(k).astype(np.float64), from_bf16(v).astype(np.float64)
        scale = 1.0 / np.sqrt(D)
        p = P.partial_attention(q.astype(np.float64), kd, vd, scale, lib=ref, rows=rows)
        # a second, disjoint partial (the "CPU side") and the merge + finalize
        q2 = rng.standard_normal(D).astype(np.float32)
        k2 = bf16(rng.standard_normal((40, D)))
        v2 = bf16(rng.standard_normal((40, D)))
        p2 = P.partial_attention(q2.astype(np.float64), from_bf16(k2), from_bf16(v2), scale, lib=ref, rows=[40])
        m = P.merge(p, p2, lib=ref)
        cases[f"attn{i}"] = dict(rows=np.array(rows, np.int32), q=q, k=k, v=v, scale=scale, o_acc=p.o_acc,
                                 max_logit=p.max_logit, denom=p.denom, count=p.count, q2=q2, k2=k2, v2=v2,
                                 o2_acc=p2.o_acc, m2=p2.max_logit, l2=p2.denom, merged_o=m.o_acc,
                                 merged_m=m.max_logit, merged_l=m.denom, final=P.finalize(m, lib=ref))
    return cases


def digest_cases(ref):
    rng = np.random.default_rng(34)
    cases = {}
    for i, rows in enumerate([1, 17, 64]):
        k = bf16(rng.standard_normal((rows, D)))
        kd = from_bf16(k).astype(np.float64)
        lo, hi = P.build_digest(kd, 0, lib=ref)
        mean = P.build_digest(kd, 1, lib=ref)
        cases[f"digest{i}"] = dict(k=k, lo=lo, hi=hi, mean=mean)
    return cases


def main():
    ref = P.ref()
    if ref is None:
        raise SystemExit("reference not available (needs /root/reference)")
    for name, cases in (("topk", topk_cases(ref)), ("attention", attention_cases(ref)),
                        ("digest", digest_cases(ref))):
        flat = {f"{c}__{k}": np.asarray(v) for c, d in cases.items() for k, v in d.items()}
        np.savez_compressed(OUT / f"golden_{name}.npz", **flat)
        print(name, len(cases), "cases")


if __name__ == "__main__":
    main()
