"""Shared test helpers: golden fixtures, bf16 round trips, synthetic unit builders."""
from __future__ import annotations

from pathlib import Path

import numpy as np
import torch

GOLDEN = Path(__file__).resolve().parent / "golden"
D, B = 128, 64


def load_golden(name: str) -> dict[str, dict[str, np.ndarray]]:
    z = np.load(GOLDEN / f"golden_{name}.npz")
    out: dict[str, dict[str, np.ndarray]] = {}
    for key in z.files:
        case, field = key.split("__", 1)
        out.setdefault(case, {})[field] = z[key]
    return out


def from_bf16(bits: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).float().numpy()


def bf16_round(x: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16).float().numpy()


def nbs_for(nb: int) -> int:
    return max(8, ((nb + 7) // 8) * 8)


def make_digests(rng, U, nbs, kind="iid", dtype=np.float32):
    """lo/hi [U][2][D][nbs] (bf16-exact values as f32)."""
    if kind == "tie":
        a = rng.integers(-2, 3, size=(U, D, nbs)).astype(np.float32)
        b = rng.integers(-2, 3, size=(U, D, nbs)).astype(np.float32)
    elif kind == "perm":
        # near-ties at the ulp level: every block is a channel permutation of
        # one of 3 base digests (values spread over 2^+-20), so with q constant
        # over channels the real sums are equal and only the reference's
        # sequential rounding orders them
        base = (rng.standard_normal((U, 3, 2, D)) * 2.0 ** rng.integers(-20, 21, size=(U, 3, 2, D))).astype(np.float32)
        a = np.empty((U, D, nbs), np.float32)
        b = np.empty((U, D, nbs), np.float32)
        for u in range(U):
            for j in range(nbs):
                perm = rng.permutation(D)
                w = rng.integers(0, 3)
                a[u, :, j], b[u, :, j] = base[u, w, 0, perm], base[u, w, 1, perm]
    elif kind == "ulp":
        # one base digest per unit; every block moves 1-3 channels by one bf16
        # ulp, so scores differ by ~2^-18 of sum |terms|: inside K1's fp32 band
        base = bf16_round(rng.standard_normal((U, 2, D)).astype(np.float32))
        a = np.repeat(base[:, 0, :, None], nbs, axis=2).copy()
        b = np.repeat(base[:, 1, :, None], nbs, axis=2).copy()
        for u in range(U):
            for j in range(nbs):
                for c in rng.integers(0, D, size=rng.integers(1, 4)):
                    for arr in (a, b):
                        bits = int(np.array([arr[u, c, j]], np.float32).view(np.uint32)[0])
                        bits = (bits + int(rng.choice([1, -1])) * 65536) & 0xFFFFFFFF
                        arr[u, c, j] = np.array([bits], np.uint32).view(np.float32)[0]
    elif kind == "huge":  # products overflow fp32 (K1 falls back to the exact path)
        a = (rng.standard_normal((U, D, nbs)) * 1e36).astype(np.float32)
        b = (rng.standard_normal((U, D, nbs)) * 1e36).astype(np.float32)
    else:
        a = rng.standard_normal((U, D, nbs)).astype(np.float32)
        b = rng.standard_normal((U, D, nbs)).astype(np.float32)
    lo, hi = np.minimum(a, b), np.maximum(a, b)
    return bf16_round(np.stack([lo, hi], axis=1))


def make_queries(rng, U, G, kind="iid"):
    if kind == "tie":
        return rng.integers(-1, 2, size=(U * G, D)).astype(np.float32)
    if kind == "perm":  # constant over channels (per head) so channel permutations keep the term multiset
        return np.repeat(rng.standard_normal((U * G, 1)), D, axis=1).astype(np.float32)
    if kind == "tinyq":  # query sums below the f32 normal range (K1's relative bound does not hold)
        return (rng.standard_normal((U * G, D)) * 1e-39).astype(np.float32)
    if kind == "huge":
        return (rng.standard_normal((U * G, D)) * 1e4).astype(np.float32)
    return rng.standard_normal((U * G, D)).astype(np.float32)
