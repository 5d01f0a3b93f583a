"""K1 parity on the GPU: selected block sets bit-exact against the reference
(golden vectors) and the oracle (seeded iid / clustered / tie-prone inputs,
ragged open blocks, k >= blocks, one block), plus the resident/CPU split."""
import numpy as np
import pytest
import torch

import py_oracle as P
from helpers import D, bf16_round, from_bf16, load_golden, make_digests, make_queries, nbs_for
from paper_2603_27138_b200 import ops

pytestmark = pytest.mark.gpu


def _gpu_topk(q, dig, n_tokens, k, G, dtype=torch.bfloat16, table=None, want_scores=True, method=0, step=0,
              last_sel=None):
    dev = torch.device("cuda")
    qd = torch.as_tensor(q, device=dev)
    qd = qd.double() if dtype == torch.float64 else qd.float()
    dd = torch.as_tensor(dig, device=dev).to(dtype).contiguous()
    nt = torch.as_tensor(n_tokens, dtype=torch.int32, device=dev)
    tb = None if table is None else torch.as_tensor(table, dtype=torch.int32, device=dev)
    r = ops.score_topk_split(qd, dd, nt, k, G, block_table=tb, want_scores=want_scores, method=method, step=step,
                             last_selected=last_sel)
    torch.cuda.synchronize()
    return {k_: v.cpu().numpy() for k_, v in r.items()}


@pytest.mark.parametrize("case", sorted(load_golden("topk")))
def test_topk_bit_exact_vs_reference_golden(cuda, case):
    c = load_golden("topk")[case]
    G, nt, k = int(c["G"]), int(c["n_tokens"]), int(c["k"])
    nb = (nt + 63) // 64
    dig = np.stack([from_bf16(c["lo"]), from_bf16(c["hi"])])[None]  # [1][2][D][nbs]
    r = _gpu_topk(c["q"], dig, [nt], k, G)
    assert r["n_sel"][0] == len(c["ids"])
    assert np.array_equal(r["sel_ids"][0, : r["n_sel"][0]], c["ids"])
    assert np.array_equal(r["scores"][0, :nb].view(np.uint64), c["scores"].view(np.uint64))


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("kind", ["iid", "tie", "perm"])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_topk_split_vs_oracle(cuda, G, kind, dtype):
    rng = np.random.default_rng(hash((G, kind, str(dtype))) % 2**32)
    U = 24
    n_tokens = rng.integers(1, 64 * 300, size=U).astype(np.int32)
    n_tokens[0], n_tokens[1], n_tokens[2] = 64, 1, 64 * 300
    nbs = nbs_for(300)
    dig = make_digests(rng, U, nbs, kind)
    q = make_queries(rng, U, G, kind)
    table = np.where(rng.random((U, nbs)) < 0.8, rng.integers(0, 10**6, size=(U, nbs)), -1).astype(np.int32)
    for k in (1, 7, 64, 300, 400):
        want = P.score_topk_split(q, dig, n_tokens, k, G, table=table, k_stride=k)
        got = _gpu_topk(q, dig, n_tokens, k, G, dtype=dtype, table=table)
        for u in range(U):
            ns = want["n_sel"][u]
            assert got["n_sel"][u] == ns
            assert np.array_equal(got["sel_ids"][u, :ns], want["sel_ids"][u, :ns]), (u, k)
            nr, nc = want["n_res"][u], want["n_cpu"][u]
            assert got["n_res"][u] == nr and got["n_cpu"][u] == nc
            assert np.array_equal(got["res_ids"][u, :nr], want["res_ids"][u, :nr])
            assert np.array_equal(got["res_slots"][u, :nr], want["res_slots"][u, :nr])
            assert np.array_equal(got["cpu_ids"][u, :nc], want["cpu_ids"][u, :nc])
            nb = (n_tokens[u] + 63) // 64
            tail = n_tokens[u] - 64 * (nb - 1)
            rows = lambda ids: sum(tail if i == nb - 1 else 64 for i in ids)  # noqa: E731
            assert got["res_tokens"][u] == rows(want["res_ids"][u, :nr])
            assert got["cpu_tokens"][u] == rows(want["cpu_ids"][u, :nc])
            assert np.array_equal(got["scores"][u, :nb].view(np.uint64), want["scores"][u, :nb].view(np.uint64))


@pytest.mark.parametrize("G", [1, 8])
@pytest.mark.parametrize("kind", ["ulp", "tinyq", "huge"])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_topk_band_edges_vs_oracle(cuda, G, kind, dtype):
    """Inputs aimed at K1's fast-score band: ulp-level score gaps (exact path
    decides), f32-subnormal query sums and fp32 overflow (whole unit exact)."""
    rng = np.random.default_rng(hash(("edge", G, kind, str(dtype))) % 2**32)
    U, nbs = 12, nbs_for(200)
    n_tokens = np.full(U, 64 * 200 - 17, np.int32)
    dig = make_digests(rng, U, nbs, "ulp" if kind == "ulp" else ("huge" if kind == "huge" else "iid"))
    q = make_queries(rng, U, G, kind if kind != "ulp" else "iid")
    for k in (1, 16, 64):
        want = P.score_topk_split(q, dig, n_tokens, k, G, k_stride=k)
        got = _gpu_topk(q, dig, n_tokens, k, G, dtype=dtype)
        for u in range(U):
            ns = want["n_sel"][u]
            assert got["n_sel"][u] == ns
            assert np.array_equal(got["sel_ids"][u, :ns], want["sel_ids"][u, :ns]), (kind, u, k)


@pytest.mark.parametrize("G", [1, 4, 8])
@pytest.mark.parametrize("kind", ["iid", "perm"])
def test_topk_bf16_queries_vs_oracle(cuda, G, kind):
    """bf16 queries (the model's own dtype; q_dtype = SCOUT_BF16): the oracle
    sees the same bf16-rounded values, selection and scores stay bit-exact."""
    rng = np.random.default_rng(hash(("bf16q", G, kind)) % 2**32)
    U, nbs = 16, nbs_for(260)
    n_tokens = rng.integers(1, 64 * 260, size=U).astype(np.int32)
    dig = make_digests(rng, U, nbs, kind)
    q = bf16_round(make_queries(rng, U, G, kind))
    table = np.where(rng.random((U, nbs)) < 0.8, rng.integers(0, 10**6, size=(U, nbs)), -1).astype(np.int32)
    dev = torch.device("cuda")
    for k in (1, 33, 64):
        want = P.score_topk_split(q, dig, n_tokens, k, G, table=table, k_stride=k)
        r = ops.score_topk_split(torch.from_numpy(q).to(dev).bfloat16(), torch.from_numpy(dig).to(dev).bfloat16(),
                                 torch.from_numpy(n_tokens).to(dev), k, G,
                                 block_table=torch.from_numpy(table).to(dev), want_scores=True)
        got = {k_: v.cpu().numpy() for k_, v in r.items()}
        for u in range(U):
            ns, nr = want["n_sel"][u], want["n_res"][u]
            assert got["n_sel"][u] == ns and got["n_res"][u] == nr
            assert np.array_equal(got["sel_ids"][u, :ns], want["sel_ids"][u, :ns]), (u, k)
            assert np.array_equal(got["res_slots"][u, :nr], want["res_slots"][u, :nr])
            nb = (n_tokens[u] + 63) // 64
            assert np.array_equal(got["scores"][u, :nb].view(np.uint64), want["scores"][u, :nb].view(np.uint64))


@pytest.mark.parametrize("nb", [513, 520, 640, 700, 1000, 2048, 2600])
def test_topk_many_blocks_vs_oracle(cuda, nb):
    """Long contexts: running scores in registers (2 quads per thread <= 1024
    blocks, 4 <= 2048) and in shared memory (> 2048). 513-640 blocks: the
    direct-load path's tail quads split over the warps' channel quarters;
    700: one tail quad per thread."""
    rng = np.random.default_rng(nb)
    U, G, nbs = 4, 8, nbs_for(nb)
    n_tokens = np.array([64 * nb, 64 * nb - 63, 64 * (nb // 2) + 5, 64 * nb - 1], np.int32)
    dig = make_digests(rng, U, nbs)
    q = make_queries(rng, U, G)
    for k in (128, 512):
        want = P.score_topk_split(q, dig, n_tokens, k, G, k_stride=k)
        got = _gpu_topk(q, dig, n_tokens, k, G)
        for u in range(U):
            ns = want["n_sel"][u]
            assert got["n_sel"][u] == ns
            assert np.array_equal(got["sel_ids"][u, :ns], want["sel_ids"][u, :ns]), (u, k)


def test_topk_generic_f64_paths(cuda):
    """Arbitrary doubles (the drop-in wrapper's path): minmax and mean, no fma."""
    rng = np.random.default_rng(7)
    U, G, nbs = 6, 2, 64
    n_tokens = np.full(U, 64 * 50, np.int32)
    q = rng.standard_normal((U * G, D)) * np.pi
    a, b = rng.standard_normal((U, D, nbs)) / 3, rng.standard_normal((U, D, nbs)) / 3
    dig = np.stack([np.minimum(a, b), np.maximum(a, b)], axis=1)
    for method, dg in ((0, dig), (1, dig[:, :1])):
        want = P.score_topk_split(q, dg, n_tokens, 9, G, method=method)
        got = _gpu_topk(q, dg, n_tokens, 9, G, dtype=torch.float64, method=method)
        assert np.array_equal(got["sel_ids"][:, :9], want["sel_ids"][:, :9])
        assert np.array_equal(got["scores"][:, :50], want["scores"][:, :50])


def test_topk_kat_embedded(cuda):
    """test_digest.cpp:46-55 KAT embedded in d=128 (zero padding adds +0.0)."""
    dig = np.zeros((1, 2, D, 8), np.float32)
    dig[0, 0, :2, 0], dig[0, 1, :2, 0] = [0.0, -2.0], [3.0, 1.0]
    q = np.zeros((1, D), np.float32)
    q[0, :2] = [1.0, -1.0]
    r = _gpu_topk(q, dig, [64], 1, 1)
    assert r["scores"][0, 0] == 5.0


def test_topk_k_zero_rejected_and_mark_selected(cuda):
    rng = np.random.default_rng(3)
    dig = make_digests(rng, 2, 16)
    q = make_queries(rng, 2, 1)
    with pytest.raises(ValueError, match="k must be >= 1"):
        _gpu_topk(q, dig, [640, 640], 0, 1)
    last = torch.full((2, 16), -1, dtype=torch.int32, device="cuda")
    r = _gpu_topk(q, dig, [640, 640], 4, 1, step=11, last_sel=last)
    last = last.cpu().numpy()
    for u in range(2):
        assert set(np.nonzero(last[u] == 11)[0]) == set(r["sel_ids"][u, :4])


def test_topk_empty_unit(cuda):
    rng = np.random.default_rng(5)
    r = _gpu_topk(make_queries(rng, 2, 1), make_digests(rng, 2, 8), [0, 128], 3, 1)
    assert r["n_sel"][0] == 0 and r["n_sel"][1] == 2


def test_topk_batch_persistent_grid_matches_single_launches(cuda):
    """scout_score_topk_split_batch over more (layer, unit) items than resident
    CTAs, on the persistent grid (SCOUT_K1_PERSIST=1, read once per process:
    run in a subprocess) and the classic one: every layer's lists equal the
    one-layer launches bit for bit."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(__file__)
    for persist in ("1", "0"):
        env = dict(os.environ, SCOUT_K1_PERSIST=persist)
        code = ("import sys; sys.path[:0] = ['../oracle', '..', '.']; "
                "import test_gpu_topk as t; t._batch_vs_single()")
        r = subprocess.run([sys.executable, "-c", code], cwd=here, env=env, capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stdout + r.stderr


def _batch_vs_single():
    from paper_2603_27138_b200 import _capi as A

    rng = np.random.default_rng(99)
    L, U, G, nb, k = 3, 700, 4, 96, 16  # 2100 items > 148 x 7 resident CTAs
    nbs = nbs_for(nb)
    dev = torch.device("cuda")
    digs = [torch.from_numpy(make_digests(rng, U, nbs, "perm" if l == 1 else "iid")).to(dev).bfloat16().contiguous()
            for l in range(L)]
    qs = [torch.from_numpy(make_queries(rng, U, G, "perm" if l == 1 else "iid")).to(dev) for l in range(L)]
    nt = torch.from_numpy(rng.integers(64 * 40, 64 * nb + 1, size=U).astype(np.int32)).to(dev)
    tabs = [torch.from_numpy(np.where(rng.random((U, nbs)) < 0.7, rng.integers(0, 10**6, size=(U, nbs)), -1)
                             .astype(np.int32)).to(dev) for _ in range(L)]
    outs = {n: torch.full((L, U, k), -7, dtype=torch.int32, device=dev) for n in ("sel", "rs", "ri", "ci")}
    cnts = {n: torch.full((L, U), -7, dtype=torch.int32, device=dev) for n in ("ns", "nr", "nc", "rt", "ct")}
    arr = (A.TopkArgs * L)()
    for i in range(L):
        a = arr[i]
        a.n_units, a.group, a.digest_dtype, a.method, a.k, a.k_stride, a.nb_stride = U, G, A.SCOUT_BF16, 0, k, k, nbs
        a.q, a.digests, a.n_tokens, a.block_table = qs[i].data_ptr(), digs[i].data_ptr(), nt.data_ptr(), tabs[i].data_ptr()
        a.sel_ids, a.res_slots, a.res_ids, a.cpu_ids = (outs[n][i].data_ptr() for n in ("sel", "rs", "ri", "ci"))
        a.n_sel, a.n_res, a.n_cpu, a.res_tokens, a.cpu_tokens = (cnts[n][i].data_ptr() for n in ("ns", "nr", "nc", "rt", "ct"))
    A.check(A.lib().scout_score_topk_split_batch(arr, L, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    for i in range(L):
        r = ops.score_topk_split(qs[i], digs[i], nt, k, G, block_table=tabs[i], k_stride=k)
        torch.cuda.synchronize()
        ns_ = r["n_sel"]
        assert torch.equal(cnts["ns"][i], ns_) and torch.equal(cnts["nr"][i], r["n_res"])
        assert torch.equal(cnts["rt"][i], r["res_tokens"]) and torch.equal(cnts["ct"][i], r["cpu_tokens"])
        for u in range(0, U, 7):
            n = int(ns_[u])
            assert torch.equal(outs["sel"][i, u, :n], r["sel_ids"][u, :n]), (i, u)
            nr = int(r["n_res"][u])
            assert torch.equal(outs["rs"][i, u, :nr], r["res_slots"][u, :nr])
            assert torch.equal(outs["ci"][i, u, :n - nr], r["cpu_ids"][u, :n - nr])


def test_topk_ring_path_parity(cuda):
    """The bulk-copy ring (SCOUT_K1_DIRECT=0, read once per process) is no
    longer the default for bf16 digests: run the oracle parity cases through it
    in a subprocess."""
    import os
    import subprocess
    import sys

    if os.environ.get("SCOUT_K1_DIRECT") == "0":
        pytest.skip("already on the ring path")
    here = os.path.dirname(__file__)
    env = dict(os.environ, SCOUT_K1_DIRECT="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "test_gpu_topk.py", "-k",
                        "split_vs_oracle or band_edges or many_blocks or bf16_queries"],
                       cwd=here, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
