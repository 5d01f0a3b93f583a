"""K6 layer-ahead query prediction (tcgen05 GEMM) against the reference's
predict_next_query(rms_normalize(x), W) (model.hpp:215-217, via oracle/_ref)
and a torch fp32 restatement on the same bf16 operands."""
import numpy as np
import pytest
import torch

import py_oracle as P
from paper_2603_27138_b200 import ops

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("hidden,n_out", [(256, 256), (640, 384), (512, 256)])
@pytest.mark.parametrize("batch", [1, 5, 32, 40])
@pytest.mark.parametrize("max_ctas", [0, 2, 4, 5])
def test_predict_query_vs_reference(cuda, hidden, n_out, batch, max_ctas):
    """max_ctas 0: one CTA per SM (tiles shared by several CTAs); 2 / 5: the
    minimum grid (= tiles: whole tiles) and a grid that splits tiles unevenly;
    4 with (512, 256): two CTAs per tile with an even chunk count, the cluster
    pairs whose K halves meet in shared memory."""
    rng = np.random.default_rng(hidden + n_out + batch + 7 * max_ctas)
    w = torch.from_numpy(rng.standard_normal((hidden, n_out)).astype(np.float32) / np.sqrt(hidden)).bfloat16()
    x = rng.standard_normal((batch, hidden)).astype(np.float32) * 3.0
    x[0, :] = 0.0 if batch > 2 else x[0, :]  # rms == 0 row: rms_normalize returns x unchanged
    qp = ops.QueryPredictor(w.cuda(), batch, max_ctas=max_ctas)
    q32, qbf = qp(torch.from_numpy(x), want=("f32", "bf16"))
    torch.cuda.synchronize()
    q32, qbf = q32.cpu(), qbf.cpu()
    wd = w.double().numpy()
    for b in range(batch):
        want = P.predict_query(x[b], wd)
        err = np.abs(q32[b].double().numpy() - want).max()
        assert err <= 1e-2 * max(np.abs(want).max(), 1e-30), (b, err)
    # the kernel's own arithmetic: bf16 x^ times bf16 W, fp32 accumulation
    xd = torch.from_numpy(x).double()
    rms = xd.pow(2).mean(1, keepdim=True).sqrt()
    xn = torch.where(rms == 0, xd, xd / torch.where(rms == 0, torch.ones_like(rms), rms)).float().bfloat16()
    ref32 = xn.double() @ w.double()
    assert torch.allclose(q32.double(), ref32, rtol=0, atol=2e-5 * ref32.abs().max().item() + 1e-30)
    assert torch.equal(qbf, q32.bfloat16())


def test_predict_query_qwen3_32b_shape_deterministic(cuda):
    """Qwen3-32B: hidden 5120 -> 64 x 128 query features, batch 32."""
    torch.manual_seed(0)
    hidden, n_out, batch = 5120, 8192, 32
    w = (torch.randn(hidden, n_out, device="cuda") / hidden ** 0.5).bfloat16()
    x = torch.randn(batch, hidden, device="cuda")
    qp = ops.QueryPredictor(w, batch)
    a = qp(x).clone()
    b = qp(x)
    torch.cuda.synchronize()
    assert torch.equal(a, b)  # k-split partials are reduced in a fixed order
    xn = (x.double() / x.double().pow(2).mean(1, keepdim=True).sqrt()).float().bfloat16()
    ref = (xn.double() @ w.double())
    assert torch.allclose(a.double(), ref, rtol=0, atol=1e-4 * ref.abs().max().item())
    for r in (0, 17, 31):
        want = P.predict_query(x[r].cpu().numpy(), w.double().cpu().numpy())
        assert np.abs(a[r].double().cpu().numpy() - want).max() <= 1e-2 * np.abs(want).max()
