"""Batch 2-3 through the batch-pair gemv_cta (x mode 2): two fp16 batch columns
share every MMA -- each weight is decoded once for both (matvec, kernel.hpp:
89-124, per column).  The per-column arithmetic is the single-column kernel's
(the same exact per-(row, block) products, epilogue, outlier scan and pair
reduction), so the pair's y must equal two single-column launches bit for
bit, and the oracle within 1e-5."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2306_03078_b200 as P
from oracle import relative_l2
from paper_2306_03078_b200 import synth

pytestmark = pytest.mark.gpu


def _run(L, x, batch):
    y = torch.full((batch, L.rows), float("nan"), device="cuda")
    L.matvec(x, y, batch=batch)
    torch.cuda.synchronize()
    return y.cpu().numpy()


@pytest.mark.parametrize("bw,bs", [(2, 2), (3, 3), (4, 4), (3, 2)])
@pytest.mark.parametrize("shape,perm", [((64, 512), False), ((160, 1000), True), ((256, 4096), False),
                                        ((96, 17000), False), ((96, 300), False), ((64, 1004), False)])
@pytest.mark.parametrize("batch", [2, 3])
def test_batch_pair_equals_single_columns(cuda, oracle_c, bw, bs, shape, perm, batch):
    m, n = shape
    s = P.encode_arrays(synth.make_layer(m, n, weight_bits=bw, scale_bits=bs, zero_bits=bs, outlier_rate=0.02,
                                         seed=bw * 11 + m + batch, permute=perm))
    L = P.Layer(s)
    assert L.info["fast_path"] == 1
    g = torch.Generator().manual_seed(m + n)
    x = (torch.randn(batch, n, generator=g) * torch.tensor([1.0, 30.0, 0.01])[:batch, None]).half().cuda()
    y = _run(L, x, batch)
    assert P.last_launch_count() == (1 if batch == 2 else 2)  # the pair, then the odd column alone
    t = oracle_c.decode(s)
    for b in range(batch):
        y1 = _run(L, x[b].contiguous(), 1)[0]
        # bit-identical unless the two plans stage a different number of a
        # cell's outliers in shared memory (the remainder is summed in a
        # second chunk sequence): then fp32 rounding order may differ
        assert np.array_equal(y[b].view(np.uint32), y1.view(np.uint32)) or np.allclose(y[b], y1, rtol=1e-6, atol=0), b
        assert relative_l2(y[b], t.matvec(x[b].float().cpu().numpy())) <= 1e-5


@pytest.mark.slow
@pytest.mark.parametrize("shape", [(8192, 22016), (24576, 8192)])
def test_batch_pair_full_size(cuda, reference, shape):
    """BASELINE configs[3] shape (and the bench's fused-QKV rows): batch 2 in one pass."""
    m, n = shape
    s = synth.random_stream(m, n, 3, 3, 3, 0.01, seed=9)
    L = P.Layer(s)
    x = torch.randn(2, n, generator=torch.Generator().manual_seed(1)).half().cuda()
    y = _run(L, x, 2)
    t = reference.decode(s)
    for b in range(2):
        assert relative_l2(y[b], t.matvec(x[b].float().cpu().numpy())) <= 1e-5
