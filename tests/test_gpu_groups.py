"""Wide statistic groups on the fast kernels: beta1, beta2 multiples of 16
(PAPER Appendix D: 3/3/3 bits, beta1 = 16, beta2 = 32; the Table-10 beta
grid) -- the loader repeats a wider group's statistics / scalars in every
16 x 16 tile it covers, so gemv_cta, gemm_tc and dequant_cells run unchanged.
Against the oracle: dequantize bit-exact, matvec within 1e-5 (exact codes)
or 1e-3 (fp16-weight tensor-core path); the device transcode equals the host
one and the export re-encodes the stream byte for byte."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2306_03078_b200 as P
from oracle import relative_l2
from paper_2306_03078_b200 import synth

pytestmark = pytest.mark.gpu

GROUPS = [(16, 32), (32, 16), (32, 32), (16, 64), (64, 128), (128, 16), (48, 80)]


@pytest.mark.parametrize("b1,b2", GROUPS)
@pytest.mark.parametrize("shape,perm", [((160, 1000), True), ((256, 4096), False), ((96, 300), False)])
def test_wide_groups_fast_path(cuda, oracle_c, b1, b2, shape, perm):
    m, n = shape
    s = P.encode_arrays(synth.make_layer(m, n, beta1=b1, beta2=b2, seed=b1 * 3 + b2 + m, permute=perm,
                                         outlier_rate=0.02))
    L = P.Layer(s)
    assert L.info["fast_path"] == 1
    t = oracle_c.decode(s)
    w = torch.empty(m, n, device="cuda")
    L.dequantize(w)
    assert np.array_equal(w.cpu().numpy().view(np.uint32), t.dequantize_full().view(np.uint32))
    x = torch.randn(5, n, generator=torch.Generator().manual_seed(n)).half().cuda()
    for batch, tol in ((1, 1e-5), (2, 1e-5), (5, 1e-3)):
        y = torch.empty(batch, m, device="cuda")
        L.matvec(x[:batch].contiguous(), y, batch=batch)
        yh = y.cpu().numpy()
        for b in range(batch):
            assert relative_l2(yh[b], t.matvec(x[b].float().cpu().numpy())) <= tol, (batch, b)
    assert L.export_stream() == s
    dh = P.Layer(s, host_transcode=True).debug_cells()
    dd = L.debug_cells()
    assert np.array_equal(dh["cell_off"], dd["cell_off"]) and np.array_equal(dh["cells"], dd["cells"])


@pytest.mark.slow
def test_appendix_d_config_full_size(cuda, reference):
    """PAPER Appendix D (3,3,3, beta1 = 16, beta2 = 32) at 8192x8192 against the
    reference's own matvec(t, x, plan)."""
    s = P.encode_arrays(synth.make_layer(8192, 8192, beta1=16, beta2=32, seed=4, outlier_rate=0.01))
    L = P.Layer(s)
    assert L.info["fast_path"] == 1
    x = torch.randn(8192, generator=torch.Generator().manual_seed(7)).half().cuda()
    y = torch.empty(8192, device="cuda")
    L.matvec(x, y)
    t = reference.decode(s)
    assert relative_l2(y.cpu().numpy(), t.matvec(x.float().cpu().numpy())) <= 1e-5
