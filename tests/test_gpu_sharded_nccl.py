"""The NCCL row-sharded path behind the C ABI (spqr_nccl_* + spqr_sharded_*,
SURVEY 8b/8e): a world-1 communicator made through spqr_nccl_unique_id /
spqr_nccl_comm_init (NCCL refuses two ranks on one GPU, so world > 1 runs only
on a multi-GPU box -- the band arithmetic for world > 1 is tested on CPU in
test_dist.py, and the band kernels per rank in test_gpu_fullsize.py).

* stacked q/k/v-style members: y comes back in [member 0; member 1; ...]
  order, bitwise equal to the stacked single-GPU handle (same kernel, same
  partition), batch 1 (in-place all-gather) and batch 2 (gather slots +
  strided compaction), fp16 and fp32 x;
* against the reference's matvec(t, x, plan) (kernel.hpp:89) per member.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2306_03078_b200 as P
from oracle import relative_l2
from paper_2306_03078_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm(cuda):
    c = P.NcclComm(P.nccl_unique_id(), 1, 0, 0)
    yield c
    c.close()


@pytest.mark.parametrize("batch", [1, 2])
@pytest.mark.parametrize("xdt", [torch.float16, torch.float32])
def test_sharded_stacked_world1_matches_stacked_layer(cuda, comm, reference, batch, xdt):
    shapes = [(256, 768, 11), (256, 768, 12), (96, 768, 13)]
    streams = [synth.random_stream(m, n, 3, 3, 3, 0.01, seed=s) for m, n, s in shapes]
    S = P.ShardedNccl(streams, comm, device=0)
    assert S.rows == sum(m for m, _, _ in shapes) and S.band == (0, S.rows)
    L = P.Layer.stacked(streams, device=0)
    g = torch.Generator().manual_seed(3)
    x = torch.randn(batch, 768, generator=g).to(xdt).cuda()
    y = torch.full((batch, S.rows), float("nan"), device="cuda")
    y_ref = torch.empty(batch, S.rows, device="cuda")
    S.matvec(x, y, batch=batch)
    L.matvec(x, y_ref, batch=batch)
    torch.cuda.synchronize()
    yh, yr = y.cpu().numpy(), y_ref.cpu().numpy()
    assert np.array_equal(yh.view(np.uint32), yr.view(np.uint32))
    xh = x.float().cpu().numpy()
    off = 0
    for (m, n, _), s in zip(shapes, streams):
        t = reference.decode(s)
        for b in range(batch):
            want = t.matvec(xh[b])
            assert relative_l2(yh[b, off:off + m], want) <= 1e-5
        off += m
    S.close()
    L.close()


def test_sharded_rejects_wrong_world(cuda, comm):
    s = synth.random_stream(64, 256, 3, 3, 3, 0.01, seed=1)
    with pytest.raises(P.SpqrError, match="ConfigInvalid"):
        P.ShardedNccl(s, type("C", (), {"rank": 0, "world": 2, "handle": comm.handle})(), device=0)


def test_band_layer_view(cuda, comm):
    s = synth.random_stream(128, 512, 3, 3, 3, 0.01, seed=4)
    S = P.ShardedNccl(s, comm, device=0)
    L = S.band_layer()
    assert L.rows == 128 and L.cols == 512
    x = torch.randn(512, device="cuda").half()
    y1, y2 = torch.empty(128, device="cuda"), torch.empty(128, device="cuda")
    L.matvec(x, y1)
    S.matvec(x, y2)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    L.close()  # a view: does not free the band
    S.matvec(x, y2)
    torch.cuda.synchronize()
    S.close()
