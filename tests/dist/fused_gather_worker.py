"""torchrun worker for tests/test_gpu.py::test_fused_gather_* (GPU): N ranks
share cuda:0 (CUDA IPC between processes of one device stands in for NVLink
peers).  Each rank holds its row band of a layer; the fused path
(spqr_matvec_gather + spqr_gather_wait) must leave the full y on every rank,
bit-identical to the band kernels' own outputs gathered over gloo, and within
1e-5 of the oracle; rounds repeat eagerly and from a replayed CUDA graph."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2306_03078_b200 as P  # noqa: E402
from paper_2306_03078_b200 import synth  # noqa: E402
from paper_2306_03078_b200.sharded import ShardedLayer, gather_rows  # noqa: E402
from oracle import oracle as O  # noqa: E402


def fail(msg):
    print(msg, flush=True)
    sys.exit(1)


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    orc = O.Oracle()
    for m, n, perm in ((1024, 2048, False), (608, 1280, True)):
        s = P.encode_arrays(synth.make_layer(m, n, outlier_rate=0.02, seed=m + n, permute=perm))
        fused = ShardedLayer(s, rank, world, 0, fused=True)
        plain = fused.layer
        r0, r1 = fused.band
        st = torch.cuda.Stream()
        xs = [torch.from_numpy(synth.random_x(n, seed=11 + i).reshape(-1)).to(dev) for i in range(4)]
        x = torch.empty_like(xs[0])
        y_band = torch.empty(r1 - r0, device=dev)

        def check(xh, y_full, tag):
            plain.matvec(xh, y_band, stream=st)
            st.synchronize()
            y_ref = gather_rows(y_band.cpu(), fused.bands)[:m].numpy()
            y = y_full.cpu().numpy()
            if not np.array_equal(y.view(np.uint32), y_ref.view(np.uint32)):
                fail(f"rank {rank} {tag}: fused != band kernels, max {np.abs(y - y_ref).max()}")
            yo = orc.decode(s).matvec(xh.float().cpu().numpy())
            rel = np.linalg.norm(y - yo) / np.linalg.norm(yo)
            if rel > 1e-5:
                fail(f"rank {rank} {tag}: rel {rel} vs oracle")

        x32 = torch.empty(n, device=dev, dtype=torch.float32)
        for i in range(3):  # eager rounds; round 2 with fp32 x (the hi/lo kernel with the gather)
            xi = x32 if i == 2 else x
            with torch.cuda.stream(st):
                xi.copy_(xs[i] if i < 2 else xs[0].float() * 1.0009765625)  # not fp16-exact
                y = fused.matvec(xi, stream=st)
            st.synchronize()
            check(xi, y, f"m={m} eager {i}")
            dist.barrier()  # nobody starts the next round while a peer still reads this one
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(st):
            x.copy_(xs[2])
        st.synchronize()
        with torch.cuda.graph(g, stream=st):
            y = fused.matvec(x, stream=st)
        for i in (2, 3):  # graph rounds (the capture itself launched nothing)
            with torch.cuda.stream(st):
                x.copy_(xs[i])
                g.replay()
            st.synchronize()
            check(x, y, f"m={m} graph {i}")
            dist.barrier()
        del g
        # back-to-back rounds, no host barrier: each rank's consumer of a
        # round's y (the D2H copy) is stream-ordered before its next band
        # kernel, and no rank stores round R into a peer's y before that
        # peer's band kernel of round R has started (gemv_cta wait_peers)
        R = 6
        outs = [torch.empty(m, dtype=torch.float32).pin_memory() for _ in range(R)]
        xr = [xs[i % 4] if i % 2 == 0 else xs[i % 4] * 0.5 for i in range(R)]
        with torch.cuda.stream(st):
            for i in range(R):
                x.copy_(xr[i])
                y = fused.matvec(x, stream=st)
                outs[i].copy_(y[:m], non_blocking=True)
        st.synchronize()
        for i in range(R):
            check(xr[i], outs[i], f"m={m} back-to-back {i}")
        dist.barrier()
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print("fused gather ok", flush=True)


if __name__ == "__main__":
    main()
