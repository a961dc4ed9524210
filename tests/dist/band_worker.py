"""torchrun worker for tests/test_dist.py (gloo, CPU): every rank takes its row
band of a layer (row_bands + slice_rows, the loader's cut), computes the band
product with the oracle (standing in for the band kernel, which needs a GPU),
and gather_rows() assembles y; rank-local result must equal the full product."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2306_03078_b200 as P  # noqa: E402
from paper_2306_03078_b200 import synth  # noqa: E402
from paper_2306_03078_b200.sharded import gather_rows, row_bands  # noqa: E402
from oracle import oracle as O  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    orc = O.Oracle()
    for m, n, perm in ((256, 512, False), (208, 544, True), (96, 272, True)):
        s = P.encode_arrays(synth.make_layer(m, n, outlier_rate=0.03, seed=m + n, permute=perm))
        x = synth.random_x(n, seed=5).reshape(-1).astype(np.float32)
        bands = row_bands(m, world)
        assert bands[0][0] == 0 and bands[-1][1] == m
        assert all(a % 32 == 0 for a, _ in bands)
        r0, r1 = bands[rank]
        y_band = orc.decode(P.slice_rows(s, r0, r1)).matvec(x) if r1 > r0 else np.zeros(0, np.float32)
        y = gather_rows(torch.from_numpy(y_band), bands)[:m].numpy()
        y_ref = orc.decode(s).matvec(x)
        if not np.array_equal(y.view(np.uint32), y_ref.view(np.uint32)):
            print(f"rank {rank}: mismatch m={m} n={n} max={np.abs(y - y_ref).max()}", flush=True)
            sys.exit(1)
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print("band gather ok", flush=True)


if __name__ == "__main__":
    main()
