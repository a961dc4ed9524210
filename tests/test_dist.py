"""Multi-process host logic of the row-sharded path (gloo, world size 2, CPU)."""
import os
import socket
import subprocess
import sys

import pytest

from paper_2306_03078_b200.sharded import row_bands

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("m,world,beta2", [(8192, 8, 16), (22016, 8, 16), (22016, 4, 16), (4096, 2, 16),
                                           (208, 2, 16), (96, 3, 16), (40, 2, 16), (8192, 8, 64), (200, 2, 48)])
def test_row_bands_cover_and_align(m, world, beta2):
    bands = row_bands(m, world, beta2=beta2)
    align = 32 * beta2 // __import__("math").gcd(32, beta2)
    assert len(bands) == world
    assert bands[0][0] == 0 and bands[-1][1] == m
    for (a, b), (c, _) in zip(bands, bands[1:]):
        assert b == c
    assert all(b > a for a, b in bands)  # no empty band
    assert all(a % align == 0 for a, _ in bands)  # never splits a cell or a statistics group
    units = [-(-(b - a) // align) for a, b in bands]
    assert max(units) - min(units) <= 1


@pytest.mark.parametrize("m,world", [(96, 4), (4, 2), (31, 2)])
def test_row_bands_refuse_empty_bands(m, world):
    with pytest.raises(ValueError):
        row_bands(m, world)


@pytest.mark.parametrize("m,world,beta2", [(8192, 8, 16), (22016, 8, 16), (44032, 3, 16), (24576, 8, 16),
                                           (208, 2, 16), (96, 3, 16), (40, 2, 16), (8192, 8, 64), (200, 2, 48)])
def test_c_abi_row_bands_match(m, world, beta2):
    """spqr_row_bands (the edges spqr_sharded_create cuts) == sharded.row_bands."""
    import paper_2306_03078_b200 as P
    assert P.c_row_bands(m, beta2, world) == row_bands(m, world, beta2=beta2)


def test_c_abi_row_bands_refuse_empty_bands():
    import paper_2306_03078_b200 as P
    with pytest.raises(P.SpqrError):
        P.c_row_bands(96, 16, 4)


def test_llama_bands_are_equal():
    for m in (4096, 8192, 11008, 22016):
        for w in (1, 2, 4, 8):
            sizes = {b - a for a, b in row_bands(m, w)}
            assert len(sizes) == 1, (m, w)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_gather_matches_full_product_world2(oracle_c):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(HERE, "dist", "band_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "band gather ok" in r.stdout
