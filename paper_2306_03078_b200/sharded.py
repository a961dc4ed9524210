"""Row-sharded multi-GPU decode: one process per GPU.

Rank r of N holds the row band `row_bands(m, N)[r]` of a layer -- its cells,
its CSR rows and the shared permutation (the loader cuts the band with
spqr_stream_slice_rows semantics) -- runs the fused kernel on it, and the y
bands are all-gathered over NCCL (torch.distributed is the plumbing).  x is
replicated: in tensor-parallel decode it arrives from the previous layer.
"""
from __future__ import annotations

import math

import torch
import torch.distributed as dist

from . import Gather, Layer, validate

CELL_ROWS = 32  # bands never split a cell (row-group pair); beta2 = 16 divides it


def row_bands(m: int, world: int, align: int = CELL_ROWS, beta2: int = 16) -> list[tuple[int, int]]:
    """Contiguous row bands aligned to lcm(`align`, beta2) rows (bands never
    split a cell or a statistics group), sizes differing by at most one unit
    (the last band also takes the ragged tail).  Every rank gets a non-empty
    band: world must not exceed the number of units."""
    if world < 1:
        raise ValueError("world must be >= 1")
    align = math.lcm(align, beta2)
    units = (m + align - 1) // align
    if world > units:
        raise ValueError(f"{world} ranks but only {units} row units of {align} rows: some band would be empty")
    out, u0 = [], 0
    for r in range(world):
        u1 = u0 + units // world + (1 if r < units % world else 0)
        out.append((min(m, u0 * align), min(m, u1 * align)))
        u0 = u1
    return out


def gather_rows(y_band: torch.Tensor, bands: list[tuple[int, int]], out: torch.Tensor | None = None,
                group=None) -> torch.Tensor:
    """All-gather the ranks' y bands (fp32, rows of this rank's band first dim)
    into the full y on every rank.  Equal bands gather in place; ragged bands
    gather padded slots and compact."""
    world = len(bands)
    m = bands[-1][1]
    sizes = [b - a for a, b in bands]
    mx = max(sizes)
    nccl = dist.get_backend(group) == "nccl"
    if all(s == mx for s in sizes):
        full = out if out is not None else torch.empty(world * mx, dtype=y_band.dtype, device=y_band.device)
        if nccl:
            dist.all_gather_into_tensor(full, y_band.contiguous(), group=group)
        else:  # gloo (CPU tests): list form
            dist.all_gather(list(full.view(world, mx)), y_band.contiguous(), group=group)
        return full
    pad = torch.zeros(mx, dtype=y_band.dtype, device=y_band.device)
    pad[: y_band.numel()] = y_band
    slots = torch.empty(world * mx, dtype=y_band.dtype, device=y_band.device)
    if nccl:
        dist.all_gather_into_tensor(slots, pad, group=group)
    else:
        dist.all_gather(list(slots.view(world, mx)), pad, group=group)
    full = out if out is not None else torch.empty(m, dtype=y_band.dtype, device=y_band.device)
    for r, (a, b) in enumerate(bands):
        full[a:b] = slots[r * mx: r * mx + (b - a)]
    return full


class _DeviceArray:
    """A raw device pointer as a torch tensor (__cuda_array_interface__, no copy)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3,
                                         "strides": None}


class FusedGather:
    """The all-gather fused into the band kernel (spqr_matvec_gather): one
    spqr_gather per rank, CUDA IPC handles exchanged over `group` (any
    torch.distributed backend -- it carries 64 bytes per rank once)."""

    def __init__(self, rows: int, bands: list[tuple[int, int]], rank: int, world: int, device: int, group=None):
        self.g = Gather(device, rows, world, rank)
        handles = [None] * world
        dist.all_gather_object(handles, self.g.handle(), group=group)
        self.g.open(handles, [a for a, _ in bands])
        self.y = torch.as_tensor(_DeviceArray(self.g.y_ptr(), rows), device=torch.device("cuda", device))

    def matvec(self, layer: Layer, x: torch.Tensor, stream=None) -> torch.Tensor:
        self.g.matvec(layer, x, stream=stream)
        self.g.wait(stream=stream)
        return self.y


class ShardedLayer:
    """This rank's band of one layer, resident on `device`.  fused=True (world
    > 1): the band kernel stores its rows into every rank's full y over P2P and
    one wait launch replaces the NCCL all-gather (the NCCL path stays the
    baseline the north star names)."""

    def __init__(self, stream: bytes, rank: int, world: int, device: int, fused: bool = False, group=None):
        info = validate(stream)
        self.rows, self.cols = info["rows"], info["cols"]
        self.bands = row_bands(self.rows, world, beta2=info["beta2"])
        self.band = self.bands[rank]
        r0, r1 = self.band
        self.layer = Layer(stream, device=device, rows=(r0, r1) if world > 1 else None)
        dev = torch.device("cuda", device)
        self.y_band = torch.empty(r1 - r0, dtype=torch.float32, device=dev)
        mx = max(b - a for a, b in self.bands)
        self.y_full = torch.empty(max(self.rows, world * mx), dtype=torch.float32, device=dev)
        self.fused = FusedGather(self.rows, self.bands, rank, world, device, group) if fused and world > 1 else None

    def matvec(self, x: torch.Tensor, stream=None, group=None) -> torch.Tensor:
        """Full y (fp32, rows) on every rank: band matvec + all-gather."""
        if self.fused is not None:
            return self.fused.matvec(self.layer, x, stream=stream)
        self.layer.matvec(x, self.y_band, stream=stream)
        if len(self.bands) == 1:
            return self.y_band
        return gather_rows(self.y_band, self.bands, out=self.y_full, group=group)[: self.rows]
