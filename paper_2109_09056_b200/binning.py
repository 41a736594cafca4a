"""Key and linked-cell binning on the GPU -- drop-in for ``particula.binning``.

Replaces ref binning.py:13-101 with the K1-K3 kernels: cell assignment with
warp-aggregated atomic counts (``pc_bin_count``), a device exclusive scan
(``pc_scan_i32``) and a stable counting-sort placement (``pc_bin_place``).
``bin_by_key`` runs LSD passes of the same stable counting sort over 16-bit
digits of the keys.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _kernels, _lib
from ._lib import call, ptr, stream
from .aosoa import FieldView, ParticleSet
from .geometry import Box


@dataclass(frozen=True)
class Permutation:
    """map[source index] = destination index (ref binning.py:13-33)."""

    map: np.ndarray

    def __post_init__(self):
        m = self.map
        if isinstance(m, torch.Tensor):
            m = m.detach().cpu().numpy()
        object.__setattr__(self, "map", np.asarray(m, dtype=np.int64))

    @property
    def n(self) -> int:
        return self.map.shape[0]

    def device_map(self, device=None) -> torch.Tensor:
        dev = device if device is not None else _lib.device()
        return torch.as_tensor(self.map, dtype=torch.int64).to(dev)

    def is_bijection(self) -> bool:
        """Range + duplicate check on the device (``pc_check_bijection``)."""
        n = self.n
        if n == 0:
            return True
        m = self.device_map()
        seen = torch.zeros(n, dtype=torch.int32, device=m.device)
        flag = torch.zeros(1, dtype=torch.int32, device=m.device)
        call("pc_check_bijection", ptr(m), n, ptr(seen), ptr(flag), stream())
        return int(flag.item()) == 0


@dataclass(frozen=True)
class CellBinning:
    cells: np.ndarray
    cell_size: np.ndarray
    origin: np.ndarray
    offsets: np.ndarray
    permutation: Permutation

    @property
    def num_cells(self) -> int:
        return int(np.prod(self.cells))


def bin_by_key(keys) -> Permutation:
    """Stable sort permutation of integer keys (ref binning.py:49-55)."""
    k = keys if isinstance(keys, torch.Tensor) else torch.as_tensor(np.asarray(keys))
    dev = _lib.device()
    k = k.to(device=dev, dtype=torch.int64).contiguous()
    n = k.numel()
    if n == 0:
        return Permutation(np.empty(0, np.int64))
    kmin = int(k.min().item())
    span = int(k.max().item()) - kmin          # unsigned span of (key - kmin)
    perm = None                                # current order[dst] = src (int32)
    shift = 0
    # LSD passes of 8-bit digits, each a stable partition (O(n) however many
    # keys share a digit -- pc_bin_place's cell stabilisation is for small cells)
    digit_bits = 8
    while True:
        cell_of = torch.empty(n, dtype=torch.int32, device=dev)
        ncells = 1 << digit_bits
        counts = torch.zeros(ncells, dtype=torch.int32, device=dev)
        call("pc_key_digits", ptr(k), ptr(perm), n, kmin, shift, ncells - 1, ptr(cell_of),
             ptr(counts), stream())
        order, _ = _kernels.stable_partition(cell_of, ncells)
        perm = order if perm is None else _kernels.gather_rows(perm, order, n)
        shift += digit_bits
        if shift >= 64 or (span >> shift) == 0:
            break
    m = torch.empty(n, dtype=torch.int64, device=dev)
    call("pc_invert_order", ptr(perm), n, ptr(m), stream())
    return Permutation(m)


def _grid_for_cells(box: Box, cell_size):
    cs = np.broadcast_to(np.asarray(cell_size, dtype=np.float64), (box.ndim,)).copy()
    if np.any(cs <= 0):
        raise ValueError("cell_size must be positive")
    nc = np.maximum(1, np.ceil((box.lengths / cs) - 1e-12).astype(np.int64))
    return cs, nc, _lib.make_grid(box.low, box.high, cs, nc)


def _positions(positions):
    if isinstance(positions, FieldView):
        return positions.device_values()
    return _kernels.as_device(positions)


def cell_indices(positions, box: Box, cell_size):
    """(cells per axis, per-particle (n, d) cell index) -- ref binning.py:58-73."""
    x = _positions(positions)
    if x.dim() == 1:
        x = x.reshape(-1, box.ndim)
    cs, nc, grid = _grid_for_cells(box, cell_size)
    n = x.shape[0]
    cell_of = torch.empty(max(n, 1), dtype=torch.int32, device=x.device)
    idx = torch.empty((max(n, 1), box.ndim), dtype=torch.int64, device=x.device)
    counts = torch.zeros(grid.ncells, dtype=torch.int32, device=x.device)
    flag = torch.zeros(1, dtype=torch.int32, device=x.device)
    call("pc_bin_count", ptr(x), n, box.ndim, grid, 1, ptr(cell_of), ptr(idx), ptr(counts),
         ptr(flag), stream())
    if int(flag.item()) & _lib.FLAG_OUTSIDE:
        raise ValueError("position outside box")
    return nc, idx[:n].cpu().numpy()


def bin_by_position(positions, box: Box, cell_size) -> CellBinning:
    """Geometric binning; the permutation groups cells contiguously in
    row-major order (ref binning.py:76-87)."""
    x = _positions(positions)
    if x.dim() == 1:
        x = x.reshape(-1, box.ndim)
    cs, nc, grid = _grid_for_cells(box, cell_size)
    n = x.shape[0]
    srt = _kernels.CellSort(x, box.ndim, grid, check_inside=True)
    if n and srt.outside():
        raise ValueError("position outside box")
    offsets = srt.cell_start.to(torch.int64).cpu().numpy()
    pmap = srt.perm_map() if n else torch.empty(0, dtype=torch.int64)
    return CellBinning(nc, cs, box.low.copy(), offsets, Permutation(pmap))


def permute(pset: ParticleSet, p: Permutation) -> None:
    """Reorder all fields so tuple i moves to index p.map[i] (ref binning.py:90-101),
    one ``pc_aosoa_permute`` launch over the whole AoSoA buffer."""
    if p.n != pset.size:
        raise ValueError(f"permutation length {p.n} != set size {pset.size}")
    if not p.is_bijection():
        raise ValueError("permutation is not a bijection")
    if pset.size == 0:
        return
    m = p.device_map(pset.device)
    bases = pset.word_bases()
    dst = torch.zeros_like(pset._buffer)
    call("pc_aosoa_permute", ptr(pset._buffer), ptr(dst), ptr(m), pset.size,
         pset.vector_length, pset._struct_bytes, ptr(bases), bases.numel(), stream())
    pset._buffer = dst
