"""Cell-accelerated Verlet lists on the GPU -- drop-in for ``particula.neighbors``.

``build_verlet`` (ref neighbors.py:100-134) runs entirely on the device:
stable counting sort of the particles into the reference's cell grid
(``nc = max(1, floor(L/(rc*ratio)))``, width ``L/nc``), a count sweep and a
fill sweep of the deduplicated 27-cell stencil with the bit-exact FP64 pair
predicate (``pc_nbr_build``), and an in-row sort so ``indices`` matches the
reference's ascending rows.  ``VerletList`` keeps the CSR on the device and
materialises the reference's numpy fields on first access.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _kernels, _lib
from ._lib import call, ptr, stream
from .aosoa import FieldView
from .geometry import Box


class VerletList:
    """Neighbor list in dense or compressed layout (ref neighbors.py:14-46).

    Constructible like the reference dataclass (numpy fields), or from device
    CSR tensors via ``from_device``; either view is produced on demand.
    """

    def __init__(self, layout, half_or_full, cutoff, counts, table=None, indices=None,
                 offsets=None):
        self.layout = layout
        self.half_or_full = half_or_full
        self.cutoff = cutoff
        self._counts = None if counts is None else np.asarray(counts, np.int64)
        self._table = None if table is None else np.asarray(table, np.int64)
        self._indices = None if indices is None else np.asarray(indices, np.int64)
        self._offsets = None if offsets is None else np.asarray(offsets, np.int64)
        self._dev = None      # (counts i32, offsets i64, index i32) on device

    @classmethod
    def from_device(cls, layout, half_or_full, cutoff, counts, offsets, index, table=None):
        obj = cls(layout, half_or_full, cutoff, None)
        obj._dev = (counts, offsets, index)
        obj._dev_table = table
        return obj

    # -- reference fields ---------------------------------------------------
    @property
    def counts(self) -> np.ndarray:
        if self._counts is None:
            self._counts = self._dev[0].to(torch.int64).cpu().numpy()
        return self._counts

    @property
    def indices(self):
        if self.layout != "compressed":
            return None
        if self._indices is None:
            self._indices = self._dev[2].to(torch.int64).cpu().numpy()
        return self._indices

    @property
    def offsets(self):
        if self.layout != "compressed":
            return None
        if self._offsets is None:
            self._offsets = self._dev[1].cpu().numpy()
        return self._offsets

    @property
    def table(self):
        if self.layout != "dense":
            return None
        if self._table is None:
            self._table = self._dev_table.cpu().numpy()
        return self._table

    @property
    def n(self) -> int:
        return self.counts.shape[0]

    @property
    def total(self) -> int:
        return int(self.counts.sum())

    def neighbors(self, i: int) -> np.ndarray:
        if self.layout == "dense":
            return self.table[i, : self.counts[i]]
        return self.indices[self.offsets[i]: self.offsets[i + 1]]

    def pairs(self):
        """All stored (i, j), ascending i then stored j (ref neighbors.py:39-46)."""
        i = np.repeat(np.arange(self.n), self.counts)
        if self.layout == "compressed":
            return i, self.indices.copy()
        return i, self.table[self.table >= 0]

    # -- device view used by md.lj_forces -------------------------------------
    def device_csr(self):
        """(counts int32, offsets int64, index int32) CUDA tensors."""
        if self._dev is not None:
            return self._dev
        dev = _lib.device()
        counts = torch.as_tensor(self.counts).to(device=dev, dtype=torch.int32)
        if self.layout == "compressed":
            offsets = torch.as_tensor(self.offsets).to(dev)
            index = torch.as_tensor(self.indices).to(device=dev, dtype=torch.int32)
        else:
            width = self.table.shape[1] if self.table.ndim == 2 else 0
            offsets = torch.arange(self.n + 1, dtype=torch.int64, device=dev) * width
            index = torch.as_tensor(self.table).to(device=dev, dtype=torch.int32).reshape(-1)
        self._dev = (counts, offsets, index.contiguous())
        return self._dev


def _validate(box, per, cutoff, layout, half_or_full, cell_ratio):
    """ref neighbors.py:107-118."""
    if cutoff <= 0:
        raise ValueError("cutoff must be positive")
    if cell_ratio < 1.0:
        raise ValueError("cell_ratio must be >= 1")
    if layout not in ("dense", "compressed"):
        raise ValueError(f"unknown layout {layout!r}")
    if half_or_full not in ("half", "full"):
        raise ValueError(f"unknown pair convention {half_or_full!r}")
    for a in np.flatnonzero(per):
        if cutoff > 0.5 * box.lengths[a]:
            raise ValueError("cutoff exceeds half the box length on a periodic axis")


def neighbor_grid(box: Box, cutoff: float, cell_ratio: float = 1.0):
    """The reference's search grid (neighbors.py:56-59)."""
    edge = cutoff * cell_ratio
    nc = np.maximum(1, np.floor(box.lengths / edge).astype(np.int64))
    width = box.lengths / nc
    return nc, width, _lib.make_grid(box.low, box.high, width, nc)


def build_verlet(positions, box: Box, periodic, cutoff: float, layout: str = "compressed",
                 half_or_full: str = "full", cell_ratio: float = 1.0) -> VerletList:
    """Pairs with minimum-image distance strictly below ``cutoff``."""
    if isinstance(positions, FieldView):
        x = positions.device_values()
    else:
        x = _kernels.as_device(positions)
    per = np.broadcast_to(np.asarray(periodic, dtype=bool), (box.ndim,)).copy()
    _validate(box, per, cutoff, layout, half_or_full, cell_ratio)
    if x.dim() != 2 or x.shape[1] != box.ndim:
        raise ValueError(f"positions must be (n, {box.ndim})")
    n = int(x.shape[0])
    dev = x.device
    s = stream()
    _nc, _w, grid = neighbor_grid(box, cutoff, cell_ratio)
    pbox = _lib.make_box(box.low, box.high, per)
    cutoff2 = float(cutoff) * float(cutoff)
    half = int(half_or_full == "half")
    counts = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
    offsets = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    if n == 0:
        index = torch.empty(0, dtype=torch.int32, device=dev)
        return _finish(layout, half_or_full, cutoff, counts[:0], offsets, index, n, 0)
    pos4 = _kernels.pack_pos4(x)                       # tags = caller index
    srt = _kernels.CellSort(pos4, 4, grid)
    sorted4 = _kernels.gather_rows(pos4, srt.order, n)
    cnt_sorted = torch.empty(n, dtype=torch.int32, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    call("pc_nbr_build", ptr(sorted4), n, ptr(srt.cell_start), grid, pbox, cutoff2, half,
         _lib.PC_NBR_COUNT, 1, ptr(cnt_sorted), None, None, 0, 0, ptr(flag), s, None, None)
    # counts in caller order -> CSR offsets; the fill writes row k at the
    # offset of its caller index, then rows are sorted ascending
    call("pc_scatter_rows", ptr(cnt_sorted), ptr(counts), ptr(srt.order), n, 4, s)
    offsets = _kernels.scan_i32(counts[:n], out_dtype=torch.int64)
    total = int(offsets[n].item())
    off_sorted = _kernels.gather_rows(offsets[:n], srt.order, n)
    index = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    call("pc_nbr_build", ptr(sorted4), n, ptr(srt.cell_start), grid, pbox, cutoff2, half,
         _lib.PC_NBR_CSR, 1, ptr(cnt_sorted), ptr(off_sorted), ptr(index), 0, 0, ptr(flag), s, None, None)
    call("pc_sort_rows", ptr(offsets), n, ptr(index), s)
    return _finish(layout, half_or_full, cutoff, counts[:n], offsets, index[:total], n, total)


def _finish(layout, half_or_full, cutoff, counts, offsets, index, n, total):
    table = None
    if layout == "dense":
        width = int(counts.max().item()) if n else 0
        table = torch.empty((n, width), dtype=torch.int64, device=counts.device)
        call("pc_csr_to_dense", ptr(offsets), n, ptr(index), width, ptr(table), stream())
    return VerletList.from_device(layout, half_or_full, cutoff, counts, offsets, index, table)


def for_each_neighbor(vlist: VerletList, i_range, kernel) -> None:
    """Host callable kernel(i, j) per stored entry, ascending i then stored j
    (ref neighbors.py:137-143)."""
    begin, end = i_range
    for i in range(begin, end):
        for j in vlist.neighbors(i):
            kernel(i, int(j))


def for_each_neighbor2(vlist: VerletList, i_range, kernel) -> None:
    """kernel(i, j, k) per ordered pair of distinct neighbors, j stored before k
    (ref neighbors.py:146-154)."""
    if vlist.half_or_full != "full":
        raise ValueError("second-level traversal requires a full list")
    begin, end = i_range
    for i in range(begin, end):
        js = vlist.neighbors(i)
        for a in range(js.size):
            for b in range(a + 1, js.size):
                kernel(i, int(js[a]), int(js[b]))


# ---- device functor traversals (include/particula_b200_traverse.cuh) -------
# the GPU form of for_each_neighbor / for_each_neighbor2 is a
# C++ device functor (a Python callable cannot run on the device); these two
# consumers ship with the library and back the parity tests.


def _traverse_args(vlist: VerletList, positions, box: Box, periodic, i_range):
    x = _kernels.as_device(positions).to(torch.float64).contiguous()
    if x.dim() != 2 or x.shape[1] != 3:
        raise ValueError("positions must be (n, 3)")
    counts, offsets, index = vlist.device_csr()
    n = int(counts.numel())
    if x.shape[0] != n:
        raise ValueError("positions and neighbor list sizes differ")
    begin, end = (0, n) if i_range is None else (int(i_range[0]), int(i_range[1]))
    per = np.broadcast_to(np.asarray(periodic, bool), (3,))
    pbox = _lib.make_box(box.low, box.high, per)
    out = torch.zeros(max(n, 1), dtype=torch.float64, device=x.device)
    return x, pbox, offsets, index, n, begin, end, out


def coordination(vlist: VerletList, positions, box: Box, periodic, r_inner: float,
                 i_range=None, team: bool = False) -> np.ndarray:
    """Per-row count of stored neighbors closer than r_inner (for_each_neighbor
    with a device pair functor; one thread or one warp per row)."""
    x, pbox, off, idx, n, b, e, out = _traverse_args(vlist, positions, box, periodic, i_range)
    call("pc_traverse_coordination", ptr(x), pbox, ptr(off), ptr(idx), n, b, e,
         float(r_inner), int(team), ptr(out), stream())
    return out[:n].cpu().numpy()


def angle_sums(vlist: VerletList, positions, box: Box, periodic, i_range=None,
               team: bool = False) -> np.ndarray:
    """Per-row sum of cos(angle j-i-k) over pairs of stored neighbors j before
    k (for_each_neighbor2 with a device three-body functor; full lists only,
    as ref neighbors.py:148-149)."""
    if vlist.half_or_full != "full":
        raise ValueError("second-level traversal requires a full list")
    x, pbox, off, idx, n, b, e, out = _traverse_args(vlist, positions, box, periodic, i_range)
    call("pc_traverse_angle_sum", ptr(x), pbox, ptr(off), ptr(idx), n, b, e, int(team),
         ptr(out), stream())
    return out[:n].cpu().numpy()
