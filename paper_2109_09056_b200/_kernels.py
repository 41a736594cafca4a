"""Thin typed wrappers over the C ABI, operating on torch CUDA tensors.

Torch is used for device memory and the current stream only; every
arithmetic step below is one of our sm_100a kernels (``pc_*``).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, stream


def as_device(a, dtype=torch.float64):
    """numpy/sequence -> contiguous CUDA tensor (CUDA tensors pass through)."""
    dev = _lib.device()
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype).to(dev)


def to_host(t):
    return t.detach().cpu().numpy()


def box_op(box, x, periodic, op):
    """Box.wrap / Box.min_image: same container type out as in."""
    is_tensor = isinstance(x, torch.Tensor)
    t = as_device(x).clone()
    d = box.ndim
    shape = t.shape
    if shape[-1] != d:
        raise ValueError(f"last axis must have {d} components")
    b = _lib.make_box(box.low, box.high, np.broadcast_to(
        np.asarray(periodic, bool), (d,)))
    rows = int(t.numel() // d)
    name = "pc_box_wrap" if op == "wrap" else "pc_box_min_image"
    call(name, ptr(t), rows, d, b, stream())
    return t if is_tensor else to_host(t)


def scan_i32(counts, out_dtype=torch.int32):
    """Exclusive scan -> n+1 entries."""
    n = counts.numel()
    out = torch.empty(n + 1, dtype=out_dtype, device=counts.device)
    tmp = torch.empty(int(_lib.load().pc_scan_tmp_bytes(n)) // 8 + 1, dtype=torch.int64,
                      device=counts.device)
    name = "pc_scan_i32" if out_dtype == torch.int32 else "pc_scan_i32_i64"
    call(name, ptr(counts), ptr(out), n, ptr(tmp), tmp.numel() * 8, stream())
    return out


def stable_partition(keys, nbins):
    """Stable partition of int32 keys in [0, nbins), nbins <= 256
    (pc_partition_hist -> scan -> pc_partition_place): (order[dst] = src,
    bin starts on the device, nbins + 1 entries)."""
    n = keys.numel()
    dev = keys.device
    nch = int(_lib.load().pc_partition_chunks(n))
    hist = torch.zeros(max(nbins * nch, 1), dtype=torch.int32, device=dev)
    order = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    if n == 0:
        return order[:0], torch.zeros(nbins + 1, dtype=torch.int32, device=dev)
    keys = keys.contiguous()
    call("pc_partition_hist", ptr(keys), n, nbins, ptr(hist), stream())
    off = scan_i32(hist[:nbins * nch])
    call("pc_partition_place", ptr(keys), n, nbins, ptr(off), ptr(order), stream())
    return order[:n], off[::nch][: nbins + 1]


class CellSort:
    """Stable counting sort of particles into a linked-cell grid.

    K1 ``pc_bin_count`` (cell id + warp-aggregated atomic counts), K2
    ``pc_scan_i32`` (cell offsets), K3 ``pc_bin_place`` (atomic placement +
    per-cell stabilisation).  ``order[dst] = src``.
    """

    def __init__(self, x, x_stride, grid, check_inside=False, stable=True, planar=None):
        dev = x.device
        # planar=(pl, ps, n): bin straight from a planar x | y | z copy
        n = planar[2] if planar is not None else (x.numel() // x_stride if x.numel() else 0)
        self.n = n
        self.grid = grid
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self.cell_of = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        counts = torch.zeros(grid.ncells, dtype=torch.int32, device=dev)
        s = stream()
        if planar is not None:
            call("pc_bin_count_planar", ptr(planar[0]), planar[1], n, grid, ptr(self.cell_of),
                 ptr(counts), ptr(self.flag), s)
        else:
            call("pc_bin_count", ptr(x), n, x_stride, grid, int(check_inside),
                 ptr(self.cell_of), None, ptr(counts), ptr(self.flag), s)
        self.counts = counts
        self.cell_start = scan_i32(counts)
        fill = torch.zeros(grid.ncells, dtype=torch.int32, device=dev)
        self.order = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        if stable:
            tmp = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
            call("pc_bin_place", ptr(self.cell_of), n, ptr(self.cell_start), grid.ncells,
                 ptr(fill), ptr(tmp), ptr(self.order), s)
        else:                        # the caller re-sorts every cell (pc_cell_zsort)
            call("pc_bin_place_unstable", ptr(self.cell_of), n, ptr(self.cell_start),
                 ptr(fill), ptr(self.order), s)

    def outside(self) -> bool:
        return bool(int(self.flag.item()) & _lib.FLAG_OUTSIDE)

    def perm_map(self):
        m = torch.empty(max(self.n, 1), dtype=torch.int64, device=self.order.device)
        call("pc_invert_order", ptr(self.order), self.n, ptr(m), stream())
        return m[:self.n]


def gather_rows(src, order, n, out=None):
    """dst[k] = src[order[k]] for k < n, row-wise (any contiguous row layout)."""
    dst = torch.empty_like(src) if out is None else out
    row_bytes = src[0].numel() * src.element_size() if src.dim() > 1 else src.element_size()
    call("pc_gather_rows", ptr(src), ptr(dst), ptr(order), n, row_bytes, stream())
    return dst


def pack_pos4(x, tags=None):
    """(n, d<=3) FP64 positions -> (n, 4) pos4 with int64 tags in slot 3."""
    x = as_device(x)
    n, d = x.shape
    p = torch.zeros((n, 4), dtype=torch.float64, device=x.device)
    if n:
        p[:, :d] = x          # device copy (plumbing)
        t = torch.arange(n, dtype=torch.int64, device=x.device) if tags is None else tags
        p[:, 3] = t.view(torch.float64) if t.dtype == torch.int64 else t
    return p
