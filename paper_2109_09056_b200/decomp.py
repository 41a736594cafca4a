"""Spatial domain decomposition -- drop-in for ``particula.decomp``.

``DomainFabric``/``decompose`` are host metadata (uniform Cartesian split,
row-major rank ids; ref decomp.py:21-70).  ``migrate``, ``build_halo``,
``halo_gather`` and ``halo_scatter`` keep the reference's in-process
list-of-rank-sets API and its deterministic ordering (arrivals by ascending
source rank, exports by (destination, local index)), with every data-sized
step on the GPU: wrap + ownership (``pc_box_wrap``, ``pc_owner_of``), stable
counting sort by owner, per-image export planning (``pc_halo_plan`` +
``pc_compact``), shifted ghost staging (``pc_gather_shift``) and the
reverse-halo accumulation (``pc_scatter_add``).  The multi-GPU MD engine
(``dist.py``) exchanges the same blocks between processes over NCCL.
"""

from __future__ import annotations

import ctypes
import itertools
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _kernels, _lib
from ._lib import call, ptr, stream
from .aosoa import ParticleSet
from .geometry import Box


@dataclass(frozen=True)
class DomainFabric:
    global_box: Box
    rank_dims: np.ndarray
    periodic: np.ndarray

    def __post_init__(self):
        dims = np.atleast_1d(np.asarray(self.rank_dims, dtype=np.int64))
        per = np.atleast_1d(np.asarray(self.periodic, dtype=bool))
        if dims.shape[0] != self.global_box.ndim or per.shape[0] != self.global_box.ndim:
            raise ValueError("rank_dims/periodic must match box dimensionality")
        if np.any(dims < 1):
            raise ValueError("rank_dims must be >= 1 per axis")
        object.__setattr__(self, "rank_dims", dims)
        object.__setattr__(self, "periodic", per)

    @property
    def n_ranks(self) -> int:
        return int(np.prod(self.rank_dims))

    @property
    def block_lengths(self) -> np.ndarray:
        return self.global_box.lengths / self.rank_dims

    def coords_of(self, rank: int) -> np.ndarray:
        return np.array(np.unravel_index(rank, tuple(self.rank_dims)))

    def rank_of(self, coords) -> int:
        return int(np.ravel_multi_index(tuple(np.asarray(coords)), tuple(self.rank_dims)))

    def local_box(self, rank: int) -> Box:
        c = self.coords_of(rank)
        bl = self.block_lengths
        low = self.global_box.low + c * bl
        high = np.where(c == self.rank_dims - 1, self.global_box.high, low + bl)
        return Box(low, high)

    def pc_grid(self):
        gb = self.global_box
        return _lib.make_grid(gb.low, gb.high, self.block_lengths, self.rank_dims)

    def owner_of(self, x):
        """Owning rank per position (ref decomp.py:58-66), on the device."""
        is_tensor = isinstance(x, torch.Tensor)
        t = _kernels.as_device(x)
        d = self.global_box.ndim
        t = t.reshape(-1, d)
        owners = _owner_tensor(self, t)
        return owners if is_tensor else owners.to(torch.int64).cpu().numpy()


def decompose(global_box: Box, rank_dims, periodic) -> DomainFabric:
    return DomainFabric(global_box, rank_dims, periodic)


def _owner_tensor(fabric: DomainFabric, x: torch.Tensor) -> torch.Tensor:
    n, d = x.shape
    owner = torch.empty(max(n, 1), dtype=torch.int32, device=x.device)
    flag = torch.zeros(1, dtype=torch.int32, device=x.device)
    call("pc_owner_of", ptr(x), n, d, fabric.pc_grid(), ptr(owner), ptr(flag), stream())
    if n and int(flag.item()) & _lib.FLAG_OUTSIDE:
        raise ValueError("position outside global box")
    return owner[:n]


def _group_by(keys: torch.Tensor, nbins: int):
    """Stable grouping of int32 keys in [0, nbins): (order, starts host)
    (ref decomp.py:97-99; pc_partition_*, O(n) at any group size)."""
    if nbins > 256:
        raise ValueError("at most 256 ranks")
    order, starts = _kernels.stable_partition(keys.to(torch.int32), nbins)
    return order, starts.cpu().numpy()[: nbins + 1]


def _field_width(pset: ParticleSet, name: str) -> int:
    return int(np.prod(pset.schema.extent(name), dtype=np.int64))


def _rows_view(t: torch.Tensor, w: int) -> torch.Tensor:
    return t.reshape(t.shape[0], w) if t.numel() else t.reshape(0, w)


def migrate(fabric: DomainFabric, sets, position_field: str = "x") -> None:
    """Move every particle to the rank whose half-open box contains it; each
    destination receives tuples sorted by (source rank, source index)
    (ref decomp.py:77-112)."""
    if len(sets) != fabric.n_ranks:
        raise ValueError("one ParticleSet per rank required")
    gb = fabric.global_box
    d = gb.ndim
    pbox = _lib.make_box(gb.low, gb.high, fabric.periodic)
    outgoing = []
    for pset in sets:
        pset.resize(pset.owned)
        pset.ghosts = 0
        data = {nm: pset.slice(nm).device_values() for nm in pset.schema.names()}
        x = data[position_field].reshape(-1, d).contiguous()
        n = x.shape[0]
        s = stream()
        if n:
            call("pc_box_wrap", ptr(x), n, d, pbox, s)
            flag = torch.zeros(1, dtype=torch.int32, device=x.device)
            call("pc_check_nonperiodic", ptr(x), n, d, pbox, ptr(flag), s)
            if int(flag.item()) & _lib.FLAG_NONPERIODIC:
                bad = int(np.flatnonzero(~fabric.periodic)[0])
                raise ValueError(f"particle outside global box on non-periodic axis {bad}")
        data[position_field] = x.reshape(data[position_field].shape)
        owners = _owner_tensor(fabric, x)
        order, starts = _group_by(owners, fabric.n_ranks)
        outgoing.append((order, starts, data))
    for r, pset in enumerate(sets):
        total = int(sum(st[r + 1] - st[r] for _, st, _ in outgoing))
        pset.resize(total)
        pset.ghosts = 0
        for nm in pset.schema.names():
            w = _field_width(pset, nm)
            view = pset.slice(nm)
            dense = torch.empty((total, w), dtype=view._tdtype, device=pset.device)
            pos = 0
            for order, st, data in outgoing:
                cnt = int(st[r + 1] - st[r])
                if cnt:
                    src = _rows_view(data[nm], w)
                    sel = order[int(st[r]): int(st[r + 1])].contiguous()
                    call("pc_gather_rows", ptr(src), ptr(dense[pos:]), ptr(sel), cnt, 8 * w,
                         stream())
                pos += cnt
            view.device_assign(dense.reshape((total, *view.extent)))


@dataclass
class HaloPlan:
    """Export records per source rank, sorted by (dest, local index)
    (ref decomp.py:123-140).  Host numpy copies mirror the reference fields;
    the device tensors drive the gather/scatter kernels."""
    fabric: DomainFabric
    width: float
    position_field: str
    export_index: list
    export_dest: list
    export_shift: list
    import_layout: list
    owned_snapshot: tuple
    dev_index: list = field(default_factory=list)    # int32 CUDA per source
    dev_shift: list = field(default_factory=list)    # (m, d) f64 CUDA per source
    dest_ranges: list = field(default_factory=list)  # per source {dest: (start, end)}

    def import_total(self, rank: int) -> int:
        return sum(c for _, c in self.import_layout[rank])

    def check_fresh(self, sets) -> None:
        if tuple(p.owned for p in sets) != self.owned_snapshot:
            raise RuntimeError("stale halo plan: particle residency changed since build")


def _halo_offsets(fabric: DomainFabric, r: int):
    """Candidate images of rank r in product order (ref decomp.py:164-194)."""
    d = fabric.global_box.ndim
    L = fabric.global_box.lengths
    dims = fabric.rank_dims
    me = fabric.coords_of(r)
    out = []
    for off in itertools.product(*[(-1, 0, 1)] * d):
        if all(o == 0 for o in off):
            continue
        tgt = me + np.array(off)
        shift = np.zeros(d)
        ok = True
        for a in range(d):
            if 0 <= tgt[a] < dims[a]:
                continue
            if not fabric.periodic[a]:
                ok = False
                break
            if tgt[a] < 0:
                tgt[a] += dims[a]
                shift[a] = L[a]
            else:
                tgt[a] -= dims[a]
                shift[a] = -L[a]
        if not ok:
            continue
        dest = fabric.rank_of(tgt)
        if dest == r:
            continue
        out.append((dest, shift))
    return out


def build_halo(fabric: DomainFabric, sets, width: float, position_field: str = "x") -> HaloPlan:
    """Plan ghost exports: particle -> every adjacent rank whose box is
    within ``width`` (best periodic image per destination), ref decomp.py:143-228."""
    bl = fabric.block_lengths
    if width <= 0:
        raise ValueError("halo width must be positive")
    if width > bl.min() * (1 + 1e-12):
        raise ValueError("halo width exceeds the smallest local box edge")
    d = fabric.global_box.ndim
    w2 = width * width
    exp_idx, exp_dest, exp_shift = [], [], []
    dev_idx, dev_shift, ranges = [], [], []
    for r, pset in enumerate(sets):
        n = pset.owned
        x = _rows_view(pset.slice(position_field).device_values(), d)[:n].contiguous()
        offs = _halo_offsets(fabric, r)
        dests = sorted(set(dst for dst, _ in offs))
        slot_of = {dst: k for k, dst in enumerate(dests)}
        ns = len(dests)
        idx_parts, off_parts, dest_parts = [], [], []
        rng = {}
        if ns and n:
            h_slot = np.array([slot_of[dst] for dst, _ in offs], np.int32)
            h_shift = np.ascontiguousarray(np.stack([s for _, s in offs]), np.float64)
            lo = np.stack([fabric.local_box(dst).low for dst, _ in offs]).astype(np.float64)
            hi = np.stack([fabric.local_box(dst).high for dst, _ in offs]).astype(np.float64)
            lo, hi = np.ascontiguousarray(lo), np.ascontiguousarray(hi)
            flags = torch.empty((ns, n), dtype=torch.int32, device=x.device)
            best = torch.empty((ns, n), dtype=torch.int8, device=x.device)
            call("pc_halo_plan", ptr(x), n, d, len(offs), h_slot.ctypes.data_as(ctypes.c_void_p),
                 h_shift.ctypes.data_as(ctypes.c_void_p), lo.ctypes.data_as(ctypes.c_void_p),
                 hi.ctypes.data_as(ctypes.c_void_p), ns, float(w2), ptr(flags), ptr(best),
                 stream())
            start = 0
            for k, dst in enumerate(dests):
                pos = _kernels.scan_i32(flags[k])
                m = int(pos[n].item())
                ix = torch.empty(max(m, 1), dtype=torch.int32, device=x.device)
                oc = torch.empty(max(m, 1), dtype=torch.int8, device=x.device)
                call("pc_compact", ptr(flags[k]), ptr(pos), n, ptr(ix), ptr(best[k]), ptr(oc),
                     stream())
                idx_parts.append(ix[:m])
                off_parts.append(oc[:m])
                dest_parts.append(np.full(m, dst, np.int64))
                rng[dst] = (start, start + m)
                start += m
            table = torch.as_tensor(h_shift).to(x.device)
            ix = torch.cat(idx_parts) if idx_parts else torch.empty(0, dtype=torch.int32)
            oc = torch.cat(off_parts).to(torch.int64)
            sh = table[oc] if oc.numel() else torch.empty((0, d), dtype=torch.float64,
                                                         device=x.device)
        else:
            ix = torch.empty(0, dtype=torch.int32, device=pset.device)
            sh = torch.empty((0, d), dtype=torch.float64, device=pset.device)
        dev_idx.append(ix.contiguous())
        dev_shift.append(sh.contiguous())
        ranges.append(rng)
        exp_idx.append(ix.to(torch.int64).cpu().numpy())
        exp_dest.append(np.concatenate(dest_parts) if dest_parts else np.empty(0, np.int64))
        exp_shift.append(sh.cpu().numpy())
    layout = [[] for _ in range(fabric.n_ranks)]
    for s in range(fabric.n_ranks):
        for dst, (a, b) in sorted(ranges[s].items()):
            if b > a:
                layout[dst].append((s, b - a))
    for lay in layout:
        lay.sort()
    return HaloPlan(fabric, width, position_field, exp_idx, exp_dest, exp_shift, layout,
                    tuple(p.owned for p in sets), dev_idx, dev_shift, ranges)


def halo_gather(plan: HaloPlan, sets, fields=None) -> None:
    """Append ghost copies after owned particles, positions shifted by their
    image; ghost slots ordered by ascending source rank; unrequested fields
    zero on ghosts (ref decomp.py:231-260)."""
    plan.check_fresh(sets)
    pf = plan.position_field
    if fields is not None and pf not in fields:
        fields = list(fields) + [pf]
    staged = []
    for s, pset in enumerate(sets):
        names = fields if fields is not None else pset.schema.names()
        data = {}
        m = plan.dev_index[s].numel()
        for nm in names:
            w = _field_width(pset, nm)
            src = _rows_view(pset.slice(nm).device_values(), w)
            out = torch.empty((m, w), dtype=src.dtype, device=pset.device)
            if m:
                if src.dtype == torch.float64:
                    sh = plan.dev_shift[s] if nm == pf else None
                    call("pc_gather_shift", ptr(src), ptr(plan.dev_index[s]), m, w, ptr(sh),
                         ptr(out), stream())
                else:
                    call("pc_gather_rows", ptr(src), ptr(out), ptr(plan.dev_index[s]), m, 8 * w,
                         stream())
            data[nm] = out
        staged.append(data)
    for r, pset in enumerate(sets):
        owned = pset.owned
        keep = {nm: pset.slice(nm).device_values()[:owned] for nm in staged[r]}
        total = plan.import_total(r)
        pset.resize(owned)
        pset.resize(owned + total)
        pset.ghosts = total
        for nm in keep:
            view = pset.slice(nm)
            w = _field_width(pset, nm)
            parts = [_rows_view(keep[nm], w)]
            for s, cnt in plan.import_layout[r]:
                a, b = plan.dest_ranges[s][r]
                parts.append(staged[s][nm][a:b])
            view.device_assign(torch.cat(parts).reshape((owned + total, *view.extent)))


def halo_scatter(plan: HaloPlan, sets, fields) -> None:
    """Sum ghost-accumulated values back onto owners in ascending destination
    order, then clear the ghosts (ref decomp.py:263-300)."""
    plan.check_fresh(sets)
    for r, pset in enumerate(sets):
        if pset.size != pset.owned + plan.import_total(r):
            raise RuntimeError("halo_scatter without matching gather")
    base = []
    for r, pset in enumerate(sets):
        b, pos = {}, pset.owned
        for s, cnt in plan.import_layout[r]:
            b[s] = pos
            pos += cnt
        base.append(b)
    for nm in fields:
        snap = [p.slice(nm).device_values() for p in sets]
        for r, pset in enumerate(sets):
            w = _field_width(pset, nm)
            local = _rows_view(snap[r].clone(), w)
            if local.dtype != torch.float64:
                raise TypeError("halo_scatter supports float64 fields")
            for dst in sorted(plan.dest_ranges[r]):
                a, b = plan.dest_ranges[r][dst]
                if b <= a:
                    continue
                src = _rows_view(snap[dst], w)[base[dst][r]: base[dst][r] + (b - a)].contiguous()
                idx = plan.dev_index[r][a:b].contiguous()
                call("pc_scatter_add", ptr(local), ptr(idx), b - a, w, ptr(src), stream())
            if pset.ghosts:
                local[pset.owned:] = 0
            view = pset.slice(nm)
            view.device_assign(local.reshape((pset.size, *view.extent)))
