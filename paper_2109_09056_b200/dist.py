"""Multi-GPU LJ MD by spatial domain decomposition (one rank per GPU).

The reference simulates its ranks in one process (ref decomp.py:1-8, md.py
MDDriver with ``rank_dims``): every rank owns a block of a uniform Cartesian
split, carries ghost copies of the particles within the halo width
``(rc + skin)(1 + 1e-9)`` of its block, migrates particles at every neighbor
rebuild and refreshes ghost positions on every other step, with the cached
halo plan (md.py:169-200).  This module is the same algorithm with one rank
per GPU:

* ``DomainEngine`` -- one rank's device-resident state and phases.  Owned and
  ghost particles share one array sorted by a local linked-cell grid that
  covers the block plus its halo (``binpos``: ghosts shifted by their
  periodic image); the FP64 pair predicate and the forces use the raw
  positions with the global minimum image, exactly the reference's ghost
  convention (md.py:181-188), so the neighbor sets are the single-domain ones.
* phases produce per-destination float64 row blocks ("outboxes") and consume
  per-source blocks ("inboxes") in ascending source order -- the reference's
  deterministic delivery (decomp.py:5-7).
* ``NCCLTransport`` moves the blocks between processes (``torch.distributed``
  send/recv batched per exchange, counts first via all_gather; NCCL over
  NVLink/NVSwitch on a B200 box, gloo in the CPU tests);
  ``FabricMD`` runs all ranks in one process on one device (the reference's
  in-process fabric) by routing the blocks directly.
"""

from __future__ import annotations

import ctypes
import itertools
import os

import numpy as np
import torch

from . import _kernels, _lib
from ._lib import call, ptr, stream
from .decomp import DomainFabric, decompose
from .geometry import Box
from .md import MDConfig, _CUTOFF_MARGIN, _lj_params, _PhaseTimer, _tile_order_kind, \
    _TILE_FUSED_ORDER, fcc_lattice, initial_velocities

MIG_W = 7     # migrate row: x, y, z, vx, vy, vz, gid (int64 bits)
HALO_W = 7    # halo row: x, y, z, gid bits, shift x, y, z


def rank_dims_for(world: int):
    """Rank grid of BASELINE configs: 1 -> 1x1x1, 2 -> 2x1x1, 4 -> 2x2x1, 8 -> 2x2x2."""
    table = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}
    if world in table:
        return table[world]
    dims = [1, 1, 1]
    w, a = world, 0
    for p in (2, 3, 5, 7):
        while w % p == 0:
            dims[a % 3] *= p
            w //= p
            a += 1
    if w != 1:
        dims[0] *= w
    return tuple(dims)


def _as_f64(t):
    return t.view(torch.float64) if t.dtype == torch.int64 else t


class DomainEngine:
    """One rank's particles and kernels (owned + ghost rows in one array)."""

    def __init__(self, cfg: MDConfig, fabric: DomainFabric, rank: int, x, v, gid, device,
                 ell_width: int = 128, planar_gather: bool = True, time_phases: bool = False,
                 tile: bool = True, deterministic: bool = False, half_list: bool = False):
        self.cfg = cfg
        self.fabric = fabric
        self.rank = rank
        self.device = torch.device(device)
        gb = fabric.global_box
        self.box = gb
        self.periodic = np.array(fabric.periodic)
        self.search = (cfg.cutoff + cfg.skin) * _CUTOFF_MARGIN
        self.halo_width = self.search
        if self.halo_width > fabric.block_lengths.min():
            raise ValueError("cutoff + skin exceeds the local box edge for this rank grid")
        self._gbox = _lib.make_box(gb.low, gb.high, self.periodic)
        self._lj = _lj_params(cfg.epsilon, cfg.sigma, cfg.cutoff)
        self._dtm = 0.5 * cfg.dt / cfg.mass
        self._search2 = self.search * self.search
        self._mi_guard = float(cfg.cutoff) * (1.0 + 1e-6) + 1e-9
        self.ell_width = -(-int(ell_width) // 4) * 4
        # deterministic mode: SELL rows in global-id order and
        # per-atom energy rows, reduced in id order by the driver
        self.deterministic = bool(deterministic)
        if self.deterministic:
            tile, planar_gather = False, True
        # Newton-3 half list (K7 + K12): each pair once on exactly one rank
        # (row i owned, neighbour j with gid_j > gid_i, ghost or owned), FP64
        # atomics on both sides, ghost forces sent back to their owners
        # (reverse halo, ref decomp.py:263-300), then the final kick
        self.half = bool(half_list)
        if self.half and self.deterministic:
            raise ValueError("the half-list engine is not deterministic (FP64 atomics)")
        if self.half:
            tile = False
        self.planar_gather = planar_gather or tile
        # tile path (pc_tile.cu, as the single-domain engine): local grid,
        # binpos-staged FP32 prefilter, raw positions + global minimum image
        # for the exact predicate and the force; SELL when the local grid has
        # < 3 cells on an axis or a tile build overflows
        self.tile = bool(tile)
        self.mode = "sell"
        self._q8 = 14
        self._tlist = None
        self._tplan = None
        self.tile_failures = 0
        # tile path: the force epilogue also runs the next step's integrate
        # block into pl_n / vel_n (as MDDriver); `_advanced` marks them valid,
        # `_pos_stale` that pos4 xyz lags behind pl
        self._advanced = False
        self._pos_stale = False
        self._time = time_phases
        self.timer = _PhaseTimer()
        self._local_grid()
        self._offsets = self._halo_offsets()
        n = int(x.shape[0])
        self.cap = 0
        self._alloc(max(64, int(n * 1.6) + 64))
        self.n_owned, self.n_total = n, n
        if n:
            self.pos[:n, :3] = x.to(self.device, torch.float64)
            self.pos[:n, 3] = gid.to(self.device, torch.int64).view(torch.float64)
            self.vel[:, :n] = v.to(self.device, torch.float64).t()
        self.is_ghost = torch.zeros(self.cap, dtype=torch.int32, device=self.device)
        self.flag = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.build_flag = torch.zeros(3, dtype=torch.int32, device=self.device)
        self.export_rows = {}     # dest -> int32 sorted rows (per-step pack)
        self.ghost_blocks = []    # [(src, int32 sorted rows)] ascending src
        self.rebuilds = 0
        self.force_events = None  # optional [(start, end)] CUDA events per force launch
        self.rebuild_events = None  # optional [(sort start, build start, end)] per rebuild

    # ---- geometry -----------------------------------------------------------
    def _local_grid(self):
        """Cells >= search over the block + halo on decomposed axes; the full
        periodic length on undecomposed axes (self-images by min image)."""
        f, gb = self.fabric, self.fabric.global_box
        lb = f.local_box(self.rank)
        lo, hi, per = np.zeros(3), np.zeros(3), np.zeros(3, bool)
        for a in range(3):
            if f.rank_dims[a] == 1:
                lo[a], hi[a], per[a] = gb.low[a], gb.high[a], bool(self.periodic[a])
            else:
                lo[a], hi[a] = lb.low[a] - self.halo_width, lb.high[a] + self.halo_width
        ext = hi - lo
        nc = np.maximum(1, np.floor(ext / self.search).astype(np.int64))
        self.lbox_lo, self.lbox_hi, self.lbox_per = lo, hi, per
        self._lbox = _lib.make_box(lo, hi, per)
        self._grid = _lib.make_grid(lo, hi, ext / nc, nc)

    def _halo_offsets(self):
        f = self.fabric
        d = 3
        L = f.global_box.lengths
        me = f.coords_of(self.rank)
        out = []
        for off in itertools.product((-1, 0, 1), repeat=d):
            if not any(off):
                continue
            tgt = me + np.array(off)
            shift = np.zeros(d)
            ok = True
            for a in range(d):
                if 0 <= tgt[a] < f.rank_dims[a]:
                    continue
                if not f.periodic[a]:
                    ok = False
                    break
                if tgt[a] < 0:
                    tgt[a] += f.rank_dims[a]
                    shift[a] = L[a]
                else:
                    tgt[a] -= f.rank_dims[a]
                    shift[a] = -L[a]
            if not ok:
                continue
            # undecomposed periodic axes wrap inside the local grid: an image
            # shifted along one of them would duplicate the local self-image
            if any(shift[a] != 0 and f.rank_dims[a] == 1 for a in range(d)):
                continue
            dest = f.rank_of(tgt)
            if dest != self.rank:
                out.append((dest, shift))
        # One slot per image (not per destination as in the API's build_halo):
        # when a block is narrower than twice the halo width a particle can be
        # needed on both sides of a neighbour's block.  The reference covers
        # that with one raw-position ghost + global min image (md.py:181-182);
        # binning ghosts in the local frame needs every image within the
        # width.  Duplicate images never pair twice: the build's binpos
        # prefilter only accepts the image adjacent to the row particle.
        # offsets grouped by destination rank (stable: product order within a
        # destination), so one compaction over all offsets yields contiguous
        # per-destination export blocks in the same order as per-offset passes
        out = sorted(out, key=lambda ds: ds[0])
        dests = [dst for dst, _ in out]
        h_slot = np.arange(len(out), dtype=np.int32)
        h_shift = np.ascontiguousarray(np.stack([s for _, s in out])) if out else np.zeros((0, 3))
        lo = np.stack([f.local_box(dst).low for dst, _ in out]) if out else np.zeros((0, 3))
        hi = np.stack([f.local_box(dst).high for dst, _ in out]) if out else np.zeros((0, 3))
        return {"dests": dests, "slot": h_slot, "shift": h_shift.astype(np.float64),
                "lo": np.ascontiguousarray(lo, np.float64),
                "hi": np.ascontiguousarray(hi, np.float64)}

    # ---- storage -------------------------------------------------------------
    def _alloc(self, cap):
        dev = self.device
        old = None
        if self.cap:
            old = (self.pos, self.vel, self.n_total)
        self.cap = int(cap)
        self.pos = torch.zeros((self.cap + 1, 4), dtype=torch.float64, device=dev)
        self.pos[self.cap, :3] = float("nan")
        self.pos[self.cap, 3] = torch.tensor(-1, dtype=torch.int64).view(torch.float64)
        self.binpos = torch.zeros_like(self.pos)
        self.vel = torch.zeros((3, self.cap), dtype=torch.float64, device=dev)
        self.frc = torch.zeros((3, self.cap), dtype=torch.float64, device=dev)
        self.cnt = torch.zeros(self.cap, dtype=torch.int32, device=dev)
        slices = -(-self.cap // 32)
        self.nbr = torch.empty(slices * self.ell_width * 32, dtype=torch.int32, device=dev)
        self.pl = None
        self._ps = -(-(self.cap + 1) // 16) * 16      # planar stride (TMA: 16-element multiple)
        if self.planar_gather:
            self.pl = torch.empty((3, self._ps), dtype=torch.float64, device=dev)
            self.pl[:, self.cap:] = float("nan")
            self.bpl = torch.empty_like(self.pl) if self.tile else None
            self._pl_n = torch.empty_like(self.pl) if self.tile else None
            self._vel_n = torch.empty_like(self.vel) if self.tile else None
        self._nblk = int(_lib.load().pc_lj_force_sell_partials(self.cap))
        self.partial = torch.zeros((self._nblk, 5), dtype=torch.float64, device=dev)
        self.diag = torch.zeros(5, dtype=torch.float64, device=dev)
        if old is not None:
            p, v, n = old
            self.pos[:n] = p[:n]
            self.vel[:, :n] = v[:, :n]

    def _ensure(self, n):
        if n > self.cap:
            keep_ghost = None
            self._alloc(int(n * 1.3) + 64)
            self.is_ghost = torch.zeros(self.cap, dtype=torch.int32, device=self.device)
            del keep_ghost

    def _t0(self):
        return self.timer.start() if self._time else None

    def _t1(self, phase, e0):
        if self._time:
            self.timer.stop(phase, e0)

    # ---- phases --------------------------------------------------------------
    def _sync_pos4(self):
        """pos4 x, y, z <- pl (the fused integrate only writes pl)."""
        if self._pos_stale:
            call("pc_pos_from_planar", ptr(self.pl), self._ps, self.n_total, ptr(self.pos),
                 stream())
            self._pos_stale = False

    def integrate(self):
        if self._advanced:          # done by the previous force epilogue
            self.pl, self._pl_n = self._pl_n, self.pl
            self.vel, self._vel_n = self._vel_n, self.vel
            self._advanced = False
            self._pos_stale = True
            return
        e0 = self._t0()
        self._sync_pos4()
        call("pc_kick_drift_wrap", ptr(self.pos), ptr(self.vel), self.cap, ptr(self.frc),
             self.cap, self.n_total, self._dtm, float(self.cfg.dt), self._gbox, ptr(self.pl),
             self._ps, stream())
        self._t1("integrate", e0)

    def migrate_out(self):
        """Drop ghosts, wrap (done in integrate), owners, stable grouping by
        owner; returns {dest: (m, 7) rows} for dest != self (decomp.py:77-99)."""
        e0 = self._t0()
        self._sync_pos4()
        # owners of every row; ghost rows get the out-of-range key n_ranks, which
        # the partition drops (decomp.py:86-88 drops ghosts before migrating),
        # so stayers and migrants are gathered straight from the current arrays
        n = self.n_total
        x = self.pos[:n, :3].contiguous()
        owner = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        flag = torch.zeros(1, dtype=torch.int32, device=self.device)
        if n:
            # ghost rows: key n_ranks, unchecked (the tile force pass does not
            # advance them; the refresh or this rebuild replaces them)
            call("pc_owner_of_domain", ptr(x), n, 3, self.fabric.pc_grid(),
                 ptr(self.is_ghost) if self.n_total != self.n_owned else None,
                 self.fabric.n_ranks, ptr(owner), ptr(flag), stream())
        # stable grouping by owner (decomp.py:97-99); the group starts and the
        # outside-box flag come back in one device->host read
        nr = self.fabric.n_ranks
        order, starts_d = _kernels.stable_partition(owner[:n], nr)
        host = torch.cat([starts_d.to(torch.int32), flag]).cpu().numpy()
        if host[nr + 1]:
            raise ValueError("position outside global box")
        starts = host[: nr + 1].astype(np.int64)
        self._mig_order, self._mig_starts = order, starts
        out = {}
        # every mover in one pack (owner order, the rank's own stayers cut out),
        # then per-destination views
        r0, r1 = int(starts[self.rank]), int(starts[self.rank + 1])
        movers = [order[: r0], order[r1: int(starts[nr])]]
        movers = [m for m in movers if m.numel()]
        if movers:
            idx = torch.cat(movers) if len(movers) > 1 else movers[0]
            buf = self._pack_mig(idx)
            for dst in range(nr):
                a, b = int(starts[dst]), int(starts[dst + 1])
                if dst == self.rank or b == a:
                    continue
                off = a if dst < self.rank else a - (r1 - r0)
                out[dst] = buf[off: off + (b - a)]
        self._t1("migrate", e0)
        return out

    def _pack_mig(self, rows):
        m = rows.numel()
        buf = torch.empty((m, MIG_W), dtype=torch.float64, device=self.device)
        rows = rows.contiguous()
        p = torch.empty((m, 4), dtype=torch.float64, device=self.device)
        _kernels.gather_rows(self.pos, rows, m, out=p)
        buf[:, 0:3] = p[:, 0:3]
        buf[:, 6] = p[:, 3]
        for a in range(3):
            tmp = torch.empty(m, dtype=torch.float64, device=self.device)
            _kernels.gather_rows(self.vel[a], rows, m, out=tmp)
            buf[:, 3 + a] = tmp
        return buf

    def migrate_in(self, inbox):
        """Arrivals by ascending source rank, own stayers at position rank
        (decomp.py:100-112); stayers are gathered straight into place."""
        e0 = self._t0()
        order, starts = self._mig_order, self._mig_starts
        parts = []                                 # (src, rows or None, m)
        for src in range(self.fabric.n_ranks):
            if src == self.rank:
                m = int(starts[src + 1]) - int(starts[src])
                if m:
                    parts.append((src, None, m))
            elif src in inbox and inbox[src].shape[0]:
                parts.append((src, inbox[src], int(inbox[src].shape[0])))
        n = sum(m for _, _, m in parts)
        self._ensure(n + 1)
        new_pos = torch.empty_like(self.pos)
        new_pos[self.cap] = self.pos[self.cap]
        new_vel = torch.empty_like(self.vel)
        at = 0
        for src, rows, m in parts:
            if rows is None:
                idx = order[int(starts[src]):int(starts[src + 1])].contiguous()
                _kernels.gather_rows(self.pos, idx, m, out=new_pos[at:at + m])
                for a in range(3):
                    _kernels.gather_rows(self.vel[a], idx, m, out=new_vel[a, at:at + m])
            else:
                new_pos[at:at + m, :3] = rows[:, 0:3]
                new_pos[at:at + m, 3] = rows[:, 6]
                new_vel[:, at:at + m] = rows[:, 3:6].t()
            at += m
        self.pos, self.vel = new_pos, new_vel
        self.n_owned = self.n_total = n
        self.is_ghost[: self.cap].zero_()
        self._t1("migrate", e0)

    def halo_out(self):
        """Export plan (best image per destination, d^2 < w^2) and the ghost
        payload per destination (decomp.py:143-228, 231-246)."""
        e0 = self._t0()
        n = self.n_owned
        o = self._offsets
        self._exports = {}
        out = {}
        ns = len(o["dests"])
        if ns == 0 or n == 0:
            self._t1("halo", e0)
            return out
        # fused selection (pc_halo_select_*): per-chunk counts per image slot,
        # one scan, then every exported particle writes its index and ghost
        # row in (slot, index) order -- one host read of the slot bounds
        vp = ctypes.c_void_p
        slot, shift = o["slot"].ctypes.data_as(vp), o["shift"].ctypes.data_as(vp)
        lo, hi = o["lo"].ctypes.data_as(vp), o["hi"].ctypes.data_as(vp)
        w2 = float(self.halo_width * self.halo_width)
        # interior of the own block (shrunk by the width, with margin): its
        # particles are farther than the width from every other block
        lb = self.fabric.local_box(self.rank)
        pad = self.halo_width * (1.0 + 1e-9) + 1e-9 * float(np.max(self.fabric.global_box.lengths))
        self._in_lo = np.ascontiguousarray(lb.low + pad, dtype=np.float64)
        self._in_hi = np.ascontiguousarray(lb.high - pad, dtype=np.float64)
        in_lo, in_hi = self._in_lo.ctypes.data_as(vp), self._in_hi.ctypes.data_as(vp)
        nch = int(_lib.load().pc_halo_select_chunks(n))
        hist = torch.empty(ns * nch, dtype=torch.int32, device=self.device)
        call("pc_halo_select_count", ptr(self.pos), n, 3, len(o["slot"]), slot, shift, lo, hi,
             ns, w2, ptr(hist), stream(), in_lo, in_hi)
        pos = _kernels.scan_i32(hist)
        starts = pos[0: ns * nch + 1: nch].cpu().numpy()        # ns + 1 per-slot bounds
        total = int(starts[ns])
        if total:
            ix_all = torch.empty(total, dtype=torch.int32, device=self.device)
            buf_all = torch.empty((total, HALO_W), dtype=torch.float64, device=self.device)
            call("pc_halo_select_place", ptr(self.pos), n, 3, len(o["slot"]), slot, shift, lo,
                 hi, ns, w2, ptr(pos), ptr(ix_all), ptr(buf_all), stream(), in_lo, in_hi)
            k = 0
            while k < ns:                                       # contiguous per destination
                dst, k1 = o["dests"][k], k
                while k1 < ns and o["dests"][k1] == dst:
                    k1 += 1
                a_, b_ = int(starts[k]), int(starts[k1])
                if b_ > a_:
                    self._exports[dst] = ix_all[a_:b_]
                    out[dst] = buf_all[a_:b_]
                k = k1
        self._t1("halo", e0)
        return out

    def halo_in(self, inbox):
        """Ghosts after owned rows by ascending source (decomp.py:247-260)."""
        e0 = self._t0()
        n = self.n_owned
        blocks = [(src, inbox[src]) for src in sorted(inbox) if inbox[src].shape[0]]
        g = sum(b.shape[0] for _, b in blocks)
        self._ensure(n + g + 1)
        self.binpos[:n] = self.pos[:n]
        at = n
        self._ghost_src = []
        for src, b in blocks:
            self._ghost_src.append((src, at, int(b.shape[0])))
            at += int(b.shape[0])
        if g:                                  # all sources' blocks at once
            b = torch.cat([blk for _, blk in blocks]) if len(blocks) > 1 else blocks[0][1]
            self.pos[n:at] = b[:, 0:4]
            self.binpos[n:at, :3] = b[:, 0:3] + b[:, 4:7]
            self.binpos[n:at, 3] = b[:, 3]
            self.vel[:, n:at] = 0.0
        self.is_ghost[: self.cap].zero_()
        self.is_ghost[n:at] = 1
        self.n_total = at
        self._t1("halo", e0)

    def sort_and_build(self):
        """Stable cell sort of owned + ghost rows on the local grid, then the
        tile (else SELL) Verlet build of all rows (ghost rows emptied)."""
        rev = self.rebuild_events
        if rev is None:
            self._sort_and_build()
            return
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        self._build_mark = ev[1]
        self._sort_and_build()
        ev[2].record()
        rev.append(tuple(ev))

    def _mark_build(self):
        m = getattr(self, "_build_mark", None)
        if m is not None:
            m.record()
            self._build_mark = None

    def _sort_and_build(self):
        n = self.n_total
        s = stream()
        e0 = self._t0()
        tile = self.tile and n > 0 and min(self._grid.nc[0], self._grid.nc[1],
                                           self._grid.nc[2]) >= 3
        srt = _kernels.CellSort(self.binpos[:n], 4, self._grid, stable=not tile)
        order = srt.order
        if tile:
            # z-sorted cells (local frame): the tile path's staged columns and
            # home rows are z-sorted slot runs (pc_tile.cu)
            order = torch.empty_like(srt.order)
            call("pc_cell_zsort", ptr(self.binpos[:, 2]), 4, ptr(srt.cell_start),
                 self._grid.ncells, ptr(srt.order), ptr(order), s)
        new_pos = torch.empty_like(self.pos)
        new_pos[self.cap] = self.pos[self.cap]
        new_bin = torch.empty_like(self.binpos)
        new_vel = torch.zeros_like(self.vel)
        new_g = torch.zeros_like(self.is_ghost)
        self._planar_done = self.pl is not None and getattr(self, "bpl", None) is not None
        if self._planar_done:
            # one pass: pos4, binpos4, velocities, ghost flags + both planar copies
            call("pc_domain_permute", ptr(order), n, ptr(self.pos), ptr(new_pos),
                 ptr(self.binpos), ptr(new_bin), ptr(self.vel), ptr(new_vel),
                 self.vel.stride(0), ptr(self.is_ghost), ptr(new_g), ptr(self.pl),
                 ptr(self.bpl), self._ps, s)
        else:
            _kernels.gather_rows(self.pos, order, n, out=new_pos)
            _kernels.gather_rows(self.binpos, order, n, out=new_bin)
            for a in range(3):
                _kernels.gather_rows(self.vel[a], order, n, out=new_vel[a])
            _kernels.gather_rows(self.is_ghost, order, n, out=new_g)
        self.pos, self.binpos, self.vel, self.is_ghost = new_pos, new_bin, new_vel, new_g
        inv = torch.empty(max(n, 1), dtype=torch.int64, device=self.device)
        call("pc_invert_order", ptr(order), n, ptr(inv), s)
        inv32 = inv[:n].to(torch.int32)
        self.export_rows = {dst: inv32[ix.to(torch.int64)].contiguous()
                            for dst, ix in getattr(self, "_exports", {}).items()}
        self.ghost_blocks = [(src, inv32[at:at + m].contiguous())
                             for src, at, m in getattr(self, "_ghost_src", [])]
        # the per-step refresh as one pack, one all-to-all, one unpack:
        # exported rows concatenated by destination rank, ghost rows by source
        world = self.fabric.n_ranks
        self.send_split = [0] * world
        self.recv_split = [0] * world
        for dst, rows in self.export_rows.items():
            self.send_split[dst] = int(rows.numel())
        for src, rows in self.ghost_blocks:
            self.recv_split[src] = int(rows.numel())
        ex = [self.export_rows[d] for d in sorted(self.export_rows)]
        gh = [rows for _, rows in self.ghost_blocks]
        self.export_all = torch.cat(ex) if ex else torch.empty(0, dtype=torch.int32,
                                                               device=self.device)
        self.ghost_all = torch.cat(gh) if gh else torch.empty(0, dtype=torch.int32,
                                                              device=self.device)
        if self.pl is not None and not self._planar_done:
            call("pc_pos_planar", ptr(self.pos), n, ptr(self.pl), self._ps, s)
        self._t1("sort", e0)
        e0 = self._t0()
        self._mark_build()
        if tile and self._tile_build(srt.cell_start):
            self.rebuilds += 1
            self._t1("neighbor", e0)
            return
        self._sell_build(srt.cell_start)
        self.rebuilds += 1
        self._t1("neighbor", e0)

    def _sell_build(self, cell_start):
        """SELL Verlet build of all rows (ghost rows emptied); also the
        fallback of a failed tile build (verify_build)."""
        n, s = self.n_total, stream()
        self.mode = "half" if self.half else "sell"
        used = ctypes.c_int32(0)
        # half list: the per-particle kernel, whose half test compares global
        # ids (gid_j > gid_i) -- the rule that puts every cross-rank pair on
        # exactly one rank; ghost rows are emptied below
        staged = not self.half
        while True:
            self.build_flag.zero_()
            if staged:
                call("pc_nbr_build_sell", ptr(self.pos), n, ptr(cell_start), self._grid,
                     self._lbox, self._search2, self.ell_width, self.cap, ptr(self.cnt),
                     ptr(self.nbr), ptr(self.build_flag), ctypes.byref(used), s,
                     ptr(self.binpos), self._gbox, 0)
            else:
                call("pc_nbr_build", ptr(self.pos), n, ptr(cell_start), self._grid,
                     self._lbox, self._search2, int(self.half), _lib.PC_NBR_SELL, 0,
                     ptr(self.cnt), None, ptr(self.nbr), self.cap, self.ell_width,
                     ptr(self.build_flag), s, ptr(self.binpos), self._gbox)
            fl = int(self.build_flag[0].item())
            if fl & _lib.FLAG_STAGE:
                staged = False
                continue
            if not (fl & _lib.FLAG_OVERFLOW):
                break
            self.ell_width = -(-(int(self.cnt[:n].max().item()) + 8) // 4) * 4
            slices = -(-self.cap // 32)
            self.nbr = torch.empty(slices * self.ell_width * 32, dtype=torch.int32,
                                   device=self.device)
        self.cnt[:n] *= (1 - self.is_ghost[:n])          # ghost rows carry no list
        if self.deterministic:
            call("pc_sell_sort_by_tag", ptr(self.pos), n, ptr(self.cnt), ptr(self.nbr),
                 self.ell_width, ptr(self.build_flag), s)
            if int(self.build_flag[0].item()) & _lib.FLAG_OVERFLOW:
                raise RuntimeError("deterministic mode: a Verlet row exceeds 256 entries")
        self.used_staged = bool(used.value)

    def _tile_build(self, cell_start) -> bool:
        """Tile round lists of all rows (ghost rows empty, pc_tile_build_domain);
        False (SELL fallback) when a neighbourhood or a row exceeds the tile
        capacities."""
        n, s, dev = self.n_total, stream(), self.device
        lib, g = _lib.load(), self._grid
        if not getattr(self, "_planar_done", False):
            call("pc_pos_planar", ptr(self.binpos), n, ptr(self.bpl), self._ps, s)
        nt = int(lib.pc_tile_count(g))
        rw = torch.empty(nt, dtype=torch.int32, device=dev)
        # rows = owned home particles only (ghost rows carry no list)
        call("pc_tile_rows_domain", ptr(cell_start), g, ptr(self.is_ghost), ptr(rw), s)
        self._rw0 = _kernels.scan_i32(rw)
        bound = n // 32 + nt + 1
        self._ntiles = nt
        if self._tlist is None or self._rounds.numel() < bound:
            self._rounds = torch.empty(bound, dtype=torch.int32, device=dev)
            self._rowidx = torch.empty(bound * 32, dtype=torch.int32, device=dev)
            self._tlist = torch.empty(bound * self._q8 * 512, dtype=torch.uint8, device=dev)
        pi = int(lib.pc_tile_plan_ints())
        if self._tplan is None or self._tplan.numel() < nt * pi:
            self._tplan = torch.empty(nt * pi, dtype=torch.int32, device=dev)
        self._nblk_tile = int(lib.pc_tile_force_partials(nt))
        # two partial blocks: the interior / boundary passes of a split step
        if self.partial.shape[0] < 2 * self._nblk_tile:
            self.partial = torch.zeros((2 * self._nblk_tile, 5), dtype=torch.float64,
                                       device=dev)
        self._tghost = torch.empty(max(nt, 1), dtype=torch.int32, device=dev)
        self.build_flag.zero_()
        kind = _tile_order_kind(self.cfg.rebuild_stride)
        fused = _TILE_FUSED_ORDER and kind == 1
        call("pc_tile_build_ordered", ptr(self.pl), self._ps, ptr(cell_start), g, self._lbox,
             self._search2, self._q8, ptr(self._rw0), ptr(self._tplan), ptr(self._rowidx),
             ptr(self._rounds), ptr(self._tlist), ptr(self.build_flag), s, ptr(self.bpl),
             self._gbox, ptr(self.is_ghost), ptr(self._tghost), 1 if fused else 0)
        # no host read of the build flags here: the step's force is launched
        # speculatively on these lists and verify_build checks the flags after
        # it (a failed build -- a neighbourhood beyond the staging area or a
        # row beyond the list capacity -- redoes list and force on SELL)
        self._spec = True
        self._spec_cell_start = cell_start
        # interior tiles (no ghost staged) first, then boundary tiles, each in
        # ascending tile order; bounds stay on the device ([0, n_int, nt])
        self._tsplit, bounds = _kernels.stable_partition(self._tghost[:nt], 2)
        self._tbounds = bounds.contiguous()          # (a strided view of the scan)
        if not fused:
            call("pc_tile_order", bound, ptr(self._rw0[nt:]), ptr(self._rounds),
                 ptr(self._tlist), self._q8, kind, s)
        self.mode = "tile"
        self.used_staged = True
        return True

    def refresh_out(self):
        """Per-step ghost refresh payload (raw x, y, z of exported rows)."""
        e0 = self._t0()
        out = {}
        for dst, rows in self.export_rows.items():
            m = rows.numel()
            buf = torch.empty((m, 3), dtype=torch.float64, device=self.device)
            if self.pl is not None:
                call("pc_halo_pack_planar", ptr(self.pl), self._ps, ptr(rows), m, ptr(buf),
                     stream())
            else:
                call("pc_halo_pack", ptr(self.pos), ptr(rows), m, ptr(buf), stream())
            out[dst] = buf
        self._t1("halo", e0)
        return out

    def refresh_pack(self):
        """The per-step refresh payload of all destinations in one buffer
        (raw x, y, z of the exported rows, destination-rank order)."""
        e0 = self._t0()
        m = int(self.export_all.numel())
        buf = torch.empty((m, 3), dtype=torch.float64, device=self.device)
        if m:
            call("pc_halo_pack_planar", ptr(self.pl), self._ps, ptr(self.export_all), m,
                 ptr(buf), stream())
        self._t1("halo", e0)
        return buf

    def refresh_unpack(self, buf):
        """Ghost rows of all sources from one received buffer (source order)."""
        e0 = self._t0()
        m = int(self.ghost_all.numel())
        if m:
            call("pc_halo_unpack", ptr(buf), ptr(self.ghost_all), m, ptr(self.pos),
                 ptr(self.pl), self._ps, stream())
        self._t1("halo", e0)

    def refresh_in(self, inbox):
        e0 = self._t0()
        for src, rows in self.ghost_blocks:
            buf = inbox[src]
            call("pc_halo_unpack", ptr(buf), ptr(rows), rows.numel(), ptr(self.pos),
                 ptr(self.pl), self._ps, stream())
        self._t1("halo", e0)

    @property
    def can_split(self) -> bool:
        """The force pass can run as interior + boundary tile passes around
        the ghost refresh (tile path only)."""
        return self.mode == "tile"

    def force(self, kick_dtm, part=None):
        """Force + fused final kick / next integrate.  part: None (all rows),
        "interior" (tiles whose staged neighbourhood holds no ghost: safe while
        the ghost refresh is in flight) or "boundary" (the rest, after the
        refresh) -- each row is computed by the same code either way, so the
        trajectory is bitwise the same as with one pass."""
        e0 = self._t0()
        ev = self.force_events
        if ev is not None:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
        if self.mode == "tile":
            npart = self._nblk_tile
            tiles = trange = None
            out = self.partial
            if part == "interior":
                tiles, trange = self._tsplit, self._tbounds[0:]
            elif part == "boundary":
                tiles, trange = self._tsplit, self._tbounds[1:]
                out = self.partial[npart:]
            elif part is not None:
                raise ValueError(f"unknown force part {part!r}")
            self._split = part is not None
            call("pc_tile_force", ptr(self.pl), self._ps, self._ntiles, ptr(self._tplan),
                 ptr(self._rowidx), ptr(self._rounds), ptr(self._tlist), self._q8, self._gbox,
                 self._lj, self._mi_guard, ptr(self.frc), self.cap, ptr(self.vel), self.cap,
                 float(kick_dtm), float(self.cfg.mass), ptr(out), ptr(self.flag),
                 ptr(self._pl_n), ptr(self._vel_n), self._dtm, float(self.cfg.dt), None,
                 None if tiles is None else ptr(tiles), None if trange is None else ptr(trange),
                 stream())
            if part != "interior":
                self._advanced = True
        elif self.half:
            # local pair forces only: owned and ghost rows accumulate (FP64
            # atomics); reverse_pack / reverse_add and kick() complete the step
            self.frc.zero_()
            call("pc_lj_force_sell_half", ptr(self.pos), self.n_total, ptr(self.cnt),
                 ptr(self.nbr), self.ell_width, self._gbox, self._lj, self._mi_guard,
                 ptr(self.frc), self.cap, ptr(self.partial), ptr(self.flag), stream())
        elif self.deterministic:
            if getattr(self, "_atom", None) is None or self._atom.shape[0] < self.cap:
                self._atom = torch.zeros((self.cap, 5), dtype=torch.float64, device=self.device)
            call("pc_lj_force_sell_atoms", ptr(self.pos), ptr(self.pl), self._ps, self.n_total,
                 ptr(self.cnt), ptr(self.nbr), self.ell_width, self._gbox, self._lj,
                 self._mi_guard, ptr(self.frc), self.cap, ptr(self.vel), self.cap,
                 float(kick_dtm), float(self.cfg.mass), ptr(self._atom), ptr(self.flag),
                 stream())
        else:
            call("pc_lj_force_sell", ptr(self.pos), ptr(self.pl), self._ps, self.n_total,
                 ptr(self.cnt), ptr(self.nbr), self.ell_width, self._gbox, self._lj,
                 self._mi_guard, ptr(self.frc), self.cap, ptr(self.vel), self.cap,
                 float(kick_dtm), float(self.cfg.mass), ptr(self.partial), ptr(self.flag),
                 stream())
        if ev is not None:
            b.record()
            ev.append((a, b))
        self._t1("force", e0)

    def save_spec(self):
        """Before the force on speculatively built tile lists: keep what that
        force changes (velocities: fused kick; error flags)."""
        if getattr(self, "_spec", False):
            self._spec_vel = self.vel.clone()
            self._spec_flag = self.flag.clone()

    def verify_build(self, kick_dtm):
        """After that force: read the tile build's flags (the rebuild's only
        host read of them, with the force already queued); on a failed build
        restore the saved state and redo the list and the force on SELL."""
        if not getattr(self, "_spec", False):
            return
        self._spec = False
        fl = int(self.build_flag[0].item())
        if fl & (_lib.FLAG_STAGE | _lib.FLAG_OVERFLOW):
            self.vel.copy_(self._spec_vel)
            self.flag.copy_(self._spec_flag)
            self._advanced = False
            self.tile_failures += 1
            self._sell_build(self._spec_cell_start)
            self.force(kick_dtm)
        self._spec_vel = self._spec_flag = None

    # ---- half list: reverse halo + kick (K12) ---------------------------------
    def reverse_out(self):
        """Ghost forces per source rank (and cleared on the ghost rows)."""
        e0 = self._t0()
        out = {}
        for src, rows in self.ghost_blocks:
            m = rows.numel()
            buf = torch.empty((m, 3), dtype=torch.float64, device=self.device)
            call("pc_halo_force_pack", ptr(self.frc), self.cap, ptr(rows), m, ptr(buf), stream())
            out[src] = buf
        self._t1("halo", e0)
        return out

    def reverse_in(self, inbox):
        """Add the forces our ghosts received on other ranks onto the owned
        rows they were exported from (halo_scatter, ref decomp.py:281-293)."""
        e0 = self._t0()
        for dst, rows in self.export_rows.items():
            if dst in inbox:
                call("pc_halo_force_add", ptr(self.frc), self.cap, ptr(rows), rows.numel(),
                     ptr(inbox[dst]), stream())
        self._t1("halo", e0)

    def reverse_pack(self):
        """All ghost forces in one buffer (ghost_all: source-rank order)."""
        m = int(self.ghost_all.numel())
        buf = torch.empty((m, 3), dtype=torch.float64, device=self.device)
        if m:
            call("pc_halo_force_pack", ptr(self.frc), self.cap, ptr(self.ghost_all), m,
                 ptr(buf), stream())
        return buf

    def reverse_add(self, buf):
        """Received ghost forces (export_all: destination-rank order) onto owners."""
        m = int(self.export_all.numel())
        if m:
            call("pc_halo_force_add", ptr(self.frc), self.cap, ptr(self.export_all), m,
                 ptr(buf), stream())

    def kick(self, kick_dtm):
        """Final half kick v += dtm f of the half-list step (ghost rows: f = 0
        after reverse_out, so their zero velocities stay) + KE partials."""
        e0 = self._t0()
        nk = int(_lib.load().pc_lj_force_blocks(self.n_total))
        if getattr(self, "partial_k", None) is None or self.partial_k.shape[0] < nk:
            self.partial_k = torch.zeros((max(nk, 1), 5), dtype=torch.float64,
                                         device=self.device)
        call("pc_kick", ptr(self.vel), self.cap, ptr(self.frc), self.cap, self.n_total,
             float(kick_dtm), float(self.cfg.mass), ptr(self.partial_k), stream())
        self._t1("integrate", e0)

    def local_diagnostics(self):
        if self.half:
            # KE / momentum from the kick partials, PE from the force partials
            nb = int(_lib.load().pc_lj_force_sell_partials(self.n_total))
            call("pc_reduce_partials", ptr(self.partial), nb, ptr(self.diag), stream())
            nk = int(_lib.load().pc_lj_force_blocks(self.n_total))
            d = torch.empty(5, dtype=torch.float64, device=self.device)
            call("pc_reduce_partials", ptr(self.partial_k), nk, ptr(d), stream())
            d[1] = self.diag[1]
            self.diag.copy_(d)
            return self.diag
        if self.mode == "tile":
            nb = self._nblk_tile * (2 if getattr(self, "_split", False) else 1)
        else:
            nb = int(_lib.load().pc_lj_force_sell_partials(self.n_total))
        call("pc_reduce_partials", ptr(self.partial), nb, ptr(self.diag), stream())
        return self.diag

    def exact_limbs(self, limbs):
        """Deterministic mode: add this rank's owned per-atom (KE, PE, px, py,
        pz) rows to the exact integer limbs (pc_exact_sum, ghost rows left
        out) -- limbs of all ranks add up to the single-domain limbs."""
        call("pc_exact_sum", ptr(self._atom), self.n_total, 5, ptr(self.is_ghost), ptr(limbs),
             stream())

    def mean_neighbors(self) -> float:
        """Mean Verlet-list length over owned rows (ghost rows are empty)."""
        n = self.n_total
        if self.mode == "tile":
            cnt = torch.zeros(n, dtype=torch.int32, device=self.device)
            table = torch.empty((n, 128), dtype=torch.int32, device=self.device)
            call("pc_tile_decode", self._ntiles, ptr(self._tplan), ptr(self._rowidx),
                 ptr(self._rounds), ptr(self._tlist), self._q8, 128, ptr(cnt), ptr(table),
                 stream())
            total = float(cnt.double().sum().item())
        else:
            total = float(self.cnt[:n].double().sum().item())
        return total / max(1, self.n_owned)

    def neighbor_rows(self):
        """Verlet rows of the current build as host lists of local row
        indices, row = current (cell-sorted) index; ghost rows are empty."""
        n = self.n_total
        out = []
        if self.mode == "tile":
            w = 128
            cnt = torch.zeros(n, dtype=torch.int32, device=self.device)
            table = torch.full((n, w), -1, dtype=torch.int32, device=self.device)
            call("pc_tile_decode", self._ntiles, ptr(self._tplan), ptr(self._rowidx),
                 ptr(self._rounds), ptr(self._tlist), self._q8, w, ptr(cnt), ptr(table),
                 stream())
            c, t = cnt.cpu().numpy(), table.cpu().numpy()
            return [t[a, :c[a]] for a in range(n)]
        Q = self.ell_width // 4
        cnt = self.cnt[:n].cpu().numpy()
        words = self.nbr.cpu().numpy()
        for a in range(n):
            k = np.arange(cnt[a])
            out.append(words[((a >> 5) * Q + (k >> 2)) * 128 + (a & 31) * 4 + (k & 3)])
        return out

    def owned_state(self):
        """(gid, x, v) of owned rows (host numpy)."""
        self._sync_pos4()
        n = self.n_total
        g = self.is_ghost[:n].cpu().numpy().astype(bool)
        p = self.pos[:n].cpu().numpy()
        v = self.vel[:, :n].cpu().numpy().T
        ids = p[:, 3].copy().view(np.int64)
        return ids[~g], p[~g, :3], v[~g]


def _diag_dict(t, n):
    ke, pe = float(t[0]), float(t[1])
    return {"KE": ke, "PE": pe, "E_total": ke + pe, "temperature": 2.0 * ke / (3.0 * n),
            "momentum": t[2:5].copy()}


def _route(outboxes):
    """In-process delivery: inbox[dst][src] = outbox[src][dst]."""
    inboxes = [dict() for _ in outboxes]
    for src, ob in enumerate(outboxes):
        for dst, buf in ob.items():
            inboxes[dst][src] = buf
    return inboxes


class _StepLogic:
    """Shared step schedule (ref md.py:219-257) over phase callbacks."""

    def _rebuild_all(self):
        self._exchange("migrate_out", "migrate_in", MIG_W)
        self._exchange("halo_out", "halo_in", HALO_W)
        for e in self._engines():
            e.sort_and_build()

    # Split the force around the ghost refresh (tile path): interior tiles'
    # pass while the all-to-all is in flight, then the boundary tiles'.  Off
    # by default (PC_OVERLAP=1 or `.overlap = True` turns it on): the split
    # costs a second launch ramp and CTA tail (+35 us per 1M-atom rank per
    # step, profiles/r02l/overlap_timing.txt), and NCCL's all-to-all runs as
    # SM kernels, which cannot start beside the persistent force kernel that
    # holds every SM's registers -- so the exchange does not actually run
    # under the interior pass.
    overlap = os.environ.get("PC_OVERLAP", "0") == "1"

    def step(self, step_index: int):
        for e in self._engines():
            e.integrate()
        if step_index % self.cfg.rebuild_stride == 0:
            self._rebuild_all()
        elif self.overlap and all(e.can_split for e in self._engines()):
            # ref md.py:192-200 (ghost refresh, then forces) with the interior
            # tiles' force overlapping the refresh: pack -> exchange in flight
            # -> interior force -> unpack -> boundary force
            self._refresh_overlapped()
            return
        else:
            self._exchange("refresh_out", "refresh_in", 3)
        self._forces(self._dtm)

    def _forces(self, dtm):
        engines = self._engines()
        for e in engines:
            e.save_spec()
            e.force(dtm)
        if engines and engines[0].half:
            self._reverse()            # ghost forces -> owners (K12)
            for e in engines:
                e.kick(dtm)
        for e in engines:              # after a rebuild: tile build flags
            e.verify_build(dtm)

    def _init_forces(self):
        self._rebuild_all()
        self._forces(0.0)


class FabricMD(_StepLogic):
    """All ranks of a rank grid in one process on one device -- the
    reference's in-process fabric (md.py MDDriver with rank_dims), with GPU
    kernels doing every data-sized step."""

    def __init__(self, cfg: MDConfig, device=None, tile: bool = True,
                 deterministic: bool = False, half_list: bool = False):
        cfg.validate()
        self.deterministic = bool(deterministic)
        self.cfg = cfg
        a = (4.0 / cfg.density) ** (1.0 / 3.0)
        self.box = Box(np.zeros(3), np.full(3, cfg.lattice_cells * a))
        self.periodic = np.array([True, True, True])
        self.fabric = decompose(self.box, cfg.rank_dims, self.periodic)
        self.n = 4 * cfg.lattice_cells ** 3
        self._dtm = 0.5 * cfg.dt / cfg.mass
        dev = device if device is not None else _lib.device()
        x = torch.as_tensor(fcc_lattice(cfg.lattice_cells, a))
        v = torch.as_tensor(initial_velocities(self.n, cfg.temperature, cfg.mass, cfg.seed))
        ids = torch.arange(self.n, dtype=torch.int64)
        self.engines = []
        for r in range(self.fabric.n_ranks):
            if r == 0:
                self.engines.append(DomainEngine(cfg, self.fabric, r, x, v, ids, dev, tile=tile,
                                                 deterministic=deterministic,
                                                 half_list=half_list))
            else:
                z = torch.zeros((0, 3), dtype=torch.float64)
                self.engines.append(DomainEngine(cfg, self.fabric, r, z, z,
                                                 torch.zeros(0, dtype=torch.int64), dev,
                                                 tile=tile, deterministic=deterministic,
                                                 half_list=half_list))
        self._init_forces()

    def _engines(self):
        return self.engines

    def _exchange(self, out_name, in_name, width):
        outs = [getattr(e, out_name)() for e in self.engines]
        for e, inbox in zip(self.engines, _route(outs)):
            getattr(e, in_name)(inbox)

    def _reverse(self):
        outs = [e.reverse_out() for e in self.engines]          # {src: ghost forces}
        for e, inbox in zip(self.engines, _route(outs)):
            e.reverse_in(inbox)

    def _refresh_overlapped(self):
        outs = [e.refresh_out() for e in self.engines]          # packs
        for e in self.engines:
            e.force(self._dtm, part="interior")
        for e, inbox in zip(self.engines, _route(outs)):
            e.refresh_in(inbox)
        for e in self.engines:
            e.force(self._dtm, part="boundary")

    def diagnostics(self):
        if self.deterministic:          # exact per-atom sums, order-independent
            dev = self.engines[0].device
            limbs = torch.zeros(20, dtype=torch.int64, device=dev)
            for e in self.engines:
                if e.n_total:
                    e.exact_limbs(limbs)
            d = torch.zeros(5, dtype=torch.float64, device=dev)
            call("pc_exact_finish", ptr(limbs), 5, ptr(d), stream())
            return _diag_dict(d.cpu().numpy(), self.n)
        tot = sum(e.local_diagnostics().cpu().numpy() for e in self.engines)
        ke, pe = float(tot[0]), float(tot[1])
        return {"KE": ke, "PE": pe, "E_total": ke + pe,
                "temperature": 2.0 * ke / (3.0 * self.n), "momentum": tot[2:5].copy()}

    def gather_state(self):
        x = np.zeros((self.n, 3))
        v = np.zeros((self.n, 3))
        for e in self.engines:
            ids, xs, vs = e.owned_state()
            x[ids] = xs
            v[ids] = vs
        return x, v


class NCCLTransport:
    """Per-destination row blocks between processes with torch.distributed:
    send counts first (all_gather of the count vector), then one batched
    isend/irecv per peer pair.  Works with nccl (GPU) and gloo (CPU tests)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

        # gloo moves host tensors only: stage device blocks through the host
        # (used to run several ranks on one GPU in tests); NCCL sends device
        # memory directly over NVLink
        self.host_staged = dist.get_backend(group) == "gloo"

    def _wire(self, t):
        return t.cpu() if self.host_staged else t

    def counts(self, outbox, device):
        send = torch.zeros(self.world, dtype=torch.int64)
        for dst, buf in outbox.items():
            send[dst] = buf.shape[0]
        send = send if self.host_staged else send.to(device)
        allc = [torch.zeros_like(send) for _ in range(self.world)]
        self.dist.all_gather(allc, send, group=self.group)
        return torch.stack(allc).cpu().numpy()        # [src, dst]

    def exchange(self, outbox, width, device, dtype=torch.float64, recv_counts=None):
        """recv_counts ({src: rows}, e.g. the ghost blocks of the current halo
        plan for the per-step refresh) skips the counts all_gather."""
        c = self.counts(outbox, device) if recv_counts is None else None
        ops, inbox = [], {}
        for peer in range(self.world):
            if peer == self.rank:
                continue
            if c is None:
                m_out = int(outbox[peer].shape[0]) if peer in outbox else 0
                m_in = int(recv_counts.get(peer, 0))
            else:
                m_out = int(c[self.rank, peer])
                m_in = int(c[peer, self.rank])
            if m_out:
                ops.append(self.dist.P2POp(self.dist.isend,
                                           self._wire(outbox[peer].contiguous()), peer,
                                           group=self.group))
            if m_in:
                buf = torch.empty((m_in, width), dtype=dtype,
                                  device="cpu" if self.host_staged else device)
                inbox[peer] = buf
                ops.append(self.dist.P2POp(self.dist.irecv, buf, peer, group=self.group))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()
        if self.host_staged:
            inbox = {k: v.to(device) for k, v in inbox.items()}
        return inbox

    def alltoall(self, send, send_split, recv_split, device):
        """One all_to_all_single of (rows, 3) float64 blocks: rows for rank r
        are send[sum(send_split[:r]) : +send_split[r]]; the received blocks
        come back in source-rank order."""
        out = torch.empty((sum(recv_split), send.shape[1] if send.dim() == 2 else 3),
                          dtype=send.dtype, device="cpu" if self.host_staged else device)
        self.dist.all_to_all_single(out, self._wire(send.contiguous()), list(recv_split),
                                    list(send_split), group=self.group)
        return out.to(device) if self.host_staged else out

    def alltoall_async(self, send, send_split, recv_split, device):
        """alltoall started without blocking the compute stream: returns
        (finish, out); finish() makes the current stream wait for the
        exchange (NCCL: a stream dependency, no host sync) and returns the
        received rows.  gloo moves host tensors, so it completes up front."""
        if self.host_staged:
            out = self.alltoall(send, send_split, recv_split, device)
            return (lambda: out), out
        out = torch.empty((sum(recv_split), send.shape[1] if send.dim() == 2 else 3),
                          dtype=send.dtype, device=device)
        work = self.dist.all_to_all_single(out, send.contiguous(), list(recv_split),
                                           list(send_split), group=self.group, async_op=True)

        def finish():
            work.wait()
            return out
        return finish, out

    def allreduce(self, t):
        w = self._wire(t)
        self.dist.all_reduce(w, group=self.group)
        if w is not t:
            t.copy_(w)
        return t


class _Raw:
    """A device address where the C-ABI shims expect a tensor (ptr(t))."""

    def __init__(self, addr: int):
        self.addr = int(addr)

    def data_ptr(self) -> int:
        return self.addr


def p2p_plan(C, me: int):
    """Addressing of one rank's peer-memory all-to-all from the split matrix
    C[src, dst] (rows src sends to dst): the rank's send buffer holds its
    rows in destination order, and every receive window holds the rows of
    all sources in source order (the all_to_all_single layout).  Returns
    {"puts": [(dst, src0, count, dst0)], "dsts", "srcs"}: the put to dst
    copies send rows [src0, src0 + count) to window rows [dst0, dst0 + count)."""
    C = np.asarray(C, np.int64)
    world = C.shape[0]
    src0 = np.concatenate(([0], np.cumsum(C[me])))[:-1]
    dsts = [d for d in range(world) if C[me, d] > 0]
    srcs = [s for s in range(world) if C[s, me] > 0]
    puts = [(d, int(src0[d]), int(C[me, d]), int(C[:me, d].sum())) for d in dsts]
    return {"puts": puts, "dsts": dsts, "srcs": srcs}


class P2PTransport(NCCLTransport):
    """NCCLTransport whose per-step all-to-alls (the ghost refresh of
    md.py:192-200 / decomp.py:231-260 and the reverse halo of
    decomp.py:263-300) move rows by direct peer-memory stores between the
    ranks' processes (CUDA IPC windows, NVLink), with device-side arrival /
    acknowledgement flags -- no NCCL kernel and no host round trip per step
    (pc_p2p_*, csrc/pc_p2p.cu).  The rebuild-time exchanges (counts,
    migrate, halo plan) stay on torch.distributed.

    A channel is prepared collectively after every rebuild with the new
    split sizes (``prepare``); windows are sized to the largest receive of
    any rank and re-allocated (all ranks together) only when that grows.
    Per call k: acknowledge step k - 1's unpack to its sources, wait until
    every destination acknowledged step k - 2 (parity reuse), store this
    rank's rows into each destination's parity-(k & 1) block, raise the
    destinations' arrival flags, wait for every source's step-k flag."""

    SPIN_LIMIT = 1 << 25          # x 200 ns: ~7 s before a wait reports failure

    def __init__(self, group=None):
        super().__init__(group)
        self._chan = {}
        self._peer_maps = {}      # (rank, handle bytes) -> mapped address

    # -- collective plan -------------------------------------------------
    def _allgather_bytes(self, b: bytes):
        out = [None] * self.world
        self.dist.all_gather_object(out, b, group=self.group)
        return out

    def prepare(self, key, send_split, recv_split, width, device):
        """Collective: every rank calls it with its own split sizes (rows to /
        from each rank, rank order).  Returns nothing; raises if a previous
        wait of this channel failed."""
        lib = _lib.load()
        torch.cuda.synchronize()
        ch = self._chan.get(key)
        if ch is not None:
            self._check(ch)
        send = np.asarray(list(send_split), np.int64)
        rows = self._allgather_bytes(send.tobytes())
        C = np.stack([np.frombuffer(r, np.int64) for r in rows])      # [src, dst]
        need = int(C.sum(axis=0).max())
        me, world = self.rank, self.world
        if ch is None or ch["cap"] < need or ch["width"] != width:
            if ch is not None:
                self.dist.barrier(group=self.group)       # nobody writes the old windows now
                self._free(ch)
            cap = int(need * 1.25) + 64
            win = ctypes.c_void_p()
            h = ctypes.create_string_buffer(int(lib.pc_p2p_handle_bytes()))
            _lib.check(lib.pc_p2p_window_alloc(cap, width, world, ctypes.byref(win), h),
                       "pc_p2p_window_alloc")
            handles = self._allgather_bytes(h.raw)
            peers = {}
            for r in range(world):
                if r == me:
                    peers[r] = int(win.value)
                    continue
                hb = handles[r]
                if (r, hb) not in self._peer_maps:
                    addr = ctypes.c_void_p()
                    buf = ctypes.create_string_buffer(hb, len(hb))
                    _lib.check(lib.pc_p2p_open(buf, ctypes.byref(addr)), "pc_p2p_open")
                    self._peer_maps[(r, hb)] = int(addr.value)
                peers[r] = self._peer_maps[(r, hb)]
            ch = {"cap": cap, "width": width, "window": int(win.value), "peers": peers,
                  "handles": handles, "step": 0,
                  "err": torch.zeros(1, dtype=torch.int32, device=device)}
            self._chan[key] = ch
        cap = ch["cap"]
        arrive = 2 * cap * width                 # flag regions, in doubles from the base
        ch["arrive_off"], ch["ack_off"] = arrive, arrive + world
        plan = p2p_plan(C, me)
        dsts, srcs = plan["dsts"], plan["srcs"]
        rec = np.dtype([("w", np.uint64), ("src0", np.int64), ("count", np.int64),
                        ("dst0", np.int64)])
        assert rec.itemsize == int(lib.pc_p2p_dest_bytes())
        tabs = []
        for par in (0, 1):
            t = np.zeros(len(dsts), rec)
            for i, (d, src0, cnt, dst0) in enumerate(plan["puts"]):
                t[i] = (ch["peers"][d], src0, cnt, dst0 + par * cap)
            tabs.append(torch.from_numpy(t.view(np.uint8).copy()).to(device))
        ack = np.zeros(len(srcs), rec)
        for i, s in enumerate(srcs):
            ack[i] = (ch["peers"][s], 0, 0, 0)
        ch.update(put=tabs, n_dst=len(dsts), max_rows=int(C[me].max()) if world else 0,
                  ack_tab=torch.from_numpy(ack.view(np.uint8).copy()).to(device),
                  n_src=len(srcs),
                  dst_ranks=torch.tensor(dsts, dtype=torch.int32, device=device),
                  src_ranks=torch.tensor(srcs, dtype=torch.int32, device=device),
                  recv_rows=int(C[:, me].sum()), send=tuple(send.tolist()),
                  recv=tuple(int(v) for v in recv_split))
        torch.cuda.synchronize()
        self.dist.barrier(group=self.group)

    def _check(self, ch):
        if int(ch["err"].item()):
            raise RuntimeError("P2P halo exchange: a peer flag wait timed out")

    def _free(self, ch):
        lib = _lib.load()
        for (r, hb), addr in list(self._peer_maps.items()):
            if r != self.rank and ch["handles"][r] == hb:
                _lib.check(lib.pc_p2p_close(ctypes.c_void_p(addr)), "pc_p2p_close")
                del self._peer_maps[(r, hb)]
        _lib.check(lib.pc_p2p_window_free(ctypes.c_void_p(ch["window"])), "pc_p2p_window_free")

    # -- per step ----------------------------------------------------------
    def channel_alltoall(self, key, send):
        """The prepared channel's all-to-all of ``send`` ((rows, width) f64,
        destination-rank order, the prepared split sizes): returns the
        received rows (source-rank order) as a device address in this rank's
        window, valid until this channel's call after next."""
        self.channel_send(key, send)
        return self.channel_recv(key)

    def channel_send(self, key, send, rows=None, planar=None):
        """First half of channel_alltoall: acknowledge, wait for the parity
        block, store, raise the arrival flags (the stream does not wait for
        the sources yet -- work enqueued next overlaps their stores).  With
        `rows` and `planar` = (tensor, stride) instead of `send`: the rows'
        x, y, z are gathered from the planar positions inside the put
        (pc_p2p_pack_put, the fused pack of SURVEY §8 K11)."""
        ch = self._chan[key]
        s = stream()
        ch["step"] += 1
        k = ch["step"]
        if k > 1:      # the previous step's rows are unpacked (stream order): acknowledge
            call("pc_p2p_signal", ptr(ch["ack_tab"]), ch["n_src"], ch["ack_off"], self.rank,
                 k - 1, s)
        if k > 2:      # destinations have unpacked step k - 2 (this parity block is free)
            call("pc_p2p_wait", ctypes.c_void_p(ch["window"]), ch["ack_off"], ptr(ch["dst_ranks"]),
                 ch["n_dst"], k - 2, ptr(ch["err"]), self.SPIN_LIMIT, s)
        tab = ch["put"][k & 1]
        if rows is not None:
            call("pc_p2p_pack_put", ptr(planar[0]), planar[1], ptr(rows), ptr(tab), ch["n_dst"],
                 ch["max_rows"], 0, 0, s)
        else:
            call("pc_p2p_put", ptr(send), ptr(tab), ch["n_dst"], ch["max_rows"], ch["width"],
                 0, 0, s)
        call("pc_p2p_signal", ptr(tab), ch["n_dst"], ch["arrive_off"], self.rank, k, s)

    def channel_recv(self, key):
        """Second half: the stream waits for every source's step flag; the
        received rows' address."""
        ch = self._chan[key]
        k = ch["step"]
        call("pc_p2p_wait", ctypes.c_void_p(ch["window"]), ch["arrive_off"], ptr(ch["src_ranks"]),
             ch["n_src"], k, ptr(ch["err"]), self.SPIN_LIMIT, stream())
        return _Raw(ch["window"] + (k & 1) * ch["cap"] * ch["width"] * 8)

    def check_errors(self):
        for ch in self._chan.values():
            self._check(ch)


def local_block(cfg: MDConfig, cells, rank_dims, rank: int):
    """This rank's block of the fcc lattice (ids = the global lattice order)
    with per-rank seeded velocities, as numpy (x, v, ids): the input of a run
    too large for one global velocity stream (DistMD(local_init=True), or
    `state=` from the host)."""
    cells = np.asarray(cells, np.int64)
    dims = np.asarray(rank_dims, np.int64)
    a = (4.0 / cfg.density) ** (1.0 / 3.0)
    c = np.array(np.unravel_index(rank, tuple(dims)), np.int64)
    per = cells // dims
    lo = c * per
    hi = np.where(c == dims - 1, cells, lo + per)
    gx, gy, gz = np.meshgrid(*[np.arange(lo[k], hi[k]) for k in range(3)], indexing="ij")
    corner = np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1)
    basis = np.array([[0, 0, 0], [0.5, 0.5, 0], [0.5, 0, 0.5], [0, 0.5, 0.5]])
    x = (corner[:, None, :] + basis[None]).reshape(-1, 3) * a
    flat = (corner[:, 0] * cells[1] + corner[:, 1]) * cells[2] + corner[:, 2]
    ids = (flat[:, None] * 4 + np.arange(4)[None]).reshape(-1).astype(np.int64)
    v = initial_velocities(x.shape[0], cfg.temperature, cfg.mass, cfg.seed * 1000003 + rank)
    return x, v, ids


class DistMD(_StepLogic):
    """One rank per GPU under torch.distributed (launch with torchrun)."""

    def __init__(self, cfg: MDConfig, cells=None, transport=None, device=None,
                 local_init: bool = False, time_phases: bool = False,
                 deterministic: bool = False, half_list: bool = False, state=None):
        """`state`: this rank's own atoms as host (ideally pinned) tensors
        (x, v, ids) -- e.g. `local_block(...)` -- instead of building them
        here; rows owned by another rank move there at the first migrate."""
        import torch.distributed as dist
        cfg.validate()
        self.cfg = cfg
        self.transport = transport if transport is not None else NCCLTransport()
        world, rank = self.transport.world, self.transport.rank
        if tuple(cfg.rank_dims) != (1, 1, 1) and int(np.prod(cfg.rank_dims)) != world:
            raise ValueError(f"rank_dims {tuple(cfg.rank_dims)} do not match the world "
                             f"size {world}")
        dims = tuple(cfg.rank_dims) if int(np.prod(cfg.rank_dims)) == world \
            else rank_dims_for(world)
        cells = np.array(cells if cells is not None else [cfg.lattice_cells] * 3, np.int64)
        a = (4.0 / cfg.density) ** (1.0 / 3.0)
        self.box = Box(np.zeros(3), cells * a)
        self.periodic = np.array([True, True, True])
        self.fabric = decompose(self.box, dims, self.periodic)
        self.n = int(4 * np.prod(cells))
        self._dtm = 0.5 * cfg.dt / cfg.mass
        self.device = torch.device(device) if device is not None else _lib.device()
        if state is not None:
            x, v, ids = (t if isinstance(t, torch.Tensor) else torch.as_tensor(t) for t in state)
        else:
            x, v, ids = self._initial(cells, a, rank, local_init)
        self.deterministic = bool(deterministic)
        self.engine = DomainEngine(cfg, self.fabric, rank, x, v, ids, self.device,
                                   time_phases=time_phases, deterministic=deterministic,
                                   half_list=half_list)
        self._init_forces()
        del dist

    def _initial(self, cells, a, rank, local_init):
        """Reference-identical global init (md.py:67-86) kept by owner, or a
        per-rank lattice block with per-rank seeded velocities (local_init,
        for runs too large to build one global velocity stream)."""
        cfg = self.cfg
        if not local_init:
            if len(set(cells.tolist())) != 1:
                raise ValueError("global init needs a cubic lattice; use local_init")
            x = fcc_lattice(int(cells[0]), a)
            v = initial_velocities(self.n, cfg.temperature, cfg.mass, cfg.seed)
            ids = np.arange(self.n, dtype=np.int64)
            owner = self.fabric.owner_of(x) if self.n else np.zeros(0, np.int64)
            keep = owner == rank
            return (torch.as_tensor(x[keep]), torch.as_tensor(v[keep]),
                    torch.as_tensor(ids[keep]))
        return tuple(torch.as_tensor(t) for t in
                     local_block(cfg, cells, self.fabric.rank_dims, rank))

    def _engines(self):
        return [self.engine]

    @property
    def _p2p(self) -> bool:
        return isinstance(self.transport, P2PTransport)

    def _rebuild_all(self):
        super()._rebuild_all()
        if self._p2p:
            # the per-step channels follow the new halo plan (collective)
            e = self.engine
            self.transport.prepare("refresh", e.send_split, e.recv_split, 3, self.device)
            if e.half:
                self.transport.prepare("reverse", e.recv_split, e.send_split, 3, self.device)

    def _p2p_refresh_send(self):
        """Refresh over the peer-memory channel: the exported rows' x, y, z
        gathered from the planar positions inside the put (fused pack), or
        packed first when the engine has no planar copy."""
        e = self.engine
        if e.pl is not None:
            self.transport.channel_send("refresh", None, rows=e.export_all,
                                        planar=(e.pl, e._ps))
        else:
            self.transport.channel_send("refresh", e.refresh_pack())

    def _reverse(self):
        """Ghost forces back to their owners: one all-to-all, the transpose of
        the per-step refresh (split sizes swapped)."""
        e = self.engine
        buf = e.reverse_pack()
        if self._p2p:
            e.reverse_add(self.transport.channel_alltoall("reverse", buf))
            return
        e.reverse_add(self.transport.alltoall(buf, e.recv_split, e.send_split, self.device))

    def _refresh_overlapped(self):
        """Pack, start the all-to-all (NCCL stream; P2P: the stores and
        flags), interior force on the compute stream meanwhile, then wait,
        unpack, boundary force."""
        e = self.engine
        if self._p2p:
            self._p2p_refresh_send()
            e.force(self._dtm, part="interior")
            e.refresh_unpack(self.transport.channel_recv("refresh"))
            e.force(self._dtm, part="boundary")
            return
        buf = e.refresh_pack()
        work, recv = self.transport.alltoall_async(buf, e.send_split, e.recv_split, self.device)
        e.force(self._dtm, part="interior")
        e.refresh_unpack(work())
        e.force(self._dtm, part="boundary")

    def _exchange(self, out_name, in_name, width):
        e = self.engine
        if out_name == "refresh_out":
            # per step: one pack, one all-to-all (sizes fixed by the halo plan
            # until the next rebuild), one unpack -- a few host calls per step
            # whatever the number of neighbour ranks
            if self._p2p:
                self._p2p_refresh_send()
                e.refresh_unpack(self.transport.channel_recv("refresh"))
                return
            buf = e.refresh_pack()
            e.refresh_unpack(self.transport.alltoall(buf, e.send_split, e.recv_split,
                                                      self.device))
            return
        out = getattr(e, out_name)()
        inbox = self.transport.exchange(out, width, self.device)
        getattr(e, in_name)(inbox)

    def diagnostics(self):
        if self._p2p:
            self.transport.check_errors()
        if self.deterministic:
            # exact integer limbs per rank, summed over ranks (20 int64): the
            # energies equal the single-domain ones bit for bit
            limbs = torch.zeros(20, dtype=torch.int64, device=self.device)
            if self.engine.n_total:
                self.engine.exact_limbs(limbs)
            self.transport.allreduce(limbs)
            d = torch.zeros(5, dtype=torch.float64, device=self.device)
            call("pc_exact_finish", ptr(limbs), 5, ptr(d), stream())
            return _diag_dict(d.cpu().numpy(), self.n)
        d = self.engine.local_diagnostics().clone()
        self.transport.allreduce(d)
        t = d.cpu().numpy()
        ke, pe = float(t[0]), float(t[1])
        return {"KE": ke, "PE": pe, "E_total": ke + pe,
                "temperature": 2.0 * ke / (3.0 * self.n), "momentum": t[2:5].copy()}
