"""Lennard-Jones NVE mini-MD on the GPU -- drop-in for ``particula.md``.

Same public surface as ref md.py (``MD_SCHEMA``, ``MDConfig``,
``fcc_lattice``, ``initial_velocities``, ``lj_pair``, ``lj_forces``,
``MDDriver``, ``run_md``) and the same step semantics (md.py:219-257):

    integrate   v += dt/2m f ; x += dt v ; wrap          pc_kick_drift_wrap
    rebuild     (every rebuild_stride) cell sort +        pc_bin_* , pc_gather_rows,
                Verlet build at (rc+skin)(1+1e-9)          pc_nbr_build (ELL)
    force       exact-rc LJ + fused final half kick +     pc_lj_force
                KE/PE/momentum block partials

Device layout (HBM, capacity ``cap``):
    pos  (cap, 4) f64   x, y, z, global id (int64 bits)  -- 32 B gathers
    vel  (3, cap) f64   planar
    frc  (3, cap) f64   planar (FP64-accumulated, antisymmetric pair terms)
    nbr  (W, cap) i32   transposed ELL Verlet list, cnt (cap,) i32

Particles are re-sorted by cell at every rebuild (physics-transparent: the
reference sums forces in global-id order and energies by id, md.py:7-11), so
the 27 stencil cells of a particle are contiguous index ranges.

The initial lattice and Gaussian velocities are built on the host exactly as
the reference does (md.py:67-86) and uploaded once.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

# round order of the tile lists (PC_TILE_ORDER overrides: 0 off, 1 round-robin, 2 class-major)
_TILE_ORDER_ENV = os.environ.get("PC_TILE_ORDER")
# PC_TILE_FUSED=1: the round-robin order applied inside the build
# (pc_tile_build_ordered) instead of the separate pc_tile_order pass -- the
# same lists, but slower: C3 build + order 7.32 vs 5.58 ms (nine build warps
# instead of ten; the order's ALU work does not hide behind the build's
# latency, profiles/r02aa)
_TILE_FUSED_ORDER = os.environ.get("PC_TILE_FUSED", "0") == "1"


def _tile_order_kind(rebuild_stride: int) -> int:
    """Round order of the tile lists: residue round-robin (1) when the list
    is reused for >= 5 steps, else the build's ascending order (0).  At C3
    the r02 order pass costs ~1.5 ms per rebuild and saves ~340 us in every
    force pass (1424 -> 1070 us): hot config (T = 3, rebuild 5) 3.69e9 vs
    3.64e9 atom-steps/s (profiles/r02ab; with the r01 order pass rebuild 5
    was a loss, r01k)."""
    if _TILE_ORDER_ENV is not None:
        return int(_TILE_ORDER_ENV)
    return 1 if rebuild_stride >= 5 else 0

from . import _kernels, _lib, aosoa, decomp
from ._lib import call, ptr, stream
from .geometry import Box, cube
from .neighbors import VerletList, neighbor_grid

MD_SCHEMA = aosoa.schema(
    x=("float64", (3,)),
    x0=("float64", (3,)),
    v=("float64", (3,)),
    f=("float64", (3,)),
    id=("int64", ()),
)

_CUTOFF_MARGIN = 1.0 + 1e-9          # ref md.py:32-34

PHASES = ("integrate", "sort", "migrate", "halo", "neighbor", "force")


@dataclass
class MDConfig:
    """ref md.py:37-64 (same fields, defaults and validation)."""
    lattice_cells: int = 4
    density: float = 0.8442
    temperature: float = 0.8
    dt: float = 0.005
    steps: int = 100
    cutoff: float = 2.5
    skin: float = 0.0
    rebuild_stride: int = 1
    sort_stride: int = 0
    seed: int = 1
    vector_length: int = 16
    rank_dims: tuple = (1, 1, 1)
    epsilon: float = 1.0
    sigma: float = 1.0
    mass: float = 1.0

    def validate(self):
        if self.rebuild_stride > 1 and self.skin <= 0:
            raise ValueError("rebuild_stride > 1 requires a positive skin")
        if self.sort_stride and self.sort_stride % self.rebuild_stride:
            raise ValueError("sort_stride must be a multiple of rebuild_stride")
        for name in ("lattice_cells", "steps", "vector_length", "rebuild_stride"):
            if getattr(self, name) < 1 and name != "steps":
                raise ValueError(f"{name} must be >= 1")
        if self.dt <= 0 or self.cutoff <= 0 or self.density <= 0:
            raise ValueError("dt, cutoff and density must be positive")


def fcc_lattice(cells: int, spacing: float) -> np.ndarray:
    """4-atom FCC basis on a cells^3 grid, ij-meshgrid order (ref md.py:67-74)."""
    basis = np.array([[0, 0, 0], [0.5, 0.5, 0], [0.5, 0, 0.5], [0, 0.5, 0.5]], dtype=np.float64)
    ax = np.arange(cells)
    gx, gy, gz = np.meshgrid(ax, ax, ax, indexing="ij")
    corners = np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1)
    return (corners[:, None, :] + basis[None, :, :]).reshape(-1, 3) * spacing


def initial_velocities(n: int, temperature: float, mass: float, seed: int) -> np.ndarray:
    """Seeded PCG64 Gaussian velocities, zero momentum, exact-T rescale (ref md.py:77-86)."""
    v = np.random.default_rng(seed).normal(size=(n, 3))
    v -= v.mean(axis=0)
    ke = 0.5 * mass * np.einsum("ij,ij->", v, v)
    if ke > 0:
        v *= np.sqrt(1.5 * n * temperature / ke)
    return v


def lj_pair(dx, r2, eps: float, sigma: float):
    """Pair energies and force on i for dx = xj - xi (ref md.py:89-96), FP64 on device."""
    is_tensor = isinstance(dx, torch.Tensor)
    d = _kernels.as_device(dx).reshape(-1, 3)
    q = _kernels.as_device(r2).reshape(-1)
    n = q.numel()
    e = torch.empty(max(n, 1), dtype=torch.float64, device=d.device)
    f = torch.empty((max(n, 1), 3), dtype=torch.float64, device=d.device)
    call("pc_lj_pair", ptr(d), ptr(q), n, float(eps), float(sigma), ptr(e), ptr(f), stream())
    e, f = e[:n], f[:n]
    return (e, f) if is_tensor else (e.cpu().numpy(), f.cpu().numpy())


def _lj_params(eps, sigma, cutoff) -> "_lib.PcLJ":
    p = _lib.PcLJ()
    p.epsilon, p.sigma = float(eps), float(sigma)
    p.cutoff2 = float(cutoff) * float(cutoff)
    p.overlap2 = (1e-10 * float(sigma)) ** 2
    return p


def lj_forces(x_phys, ids, owned: int, vlist: VerletList, box: Box, periodic, eps: float,
              sigma: float, cutoff: float):
    """Canonical LJ forces / per-particle energies for the first ``owned`` rows
    (ref md.py:99-126): exact-cutoff re-filter in FP64, each pair energy booked
    on the smaller global id.  FP32 pair arithmetic (tolerance 1e-5)."""
    is_tensor = isinstance(x_phys, torch.Tensor)
    x = _kernels.as_device(x_phys)
    tags = _kernels.as_device(ids, dtype=torch.int64)
    pos4 = _kernels.pack_pos4(x, tags)
    counts, offsets, index = vlist.device_csr()
    per = np.broadcast_to(np.asarray(periodic, bool), (box.ndim,))
    pbox = _lib.make_box(box.low, box.high, per)
    owned = int(owned)
    dev = x.device
    f64 = torch.zeros((max(owned, 1), 3), dtype=torch.float64, device=dev)
    pe = torch.zeros(max(owned, 1), dtype=torch.float64, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    call("pc_lj_force", ptr(pos4), owned, ptr(counts), ptr(offsets), ptr(index), 0, pbox,
         _lj_params(eps, sigma, cutoff), None, 0, ptr(f64), ptr(pe), None, 0, 0.0, 1.0, None,
         ptr(flag), stream())
    if int(flag.item()) & _lib.FLAG_OVERLAP:
        raise FloatingPointError("overlapping particles in LJ kernel")
    f64, pe = f64[:owned], pe[:owned]
    return (f64, pe) if is_tensor else (f64.cpu().numpy(), pe.cpu().numpy())


class _PhaseTimer:
    """Per-phase CUDA-event timing in the reference's six buckets (md.py:158-159)."""

    def __init__(self):
        self.totals = {k: 0.0 for k in PHASES}
        self._pending = []

    def start(self):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    def stop(self, phase, e0):
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()
        self._pending.append((phase, e0, e1))
        if len(self._pending) > 4096:
            self.resolve()

    def resolve(self):
        if self._pending:
            self._pending[-1][2].synchronize()
            for phase, a, b in self._pending:
                self.totals[phase] += a.elapsed_time(b) * 1e-3
            self._pending = []
        return dict(self.totals)

    def reset(self):
        self.resolve()
        self.totals = {k: 0.0 for k in PHASES}


class MDDriver:
    """Device-resident velocity-Verlet LJ driver (ref md.py:129-292).

    ``rank_dims`` is validated exactly as the reference does (halo width vs
    block edge, md.py:140-142); one driver owns the whole box on one GPU --
    the physics is decomposition-independent by the reference's own contract
    (md.py:7-11).  Multi-GPU runs use ``paper_2109_09056_b200.dist``.
    """

    def __init__(self, cfg: MDConfig, device=None, ell_width: int = 128,
                 time_phases: bool = True, state=None, planar_gather: bool = True,
                 tile: bool = True, half_list: bool = False, deterministic: bool = False):
        cfg.validate()
        # deterministic mode: SELL rows in global-id order,
        # per-atom energies reduced in id order -- bitwise equal to FabricMD /
        # DistMD(deterministic=True) on any rank grid
        self.deterministic = bool(deterministic)
        if self.deterministic:
            tile, half_list = False, False
        self.cfg = cfg
        a = (4.0 / cfg.density) ** (1.0 / 3.0)
        self.box = cube(cfg.lattice_cells * a)
        self.periodic = np.array([True, True, True])
        self.n = 4 * cfg.lattice_cells ** 3
        self.fabric = decomp.decompose(self.box, cfg.rank_dims, self.periodic)
        halo_w = (cfg.cutoff + cfg.skin) * _CUTOFF_MARGIN
        if halo_w > self.fabric.block_lengths.min():
            raise ValueError("cutoff + skin exceeds the local box edge for this rank grid")
        self.halo_width = halo_w
        self.search = (cfg.cutoff + cfg.skin) * _CUTOFF_MARGIN
        if self.search > 0.5 * self.box.lengths.min():
            raise ValueError("cutoff exceeds half the box length on a periodic axis")
        self.device = torch.device(device) if device is not None else _lib.device()
        self._pbox = _lib.make_box(self.box.low, self.box.high, self.periodic)
        self._lj = _lj_params(cfg.epsilon, cfg.sigma, cfg.cutoff)
        _nc, _w, self._grid = neighbor_grid(self.box, self.search)
        self._search2 = self.search * self.search
        self._dtm = 0.5 * cfg.dt / cfg.mass
        self._time = time_phases
        self._timer = _PhaseTimer()
        self.ell_width = int(ell_width)

        n = self.n
        self.cap = n
        dev = self.device
        if state is None:
            x = torch.as_tensor(fcc_lattice(cfg.lattice_cells, a))
            v = torch.as_tensor(initial_velocities(n, cfg.temperature, cfg.mass, cfg.seed))
        else:       # host (ideally pinned) x, v in global-id order
            x, v = (t if isinstance(t, torch.Tensor) else torch.as_tensor(t) for t in state)
        # ingest through the reference's particle store: an AoSoA set of
        # MD_SCHEMA with the configured vector length V (ref md.py:147-153,
        # aosoa.py:63-142) in HBM, then the engine's SoA working arrays are
        # extracted from it (pc_aosoa_field).  V shapes the store, never the
        # physics: the step loop runs on the SoA copies (ref test_md.py:86-91)
        xd = x.to(dev, torch.float64, non_blocking=True)
        if state is not None:
            # caller positions: the reference's initial migrate wraps them into
            # the box (decomp.py:90-91); the lattice path is already in [0, L)
            if xd.data_ptr() == x.data_ptr():
                xd = xd.clone()
            xd = xd.contiguous()
            call("pc_box_wrap", ptr(xd), n, 3, self._pbox, stream())
        store = aosoa.create(MD_SCHEMA, cfg.vector_length, n, device=dev)
        store.slice("x").device_assign(xd)
        store.slice("x0").device_assign(xd)
        store.slice("v").device_assign(v.to(dev, torch.float64, non_blocking=True))
        store.slice("id").device_assign(torch.arange(n, dtype=torch.int64, device=dev))
        xd = store.slice("x").device_values()
        vd = store.slice("v").device_values()
        ids = store.slice("id").device_values()
        del store
        # pos has one extra row: the SELL padding target (NaN position, tag -1)
        self.pos = self._new_pos()
        self.pos[:n] = _kernels.pack_pos4(xd, ids)
        self._pos_alt = self._new_pos()
        self.vel = vd.t().contiguous()                                   # (3, n)
        self._vel_alt = torch.empty_like(self.vel)
        self.force_events = None      # optional list collecting (start, end) per force launch
        self.rebuild_events = None    # optional list: (sort start, build start, end) per rebuild
        self.frc = torch.zeros((3, n), dtype=torch.float64, device=dev)
        self.cnt = torch.zeros(n, dtype=torch.int32, device=dev)
        self.ell_width = -(-self.ell_width // 4) * 4
        self.nbr = self._new_nbr()
        # minimum image only within this distance of a periodic face (exact:
        # see pc_lj_force_sell in include/particula_b200.h)
        self._mi_guard = float(cfg.cutoff) * (1.0 + 1e-6) + 1e-9
        self.used_staged = None
        # tile-staged path (pc_tile.cu, the default): TMA-staged shared-memory
        # neighbourhoods + 16-bit slot lists in per-warp rounds; falls back to
        # the SELL path for grids with < 3 cells on an axis or extreme density
        self.tile = bool(tile) and not half_list
        # Newton-3 half list (pc_lj_force_sell_half): each pair once, FP64
        # atomics for the neighbour side, kick as a separate pass
        self.half_list = bool(half_list)
        self._ke_in_k = False
        self.partial_k = torch.zeros((int(_lib.load().pc_lj_force_blocks(n)), 5),
                                     dtype=torch.float64, device=dev)
        self.diag_k = torch.zeros(5, dtype=torch.float64, device=dev)
        self.mode = "sell"
        self._tlist = None
        self._tplan = None
        self._spec = False              # tile build issued, flags not yet checked
        self.tile_failures = 0
        self._q8 = 14                   # 112 rounds: the tile build's row capacity
        # planar x|y|z copy (stride _ps: a multiple of 16 elements, NaN rows
        # from cap on) -- the TMA staging source of the tile path and the
        # gather source of the SELL force kernel (24 B in 8-B items)
        self.planar_gather = planar_gather
        self._ps = -(-(self.cap + 1) // 16) * 16
        self.pl = torch.empty((3, self._ps), dtype=torch.float64, device=dev)
        self.pl[:, self.cap:] = float("nan")
        # tile path: the force epilogue also performs the next step's
        # integrate block into these (pc_tile_force, fused); `_advanced`
        # marks them valid, `_pos_stale` that pos4 xyz lags behind pl
        self._pl_n = self.pl.clone()
        self._vel_n = None
        self._advanced = False
        self._pos_stale = False
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)        # force errors
        self.build_flag = torch.zeros(3, dtype=torch.int32, device=dev)  # flags, need, rounds
        self._nblk = int(_lib.load().pc_lj_force_sell_partials(n))   # per-warp rows
        self.partial = torch.zeros((self._nblk, 5), dtype=torch.float64, device=dev)
        self.diag = torch.zeros(5, dtype=torch.float64, device=dev)
        self._ke_fresh = False
        self.rebuilds = 0
        # the lattice lies in [0, L): the reference's initial migrate wrap
        # (decomp.py:90-91) is the identity on it
        # the rebuild bins from the planar copy: fill it from the initial pos4
        call("pc_pos_planar", ptr(self.pos), n, ptr(self.pl), self._ps, stream())
        self._rebuild()
        self._force_step(kick_dtm=0.0)
        self._timer.reset()

    # -- phases ------------------------------------------------------------
    def _t0(self):
        return self._timer.start() if self._time else None

    def _t1(self, phase, e0):
        if self._time:
            self._timer.stop(phase, e0)

    def _new_pos(self):
        p = torch.empty((self.cap + 1, 4), dtype=torch.float64, device=self.device)
        p[self.cap, :3] = float("nan")
        p[self.cap, 3] = torch.tensor(-1, dtype=torch.int64).view(torch.float64)
        return p

    def _new_nbr(self):
        slices = -(-self.cap // 32)
        return torch.empty(slices * self.ell_width * 32, dtype=torch.int32, device=self.device)

    def _sync_pos4(self):
        """pos4 x, y, z <- pl (the fused tile integrate only writes pl)."""
        if self._pos_stale:
            call("pc_pos_from_planar", ptr(self.pl), self._ps, self.n, ptr(self.pos), stream())
            self._pos_stale = False

    def _rebuild(self):
        """Cell sort of all particle fields + SELL Verlet build (md.py:169-188)."""
        n, s = self.n, stream()
        e0 = self._t0()
        rev = self.rebuild_events
        if rev is not None:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            ev[0].record()
        zsort = self.tile and min(self._grid.nc[0], self._grid.nc[1], self._grid.nc[2]) >= 3
        # binning, the z-sort and the permute read the planar positions (always
        # current; pos4 x, y, z may lag behind after fused integrate steps).
        # The z-sort re-ranks every cell: the placement need not be stable.
        srt = _kernels.CellSort(self.pos[:n], 4, self._grid, stable=not zsort,
                                planar=(self.pl, self._ps, n))
        order = srt.order
        if zsort:
            # z-sorted cells: staged columns / home rows of the tile path are
            # z-sorted slot runs (pc_tile.cu)
            order = torch.empty_like(srt.order)
            call("pc_cell_zsort", ptr(self.pl[2]), 1, ptr(srt.cell_start), self._grid.ncells,
                 ptr(srt.order), ptr(order), s)
        # pos4 (all fields current again), velocities and the planar staging
        # copy in one pass; the new planar rows go to the spare planar buffer
        call("pc_md_permute", ptr(order), n, ptr(self.pl), self._ps, ptr(self.pos),
             ptr(self._pos_alt), ptr(self.vel), ptr(self._vel_alt), self.vel.stride(0),
             ptr(self._pl_n), s)
        self.pos, self._pos_alt = self._pos_alt, self.pos
        self.vel, self._vel_alt = self._vel_alt, self.vel
        self.pl, self._pl_n = self._pl_n, self.pl
        self._pos_stale = False
        self._t1("sort", e0)
        e0 = self._t0()
        if rev is not None:
            ev[1].record()
        self._cell_start = srt.cell_start
        if not (self.tile and self._tile_build(srt.cell_start)):
            self._sell_build(srt.cell_start)
        if rev is not None:
            ev[2].record()
            rev.append(tuple(ev))
        self._t1("neighbor", e0)
        self.rebuilds += 1

    def _sell_build(self, cell_start):
        """SELL Verlet build (staged, or per particle for dense grids)."""
        n, s = self.n, stream()
        self.mode = "half" if self.half_list else "sell"
        self._nblk = int(_lib.load().pc_lj_force_sell_partials(n))
        used = ctypes.c_int32(0)
        staged = True
        half = int(self.half_list)
        while True:
            self.build_flag.zero_()
            if staged:
                call("pc_nbr_build_sell", ptr(self.pos), n, ptr(cell_start), self._grid,
                     self._pbox, self._search2, self.ell_width, self.cap, ptr(self.cnt),
                     ptr(self.nbr), ptr(self.build_flag), ctypes.byref(used), s, None, None,
                     half)
            else:
                call("pc_nbr_build", ptr(self.pos), n, ptr(cell_start), self._grid,
                     self._pbox, self._search2, half, _lib.PC_NBR_SELL, 0, ptr(self.cnt), None,
                     ptr(self.nbr), self.cap, self.ell_width, ptr(self.build_flag), s, None,
                     None)
                used.value = 0
            fl = int(self.build_flag[0].item())
            if fl & _lib.FLAG_STAGE:          # dense neighbourhood: per-particle kernel
                staged = False
                continue
            if not (fl & _lib.FLAG_OVERFLOW):
                break
            # no silent truncation (SPEC neighbors: grow and rebuild)
            self.ell_width = -(-(int(self.cnt[:n].max().item()) + 8) // 4) * 4
            self.nbr = self._new_nbr()
        self.used_staged = bool(used.value)
        if self.deterministic:
            call("pc_sell_sort_by_tag", ptr(self.pos), n, ptr(self.cnt), ptr(self.nbr),
                 self.ell_width, ptr(self.build_flag), s)
            if int(self.build_flag[0].item()) & _lib.FLAG_OVERFLOW:
                raise RuntimeError("deterministic mode: a Verlet row exceeds 256 entries")

    def _tile_build(self, cell_start) -> bool:
        """Issue the tile round-list build (pc_tile.cu) without a host sync.
        Capacities are static (row-warps bounded by n/32 + tiles, rounds by
        the build's row capacity), so the only failures are a neighbourhood
        beyond the staging area or a row beyond the hit capacity; the build
        flags are checked after the (speculative) force launch of the same
        step, `_verify_tile_build`, which falls back to the SELL path.
        False when this grid does not fit the tile path at all."""
        g = self._grid
        if min(g.nc[0], g.nc[1], g.nc[2]) < 3 or g.ndim != 3:
            return False
        lib, s, dev = _lib.load(), stream(), self.device
        nt = int(lib.pc_tile_count(g))
        rw = torch.empty(nt, dtype=torch.int32, device=dev)
        call("pc_tile_rows", ptr(cell_start), g, ptr(rw), s)
        self._rw0 = _kernels.scan_i32(rw)
        bound = self.n // 32 + nt + 1
        self._ntiles = nt
        if self._tlist is None or self._rounds.numel() < bound:
            self._rounds = torch.empty(bound, dtype=torch.int32, device=dev)
            self._rowidx = torch.empty(bound * 32, dtype=torch.int32, device=dev)
            self._tlist = torch.empty(bound * self._q8 * 512, dtype=torch.uint8, device=dev)
        if self._tplan is None or self._tplan.numel() < nt * int(lib.pc_tile_plan_ints()):
            self._tplan = torch.empty(nt * int(lib.pc_tile_plan_ints()), dtype=torch.int32,
                                      device=dev)
        npart = int(lib.pc_tile_force_partials(nt))
        if self.partial.shape[0] < npart:
            self.partial = torch.zeros((npart, 5), dtype=torch.float64, device=dev)
        if getattr(self, "_vir_part", None) is None or self._vir_part.shape[0] < npart:
            # pair virial partials (column 0; pc_tile_force), reduced on demand
            self._vir_part = torch.zeros((npart, 5), dtype=torch.float64, device=dev)
            self._vir = torch.zeros(5, dtype=torch.float64, device=dev)
        self.build_flag.zero_()
        # bank-conflict-aware round order (lists unchanged as sets): fused into
        # the build (default) or as the separate pc_tile_order pass
        kind = _tile_order_kind(self.cfg.rebuild_stride)
        fused = _TILE_FUSED_ORDER and kind == 1
        call("pc_tile_build_ordered", ptr(self.pl), self._ps, ptr(cell_start), g, self._pbox,
             self._search2, self._q8, ptr(self._rw0), ptr(self._tplan), ptr(self._rowidx),
             ptr(self._rounds), ptr(self._tlist), ptr(self.build_flag), s, None, None, None,
             None, 1 if fused else 0)
        if not fused:
            call("pc_tile_order", bound, ptr(self._rw0[nt:]), ptr(self._rounds),
                 ptr(self._tlist), self._q8, kind, s)
        self.mode = "tile"
        self._nblk = npart
        self._spec = True
        return True

    def _verify_tile_build(self, saved):
        """Host check of the tile build flags after the speculative force was
        launched (the GPU keeps running meanwhile); on failure restore the
        state the force touched and redo the step's list + force on the SELL
        path."""
        self._spec = False
        fl = int(self.build_flag[0].item())
        if not fl & (_lib.FLAG_STAGE | _lib.FLAG_OVERFLOW):
            return
        vel, flag, kick_dtm = saved
        self.vel.copy_(vel)
        self.flag.copy_(flag)
        self._advanced = False
        self.tile_failures += 1
        self._sell_build(self._cell_start)
        self._force(kick_dtm)

    def _force_step(self, kick_dtm):
        """Force of this step; after a tile build, speculative (see
        _verify_tile_build)."""
        if self._spec:
            saved = (self.vel.clone(), self.flag.clone(), kick_dtm)
            self._force(kick_dtm)
            self._verify_tile_build(saved)
        else:
            self._force(kick_dtm)

    def _force(self, kick_dtm):
        e0 = self._t0()
        if self.force_events is not None:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
        if self.mode == "tile":
            if self._vel_n is None:
                self._vel_n = torch.empty_like(self.vel)
            call("pc_tile_force", ptr(self.pl), self._ps, self._ntiles, ptr(self._tplan),
                 ptr(self._rowidx), ptr(self._rounds), ptr(self._tlist), self._q8, self._pbox,
                 self._lj, self._mi_guard, ptr(self.frc), self.cap, ptr(self.vel), self.cap,
                 float(kick_dtm), float(self.cfg.mass), ptr(self.partial), ptr(self.flag),
                 ptr(self._pl_n), ptr(self._vel_n), self._dtm, float(self.cfg.dt),
                 ptr(self._vir_part), None, None, stream())
            self._advanced = True
        elif self.mode == "half":
            self.frc.zero_()
            call("pc_lj_force_sell_half", ptr(self.pos), self.n, ptr(self.cnt), ptr(self.nbr),
                 self.ell_width, self._pbox, self._lj, self._mi_guard, ptr(self.frc), self.cap,
                 ptr(self.partial), ptr(self.flag), stream())
        elif self.deterministic:
            if getattr(self, "_atom", None) is None:
                self._atom = torch.zeros((self.n, 5), dtype=torch.float64, device=self.device)
            call("pc_lj_force_sell_atoms", ptr(self.pos), ptr(self.pl), self._ps, self.n,
                 ptr(self.cnt), ptr(self.nbr), self.ell_width, self._pbox, self._lj,
                 self._mi_guard, ptr(self.frc), self.cap, ptr(self.vel), self.cap,
                 float(kick_dtm), float(self.cfg.mass), ptr(self._atom), ptr(self.flag),
                 stream())
        else:
            call("pc_lj_force_sell", ptr(self.pos), ptr(self.pl) if self.planar_gather else None,
                 self._ps, self.n,
                 ptr(self.cnt), ptr(self.nbr),
                 self.ell_width, self._pbox, self._lj, self._mi_guard, ptr(self.frc), self.cap,
                 ptr(self.vel), self.cap, float(kick_dtm), float(self.cfg.mass),
                 ptr(self.partial), ptr(self.flag), stream())
        if self.force_events is not None:
            b.record()
            self.force_events.append((a, b))
        self._t1("force", e0)
        if self.mode == "half":      # atomics finish f: final kick + KE partials separately
            e0 = self._t0()
            call("pc_kick", ptr(self.vel), self.cap, ptr(self.frc), self.cap, self.n,
                 float(kick_dtm), float(self.cfg.mass), ptr(self.partial_k), stream())
            self._t1("integrate", e0)
            self._ke_in_k = True
        else:
            self._ke_in_k = False
        self._ke_fresh = True

    def _integrate(self):
        if self._advanced:          # done by the previous force epilogue
            self.pl, self._pl_n = self._pl_n, self.pl
            self.vel, self._vel_n = self._vel_n, self.vel
            self._advanced = False
            self._pos_stale = True
            return
        e0 = self._t0()
        self._sync_pos4()
        call("pc_kick_drift_wrap", ptr(self.pos), ptr(self.vel), self.cap, ptr(self.frc),
             self.cap, self.n, self._dtm, float(self.cfg.dt), self._pbox, ptr(self.pl),
             self._ps, stream())
        self._t1("integrate", e0)

    def step(self, step_index: int):
        """One velocity-Verlet step (ref md.py:219-257)."""
        self._integrate()
        if step_index % self.cfg.rebuild_stride == 0:
            self._rebuild()
        self._force_step(kick_dtm=self._dtm)

    def check_errors(self):
        fl = int(self.flag.item())
        if fl & _lib.FLAG_OVERLAP:
            raise FloatingPointError("overlapping particles in LJ kernel")

    # -- diagnostics --------------------------------------------------------
    def device_diagnostics(self, out=None) -> torch.Tensor:
        """(KE, PE, px, py, pz) on the device, no host sync; `out`: a 5-double
        device row to reduce into (run_md's history) instead of self.diag."""
        if self.deterministic:
            if not self._ke_fresh:   # per-atom rows again (v unchanged: zero kick)
                self._force(0.0)
            # per-atom rows summed exactly (integer limbs, pc_exact_sum): the
            # result does not depend on the order or the decomposition
            limbs = torch.zeros(20, dtype=torch.int64, device=self.device)
            call("pc_exact_sum", ptr(self._atom), self.n, 5, None, ptr(limbs), stream())
            d = self.diag if out is None else out
            call("pc_exact_finish", ptr(limbs), 5, ptr(d), stream())
            return d
        if not self._ke_fresh:       # velocities changed outside a force pass
            call("pc_kick", ptr(self.vel), self.cap, ptr(self.frc), self.cap, self.n, 0.0,
                 float(self.cfg.mass), ptr(self.partial_k), stream())
            self._ke_in_k = True
            self._ke_fresh = True
        if self._ke_in_k:            # KE / momentum from the kick partials, PE from force
            call("pc_reduce_partials", ptr(self.partial), self._nblk, ptr(self.diag), stream())
            nk = int(_lib.load().pc_lj_force_blocks(self.n))
            call("pc_reduce_partials", ptr(self.partial_k), nk, ptr(self.diag_k), stream())
            self.diag_k[1] = self.diag[1]
            if out is not None:
                out.copy_(self.diag_k)
                return out
            return self.diag_k
        d = self.diag if out is None else out
        call("pc_reduce_partials", ptr(self.partial), self._nblk, ptr(d), stream())
        return d

    def device_virial(self):
        """Pair virial W = sum over pairs of r.F of the last force pass (tile
        path; FP64 per-warp partials, one fixed reduction), or None on the
        SELL paths."""
        if self.mode != "tile":
            return None
        call("pc_reduce_partials", ptr(self._vir_part), self._nblk, ptr(self._vir), stream())
        return self._vir[0]

    def diagnostics(self):
        """Global energies (ref md.py:261-277), plus the pair virial W and the
        pressure P = (2 KE + W) / (3 V) where the force path computes W (the
        reference reports neither)."""
        d = self.device_diagnostics().cpu().numpy()
        self.check_errors()
        ke, pe = float(d[0]), float(d[1])
        out = {"KE": ke, "PE": pe, "E_total": ke + pe,
               "temperature": 2.0 * ke / (3.0 * self.n),
               "momentum": d[2:5].copy()}
        w = self.device_virial()
        if w is not None:
            out["virial"] = float(w.item())
            out["pressure"] = (2.0 * ke + out["virial"]) / (3.0 * float(np.prod(self.box.lengths)))
        return out

    def gather_state(self):
        """Positions and velocities in global-id order (ref md.py:279-287)."""
        self._sync_pos4()
        p = self.pos[: self.n].cpu().numpy()
        ids = p[:, 3].view(np.int64)
        x = np.zeros((self.n, 3))
        v = np.zeros((self.n, 3))
        x[ids] = p[:, :3]
        v[ids] = self.vel[:, : self.n].cpu().numpy().T
        return x, v

    def verlet_sets(self):
        """The current Verlet list (search radius) as a CSR over global ids:
        (counts, offsets, indices), rows in id order, row entries sorted --
        the layout of ref neighbors.build_verlet for parity checks."""
        n, Q = self.n, self.ell_width // 4
        gid = self.pos[:n, 3].contiguous().view(torch.int64).cpu().numpy()
        if self.mode == "tile":
            cnt_t, table = self._tile_rows()
            cnt = cnt_t.to(torch.int64).cpu().numpy()
            a = np.repeat(np.arange(n), cnt)
            k = np.arange(a.size) - np.repeat(np.cumsum(cnt) - cnt, cnt)
            j = table.cpu().numpy()[a, k]
        else:
            cnt = self.cnt[:n].to(torch.int64).cpu().numpy()
            a = np.repeat(np.arange(n), cnt)
            k = np.arange(a.size) - np.repeat(np.cumsum(cnt) - cnt, cnt)
            words = self.nbr.cpu().numpy()
            w = ((a >> 5) * Q + (k >> 2)) * 128 + (a & 31) * 4 + (k & 3)
            j = words[w]
        rows_gid, nb_gid = gid[a], gid[j]
        o = np.lexsort((nb_gid, rows_gid))
        counts = np.bincount(rows_gid, minlength=n)
        offsets = np.concatenate(([0], np.cumsum(counts)))
        return counts, offsets, nb_gid[o]

    def _tile_rows(self, width: int = 128):
        """Tile lists as (count, table): row = cell-sorted particle index,
        table[row, :count[row]] its neighbours (pc_tile_decode)."""
        n = self.n
        cnt = torch.zeros(n, dtype=torch.int32, device=self.device)
        table = torch.full((n, width), -1, dtype=torch.int32, device=self.device)
        call("pc_tile_decode", self._ntiles, ptr(self._tplan), ptr(self._rowidx),
             ptr(self._rounds), ptr(self._tlist), self._q8, width, ptr(cnt), ptr(table),
             stream())
        return cnt, table

    def mean_neighbors(self) -> float:
        """Mean Verlet-list length of the current build."""
        if self.mode == "tile":
            cnt, _ = self._tile_rows()
            return float(cnt.double().mean().item())
        return float(self.cnt[: self.n].double().mean().item())

    def negate_velocities(self):
        self.vel.neg_()
        self._advanced = False      # the pre-integrated next state is stale
        self._ke_fresh = False

    @property
    def timings(self):
        return self._timer.resolve()

    @timings.setter
    def timings(self, value):
        self._timer.reset()
        for k, v in dict(value).items():
            self._timer.totals[k] = float(v)


def run_md(cfg: MDConfig, state=None, time_phases: bool = True, deterministic: bool = False,
           **driver_options):
    """Run the NVE loop; returns (per-step diagnostic rows, phase timings)
    (ref md.py:295-307).  The per-step energies are reduced on the device
    into a history buffer and read back once after the loop (the reference
    returns the rows only at the end as well), so the step loop never waits
    for the host.  An overlap detected in any step raises FloatingPointError
    after the loop.  `state`: optional host (x, v) in global-id order.
    `deterministic`: the id-ordered engine, bitwise equal to
    FabricMD / DistMD(deterministic=True) on any rank grid.  `driver_options`:
    MDDriver's engine choices (tile, half_list, planar_gather)."""
    drv = MDDriver(cfg, state=state, time_phases=time_phases, deterministic=deterministic,
                   **driver_options)
    drv.timings = {k: 0.0 for k in PHASES}
    hist = torch.empty((cfg.steps + 1, 5), dtype=torch.float64, device=drv.device)
    drv.device_diagnostics(out=hist[0])
    for s in range(1, cfg.steps + 1):
        drv.step(s)
        drv.device_diagnostics(out=hist[s])
    h = hist.cpu().numpy()
    drv.check_errors()
    rows = []
    for s in range(cfg.steps + 1):
        ke, pe = float(h[s, 0]), float(h[s, 1])
        rows.append(dict(step=s, KE=ke, PE=pe, E_total=ke + pe,
                         temperature=2.0 * ke / (3.0 * drv.n)))
    return rows, drv.timings
