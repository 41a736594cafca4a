"""CPU oracle for the LJ short-range MD hot path -- TEST INFRASTRUCTURE ONLY.

This module restates, in plain numpy, the algorithms of the reference package
``particula`` (/root/reference/pkg/src/particula, arXiv 2109.09056 proxy) that
lie on the north-star path: periodic geometry, linked-cell binning, Verlet
neighbor lists, the Lennard-Jones force, the simulated-rank migrate/halo
exchange and the velocity-Verlet MD driver.  Every function cites the
reference ``file:line`` it follows.

Who may use it: ``tests/`` (as the parity checker), ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs.  The product
package ``paper_2109_09056_b200`` never imports, calls or links anything in
``oracle/``; its CUDA path fails loudly when the extension is missing.

Parity pin: ``tests/test_oracle_golden.py`` checks each function below against
golden vectors produced by running the reference itself
(``tests/golden/make_golden.py``, committed with the fixtures).

Arithmetic contract (the bits that make the GPU neighbor lists bit-exact):
  * min-image is ``dx - L*round_half_even(dx/L)`` (geometry.py:51-58);
  * |dx|^2 is numpy's ``einsum`` over the last axis of a C-contiguous array,
    which on this numpy build evaluates ``(dx0*dx0 + dx2*dx2) + dx1*dx1``
    without FMA (asserted by ``einsum_order_ok``);
  * the pair test is the strict ``r2 < cutoff*cutoff`` in FP64.
"""

from __future__ import annotations

import itertools
import time
from dataclasses import dataclass

import numpy as np

# ---------------------------------------------------------------------------
# geometry (ref: geometry.py)
# ---------------------------------------------------------------------------


def box_wrap(x, low, high, periodic):
    """Periodic wrap into [low, high) -- ref geometry.py:40-49.

    ``low + mod(x - low, L)`` per periodic axis, then a value that rounded up
    to ``high`` is folded back to ``low``.
    """
    out = np.array(x, dtype=np.float64, copy=True)
    low = np.asarray(low, np.float64)
    high = np.asarray(high, np.float64)
    length = high - low
    for a in np.flatnonzero(np.asarray(periodic, bool)):
        col = low[a] + np.mod(out[..., a] - low[a], length[a])
        out[..., a] = np.where(col >= high[a], low[a], col)
    return out


def box_min_image(dx, length, periodic):
    """Minimum image ``dx - L*round(dx/L)`` (half-even) -- ref geometry.py:51-58."""
    out = np.array(dx, dtype=np.float64, copy=True)
    length = np.asarray(length, np.float64)
    for a in np.flatnonzero(np.asarray(periodic, bool)):
        out[..., a] -= length[a] * np.round(out[..., a] / length[a])
    return out


def sqnorm(dx):
    """|dx|^2 over the last axis exactly as the reference evaluates it
    (``np.einsum`` on a C-contiguous array; neighbors.py:92, md.py:115)."""
    dx = np.ascontiguousarray(dx, dtype=np.float64)
    return np.einsum("...k,...k->...", dx, dx)


def einsum_order_ok(samples: int = 200_000, seed: int = 0) -> bool:
    """Self-check of the numpy build: einsum |dx|^2 == (x^2 + z^2) + y^2.

    The CUDA kernels hard-code this evaluation order (no FMA); if a different
    numpy build sums differently the bit-exact neighbor claim must be re-pinned.
    """
    rng = np.random.default_rng(seed)
    d = rng.normal(size=(samples, 3)) * 1.7
    explicit = (d[:, 0] * d[:, 0] + d[:, 2] * d[:, 2]) + d[:, 1] * d[:, 1]
    return bool(np.array_equal(sqnorm(d), explicit))


# ---------------------------------------------------------------------------
# binning (ref: binning.py)
# ---------------------------------------------------------------------------


def stable_key_permutation(keys):
    """``map[src] = dst`` of the stable sort of ``keys`` -- ref binning.py:49-55."""
    keys = np.asarray(keys)
    src_of_dst = np.argsort(keys, kind="stable")
    dst = np.empty(keys.shape[0], dtype=np.int64)
    dst[src_of_dst] = np.arange(keys.shape[0], dtype=np.int64)
    return dst


def is_bijection(m, n):
    """ref binning.py:26-33."""
    m = np.asarray(m, np.int64)
    if m.shape[0] != n:
        return False
    if m.size and (m.min() < 0 or m.max() >= n):
        return False
    hit = np.zeros(n, bool)
    hit[m] = True
    return bool(hit.all())


def cell_indices(x, low, high, cell_size):
    """Half-open linked-cell coordinates -- ref binning.py:58-73.

    ``nc = max(1, ceil(L/cs - 1e-12))``, ``idx = min(floor((x-low)/cs), nc-1)``.
    Raises ValueError for non-positive cell size or a point outside the box.
    """
    x = np.asarray(x, np.float64)
    low = np.asarray(low, np.float64)
    high = np.asarray(high, np.float64)
    d = low.shape[0]
    cs = np.broadcast_to(np.asarray(cell_size, np.float64), (d,))
    if np.any(cs <= 0):
        raise ValueError("cell_size must be positive")
    if np.any(x < low) or np.any(x > high):
        raise ValueError("position outside box")
    nc = np.maximum(1, np.ceil(((high - low) / cs) - 1e-12).astype(np.int64))
    idx = np.minimum(np.floor((x - low) / cs).astype(np.int64), nc - 1)
    return nc, idx


def bin_by_position(x, low, high, cell_size):
    """Geometric binning -> (cells per axis, offsets, permutation map)
    -- ref binning.py:76-87 (row-major flat cell id, bincount, stable order)."""
    x = np.asarray(x, np.float64)
    nc, idx = cell_indices(x, low, high, cell_size)
    flat = np.ravel_multi_index(tuple(idx.T), tuple(nc)) if x.shape[0] else \
        np.empty(0, np.int64)
    counts = np.bincount(flat, minlength=int(np.prod(nc)))
    offsets = np.concatenate(([0], np.cumsum(counts))).astype(np.int64)
    return nc, offsets, stable_key_permutation(flat)


def apply_permutation(values, perm_map):
    """Row i moves to ``perm_map[i]`` -- ref binning.py:90-101."""
    values = np.asarray(values)
    out = np.empty_like(values)
    out[np.asarray(perm_map, np.int64)] = values
    return out


# ---------------------------------------------------------------------------
# neighbors (ref: neighbors.py)
# ---------------------------------------------------------------------------


def _axis_stencil(nc_a: int, periodic_a: bool):
    """Distinct stencil offsets along one axis.  On a periodic axis with fewer
    than three cells, offsets alias the same cell; the reference removes the
    duplicates with a set of flat cell ids (neighbors.py:76-89), which is the
    same as keeping the first offset of each residue class here."""
    if not periodic_a:
        return [-1, 0, 1]
    seen, keep = set(), []
    for o in (-1, 0, 1):
        r = o % nc_a
        if r not in seen:
            seen.add(r)
            keep.append(o)
    return keep


def neighbor_pairs(x, low, high, periodic, cutoff, cell_ratio=1.0, chunk=16384, rows=None):
    """All ordered (i, j), i != j, with min-image r^2 < cutoff^2, as arrays
    sorted by (i, j) -- the full-convention sets of ref neighbors.py:49-97.

    Same cell grid as the reference (``nc = max(1, floor(L/(rc*ratio)))``,
    width ``L/nc``, clipped floor) and the same FP64 predicate, evaluated
    vectorised over candidate pairs instead of a Python loop over cells.
    ``rows``: only the rows i in this index array (sampled parity checks of
    multi-million-atom systems; the row sets are the full-list rows).
    """
    x = np.ascontiguousarray(x, np.float64)
    n, d = x.shape
    low = np.asarray(low, np.float64)
    high = np.asarray(high, np.float64)
    per = np.asarray(periodic, bool)
    length = high - low
    if n == 0:
        return np.empty(0, np.int64), np.empty(0, np.int64)
    nc = np.maximum(1, np.floor(length / (cutoff * cell_ratio)).astype(np.int64))
    idx = np.clip(np.floor((x - low) / (length / nc)).astype(np.int64), 0, nc - 1)
    flat = np.ravel_multi_index(tuple(idx.T), tuple(nc))
    ncells = int(np.prod(nc))
    order = np.argsort(flat, kind="stable")
    counts = np.bincount(flat, minlength=ncells)
    start = np.concatenate(([0], np.cumsum(counts)))
    rc2 = cutoff * cutoff
    offs = list(itertools.product(*[_axis_stencil(int(nc[a]), bool(per[a]))
                                    for a in range(d)]))
    out_i, out_j = [], []
    sel = (np.arange(n, dtype=np.int64) if rows is None
           else np.unique(np.asarray(rows, np.int64)))
    for b in range(0, sel.size, chunk):
        ids = sel[b:b + chunk]
        ci = idx[ids]
        cand_i, cand_j = [], []
        for off in offs:
            cc = ci + np.asarray(off, np.int64)
            ok = np.ones(ids.shape[0], bool)
            for a in range(d):
                if per[a]:
                    cc[:, a] %= nc[a]
                else:
                    ok &= (cc[:, a] >= 0) & (cc[:, a] < nc[a])
            src = ids[ok]
            cflat = np.ravel_multi_index(tuple(cc[ok].T), tuple(nc))
            lens = counts[cflat]
            tot = int(lens.sum())
            if tot == 0:
                continue
            rep_i = np.repeat(src, lens)
            base = np.repeat(start[cflat] - (np.cumsum(lens) - lens), lens)
            rep_j = order[base + np.arange(tot)]
            cand_i.append(rep_i)
            cand_j.append(rep_j)
        if not cand_i:
            continue
        ci_all = np.concatenate(cand_i)
        cj_all = np.concatenate(cand_j)
        keep = ci_all != cj_all
        ci_all, cj_all = ci_all[keep], cj_all[keep]
        dx = box_min_image(x[cj_all] - x[ci_all], length, per)
        hit = sqnorm(dx) < rc2
        out_i.append(ci_all[hit])
        out_j.append(cj_all[hit])
    if not out_i:
        return np.empty(0, np.int64), np.empty(0, np.int64)
    pi = np.concatenate(out_i)
    pj = np.concatenate(out_j)
    o = np.lexsort((pj, pi))
    return pi[o], pj[o]


def neighbor_sets_cell_loop(x, low, high, periodic, cutoff, cell_ratio=1.0):
    """Per-row sorted neighbor arrays (full convention, no self), restating the
    reference's loop structure -- ref neighbors.py:49-97: a Python loop over
    cells; per cell the union of its stencil cells' members (``np.unique``),
    one vectorised min-image distance block (mine x candidates), and a Python
    loop over the cell's rows that slices each row's hits.

    Same sets as ``neighbor_pairs`` (tests/test_oracle_golden.py).  It exists so
    that ``bench.py --impl reference`` pays the reference's own cost profile
    (per-cell and per-row interpreter work) rather than the vectorised port's.
    """
    x = np.ascontiguousarray(x, np.float64)
    n, d = x.shape
    low = np.asarray(low, np.float64)
    length = np.asarray(high, np.float64) - low
    per = np.asarray(periodic, bool)
    nc = np.maximum(1, np.floor(length / (cutoff * cell_ratio)).astype(np.int64))
    idx = np.clip(np.floor((x - low) / (length / nc)).astype(np.int64), 0, nc - 1)
    flat = (np.ravel_multi_index(tuple(idx.T), tuple(nc)) if n
            else np.empty(0, np.int64))
    ncells = int(np.prod(nc))
    order = np.argsort(flat, kind="stable")
    counts = np.bincount(flat, minlength=ncells)
    start = np.concatenate(([0], np.cumsum(counts)))
    members = [order[start[c]:start[c + 1]] for c in range(ncells)]
    stencil = list(itertools.product(*[(-1, 0, 1)] * d))
    rc2 = cutoff * cutoff
    out = [np.empty(0, np.int64)] * n
    for c in range(ncells):
        mine = members[c]
        if mine.size == 0:
            continue
        cc = np.array(np.unravel_index(c, tuple(nc)))
        cells = set()
        for off in stencil:
            cell = cc + np.array(off)
            ok = True
            for a in range(d):
                if per[a]:
                    cell[a] %= nc[a]
                elif not 0 <= cell[a] < nc[a]:
                    ok = False
                    break
            if ok:
                cells.add(int(np.ravel_multi_index(tuple(cell), tuple(nc))))
        cand = np.unique(np.concatenate([members[k] for k in sorted(cells)]))
        dx = box_min_image(x[cand][None, :, :] - x[mine][:, None, :], length, per)
        hit = sqnorm(dx) < rc2
        for row, i in enumerate(mine):
            js = cand[hit[row]]
            out[int(i)] = js[js != i]
    return out


def neighbor_pairs_cell_loop(x, low, high, periodic, cutoff, cell_ratio=1.0):
    """``neighbor_pairs`` through the per-cell loop: the sets concatenated into
    CSR rows and expanded to (i, j) as ref neighbors.py:119-127 and
    VerletList.pairs (neighbors.py:39-46) do."""
    sets = neighbor_sets_cell_loop(x, low, high, periodic, cutoff, cell_ratio)
    cnt = np.array([js.size for js in sets], np.int64)
    pj = np.concatenate(sets) if sets else np.empty(0, np.int64)
    pi = np.repeat(np.arange(len(sets), dtype=np.int64), cnt)
    return pi, pj.astype(np.int64)


def validate_verlet_args(low, high, periodic, cutoff, layout, half_or_full,
                         cell_ratio):
    """Argument checks of ref neighbors.py:107-118 (ValueError)."""
    if cutoff <= 0:
        raise ValueError("cutoff must be positive")
    if cell_ratio < 1.0:
        raise ValueError("cell_ratio must be >= 1")
    if layout not in ("dense", "compressed"):
        raise ValueError(f"unknown layout {layout!r}")
    if half_or_full not in ("half", "full"):
        raise ValueError(f"unknown pair convention {half_or_full!r}")
    length = np.asarray(high, np.float64) - np.asarray(low, np.float64)
    for a in np.flatnonzero(np.asarray(periodic, bool)):
        if cutoff > 0.5 * length[a]:
            raise ValueError("cutoff exceeds half the box length on a periodic axis")


def build_verlet(x, low, high, periodic, cutoff, layout="compressed",
                 half_or_full="full", cell_ratio=1.0):
    """Verlet list -- ref neighbors.py:100-134.

    Returns a dict with ``counts`` and either ``indices``/``offsets`` (CSR,
    int64) or ``table`` (n x max, -1 padded).  Rows list neighbor indices in
    ascending order; ``half`` keeps j > i.
    """
    x = np.asarray(x, np.float64)
    validate_verlet_args(low, high, periodic, cutoff, layout, half_or_full,
                         cell_ratio)
    n = x.shape[0]
    pi, pj = neighbor_pairs(x, low, high, periodic, cutoff, cell_ratio)
    if half_or_full == "half":
        keep = pj > pi
        pi, pj = pi[keep], pj[keep]
    counts = np.bincount(pi, minlength=n).astype(np.int64)
    res = {"layout": layout, "half_or_full": half_or_full, "cutoff": cutoff,
           "counts": counts}
    if layout == "compressed":
        res["indices"] = pj.astype(np.int64)
        res["offsets"] = np.concatenate(([0], np.cumsum(counts))).astype(np.int64)
    else:
        width = int(counts.max()) if n else 0
        table = np.full((n, width), -1, np.int64)
        first = np.concatenate(([0], np.cumsum(counts)))[:-1]
        col = np.arange(pi.shape[0]) - np.repeat(first, counts)
        table[pi, col] = pj
        res["table"] = table
    return res


def rows_from_csr(counts, indices):
    """Per-row arrays from a CSR list (helper for comparisons)."""
    off = np.concatenate(([0], np.cumsum(counts)))
    return [indices[off[i]:off[i + 1]] for i in range(len(counts))]


def brute_force_sets(x, length, periodic, cutoff):
    """O(N^2) oracle of ref tests/test_neighbors.py:8-18 (small n only)."""
    x = np.asarray(x, np.float64)
    out = []
    for i in range(x.shape[0]):
        dx = box_min_image(x - x[i], length, periodic)
        js = np.flatnonzero(sqnorm(dx) < cutoff * cutoff)
        out.append(np.sort(js[js != i]))
    return out


# ---------------------------------------------------------------------------
# LJ force (ref: md.py)
# ---------------------------------------------------------------------------


def lj_pair(dx, r2, eps, sigma):
    """Truncated (unshifted) LJ pair energy and the force on i, dx = xj - xi
    -- ref md.py:89-96."""
    sr2 = sigma * sigma / r2
    sr6 = sr2 * sr2 * sr2
    sr12 = sr6 * sr6
    e = 4.0 * eps * (sr12 - sr6)
    fmag = 24.0 * eps * (2.0 * sr12 - sr6) / r2
    return e, -fmag[:, None] * dx


def lj_forces(x, ids, owned, pair_i, pair_j, length, periodic, eps, sigma,
              cutoff):
    """Canonical LJ forces / per-particle energies for rows < owned
    -- ref md.py:99-126.

    Pairs accumulate in ascending (gid_i, gid_j) order after the exact-cutoff
    re-filter; each pair energy is booked once, on the smaller gid.
    """
    x = np.asarray(x, np.float64)
    ids = np.asarray(ids, np.int64)
    sel = pair_i < owned
    ii, jj = pair_i[sel], pair_j[sel]
    o = np.lexsort((ids[jj], ids[ii]))
    ii, jj = ii[o], jj[o]
    dx = box_min_image(x[jj] - x[ii], length, periodic)
    r2 = sqnorm(dx)
    keep = r2 < cutoff * cutoff
    ii, jj, dx, r2 = ii[keep], jj[keep], dx[keep], r2[keep]
    if r2.size and r2.min() < (1e-10 * sigma) ** 2:
        raise FloatingPointError("overlapping particles in LJ kernel")
    e, fv = lj_pair(dx, r2, eps, sigma)
    forces = np.zeros((owned, 3))
    np.add.at(forces, ii, fv)
    pe = np.zeros(owned)
    upper = ids[jj] > ids[ii]
    np.add.at(pe, ii[upper], e[upper])
    return forces, pe


# ---------------------------------------------------------------------------
# Ewald real-space pass (ref: longrange.py) -- SURVEY §8(f3), the only other
# consumer of the half Verlet list.  erfc is scipy.special.erfc, the
# reference's own third-party dependency (longrange.py:14; scipy 1.18.1 here).
# ---------------------------------------------------------------------------


def ewald_real_space(x, q, length, alpha, r_cut, pair_i=None, pair_j=None):
    """erfc-screened Coulomb pair sum over half-list pairs (or all pairs)
    -- ref longrange.py:47-72.  Returns (energy, forces)."""
    from scipy.special import erfc
    x = np.asarray(x, np.float64)
    q = np.asarray(q, np.float64)
    n = x.shape[0]
    if pair_i is None:
        ii, jj = np.triu_indices(n, k=1)
    else:
        ii, jj = np.asarray(pair_i, np.int64), np.asarray(pair_j, np.int64)
    dx = x[jj] - x[ii]
    dx -= length * np.round(dx / length)
    r2 = sqnorm(dx)
    sel = r2 < r_cut * r_cut
    ii, jj, dx, r2 = ii[sel], jj[sel], dx[sel], r2[sel]
    r = np.sqrt(r2)
    if r.size and r.min() < 1e-10:
        raise ValueError("overlapping charges in real-space sum")
    qq = q[ii] * q[jj]
    er = erfc(alpha * r)
    energy = float(np.sum(qq * er / r))
    mag = qq * (er / r2 + 2 * alpha / np.sqrt(np.pi) * np.exp(-(alpha * r) ** 2) / r)
    fvec = (mag / r)[:, None] * dx
    forces = np.zeros_like(x)
    np.add.at(forces, jj, fvec)
    np.add.at(forces, ii, -fvec)
    return energy, forces


def fcc_lattice(cells, spacing):
    """4-atom FCC basis on a cells^3 grid, ij meshgrid order -- ref md.py:67-74."""
    basis = np.array([[0.0, 0.0, 0.0], [0.5, 0.5, 0.0],
                      [0.5, 0.0, 0.5], [0.0, 0.5, 0.5]])
    r = np.arange(cells)
    gx, gy, gz = np.meshgrid(r, r, r, indexing="ij")
    corner = np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1)
    return (corner[:, None, :] + basis[None, :, :]).reshape(-1, 3) * spacing


def initial_velocities(n, temperature, mass, seed):
    """PCG64 Gaussian velocities, zero momentum, exact-T rescale -- ref md.py:77-86."""
    v = np.random.default_rng(seed).normal(size=(n, 3))
    v -= v.mean(axis=0)
    ke = 0.5 * mass * np.einsum("ij,ij->", v, v)
    if ke > 0:
        v *= np.sqrt(1.5 * n * temperature / ke)
    return v


# ---------------------------------------------------------------------------
# decomposition (ref: decomp.py) -- ranks are dicts of numpy arrays
# ---------------------------------------------------------------------------


class Fabric:
    """Uniform Cartesian rank split, row-major ids -- ref decomp.py:21-66."""

    def __init__(self, low, high, dims, periodic):
        self.low = np.asarray(low, np.float64)
        self.high = np.asarray(high, np.float64)
        self.dims = np.asarray(dims, np.int64)
        self.periodic = np.asarray(periodic, bool)
        if np.any(self.dims < 1):
            raise ValueError("rank_dims must be >= 1 per axis")

    @property
    def n_ranks(self):
        return int(np.prod(self.dims))

    @property
    def lengths(self):
        return self.high - self.low

    @property
    def block_lengths(self):
        return self.lengths / self.dims

    def coords_of(self, r):
        return np.array(np.unravel_index(r, tuple(self.dims)))

    def rank_of(self, c):
        return int(np.ravel_multi_index(tuple(np.asarray(c)), tuple(self.dims)))

    def local_box(self, r):
        c = self.coords_of(r)
        lo = self.low + c * self.block_lengths
        hi = np.where(c == self.dims - 1, self.high, lo + self.block_lengths)
        return lo, hi

    def owner_of(self, x):
        x = np.asarray(x, np.float64)
        if np.any(x < self.low) or np.any(x > self.high):
            raise ValueError("position outside global box")
        c = np.floor((x - self.low) / self.block_lengths).astype(np.int64)
        c = np.minimum(c, self.dims - 1)
        if x.shape[0] == 0:
            return np.empty(0, np.int64)
        return np.ravel_multi_index(tuple(c.T), tuple(self.dims))


class RankStore:
    """One rank's particles: owned rows first, then ``ghosts`` ghost rows."""

    def __init__(self, fields: dict, ghosts: int = 0):
        self.f = {k: np.array(v) for k, v in fields.items()}
        self.ghosts = ghosts

    @property
    def size(self):
        return next(iter(self.f.values())).shape[0]

    @property
    def owned(self):
        return self.size - self.ghosts

    def truncate_ghosts(self):
        o = self.owned
        self.f = {k: v[:o].copy() for k, v in self.f.items()}
        self.ghosts = 0


def migrate(fab: Fabric, ranks, position_field="x"):
    """Redistribute particles to owners; arrivals ordered by (src rank, src
    index) -- ref decomp.py:77-112."""
    outgoing = []
    for st in ranks:
        st.truncate_ghosts()
        data = {k: v for k, v in st.f.items()}
        x = box_wrap(data[position_field], fab.low, fab.high, fab.periodic)
        for a in np.flatnonzero(~fab.periodic):
            if np.any(x[:, a] < fab.low[a]) or np.any(x[:, a] > fab.high[a]):
                raise ValueError(f"particle outside global box on non-periodic axis {a}")
        data[position_field] = x
        outgoing.append((fab.owner_of(x), data))
    for r, st in enumerate(ranks):
        new = {}
        for k in st.f:
            new[k] = np.concatenate([data[k][own == r] for own, data in outgoing],
                                    axis=0)
        st.f = new
        st.ghosts = 0


def _dist2_to_box(x, lo, hi):
    """ref decomp.py:115-120."""
    d = np.maximum(lo - x, 0.0) + np.maximum(x - hi, 0.0)
    return sqnorm(d)


def build_halo(fab: Fabric, ranks, width, position_field="x"):
    """Export plan: per (particle, adjacent rank) best periodic image, export
    iff d^2 < w^2 -- ref decomp.py:143-228.  Returns a dict plan."""
    bl = fab.block_lengths
    if width <= 0:
        raise ValueError("halo width must be positive")
    if width > bl.min() * (1 + 1e-12):
        raise ValueError("halo width exceeds the smallest local box edge")
    d = fab.low.shape[0]
    w2 = width * width
    exp_idx, exp_dest, exp_shift = [], [], []
    for r, st in enumerate(ranks):
        x = st.f[position_field][:st.owned]
        n = x.shape[0]
        me = fab.coords_of(r)
        best = {}
        for off in itertools.product(*[(-1, 0, 1)] * d):
            if not any(off):
                continue
            tgt = me + np.asarray(off)
            shift = np.zeros(d)
            valid = True
            for a in range(d):
                if 0 <= tgt[a] < fab.dims[a]:
                    continue
                if not fab.periodic[a]:
                    valid = False
                    break
                if tgt[a] < 0:
                    tgt[a] += fab.dims[a]
                    shift[a] = fab.lengths[a]
                else:
                    tgt[a] -= fab.dims[a]
                    shift[a] = -fab.lengths[a]
            if not valid:
                continue
            dest = fab.rank_of(tgt)
            if dest == r:
                continue
            lo, hi = fab.local_box(dest)
            d2 = _dist2_to_box(x + shift, lo, hi)
            if dest in best:
                b2, bs = best[dest]
                better = d2 < b2
                best[dest] = (np.where(better, d2, b2),
                              np.where(better[:, None], shift, bs))
            else:
                best[dest] = (d2, np.broadcast_to(shift, (n, d)).copy())
        ii, dd, ss = [], [], []
        for dest in sorted(best):
            b2, bs = best[dest]
            sel = np.flatnonzero(b2 < w2)
            ii.append(sel)
            dd.append(np.full(sel.size, dest, np.int64))
            ss.append(bs[sel])
        exp_idx.append(np.concatenate(ii) if ii else np.empty(0, np.int64))
        exp_dest.append(np.concatenate(dd) if dd else np.empty(0, np.int64))
        exp_shift.append(np.concatenate(ss, axis=0) if ss else np.empty((0, d)))
    layout = [[] for _ in range(fab.n_ranks)]
    for s in range(fab.n_ranks):
        for dest in np.unique(exp_dest[s]):
            layout[int(dest)].append((s, int((exp_dest[s] == dest).sum())))
    for lay in layout:
        lay.sort()
    return {"width": width, "position_field": position_field,
            "export_index": exp_idx, "export_dest": exp_dest,
            "export_shift": exp_shift, "import_layout": layout,
            "owned_snapshot": tuple(st.owned for st in ranks)}


def halo_gather(plan, ranks, fields=None):
    """Rebuild the ghost tail: ascending source rank, positions shifted,
    unrequested fields zero -- ref decomp.py:231-260."""
    if tuple(st.owned for st in ranks) != plan["owned_snapshot"]:
        raise RuntimeError("stale halo plan: particle residency changed since build")
    pf = plan["position_field"]
    if fields is not None and pf not in fields:
        fields = list(fields) + [pf]
    staged = []
    for s, st in enumerate(ranks):
        names = fields if fields is not None else list(st.f)
        data = {k: st.f[k][:st.owned][plan["export_index"][s]] for k in names}
        data[pf] = data[pf] + plan["export_shift"][s]
        staged.append(data)
    for r, st in enumerate(ranks):
        st.truncate_ghosts()
        total = sum(c for _, c in plan["import_layout"][r])
        for k, v in st.f.items():
            ghost = np.zeros((total,) + v.shape[1:], v.dtype)
            pos = 0
            for s, c in plan["import_layout"][r]:
                if k in staged[s]:
                    ghost[pos:pos + c] = staged[s][k][plan["export_dest"][s] == r]
                pos += c
            st.f[k] = np.concatenate([v, ghost], axis=0)
        st.ghosts = total


def halo_scatter(plan, ranks, fields):
    """Add ghost values back to owners in ascending dest order, then zero the
    ghosts -- ref decomp.py:263-300."""
    if tuple(st.owned for st in ranks) != plan["owned_snapshot"]:
        raise RuntimeError("stale halo plan: particle residency changed since build")
    for r, st in enumerate(ranks):
        if st.size != st.owned + sum(c for _, c in plan["import_layout"][r]):
            raise RuntimeError("halo_scatter without matching gather")
    base = []
    for r, st in enumerate(ranks):
        b, pos = {}, st.owned
        for s, c in plan["import_layout"][r]:
            b[s] = pos
            pos += c
        base.append(b)
    for k in fields:
        snap = [st.f[k].copy() for st in ranks]
        for r, st in enumerate(ranks):
            loc = st.f[k].copy()
            dests = plan["export_dest"][r]
            for dest in np.unique(dests):
                sel = dests == dest
                b0 = base[int(dest)][r]
                np.add.at(loc, plan["export_index"][r][sel],
                          snap[int(dest)][b0:b0 + int(sel.sum())])
            st.f[k] = loc
        for st in ranks:
            if st.ghosts:
                st.f[k][st.owned:] = 0


# ---------------------------------------------------------------------------
# MD driver (ref: md.py)
# ---------------------------------------------------------------------------

CUTOFF_MARGIN = 1.0 + 1e-9          # ref md.py:32-34


@dataclass
class MDConfig:
    """Field names and defaults of ref md.py:37-64."""
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
        """ref md.py:55-64."""
        if self.rebuild_stride > 1 and self.skin <= 0:
            raise ValueError("rebuild_stride > 1 requires a positive skin")
        if self.sort_stride and self.sort_stride % self.rebuild_stride:
            raise ValueError("sort_stride must be a multiple of rebuild_stride")
        for name in ("lattice_cells", "vector_length", "rebuild_stride"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be >= 1")
        if self.dt <= 0 or self.cutoff <= 0 or self.density <= 0:
            raise ValueError("dt, cutoff and density must be positive")


class MDOracle:
    """Velocity-Verlet LJ NVE on a simulated rank fabric -- ref md.py:129-292."""

    def __init__(self, cfg: MDConfig, cell_loop: bool = False):
        cfg.validate()
        self.cfg = cfg
        # cell_loop: neighbor lists through the reference's per-cell loop
        # (neighbor_pairs_cell_loop; same pairs, the reference's cost profile)
        self._pairs_fn = neighbor_pairs_cell_loop if cell_loop else neighbor_pairs
        a = (4.0 / cfg.density) ** (1.0 / 3.0)
        L = cfg.lattice_cells * a
        self.low = np.zeros(3)
        self.high = np.full(3, float(L))
        self.length = self.high - self.low
        self.periodic = np.array([True, True, True])
        self.n = 4 * cfg.lattice_cells ** 3
        self.fab = Fabric(self.low, self.high, cfg.rank_dims, self.periodic)
        hw = (cfg.cutoff + cfg.skin) * CUTOFF_MARGIN
        if hw > self.fab.block_lengths.min():
            raise ValueError("cutoff + skin exceeds the local box edge for this rank grid")
        self.halo_width = hw
        x = fcc_lattice(cfg.lattice_cells, a)
        v = initial_velocities(self.n, cfg.temperature, cfg.mass, cfg.seed)
        empty = lambda m: {"x": np.zeros((m, 3)), "x0": np.zeros((m, 3)),
                           "v": np.zeros((m, 3)), "f": np.zeros((m, 3)),
                           "id": np.zeros(m, np.int64)}
        self.ranks = [RankStore(empty(0)) for _ in range(self.fab.n_ranks)]
        s0 = empty(self.n)
        s0["x"][:] = x
        s0["v"][:] = v
        s0["id"][:] = np.arange(self.n)
        self.ranks[0] = RankStore(s0)
        migrate(self.fab, self.ranks)
        self.plan = None
        self.pairs = None
        self.pe_rows = {}
        self.timings = {k: 0.0 for k in
                        ("integrate", "sort", "migrate", "halo", "neighbor", "force")}
        self._rebuild_and_force()

    def _rebuild_and_force(self):
        """ref md.py:169-190."""
        t0 = time.perf_counter()
        migrate(self.fab, self.ranks)
        self.timings["migrate"] += time.perf_counter() - t0
        for st in self.ranks:
            st.f["x0"] = st.f["x"].copy()
        t0 = time.perf_counter()
        self.plan = build_halo(self.fab, self.ranks, self.halo_width)
        halo_gather(self.plan, self.ranks, fields=["x0", "id"])
        self.timings["halo"] += time.perf_counter() - t0
        t0 = time.perf_counter()
        search = (self.cfg.cutoff + self.cfg.skin) * CUTOFF_MARGIN
        self.pairs = [self._pairs_fn(st.f["x0"], self.low, self.high,
                                     self.periodic, search) for st in self.ranks]
        self.timings["neighbor"] += time.perf_counter() - t0
        self._forces()

    def _refresh_ghosts_and_force(self):
        """ref md.py:192-200."""
        for st in self.ranks:
            x0 = st.f["x"].copy()
            x0[st.owned:] = 0.0
            st.f["x0"] = x0
        t0 = time.perf_counter()
        halo_gather(self.plan, self.ranks, fields=["x0", "id"])
        self.timings["halo"] += time.perf_counter() - t0
        self._forces()

    def _forces(self):
        """ref md.py:202-215."""
        t0 = time.perf_counter()
        c = self.cfg
        for r, st in enumerate(self.ranks):
            pi, pj = self.pairs[r]
            f, pe = lj_forces(st.f["x0"], st.f["id"], st.owned, pi, pj,
                              self.length, self.periodic, c.epsilon, c.sigma,
                              c.cutoff)
            full = np.zeros((st.size, 3))
            full[:st.owned] = f
            st.f["f"] = full
            self.pe_rows[r] = pe
        self.timings["force"] += time.perf_counter() - t0

    def step(self, s):
        """ref md.py:219-257."""
        c = self.cfg
        dtm = 0.5 * c.dt / c.mass
        t0 = time.perf_counter()
        for st in self.ranks:
            o = st.owned
            v = st.f["v"].copy()
            x = st.f["x"].copy()
            v[:o] += dtm * st.f["f"][:o]
            x[:o] += c.dt * v[:o]
            st.f["v"] = v
            st.f["x"] = box_wrap(x, self.low, self.high, self.periodic)
        self.timings["integrate"] += time.perf_counter() - t0
        if s % c.rebuild_stride == 0:
            if c.sort_stride and s % c.sort_stride == 0:
                t0 = time.perf_counter()
                for st in self.ranks:
                    st.truncate_ghosts()
                    if st.owned < 2:
                        continue
                    xs = box_wrap(st.f["x"], self.low, self.high, self.periodic)
                    _, _, pm = bin_by_position(xs, self.low, self.high, c.cutoff)
                    st.f = {k: apply_permutation(v, pm) for k, v in st.f.items()}
                self.timings["sort"] += time.perf_counter() - t0
            self._rebuild_and_force()
        else:
            self._refresh_ghosts_and_force()
        t0 = time.perf_counter()
        for st in self.ranks:
            o = st.owned
            v = st.f["v"].copy()
            v[:o] += dtm * st.f["f"][:o]
            st.f["v"] = v
        self.timings["integrate"] += time.perf_counter() - t0

    def diagnostics(self):
        """Energies summed in global-id order -- ref md.py:261-277."""
        c = self.cfg
        ke_g = np.zeros(self.n)
        pe_g = np.zeros(self.n)
        mom = np.zeros((self.n, 3))
        for r, st in enumerate(self.ranks):
            o = st.owned
            ids = st.f["id"][:o]
            v = st.f["v"][:o]
            ke_g[ids] = 0.5 * c.mass * np.einsum("ij,ij->i", v, v)
            mom[ids] = c.mass * v
            pe_g[ids] = self.pe_rows[r]
        ke = float(np.sum(ke_g))
        pe = float(np.sum(pe_g))
        return {"KE": ke, "PE": pe, "E_total": ke + pe,
                "temperature": 2.0 * ke / (3.0 * self.n),
                "momentum": mom.sum(axis=0)}

    def gather_state(self):
        """ref md.py:279-287."""
        x = np.zeros((self.n, 3))
        v = np.zeros((self.n, 3))
        for st in self.ranks:
            o = st.owned
            x[st.f["id"][:o]] = st.f["x"][:o]
            v[st.f["id"][:o]] = st.f["v"][:o]
        return x, v

    def negate_velocities(self):
        """ref md.py:289-292."""
        for st in self.ranks:
            st.f["v"] = -st.f["v"]


def run_md(cfg: MDConfig):
    """ref md.py:295-307: rows of step/KE/PE/E_total/temperature + timings."""
    drv = MDOracle(cfg)
    drv.timings = {k: 0.0 for k in drv.timings}
    d = drv.diagnostics()
    rows = [dict(step=0, KE=d["KE"], PE=d["PE"], E_total=d["E_total"],
                 temperature=d["temperature"])]
    for s in range(1, cfg.steps + 1):
        drv.step(s)
        d = drv.diagnostics()
        rows.append(dict(step=s, KE=d["KE"], PE=d["PE"], E_total=d["E_total"],
                         temperature=d["temperature"]))
    return rows, dict(drv.timings)
