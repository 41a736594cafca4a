"""GPU parity at the benchmarked sizes (VERDICT r1 "next" #1).

The MD engine's tile path -- the configuration bench.py measures -- against
the CPU oracle on identical positions:

* C2 (fcc 64^3 = 1,048,576 atoms, the configs[1] workload): the whole
  Verlet list of the step-20 rebuild equals the oracle's ``build_verlet`` on
  the step-20 positions as sorted per-particle sets, bit for bit; five steps
  later every atom's force is within 1e-5 * max(|F_ref,i|_inf, F_rms) and PE
  within 1e-6.
* C3 (fcc 128^3 = 8,388,608 atoms, the BASELINE metric's configuration):
  the same checks on a random 100k-row sample (the oracle restricted to those
  rows), plus the tile path's FP32-per-pair / FP64-per-row energies against
  the SELL path's FP64 energies on the same state (1e-6).
* Hot C4 (T = 3.0, rebuild every 5 steps) at 32^3 (131k atoms), full checks.

References: ref neighbors.py:49-97 (sets), md.py:99-126 (forces / PE).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FORCE_TOL = 1e-5
ENERGY_TOL = 1e-6


@pytest.fixture(scope="module")
def pc():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2109_09056_b200 as pkg
    return pkg


def _err_ratio(f, fref):
    frms = np.sqrt((fref ** 2).sum(1).mean())
    tol = FORCE_TOL * np.maximum(np.abs(fref).max(1), frms)
    return float((np.abs(f - fref).max(1) / tol).max())


def _engine(pc, cells, temp, rebuild, steps, seed=5):
    cfg = pc.md.MDConfig(lattice_cells=cells, density=0.8442, temperature=temp, cutoff=2.5,
                         skin=0.3, rebuild_stride=rebuild, seed=seed, steps=0)
    drv = pc.md.MDDriver(cfg, time_phases=False)
    _advance(drv, 0, steps)
    assert drv.mode == "tile" and drv.tile_failures == 0
    return drv


def _advance(drv, s0, s1):
    for s in range(s0 + 1, s1 + 1):
        drv.step(s)


def _gid(drv):
    import torch
    return drv.pos[: drv.n, 3].contiguous().view(torch.int64).cpu().numpy()


def _forces_by_gid(drv, gid):
    f = np.empty((drv.n, 3))
    f[gid] = drv.frc[:, : drv.n].cpu().numpy().T
    return f


def _sampled_rows(drv, gid, sample):
    """Tile-list rows of the particles with global ids `sample`: {gid: sorted
    neighbour gids} (decoded on the device, only the sampled rows copied)."""
    import torch
    cnt, table = drv._tile_rows()
    inv = np.empty(drv.n, np.int64)
    inv[gid] = np.arange(drv.n)
    loc = torch.as_tensor(inv[sample], device=drv.device)
    c = cnt[loc].cpu().numpy()
    t = table[loc].cpu().numpy()
    return [np.sort(gid[t[k, : c[k]]]) for k in range(sample.size)]


def _check_sets(oracle, drv, x, gid, rows=None):
    pi, pj = oracle.neighbor_pairs(x, drv.box.low, drv.box.high, [True] * 3, drv.search,
                                   rows=rows)
    if rows is None:
        counts, offsets, idx = drv.verlet_sets()
        assert np.array_equal(counts, np.bincount(pi, minlength=drv.n))
        assert np.array_equal(idx, pj)
        return
    mine = _sampled_rows(drv, gid, rows)
    starts = np.searchsorted(pi, rows)
    ends = np.searchsorted(pi, rows, side="right")
    for k in range(rows.size):
        assert np.array_equal(mine[k], pj[starts[k]:ends[k]]), f"row {rows[k]}"


def _check_forces(oracle, drv, x, f, rows=None):
    pi, pj = oracle.neighbor_pairs(x, drv.box.low, drv.box.high, [True] * 3,
                                   2.5 * 1.0000001, rows=rows)
    fref, peref = oracle.lj_forces(x, np.arange(drv.n), drv.n, pi, pj, drv.box.lengths,
                                   [True] * 3, 1.0, 1.0, 2.5)
    sel = slice(None) if rows is None else rows
    assert _err_ratio(f[sel], fref[sel]) < 1.0
    return peref


def test_c2_full_lists_forces_energy(pc, oracle):
    """C2 (configs[1]): whole list bit-exact at the step-20 rebuild; all
    forces and PE five steps later."""
    drv = _engine(pc, 64, 1.44, 20, 20)       # the list of the step-20 rebuild
    x, _ = drv.gather_state()
    _check_sets(oracle, drv, x, _gid(drv))
    _advance(drv, 20, 25)                     # forces 5 steps into the list's life
    x, _ = drv.gather_state()
    gid = _gid(drv)
    f = _forces_by_gid(drv, gid)
    peref = _check_forces(oracle, drv, x, f)
    d = drv.diagnostics()
    assert abs(d["PE"] - peref.sum()) <= ENERGY_TOL * abs(peref.sum())
    assert np.abs(f.sum(0)).max() < 1e-8


def test_c3_sampled_rows(pc, oracle):
    """C3, the metric's size (8.4M atoms): 100k sampled rows -- lists
    bit-exact and forces within tolerance; tile vs SELL-path energies."""
    drv = _engine(pc, 128, 1.44, 20, 20)
    x, _ = drv.gather_state()
    rows = np.sort(np.random.default_rng(11).choice(drv.n, 100_000, replace=False))
    _check_sets(oracle, drv, x, _gid(drv), rows)
    _advance(drv, 20, 25)
    x, _ = drv.gather_state()
    gid = _gid(drv)
    f = _forces_by_gid(drv, gid)
    _check_forces(oracle, drv, x, f, rows)
    d_tile = drv.diagnostics()
    assert np.abs(f.sum(0)).max() < 1e-7
    # the same state through the SELL path (FP64 LJ, FP64 per-row energies)
    x, v = drv.gather_state()
    cfg = pc.md.MDConfig(lattice_cells=128, density=0.8442, temperature=1.44, cutoff=2.5,
                         skin=0.3, rebuild_stride=20, seed=5, steps=0)
    del drv
    ref = pc.md.MDDriver(cfg, state=(x, v), tile=False, time_phases=False)
    d_sell = ref.diagnostics()
    assert abs(d_tile["PE"] - d_sell["PE"]) <= ENERGY_TOL * abs(d_sell["PE"])
    assert abs(d_tile["KE"] - d_sell["KE"]) <= 1e-12 * abs(d_sell["KE"])


def test_hot_c4_32cubed(pc, oracle):
    """Hot liquid (T = 3.0, rebuild every 5 steps) at 32^3 = 131k atoms,
    whole list bit-exact at the step-15 rebuild (the third), forces and PE
    two steps later."""
    drv = _engine(pc, 32, 3.0, 5, 15)
    x, _ = drv.gather_state()
    _check_sets(oracle, drv, x, _gid(drv))
    _advance(drv, 15, 17)
    x, _ = drv.gather_state()
    gid = _gid(drv)
    f = _forces_by_gid(drv, gid)
    peref = _check_forces(oracle, drv, x, f)
    d = drv.diagnostics()
    assert abs(d["PE"] - peref.sum()) <= ENERGY_TOL * abs(peref.sum())


@pytest.mark.timeout(300)
def test_partial_staging_overflow_no_hang(pc, oracle):
    """some tiles overflow the staging area, others do not,
    with > 4 tiles per force CTA -- the speculative tile force must not hang
    (an overflowing tile keeps one empty row-warp that releases its staging
    buffer) and the step falls back to the SELL path with correct forces.
    40^3 fcc cells; the lower 85 % of the atoms (in x) are compressed into 60 %
    of the box (rho ~ 1.2: ~2700-slot neighbourhoods > 2304), the rest spread
    over the remaining 40 %."""
    import torch
    cells = 40
    a = (4.0 / 0.8442) ** (1.0 / 3.0)
    L = cells * a
    x = pc.md.fcc_lattice(cells, a)
    t = x[:, 0] / L
    cut = 0.853
    x[:, 0] = np.where(t < cut, t * (0.6 / cut), 0.6 + (t - cut) * (0.4 / (1 - cut))) * L
    x[:, 0] = np.minimum(x[:, 0], np.nextafter(L, 0))
    v = pc.md.initial_velocities(x.shape[0], 1.0, 1.0, 2)
    cfg = pc.md.MDConfig(lattice_cells=cells, density=0.8442, temperature=1.0, cutoff=2.5,
                         skin=0.3, rebuild_stride=10, seed=2, steps=0)
    drv = pc.md.MDDriver(cfg, state=(x, v), time_phases=False)
    assert drv.tile_failures >= 1 and drv.mode == "sell"
    ntiles = int(pc._lib.load().pc_tile_count(drv._grid))
    assert ntiles >= 5 * 148
    for s in range(1, 3):
        drv.step(s)
    xs, _ = drv.gather_state()
    gid = drv.pos[: drv.n, 3].contiguous().view(torch.int64).cpu().numpy()
    f = np.empty((drv.n, 3))
    f[gid] = drv.frc[:, : drv.n].cpu().numpy().T
    _check_forces(oracle, drv, xs, f)
