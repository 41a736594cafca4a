"""GPU parity: the CUDA path (through the C ABI) vs golden vectors produced by
the reference and vs the pinned CPU oracle.  Run with ``-m gpu`` on a B200.

Bars: bit-exact for binning, permutations, neighbor lists and the geometry
helpers; forces per atom within 1e-5 * max(|F_ref,i|_inf, F_rms) (the
north_star FP32 tolerance); energies within 1e-6 relative.
"""

import hashlib
import json

import numpy as np
import pytest

from conftest import load_cases, load_flat

pytestmark = pytest.mark.gpu

FORCE_TOL = 1e-5        # relative, per atom, vs max(|F_ref,i|_inf, F_rms)
ENERGY_TOL = 1e-6       # relative, per evaluation


@pytest.fixture(scope="module")
def pc():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2109_09056_b200 as pkg
    return pkg


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def force_err_ratio(f, fref):
    frms = np.sqrt((fref ** 2).sum(1).mean())
    tol = FORCE_TOL * np.maximum(np.abs(fref).max(1), frms)
    return float((np.abs(f - fref).max(1) / tol).max())


# ---------------------------------------------------------------- geometry
def test_box_wrap_min_image_bit_exact(pc, oracle):
    rng = np.random.default_rng(1)
    box = pc.geometry.Box([-1.0, 0.0, 2.0], [3.0, 5.5, 4.25])
    L = box.lengths
    x = box.low + rng.uniform(-3, 4, (5000, 3)) * L
    x[:10] = box.high            # exactly on the upper face
    per = [True, False, True]
    got = box.wrap(x, per)
    ref = oracle.box_wrap(x, box.low, box.high, per)
    assert np.array_equal(got, ref)
    d = rng.uniform(-2.5, 2.5, (5000, 3)) * L
    assert np.array_equal(box.min_image(d, per), oracle.box_min_image(d, L, per))


# ---------------------------------------------------------------- binning
BN = load_cases("binning.npz")


@pytest.mark.parametrize("case", [k for k in sorted(BN) if k.startswith("d")])
def test_binning_bit_exact(pc, case):
    c = BN[case]
    box = pc.geometry.Box(c["low"], c["high"])
    nc, idx = pc.binning.cell_indices(c["x"], box, float(c["cs"]))
    assert np.array_equal(nc, c["nc"]) and np.array_equal(idx, c["idx"])
    cb = pc.binning.bin_by_position(c["x"], box, float(c["cs"]))
    assert np.array_equal(cb.offsets, c["offsets"])
    assert np.array_equal(cb.permutation.map, c["map"])
    assert cb.permutation.is_bijection()


def test_bin_by_key_stable(pc):
    c = BN["keys300"]
    assert np.array_equal(pc.binning.bin_by_key(c["keys"]).map, c["map"])
    keys = np.array([3, 1, 3, 0, 1, 3])
    p = pc.binning.bin_by_key(keys)
    srt = np.empty_like(keys)
    srt[p.map] = keys
    assert np.array_equal(srt, np.sort(keys))
    wide = np.random.default_rng(3).integers(-2**60, 2**60, 5000)
    pw = pc.binning.bin_by_key(wide)
    assert np.array_equal(np.argsort(pw.map), np.argsort(wide, kind="stable"))


def test_bin_by_key_large_equal_groups(pc):
    """Few distinct keys over many elements (every digit bin holds ~n/3):
    stable and O(n) (pc_partition_*), vs numpy's stable argsort."""
    keys = np.random.default_rng(4).integers(0, 3, 400_000)
    p = pc.binning.bin_by_key(keys)
    assert np.array_equal(np.argsort(p.map), np.argsort(keys, kind="stable"))
    same = np.full(100_000, 7)
    assert np.array_equal(pc.binning.bin_by_key(same).map, np.arange(100_000))


def test_group_by_owner_ranks_1m(pc):
    """Grouping 1M particles by owner rank (ref decomp.py:97-99): stable."""
    import torch
    from paper_2109_09056_b200.decomp import _group_by
    own = np.random.default_rng(5).integers(0, 8, 1 << 20).astype(np.int32)
    order, starts = _group_by(torch.as_tensor(own).cuda(), 8)
    ref = np.argsort(own, kind="stable")
    assert np.array_equal(order.cpu().numpy(), ref)
    assert np.array_equal(starts, np.concatenate(([0], np.cumsum(np.bincount(own, minlength=8)))))


def test_cell_indices_rejects_outside(pc):
    box = pc.geometry.Box([0.0], [1.0])
    with pytest.raises(ValueError):
        pc.binning.cell_indices(np.array([[1.5]]), box, 0.5)


def test_permute_all_fields(pc):
    rng = np.random.default_rng(1)
    for V in (1, 3, 4, 16, 64):
        sch = pc.aosoa.schema(x=("float64", (3,)), s=("float64", (3, 3)), id=("int64", ()))
        p = pc.aosoa.create(sch, V, 30)
        x = rng.random((30, 3))
        s = rng.random((30, 3, 3))
        p.slice("x").copy_in(x)
        p.slice("s").copy_in(s)
        p.slice("id").copy_in(np.arange(30, dtype=np.int64))
        perm = pc.binning.bin_by_key(rng.integers(0, 5, 30))
        pc.binning.permute(p, perm)
        ids = p.slice("id").copy_out()
        xo, so = p.slice("x").copy_out(), p.slice("s").copy_out()
        for i in range(30):
            assert ids[perm.map[i]] == i
            assert np.array_equal(xo[perm.map[i]], x[i])
            assert np.array_equal(so[perm.map[i]], s[i])
    p = pc.aosoa.create(pc.aosoa.schema(m=("float64", ())), 2, 3)
    with pytest.raises(ValueError):
        pc.binning.permute(p, pc.binning.Permutation(np.array([0, 0, 1])))
    with pytest.raises(ValueError):
        pc.binning.permute(p, pc.binning.Permutation(np.array([0, 1])))


# ---------------------------------------------------------------- aosoa
@pytest.mark.parametrize("V", [1, 2, 5, 16, 17])
@pytest.mark.parametrize("n", [0, 1, 7, 40])
def test_aosoa_roundtrip(pc, V, n):
    sch = pc.aosoa.schema(x=("float64", (3,)), m=("float64", ()),
                          stress=("float64", (3, 3)), id=("int64", ()))
    p = pc.aosoa.create(sch, V, n)
    assert p.capacity == -(-n // V) * V
    rng = np.random.default_rng(n * 31 + V)
    vals = {"x": rng.random((n, 3)), "m": rng.random(n), "stress": rng.random((n, 3, 3)),
            "id": rng.integers(-2**40, 2**40, n)}
    for k, v in vals.items():
        assert np.all(p.slice(k).copy_out() == 0)
        p.slice(k).copy_in(v)
    for k, v in vals.items():
        assert np.array_equal(p.slice(k).copy_out(), v)
    if n:
        assert np.array_equal(p.slice("stress")[n - 1], vals["stress"][n - 1])
        assert p.slice("x")[0, 2] == vals["x"][0, 2]
        p.slice("m")[0] = 5.0
        assert p.slice("m")[0] == 5.0
        p.resize(n + 3)
        assert np.array_equal(p.slice("x").copy_out()[:n], vals["x"])
        assert np.all(p.slice("x").copy_out()[n:] == 0)
        q = pc.aosoa.create(sch, 4, n + 3)
        pc.aosoa.deep_copy(q, p)
        assert np.array_equal(q.slice("stress").copy_out(), p.slice("stress").copy_out())


# ---------------------------------------------------------------- neighbors
NB = load_cases("neighbors.npz")


@pytest.mark.parametrize("case", sorted(NB))
def test_neighbor_lists_bit_exact(pc, case):
    c = NB[case]
    box = pc.geometry.Box(c["low"], c["high"])
    for layout in ("compressed", "dense"):
        for conv in ("full", "half"):
            vl = pc.neighbors.build_verlet(c["x"], box, c["periodic"], float(c["cutoff"]),
                                           layout=layout, half_or_full=conv,
                                           cell_ratio=float(c["ratio"]))
            key = f"{layout}_{conv}"
            assert np.array_equal(vl.counts, c[f"{key}_counts"]), key
            if layout == "compressed":
                assert np.array_equal(vl.indices, c[f"{key}_indices"]), key
                assert np.array_equal(vl.offsets, c[f"{key}_offsets"]), key
            else:
                assert np.array_equal(vl.table, c[f"{key}_table"]), key


def test_neighbor_argument_errors(pc):
    box = pc.geometry.cube(2.0)
    x = np.zeros((1, 3))
    for kw in (dict(cutoff=-1.0), dict(cutoff=1.5), dict(cutoff=0.5, layout="sparse"),
               dict(cutoff=0.5, cell_ratio=0.5), dict(cutoff=0.5, half_or_full="x")):
        cutoff = kw.pop("cutoff")
        with pytest.raises(ValueError):
            pc.neighbors.build_verlet(x, box, [True] * 3, cutoff, **kw)


def test_neighbor_properties(pc, oracle):
    rng = np.random.default_rng(7)
    box = pc.geometry.cube(3.0)
    x = rng.random((100, 3)) * 3.0
    half = pc.neighbors.build_verlet(x, box, [True] * 3, 0.9, half_or_full="half")
    full = pc.neighbors.build_verlet(x, box, [True] * 3, 0.9, half_or_full="full")
    assert 2 * half.total == full.total
    i, j = half.pairs()
    assert np.all(j > i)
    seen = []
    pc.neighbors.for_each_neighbor(full, (0, 100), lambda a, b: seen.append((a, b)))
    ii, jj = full.pairs()
    assert seen == list(zip(ii.tolist(), jj.tolist()))
    trip = []
    pc.neighbors.for_each_neighbor2(full, (0, 100), lambda a, b, c: trip.append(a))
    assert len(trip) == int(sum(k * (k - 1) // 2 for k in full.counts))
    # rebuild idempotence
    again = pc.neighbors.build_verlet(x, box, [True] * 3, 0.9)
    assert np.array_equal(again.indices, full.indices)


@pytest.mark.parametrize("seed", range(20))
def test_criterion1_oracle_20_seeds(pc, oracle, seed):
    """ref tests/test_acceptance.py:22-50 at full size, all four variants."""
    n = 1000
    rc = (30 * 3 / (4 * np.pi * n)) ** (1 / 3)
    x = np.random.default_rng(seed).random((n, 3))
    ref = oracle.build_verlet(x, np.zeros(3), np.ones(3), [True] * 3, rc)
    box = pc.geometry.cube(1.0)
    for layout in ("dense", "compressed"):
        for conv in ("half", "full"):
            vl = pc.neighbors.build_verlet(x, box, [True] * 3, rc, layout=layout,
                                           half_or_full=conv)
            want = oracle.build_verlet(x, np.zeros(3), np.ones(3), [True] * 3, rc,
                                       layout=layout, half_or_full=conv)
            assert np.array_equal(vl.counts, want["counts"])
            if layout == "compressed":
                assert np.array_equal(vl.indices, want["indices"])
            else:
                assert np.array_equal(vl.table, want["table"])
    assert abs(ref["counts"].mean() - 30) < 3


# ---------------------------------------------------------------- LJ forces
LJ = load_flat("lj.npz")


@pytest.mark.parametrize("name", ["c8", "c16"])
def test_lj_forces_within_tolerance(pc, name):
    x0, ids, L = LJ[f"{name}_x0"], LJ[f"{name}_ids"], LJ[f"{name}_L"]
    box = pc.geometry.Box(np.zeros(3), L)
    vl = pc.neighbors.build_verlet(x0, box, [True] * 3, float(LJ[f"{name}_search"]))
    assert np.array_equal(vl.counts, LJ[f"{name}_counts"])
    assert _digest(vl.offsets, vl.indices) == str(LJ[f"{name}_csr_digest"])
    f, pe = pc.md.lj_forces(x0, ids, x0.shape[0], vl, box, [True] * 3, 1.0, 1.0, 2.5)
    fref, peref = LJ[f"{name}_f"], LJ[f"{name}_pe"]
    assert force_err_ratio(f, fref) < 1.0
    assert abs(pe.sum() - peref.sum()) <= ENERGY_TOL * abs(peref.sum())
    assert np.max(np.abs(pe - peref)) < 1e-5 * np.abs(peref).max()
    # exact antisymmetry of FP64-accumulated pair forces: net force ~ 0
    assert np.abs(f.sum(0)).max() < 1e-9


def test_lj_forces_dense_layout_and_overlap(pc):
    x0, ids, L = LJ["c8_x0"], LJ["c8_ids"], LJ["c8_L"]
    box = pc.geometry.Box(np.zeros(3), L)
    vl = pc.neighbors.build_verlet(x0, box, [True] * 3, float(LJ["c8_search"]),
                                   layout="dense")
    f, pe = pc.md.lj_forces(x0, ids, x0.shape[0], vl, box, [True] * 3, 1.0, 1.0, 2.5)
    assert force_err_ratio(f, LJ["c8_f"]) < 1.0
    x = np.array([[1.0, 1.0, 1.0], [1.0, 1.0, 1.0 + 1e-12], [5.0, 5.0, 5.0]])
    b = pc.geometry.cube(10.0)
    v2 = pc.neighbors.build_verlet(x, b, [True] * 3, 2.5)
    with pytest.raises(FloatingPointError):
        pc.md.lj_forces(x, np.arange(3), 3, v2, b, [True] * 3, 1.0, 1.0, 2.5)


def test_lj_pair_reference_points(pc):
    e, _ = pc.md.lj_pair(np.array([[1.0, 0.0, 0.0]]), np.array([1.0]), 1.0, 1.0)
    assert abs(e[0]) < 1e-14
    rm = 2.0 ** (1 / 6)
    e, f = pc.md.lj_pair(np.array([[rm, 0.0, 0.0]]), np.array([rm * rm]), 1.0, 1.0)
    assert abs(e[0] + 1.0) < 1e-14 and np.max(np.abs(f)) < 1e-12


# ---------------------------------------------------------------- MD driver
MD = load_flat("md.npz")


def _series(rows):
    return np.array([[r["KE"], r["PE"], r["E_total"], r["temperature"]] for r in rows])


def test_md_initial_state_bit_exact(pc):
    drv = pc.md.MDDriver(pc.md.MDConfig(lattice_cells=4, density=1.1, cutoff=2.3, seed=2,
                                        steps=0))
    x, v = drv.gather_state()
    assert np.array_equal(x, MD["crit3_x_init"]) and np.array_equal(v, MD["crit3_v_init"])
    d = drv.diagnostics()
    ref = MD["crit3_series"][0]
    assert abs(d["KE"] - ref[0]) <= 1e-13 * abs(ref[0])
    assert abs(d["PE"] - ref[1]) <= ENERGY_TOL * abs(ref[1])


@pytest.mark.parametrize("name", ["crit3", "skin_sort", "hot", "c1"])
def test_md_energy_series(pc, name):
    """Energy series vs the reference run: per step relative 1e-5 on E_total
    (the trajectories separate chaotically from FP32-rounding seeds; within
    100-200 steps the separation stays well below this) and the same drift."""
    kw = json.loads(str(MD[f"{name}_config"]))
    rows, timings = pc.md.run_md(pc.md.MDConfig(**kw))
    got, ref = _series(rows), MD[f"{name}_series"]
    assert got.shape == ref.shape
    rel = np.abs(got[:, 2] - ref[:, 2]) / np.abs(ref[:, 2])
    assert rel.max() < 1e-5, rel.max()
    drift_got = abs(got[-1, 2] - got[0, 2]) / abs(got[0, 2])
    drift_ref = abs(ref[-1, 2] - ref[0, 2]) / abs(ref[0, 2])
    assert abs(drift_got - drift_ref) < 1e-5
    assert set(timings) == {"integrate", "sort", "migrate", "halo", "neighbor", "force"}


def test_md_momentum_and_reversal(pc):
    cfg = pc.md.MDConfig(lattice_cells=3, density=1.1, temperature=0.8, dt=0.005, steps=0,
                         cutoff=2.0, seed=2)
    drv = pc.md.MDDriver(cfg)
    x0, v0 = drv.gather_state()
    for s in range(1, 51):
        drv.step(s)
    assert np.max(np.abs(drv.diagnostics()["momentum"])) < 1e-9
    drv.negate_velocities()
    for s in range(51, 101):
        drv.step(s)
    x1, v1 = drv.gather_state()
    dx = x1 - x0
    L = drv.box.lengths
    dx -= L * np.round(dx / L)
    assert np.max(np.abs(dx)) < 1e-6
    assert np.max(np.abs(v1 + v0)) < 1e-6


def test_md_nve_drift_criterion4(pc):
    """ref tests/test_acceptance.py:97-123: 1000-step drift < 1e-4."""
    cfg = pc.md.MDConfig(lattice_cells=4, density=1.1, cutoff=2.3, seed=2, dt=0.005,
                         steps=1000)
    rows, _ = pc.md.run_md(cfg)
    e0 = rows[0]["E_total"]
    assert abs(rows[-1]["E_total"] - e0) / abs(e0) < 1e-4


def test_md_config_validation(pc):
    with pytest.raises(ValueError):
        pc.md.MDConfig(rebuild_stride=5).validate()
    with pytest.raises(ValueError):
        pc.md.MDConfig(skin=0.3, rebuild_stride=4, sort_stride=6).validate()
    with pytest.raises(ValueError):
        pc.md.MDConfig(dt=-0.1).validate()
    with pytest.raises(ValueError):
        pc.md.run_md(pc.md.MDConfig(lattice_cells=2))


def test_md_skin_and_stride_equivalence(pc):
    base = dict(lattice_cells=3, density=1.1, temperature=0.8, dt=0.005, cutoff=2.0, seed=2)
    ref, _ = pc.md.run_md(pc.md.MDConfig(steps=60, **base))
    rows, _ = pc.md.run_md(pc.md.MDConfig(steps=60, skin=0.2, rebuild_stride=5, **base))
    for a, b in zip(ref, rows):
        assert abs(a["E_total"] - b["E_total"]) < 1e-9 * abs(b["E_total"])


@pytest.mark.parametrize("cells,temp", [(16, 1.44), (8, 3.0), (6, 1.44)])
def test_md_verlet_list_bit_exact(pc, oracle, cells, temp):
    """The MD engine's SELL list (staged FP32-prefilter build when every axis
    has >= 3 cells) equals the oracle's list on the same positions, bit-exact,
    at init and after 25 steps (one rebuild at step 20)."""
    cfg = pc.md.MDConfig(lattice_cells=cells, density=0.8442, temperature=temp, cutoff=2.5,
                         skin=0.3, rebuild_stride=20, seed=3, steps=0)
    drv = pc.md.MDDriver(cfg, tile=True)
    for stage in range(2):
        if stage:
            for s in range(1, 21):
                drv.step(s)
        x, _ = drv.gather_state()
        counts, offsets, idx = drv.verlet_sets()
        ref = oracle.build_verlet(x, drv.box.low, drv.box.high, [True] * 3, drv.search)
        assert np.array_equal(counts, ref["counts"])
        assert np.array_equal(idx, ref["indices"])
    nc = int(np.floor(drv.box.lengths[0] / drv.search))
    if nc < 3:
        assert drv.mode == "sell"
    elif cells >= 16:       # small boxes with wide cells may exceed the staging area
        assert drv.mode == "tile"


@pytest.mark.parametrize("noise", [0.0, 1e-7])
def test_md_tile_list_pairs_at_search_radius(pc, oracle, noise):
    """fcc lattice whose fifth neighbour shell lies AT the search radius
    (a = 2.8 / sqrt(5/2)): 24 pairs per atom sit inside the tile build's FP32
    band, where the reference's FP64 predicate decides, on both sides of it
    with the noise.  The tile list equals the oracle's, bit-exact."""
    cells = 16
    a = 2.8 / np.sqrt(2.5)
    x = pc.md.fcc_lattice(cells, a)
    L = cells * a
    x = np.mod(x + np.random.default_rng(5).normal(0.0, noise, x.shape), L) if noise else x
    v = np.zeros_like(x)
    cfg = pc.md.MDConfig(lattice_cells=cells, density=4.0 / a ** 3, temperature=1.0,
                         cutoff=2.5, skin=0.3, rebuild_stride=20, seed=3, steps=0)
    drv = pc.md.MDDriver(cfg, state=(x, v), tile=True)
    assert drv.mode == "tile"
    xs, _ = drv.gather_state()
    counts, offsets, idx = drv.verlet_sets()
    ref = oracle.build_verlet(xs, drv.box.low, drv.box.high, [True] * 3, drv.search)
    assert np.array_equal(counts, ref["counts"])
    assert np.array_equal(idx, ref["indices"])
    # shells 1-4 (54 neighbours) always in, shell 5 (24) decided at the boundary
    assert 54 <= counts.min() and counts.max() <= 78
    if noise:
        assert 54 < counts.mean() < 78


@pytest.mark.parametrize("cells,temp", [(16, 1.44), (6, 3.0)])
def test_md_sell_path_verlet_bit_exact(pc, oracle, cells, temp):
    """Same check for the SELL fallback path (staged SELL build)."""
    cfg = pc.md.MDConfig(lattice_cells=cells, density=0.8442, temperature=temp, cutoff=2.5,
                         skin=0.3, rebuild_stride=20, seed=3, steps=0)
    drv = pc.md.MDDriver(cfg, tile=False)
    for s in range(1, 21):
        drv.step(s)
    x, _ = drv.gather_state()
    counts, offsets, idx = drv.verlet_sets()
    ref = oracle.build_verlet(x, drv.box.low, drv.box.high, [True] * 3, drv.search)
    assert np.array_equal(counts, ref["counts"]) and np.array_equal(idx, ref["indices"])
    assert drv.mode == "sell"


def test_md_tile_vs_sell_paths(pc):
    """The tile and SELL force paths integrate the same trajectory (FP32 LJ
    magnitude vs FP64 magnitude: 1e-6 relative on E_total over 60 steps)."""
    kw = dict(lattice_cells=12, density=0.8442, temperature=1.44, cutoff=2.5, skin=0.3,
              rebuild_stride=20, seed=4, steps=60)
    def series(tile):
        drv = pc.md.MDDriver(pc.md.MDConfig(**kw), tile=tile)
        out = [drv.diagnostics()["E_total"]]
        for s in range(1, 61):
            drv.step(s)
            out.append(drv.diagnostics()["E_total"])
        return np.array(out), drv.mode
    ea, ma = series(True)
    eb, mb = series(False)
    assert (ma, mb) == ("tile", "sell")
    assert np.max(np.abs(ea - eb) / np.abs(ea)) < 1e-6


def test_md_half_list_path(pc, oracle):
    """Newton-3 half list (one entry per unordered pair) integrates the same
    energy series as the full list (atomics reorder FP64 sums: 1e-9)."""
    kw = dict(lattice_cells=10, density=0.8442, temperature=1.44, cutoff=2.5, skin=0.3,
              rebuild_stride=20, seed=6, steps=0)

    def series(half):
        # full list on the SELL path: the same FP64 LJ magnitude as the half kernel
        drv = pc.md.MDDriver(pc.md.MDConfig(**kw), half_list=half, tile=False)
        out = [drv.diagnostics()["E_total"]]
        for s in range(1, 41):
            drv.step(s)
            d = drv.diagnostics()
            out.append(d["E_total"])
        return np.array(out), drv, d
    ef, _, _ = series(False)
    eh, drv, d = series(True)
    assert drv.mode == "half"
    assert np.max(np.abs(ef - eh) / np.abs(ef)) < 1e-9
    assert np.max(np.abs(d["momentum"])) < 1e-9
    # half list content: each unordered pair of the (last rebuild's) full
    # list exactly once
    drv2 = pc.md.MDDriver(pc.md.MDConfig(**kw), half_list=True)
    counts, offsets, idx = drv2.verlet_sets()
    rows = np.repeat(np.arange(drv2.n), counts)
    pairs = set(zip(np.minimum(rows, idx).tolist(), np.maximum(rows, idx).tolist()))
    assert len(pairs) == idx.size
    p = drv2.pos[: drv2.n].cpu().numpy()
    x = np.empty((drv2.n, 3))
    x[p[:, 3].copy().view(np.int64)] = p[:, :3]
    ref = oracle.build_verlet(x, drv2.box.low, drv2.box.high, [True] * 3, drv2.search,
                              half_or_full="half")
    assert idx.size == ref["indices"].size


@pytest.mark.parametrize("cells,temp,steps", [(12, 1.44, 25), (12, 3.0, 7), (16, 1.44, 45)])
def test_md_engine_forces_vs_oracle(pc, oracle, cells, temp, steps):
    """The MD engine's force array (tile path: FP32 LJ magnitude, FP64
    accumulation) against the oracle's FP64 lj_forces on the same positions,
    per atom within 1e-5 * max(|F_ref,i|_inf, F_rms), several steps after a
    rebuild; net force ~ 0 (exact pair antisymmetry)."""
    cfg = pc.md.MDConfig(lattice_cells=cells, density=0.8442, temperature=temp, cutoff=2.5,
                         skin=0.3, rebuild_stride=20, seed=5, steps=0)
    drv = pc.md.MDDriver(cfg)
    assert drv.mode == "tile"
    for s in range(1, steps + 1):
        drv.step(s)
    x, _ = drv.gather_state()
    ids = drv.pos[: drv.n, 3].contiguous().view(__import__("torch").int64).cpu().numpy()
    f = np.empty((drv.n, 3))
    f[ids] = drv.frc[:, : drv.n].cpu().numpy().T
    pi, pj = oracle.neighbor_pairs(x, drv.box.low, drv.box.high, [True] * 3, 2.5 * 1.0000001)
    fref, peref = oracle.lj_forces(x, np.arange(drv.n), drv.n, pi, pj, drv.box.lengths,
                                   [True] * 3, 1.0, 1.0, 2.5)
    assert force_err_ratio(f, fref) < 1.0
    assert np.abs(f.sum(0)).max() < 1e-9
    d = drv.diagnostics()
    assert abs(d["PE"] - peref.sum()) <= ENERGY_TOL * abs(peref.sum())


@pytest.mark.gpu
@pytest.mark.parametrize("cells,temp", [(16, 1.44), (24, 3.0)])
def test_tile_fused_round_order_equals_order_pass(pc, cells, temp, monkeypatch):
    """The residue round-robin order applied inside the build
    (pc_tile_build_ordered, kind 1; the default for rebuild strides >= 8)
    writes the same list words as the build followed by the separate
    pc_tile_order pass: same rounds per row-warp, same slots in the same
    rounds, bit for bit."""
    import torch
    cfg = dict(lattice_cells=cells, density=0.8442, temperature=temp, cutoff=2.5, skin=0.3,
               rebuild_stride=20, seed=11, steps=0)
    lists = []
    for fused in (True, False):
        monkeypatch.setattr(pc.md, "_TILE_FUSED_ORDER", fused)
        drv = pc.md.MDDriver(pc.md.MDConfig(**cfg))
        assert drv.mode == "tile" and drv.tile_failures == 0
        torch.cuda.synchronize()
        nt = drv._ntiles
        nrw = int(drv._rw0[nt].item())
        rounds = drv._rounds[:nrw].cpu().numpy()
        words = drv._tlist.view(torch.int32)[: nrw * drv._q8 * 128].cpu().numpy()
        words = words.reshape(nrw, drv._q8, 128)
        lists.append((rounds, words, drv._rowidx[: nrw * 32].cpu().numpy()))
    (ra, wa, ia), (rb, wb, ib) = lists
    assert np.array_equal(ra, rb) and np.array_equal(ia, ib)
    for rw in range(len(ra)):
        g = (int(ra[rw]) + 7) // 8
        assert np.array_equal(wa[rw, :g], wb[rw, :g]), rw


@pytest.mark.gpu
@pytest.mark.parametrize("cells,temp", [(12, 1.44), (16, 3.0)])
def test_md_engine_virial_vs_oracle(pc, oracle, cells, temp):
    """The pair virial W = sum over pairs of r.F (tile force kernel: per-row
    FP32 sums of u = 2 sr12 - sr6, FP64 per-warp partials, one fixed
    reduction; north_star's "FP64 energy/virial reduction") against the FP64
    pair sum over the oracle's neighbour pairs on the same positions, and the
    pressure (2 KE + W) / 3V of the same diagnostics call."""
    cfg = pc.md.MDConfig(lattice_cells=cells, density=0.8442, temperature=temp, cutoff=2.5,
                         skin=0.3, rebuild_stride=20, seed=7, steps=0)
    drv = pc.md.MDDriver(cfg)
    assert drv.mode == "tile"
    for s in range(1, 8):
        drv.step(s)
    x, _ = drv.gather_state()
    d = drv.diagnostics()
    pi, pj = oracle.neighbor_pairs(x, drv.box.low, drv.box.high, [True] * 3, 2.5 * 1.0000001)
    L = drv.box.lengths
    dx = x[pj] - x[pi]
    dx -= L * np.round(dx / L)
    r2 = np.einsum("ij,ij->i", dx, dx)
    r2 = r2[r2 < 6.25]
    sr6 = (1.0 / r2) ** 3
    w_ref = 0.5 * np.sum(24.0 * (2.0 * sr6 * sr6 - sr6))      # ordered pairs: each twice
    assert abs(d["virial"] - w_ref) <= 1e-6 * abs(w_ref) + 1e-9 * len(r2)
    # P = (2 KE + W) / 3V is a difference of large terms in a hot liquid: its
    # tolerance is the virial's, carried through
    p_ref = (2.0 * d["KE"] + w_ref) / (3.0 * np.prod(L))
    assert abs(d["pressure"] - p_ref) <= (1e-6 * abs(w_ref) + 1e-9 * len(r2)) / (3.0 * np.prod(L))


def test_md_engine_empty_tiles(pc, oracle):
    """A lattice at the usual density filling half the box volume (a corner
    cube; the rest vacuum): whole tiles have no rows (28^3 cells: ~5 tiles per
    CTA, many empty).  The staging ring must pass over them (they are never
    waited on) and the forces must match the oracle's on the tile path."""
    import torch
    cells = 28
    a = (4.0 / 0.8442) ** (1.0 / 3.0)
    x = pc.md.fcc_lattice(cells, a)
    v = pc.md.initial_velocities(x.shape[0], 1.44, 1.0, 3)
    cfg = pc.md.MDConfig(lattice_cells=cells, density=0.4221, temperature=1.44, cutoff=2.5,
                         skin=0.3, rebuild_stride=10, seed=3, steps=0)
    drv = pc.md.MDDriver(cfg, state=(x, v))
    assert drv.mode == "tile"
    assert x.max() + 2.8 < drv.box.high[0]          # vacuum wider than the search radius
    for s in range(1, 16):
        drv.step(s)
    xs, _ = drv.gather_state()
    ids = drv.pos[: drv.n, 3].contiguous().view(torch.int64).cpu().numpy()
    f = np.empty((drv.n, 3))
    f[ids] = drv.frc[:, : drv.n].cpu().numpy().T
    pi, pj = oracle.neighbor_pairs(xs, drv.box.low, drv.box.high, [True] * 3, 2.5 * 1.0000001)
    fref, _ = oracle.lj_forces(xs, np.arange(drv.n), drv.n, pi, pj, drv.box.lengths,
                               [True] * 3, 1.0, 1.0, 2.5)
    assert force_err_ratio(f, fref) < 1.0
    assert drv.tile_failures == 0


def test_md_engine_non_unit_sigma_epsilon(pc, oracle):
    """sigma != 1 takes the tile force kernel's general-sigma instantiation;
    epsilon scales forces and energies (ref md.py:89-96) -- vs the oracle's
    FP64 lj_forces on the same positions."""
    import torch
    cfg = pc.md.MDConfig(lattice_cells=12, density=0.7, temperature=1.2, cutoff=2.6, skin=0.3,
                         rebuild_stride=10, seed=4, steps=0, sigma=1.05, epsilon=0.8)
    drv = pc.md.MDDriver(cfg)
    assert drv.mode == "tile"
    for s in range(1, 13):
        drv.step(s)
    x, _ = drv.gather_state()
    ids = drv.pos[: drv.n, 3].contiguous().view(torch.int64).cpu().numpy()
    f = np.empty((drv.n, 3))
    f[ids] = drv.frc[:, : drv.n].cpu().numpy().T
    pi, pj = oracle.neighbor_pairs(x, drv.box.low, drv.box.high, [True] * 3, 2.6 * 1.0000001)
    fref, peref = oracle.lj_forces(x, np.arange(drv.n), drv.n, pi, pj, drv.box.lengths,
                                   [True] * 3, 0.8, 1.05, 2.6)
    assert force_err_ratio(f, fref) < 1.0
    d = drv.diagnostics()
    assert abs(d["PE"] - peref.sum()) <= ENERGY_TOL * abs(peref.sum())


def test_md_engine_tile_overflow_falls_back(pc, oracle):
    """Dense system (rho = 1.4, ~3000-slot tile neighbourhoods > the 2304-slot
    staging capacity): the speculatively launched tile force is discarded, the
    velocities restored and the step redone on the SELL path -- forces still
    match the oracle."""
    import torch
    cfg = pc.md.MDConfig(lattice_cells=12, density=1.4, temperature=1.0, cutoff=2.5, skin=0.3,
                         rebuild_stride=10, seed=6, steps=0)
    drv = pc.md.MDDriver(cfg)
    assert drv.tile_failures >= 1 and drv.mode == "sell"
    e0 = drv.diagnostics()["E_total"]
    for s in range(1, 21):
        drv.step(s)
    x, _ = drv.gather_state()
    ids = drv.pos[: drv.n, 3].contiguous().view(torch.int64).cpu().numpy()
    f = np.empty((drv.n, 3))
    f[ids] = drv.frc[:, : drv.n].cpu().numpy().T
    pi, pj = oracle.neighbor_pairs(x, drv.box.low, drv.box.high, [True] * 3, 2.5 * 1.0000001)
    fref, _ = oracle.lj_forces(x, np.arange(drv.n), drv.n, pi, pj, drv.box.lengths,
                               [True] * 3, 1.0, 1.0, 2.5)
    assert force_err_ratio(f, fref) < 1.0
    assert abs(drv.diagnostics()["E_total"] - e0) < 1e-2 * abs(e0)


def test_md_engine_overlap_raises(pc):
    """Two coincident particles (r = 0) on the tile path: the exact per-pair
    r^2 < (1e-10 sigma)^2 test flags it (ref md.py:117-119 FloatingPointError);
    a finiteness check of the FP32 force would miss it (r^2 = 0 narrows to a
    finite value)."""
    cells = 12
    a = (4.0 / 0.8442) ** (1.0 / 3.0)
    x = pc.md.fcc_lattice(cells, a)
    x[1] = x[0]
    v = pc.md.initial_velocities(x.shape[0], 1.0, 1.0, 1)
    cfg = pc.md.MDConfig(lattice_cells=cells, density=0.8442, temperature=1.0, cutoff=2.5,
                         skin=0.3, rebuild_stride=10, seed=1, steps=0)
    drv = pc.md.MDDriver(cfg, state=(x, v))
    assert drv.mode == "tile"
    with pytest.raises(FloatingPointError):
        drv.check_errors()


_ORDER_HASH = r"""
import hashlib, sys, numpy as np, torch
import paper_2109_09056_b200 as pc
cfg = pc.md.MDConfig(lattice_cells=int(sys.argv[1]), density=0.8442, temperature=float(sys.argv[2]),
                     cutoff=2.5, skin=0.3, rebuild_stride=20, seed=13, steps=0)
drv = pc.md.MDDriver(cfg)
assert drv.mode == "tile"
torch.cuda.synchronize()
nt = drv._ntiles
nrw = int(drv._rw0[nt].item())
rounds = drv._rounds[:nrw].cpu().numpy()
words = drv._tlist.view(torch.int32)[: nrw * drv._q8 * 128].cpu().numpy().reshape(nrw, drv._q8, 128)
h = hashlib.sha256(rounds.tobytes())
for rw in range(nrw):
    h.update(words[rw, : (int(rounds[rw]) + 7) // 8].tobytes())
print(h.hexdigest())
"""


@pytest.mark.gpu
@pytest.mark.parametrize("cells,temp", [(16, 1.44), (24, 3.0)])
def test_tile_order_rewrite_same_rounds(cells, temp):
    """The r02 round-robin order kernel (tile_order_rr_kernel, default) emits
    the same list words as the r01 kernel (PC_TILE_ORDER_IMPL=1): one hash
    over every row-warp's rounds from two processes."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = []
    for impl in ("1", "2"):
        env = dict(os.environ, PC_TILE_ORDER_IMPL=impl, PC_TILE_FUSED="0", PYTHONPATH=root)
        r = subprocess.run([sys.executable, "-c", _ORDER_HASH, str(cells), str(temp)], env=env,
                           capture_output=True, text=True, timeout=300, cwd=root)
        assert r.returncode == 0, r.stderr[-2000:]
        out.append(r.stdout.strip().splitlines()[-1])
    assert out[0] == out[1]
