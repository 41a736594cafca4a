"""GPU parity of the decomposition API (migrate / build_halo / halo_gather /
halo_scatter) against the reference's own outputs (tests/golden/decomp.npz)
and the behaviours ref tests/test_decomp.py checks."""

import numpy as np
import pytest

from conftest import load_cases

pytestmark = pytest.mark.gpu

DC = load_cases("decomp.npz")


@pytest.fixture(scope="module")
def pc():
    import torch
    assert torch.cuda.is_available()
    import paper_2109_09056_b200 as pkg
    return pkg


def _sets(pc, fabric, x, V=4, f=None):
    sch = pc.aosoa.schema(x=("float64", (3,)), f=("float64", (3,)), id=("int64", ()))
    sets = [pc.aosoa.create(sch, V, 0) for _ in range(fabric.n_ranks)]
    sets[0].resize(x.shape[0])
    sets[0].slice("x").copy_in(x)
    if f is not None:
        sets[0].slice("f").copy_in(f)
    sets[0].slice("id").copy_in(np.arange(x.shape[0], dtype=np.int64))
    return sets


@pytest.mark.parametrize("case", sorted(DC))
def test_decomp_bit_exact(pc, case):
    c = DC[case]
    L = float(c["L"])
    dims = tuple(int(v) for v in c["dims"])
    fabric = pc.decomp.decompose(pc.geometry.cube(L), dims, [True] * 3)
    sets = _sets(pc, fabric, c["x"])
    pc.decomp.migrate(fabric, sets)
    for r, p in enumerate(sets):
        assert p.ghosts == 0
        assert np.array_equal(p.slice("id").copy_out(), c[f"mig_ids_{r}"])
        assert np.array_equal(p.slice("x").copy_out(), c[f"mig_x_{r}"])
    plan = pc.decomp.build_halo(fabric, sets, float(c["width"]))
    for r in range(fabric.n_ranks):
        assert np.array_equal(plan.export_index[r], c[f"exp_index_{r}"])
        assert np.array_equal(plan.export_dest[r], c[f"exp_dest_{r}"])
        assert np.array_equal(plan.export_shift[r], c[f"exp_shift_{r}"])
        lay = np.array(plan.import_layout[r], np.int64).reshape(-1, 2)
        assert np.array_equal(lay, c[f"imp_layout_{r}"])
    pc.decomp.halo_gather(plan, sets)
    for r, p in enumerate(sets):
        assert p.ghosts == int(c[f"gat_ghosts_{r}"])
        assert np.array_equal(p.slice("x").copy_out(), c[f"gat_x_{r}"])
        assert np.array_equal(p.slice("id").copy_out(), c[f"gat_id_{r}"])
        p.slice("f").copy_in(np.full((p.size, 3), 1.0) + np.arange(p.size)[:, None] * 1e-3)
    pc.decomp.halo_scatter(plan, sets, ["f"])
    for r, p in enumerate(sets):
        assert np.array_equal(p.slice("f").copy_out(), c[f"sca_f_{r}"])


def test_fabric_and_owner(pc):
    f = pc.decomp.decompose(pc.geometry.cube(2.0), (2, 1, 1), [True] * 3)
    owners = f.owner_of(np.array([[0.5, 0.1, 0.1], [1.5, 0.1, 0.1],
                                  [1.0, 0.0, 0.0], [2.0, 0.3, 0.3]]))
    assert owners.tolist() == [0, 1, 1, 1]
    with pytest.raises(ValueError):
        f.owner_of(np.array([[2.5, 0.1, 0.1]]))
    with pytest.raises(ValueError):
        pc.decomp.decompose(pc.geometry.cube(1.0), (0, 1, 1), [True] * 3)


def test_migrate_wraps_and_conserves(pc):
    rng = np.random.default_rng(11)
    fabric = pc.decomp.decompose(pc.geometry.cube(4.0), (2, 2, 2), [True] * 3)
    x = rng.random((500, 3)) * 4.0
    sets = _sets(pc, fabric, x)
    pc.decomp.migrate(fabric, sets)
    total = 0
    for r, p in enumerate(sets):
        xr = p.slice("x").copy_out()
        assert np.all(fabric.owner_of(xr) == r)
        assert np.array_equal(x[p.slice("id").copy_out()], xr)
        total += p.size
    assert total == 500
    fab2 = pc.decomp.decompose(pc.geometry.cube(2.0), (2, 1, 1), [True] * 3)
    s2 = _sets(pc, fab2, np.array([[2.3, 0.5, 0.5]]))
    pc.decomp.migrate(fab2, s2)
    assert s2[0].size == 1 and s2[1].size == 0
    assert np.allclose(s2[0].slice("x").copy_out(), [[0.3, 0.5, 0.5]])


def test_nonperiodic_stray_rejected(pc):
    box = pc.geometry.Box([0.0] * 3, [2.0] * 3)
    fabric = pc.decomp.decompose(box, (2, 1, 1), [False, True, True])
    sets = _sets(pc, fabric, np.array([[2.5, 0.5, 0.5]]))
    with pytest.raises(ValueError):
        pc.decomp.migrate(fabric, sets)


def test_stale_plan_and_width(pc):
    fabric = pc.decomp.decompose(pc.geometry.cube(4.0), (2, 1, 1), [True] * 3)
    sets = _sets(pc, fabric, np.array([[0.5, 0.5, 0.5], [2.5, 0.5, 0.5]]))
    pc.decomp.migrate(fabric, sets)
    plan = pc.decomp.build_halo(fabric, sets, width=0.5)
    sets[0].resize(sets[0].size + 1)
    with pytest.raises(RuntimeError):
        pc.decomp.halo_gather(plan, sets)
    fab8 = pc.decomp.decompose(pc.geometry.cube(4.0), (2, 2, 2), [True] * 3)
    with pytest.raises(ValueError):
        pc.decomp.build_halo(fab8, _sets(pc, fab8, np.zeros((0, 3))), width=2.5)


def test_scatter_accumulates_back_to_owner(pc):
    fabric = pc.decomp.decompose(pc.geometry.cube(4.0), (2, 1, 1), [True] * 3)
    x = np.array([[1.9, 1.0, 1.0], [2.1, 1.0, 1.0], [1.0, 3.0, 3.0]])
    sets = _sets(pc, fabric, x)
    pc.decomp.migrate(fabric, sets)
    plan = pc.decomp.build_halo(fabric, sets, width=0.5)
    pc.decomp.halo_gather(plan, sets)
    for p in sets:
        p.slice("f").copy_in(np.ones((p.size, 3)))
    pc.decomp.halo_scatter(plan, sets, ["f"])
    got = {}
    for p in sets:
        ids = p.slice("id").copy_out()[: p.owned]
        f = p.slice("f").copy_out()[: p.owned]
        for i, row in zip(ids, f):
            got[int(i)] = row[0]
    assert got[0] == 2.0 and got[1] == 2.0 and got[2] == 1.0
