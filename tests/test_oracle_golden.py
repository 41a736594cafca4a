"""Pin the CPU oracle against golden vectors produced by the reference itself.

These run without a GPU.  If any of them fails, every GPU parity claim that
uses the oracle is void.
"""

import hashlib
import json

import numpy as np
import pytest

from conftest import load_cases, load_flat


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def test_numpy_einsum_order(oracle):
    # the CUDA predicate hard-codes (x^2 + z^2) + y^2 without FMA
    assert oracle.einsum_order_ok()


NB = load_cases("neighbors.npz")


@pytest.mark.parametrize("case", sorted(NB))
def test_neighbor_lists_bit_exact(oracle, case):
    c = NB[case]
    for layout in ("compressed", "dense"):
        for conv in ("full", "half"):
            got = oracle.build_verlet(c["x"], c["low"], c["high"], c["periodic"],
                                      float(c["cutoff"]), layout=layout,
                                      half_or_full=conv,
                                      cell_ratio=float(c["ratio"]))
            key = f"{layout}_{conv}"
            assert np.array_equal(got["counts"], c[f"{key}_counts"])
            if layout == "compressed":
                assert np.array_equal(got["indices"], c[f"{key}_indices"])
                assert np.array_equal(got["offsets"], c[f"{key}_offsets"])
            else:
                assert np.array_equal(got["table"], c[f"{key}_table"])


@pytest.mark.parametrize("case", sorted(NB))
def test_neighbor_cell_loop_matches_golden(oracle, case):
    # the per-cell-loop restatement timed by bench.py --impl reference gives
    # the reference's own full sets (golden CSR) bit for bit
    c = NB[case]
    pi, pj = oracle.neighbor_pairs_cell_loop(c["x"], c["low"], c["high"], c["periodic"],
                                             float(c["cutoff"]), float(c["ratio"]))
    assert np.array_equal(np.bincount(pi, minlength=len(c["x"])), c["compressed_full_counts"])
    assert np.array_equal(pj, c["compressed_full_indices"])


def test_md_cell_loop_series_bit_exact(oracle):
    kw = json.loads(str(MD["crit3_config"]))
    kw["steps"] = 20
    drv = oracle.MDOracle(oracle.MDConfig(**kw), cell_loop=True)
    ref = oracle.MDOracle(oracle.MDConfig(**kw))
    for s in range(1, 21):
        drv.step(s)
        ref.step(s)
    xa, va = drv.gather_state()
    xb, vb = ref.gather_state()
    assert np.array_equal(xa, xb) and np.array_equal(va, vb)


def test_neighbor_brute_force_agrees(oracle):
    c = NB["rand300"]
    L = c["high"] - c["low"]
    ref = oracle.brute_force_sets(c["x"], L, c["periodic"], float(c["cutoff"]))
    got = oracle.build_verlet(c["x"], c["low"], c["high"], c["periodic"],
                              float(c["cutoff"]))
    rows = oracle.rows_from_csr(got["counts"], got["indices"])
    for a, b in zip(ref, rows):
        assert np.array_equal(a, np.sort(b))


def test_verlet_argument_errors(oracle):
    low, high = np.zeros(3), np.full(3, 2.0)
    x = np.zeros((1, 3))
    for kw in (dict(cutoff=-1.0), dict(cutoff=1.5), dict(cutoff=0.5, layout="sparse"),
               dict(cutoff=0.5, cell_ratio=0.5), dict(cutoff=0.5, half_or_full="x")):
        cutoff = kw.pop("cutoff")
        with pytest.raises(ValueError):
            oracle.build_verlet(x, low, high, [True] * 3, cutoff, **kw)


BN = load_cases("binning.npz")


@pytest.mark.parametrize("case", [k for k in sorted(BN) if k.startswith("d")])
def test_binning_bit_exact(oracle, case):
    c = BN[case]
    nc, idx = oracle.cell_indices(c["x"], c["low"], c["high"], float(c["cs"]))
    assert np.array_equal(nc, c["nc"]) and np.array_equal(idx, c["idx"])
    nc2, offsets, pmap = oracle.bin_by_position(c["x"], c["low"], c["high"],
                                                float(c["cs"]))
    assert np.array_equal(offsets, c["offsets"])
    assert np.array_equal(pmap, c["map"])


def test_bin_by_key(oracle):
    c = BN["keys300"]
    assert np.array_equal(oracle.stable_key_permutation(c["keys"]), c["map"])
    assert oracle.is_bijection(c["map"], 300)
    assert not oracle.is_bijection(np.array([0, 0, 1]), 3)


LJ = load_flat("lj.npz")


@pytest.mark.parametrize("name", ["c8", "c16"])
def test_lj_forces_bit_exact(oracle, name):
    x0, ids, L = LJ[f"{name}_x0"], LJ[f"{name}_ids"], LJ[f"{name}_L"]
    search = float(LJ[f"{name}_search"])
    per = np.array([True] * 3)
    vl = oracle.build_verlet(x0, np.zeros(3), L, per, search)
    assert np.array_equal(vl["counts"], LJ[f"{name}_counts"])
    assert _digest(vl["offsets"], vl["indices"]) == str(LJ[f"{name}_csr_digest"])
    pi = np.repeat(np.arange(x0.shape[0]), vl["counts"])
    f, pe = oracle.lj_forces(x0, ids, x0.shape[0], pi, vl["indices"], L, per,
                             1.0, 1.0, 2.5)
    assert np.array_equal(f, LJ[f"{name}_f"])
    assert np.array_equal(pe, LJ[f"{name}_pe"])


def test_lj_pair_reference_points(oracle):
    # ref tests/test_md.py:33-42
    e, _ = oracle.lj_pair(np.array([[1.0, 0, 0]]), np.array([1.0]), 1.0, 1.0)
    assert abs(e[0]) < 1e-14
    rm = 2.0 ** (1 / 6)
    e, f = oracle.lj_pair(np.array([[rm, 0, 0]]), np.array([rm * rm]), 1.0, 1.0)
    assert abs(e[0] + 1.0) < 1e-14 and np.max(np.abs(f)) < 1e-12


DC = load_cases("decomp.npz")


@pytest.mark.parametrize("case", sorted(DC))
def test_decomp_bit_exact(oracle, case):
    c = DC[case]
    L = float(c["L"])
    dims = tuple(int(d) for d in c["dims"])
    fab = oracle.Fabric(np.zeros(3), np.full(3, L), dims, [True] * 3)
    n = c["x"].shape[0]
    rng_f = None  # f payload is checked through ids (random in the fixture)
    ranks = [oracle.RankStore({"x": np.zeros((0, 3)), "f": np.zeros((0, 3)),
                               "id": np.zeros(0, np.int64)})
             for _ in range(fab.n_ranks)]
    ranks[0] = oracle.RankStore({"x": c["x"], "f": np.zeros((n, 3)),
                                 "id": np.arange(n, dtype=np.int64)})
    oracle.migrate(fab, ranks)
    for r, st in enumerate(ranks):
        assert np.array_equal(st.f["id"], c[f"mig_ids_{r}"])
        assert np.array_equal(st.f["x"], c[f"mig_x_{r}"])
    plan = oracle.build_halo(fab, ranks, float(c["width"]))
    for r in range(fab.n_ranks):
        assert np.array_equal(plan["export_index"][r], c[f"exp_index_{r}"])
        assert np.array_equal(plan["export_dest"][r], c[f"exp_dest_{r}"])
        assert np.array_equal(plan["export_shift"][r], c[f"exp_shift_{r}"])
        lay = np.array(plan["import_layout"][r], np.int64).reshape(-1, 2)
        assert np.array_equal(lay, c[f"imp_layout_{r}"])
    oracle.halo_gather(plan, ranks)
    for r, st in enumerate(ranks):
        assert np.array_equal(st.f["x"], c[f"gat_x_{r}"])
        assert np.array_equal(st.f["id"], c[f"gat_id_{r}"])
        assert st.ghosts == int(c[f"gat_ghosts_{r}"])
        st.f["f"] = np.full((st.size, 3), 1.0) + np.arange(st.size)[:, None] * 1e-3
    oracle.halo_scatter(plan, ranks, ["f"])
    for r, st in enumerate(ranks):
        assert np.array_equal(st.f["f"], c[f"sca_f_{r}"])


MD = load_flat("md.npz")


@pytest.mark.parametrize("name", ["crit3", "skin_sort", "hot"])
def test_md_energy_series_bit_exact(oracle, name):
    kw = json.loads(str(MD[f"{name}_config"]))
    rows, _ = oracle.run_md(oracle.MDConfig(**kw))
    got = np.array([[r["KE"], r["PE"], r["E_total"], r["temperature"]]
                    for r in rows])
    assert np.array_equal(got, MD[f"{name}_series"])


def test_md_distributed_fabric_bit_exact(oracle):
    rows, _ = oracle.run_md(oracle.MDConfig(lattice_cells=4, density=1.1,
                                            cutoff=2.3, seed=2, steps=20,
                                            rank_dims=(2, 2, 2)))
    got = np.array([[r["KE"], r["PE"], r["E_total"], r["temperature"]]
                    for r in rows])
    assert np.array_equal(got, MD["crit3_222_series"])
    assert np.array_equal(got, MD["crit3_series"][:21])


def test_md_trajectory_bit_exact(oracle):
    drv = oracle.MDOracle(oracle.MDConfig(lattice_cells=4, density=1.1,
                                          cutoff=2.3, seed=2, steps=0))
    x, v = drv.gather_state()
    assert np.array_equal(x, MD["crit3_x_init"]) and np.array_equal(v, MD["crit3_v_init"])
    for s in range(1, 51):
        drv.step(s)
    x, v = drv.gather_state()
    assert np.array_equal(x, MD["crit3_x50"]) and np.array_equal(v, MD["crit3_v50"])


@pytest.mark.slow
def test_md_c1_series_bit_exact(oracle):
    kw = json.loads(str(MD["c1_config"]))
    kw["steps"] = 20
    rows, _ = oracle.run_md(oracle.MDConfig(**kw))
    got = np.array([[r["KE"], r["PE"], r["E_total"], r["temperature"]]
                    for r in rows])
    assert np.array_equal(got, MD["c1_series"][:21])


EW = load_flat("ewald.npz")


@pytest.mark.parametrize("name", ["rand400", "nacl216"])
def test_ewald_real_space_bit_exact(oracle, name):
    """Oracle real-space pass == the reference's _real_space (longrange.py:47-72),
    on the reference's half-list pairs and on all pairs."""
    g = lambda k: EW[f"{name}_{k}"]  # noqa: E731
    e, f = oracle.ewald_real_space(g("x"), g("q"), float(g("L")), float(g("alpha")),
                                   float(g("rcut")), g("pi"), g("pj"))
    assert e == float(g("energy"))
    assert np.array_equal(f, g("forces"))
    e2, f2 = oracle.ewald_real_space(g("x"), g("q"), float(g("L")), float(g("alpha")),
                                     float(g("rcut")))
    assert e2 == float(g("energy_all"))
    assert np.array_equal(f2, g("forces_all"))
    # the half list covers every pair within r_cut: same physics either way
    assert abs(e - e2) <= 1e-12 * abs(e2)
