"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

The reference is imported read-only under the alias ``particula_ref`` (it uses
only relative imports) and executed unchanged; its outputs are frozen into
``tests/golden/*.npz`` so that the oracle (``oracle/particula_oracle.py``) and
the CUDA path can be checked on a GPU box that has no /root/reference.
"""

from __future__ import annotations

import hashlib
import importlib.util
import json
import os
import sys

import numpy as np

REF_PKG = "/root/reference/pkg/src/particula"
OUT = os.path.dirname(os.path.abspath(__file__))


def load_reference():
    spec = importlib.util.spec_from_file_location(
        "particula_ref", os.path.join(REF_PKG, "__init__.py"),
        submodule_search_locations=[REF_PKG])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["particula_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def neighbor_cases(ref):
    from particula_ref import neighbors
    from particula_ref.geometry import Box, cube
    cases = {}

    def add(name, x, box, per, cutoff, ratio=1.0):
        rec = {"x": x, "low": box.low, "high": box.high,
               "periodic": np.asarray(per, bool),
               "cutoff": np.float64(cutoff), "ratio": np.float64(ratio)}
        for layout in ("compressed", "dense"):
            for conv in ("full", "half"):
                vl = neighbors.build_verlet(x, box, per, cutoff, layout=layout,
                                            half_or_full=conv, cell_ratio=ratio)
                key = f"{layout}_{conv}"
                rec[f"{key}_counts"] = vl.counts
                if layout == "compressed":
                    rec[f"{key}_indices"] = vl.indices
                    rec[f"{key}_offsets"] = vl.offsets
                else:
                    rec[f"{key}_table"] = vl.table
        cases[name] = rec

    rng = np.random.default_rng(42)          # ref tests/test_neighbors.py:21-33
    add("rand300", rng.random((300, 3)) * 4.0, cube(4.0), [True] * 3, 0.8)
    rng = np.random.default_rng(7)
    add("rand100_nc3", rng.random((100, 3)) * 3.0, cube(3.0), [True] * 3, 0.9)
    rng = np.random.default_rng(11)          # nc = 2 on every axis: stencil aliasing
    add("rand120_nc2", rng.random((120, 3)) * 3.0, cube(3.0), [True] * 3, 1.2)
    rng = np.random.default_rng(12)          # nc = 1 through cell_ratio
    add("rand80_nc1", rng.random((80, 3)) * 2.0, cube(2.0), [True] * 3, 0.9, 2.5)
    rng = np.random.default_rng(13)          # mixed periodicity, offset box
    box = Box([-1.0, 0.5, 2.0], [3.0, 4.0, 5.5])
    x = box.low + rng.random((400, 3)) * box.lengths
    add("mixed400", x, box, [True, False, True], 0.7, 1.3)
    add("pair_nonper", np.array([[0.05, 1.0, 1.0], [1.95, 1.0, 1.0]]),
        Box([0.0] * 3, [2.0] * 3), [False, True, True], 0.5)
    add("pair_strict", np.array([[1.0, 1.0, 1.0], [2.0, 1.0, 1.0]]), cube(10.0),
        [True] * 3, 1.0)
    n = 1000                                  # ref tests/test_acceptance.py:22-50
    rc = (30 * 3 / (4 * np.pi * n)) ** (1 / 3)
    for seed in range(3):
        add(f"crit1_seed{seed}", np.random.default_rng(seed).random((n, 3)),
            cube(1.0), [True] * 3, rc)
    # integer-ratio box (L/rc = 5): cell width equals the cutoff exactly
    rng = np.random.default_rng(21)
    add("lattice_exact", np.round(rng.random((500, 3)) * 40) / 10.0, cube(4.0),
        [True] * 3, 0.8)
    return cases


def binning_cases(ref):
    from particula_ref import binning
    from particula_ref.geometry import Box
    cases = {}
    rng = np.random.default_rng(5)
    for d, n, cs in ((1, 50, 0.3), (2, 120, 0.25), (3, 400, 0.5), (3, 1000, 0.37)):
        box = Box(np.zeros(d), np.full(d, 2.0))
        x = rng.random((n, d)) * 2.0
        x[0] = 2.0                                 # upper face clamps down
        x[1] = 0.0
        cb = binning.bin_by_position(x, box, cs)
        nc, idx = binning.cell_indices(x, box, cs)
        cases[f"d{d}_n{n}"] = {"x": x, "low": box.low, "high": box.high,
                               "cs": np.float64(cs), "nc": nc, "idx": idx,
                               "offsets": cb.offsets, "map": cb.permutation.map}
    keys = rng.integers(0, 7, 300)
    cases["keys300"] = {"keys": keys, "map": binning.bin_by_key(keys).map}
    return cases


def lj_case(ref, cells, steps, name):
    from particula_ref import md
    cfg = md.MDConfig(lattice_cells=cells, density=0.8442, temperature=1.44,
                      dt=0.005, cutoff=2.5, skin=0.3, rebuild_stride=20, seed=1,
                      steps=0)
    drv = md.MDDriver(cfg)
    for s in range(1, steps + 1):
        drv.step(s)
    p = drv.sets[0]
    x0 = p.slice("x0").copy_out()
    ids = p.slice("id").copy_out()
    search = (cfg.cutoff + cfg.skin) * md._CUTOFF_MARGIN
    vl = ref.neighbors.build_verlet(x0, drv.box, drv.periodic, search)
    f, pe = md.lj_forces(x0, ids, p.owned, vl, drv.box, drv.periodic, 1.0, 1.0, 2.5)
    return {f"{name}_x0": x0, f"{name}_ids": ids, f"{name}_L": drv.box.lengths,
            f"{name}_search": np.float64(search),
            f"{name}_counts": vl.counts,
            f"{name}_csr_digest": np.array(digest(vl.offsets, vl.indices)),
            f"{name}_f": f, f"{name}_pe": pe}


def md_series(ref):
    from particula_ref import md
    out = {}
    configs = {
        # ref tests/test_acceptance.py:79-92 (criterion 3 configuration)
        "crit3": dict(lattice_cells=4, density=1.1, cutoff=2.3, seed=2, steps=200),
        # skin + deferred rebuild + sort (ref tests/test_md.py:94-105)
        "skin_sort": dict(lattice_cells=3, density=1.1, temperature=0.8,
                          cutoff=2.0, seed=2, steps=40, skin=0.2,
                          rebuild_stride=5, sort_stride=10),
        # BASELINE configs[0]: fcc 16^3, T=1.44, rc 2.5, skin 0.3, rebuild 20
        "c1": dict(lattice_cells=16, density=0.8442, temperature=1.44,
                   cutoff=2.5, skin=0.3, rebuild_stride=20, seed=1, steps=100),
        # hot liquid regime (BASELINE configs[3]) at 6^3
        "hot": dict(lattice_cells=6, density=0.8442, temperature=3.0,
                    cutoff=2.5, skin=0.3, rebuild_stride=5, sort_stride=5,
                    seed=1, steps=40),
    }
    for name, kw in configs.items():
        rows, _ = md.run_md(md.MDConfig(**kw))
        out[f"{name}_series"] = np.array([[r["KE"], r["PE"], r["E_total"],
                                           r["temperature"]] for r in rows])
        out[f"{name}_config"] = np.array(json.dumps(kw))
    # state after 50 steps for trajectory comparisons (crit3 config)
    drv = md.MDDriver(md.MDConfig(lattice_cells=4, density=1.1, cutoff=2.3,
                                  seed=2, steps=0))
    x0, v0 = drv.gather_state()
    out["crit3_x_init"], out["crit3_v_init"] = x0, v0
    for s in range(1, 51):
        drv.step(s)
    out["crit3_x50"], out["crit3_v50"] = drv.gather_state()
    # distributed fabric == serial (ref tests/test_md.py:77-83)
    rows, _ = md.run_md(md.MDConfig(lattice_cells=4, density=1.1, cutoff=2.3,
                                    seed=2, steps=20, rank_dims=(2, 2, 2)))
    out["crit3_222_series"] = np.array([[r["KE"], r["PE"], r["E_total"],
                                         r["temperature"]] for r in rows])
    return out


def decomp_cases(ref):
    from particula_ref import aosoa, decomp
    from particula_ref.geometry import cube
    schema = aosoa.schema(x=("float64", (3,)), f=("float64", (3,)),
                          id=("int64", ()))
    cases = {}
    for name, L, dims, n, width, seed in (("d222", 6.0, (2, 2, 2), 300, 1.2, 3),
                                          ("d221", 6.0, (2, 2, 1), 400, 1.0, 2),
                                          ("d211", 4.0, (2, 1, 1), 200, 0.9, 4),
                                          ("d311", 9.0, (3, 1, 1), 300, 1.1, 6)):
        fabric = decomp.decompose(cube(L), dims, [True] * 3)
        rng = np.random.default_rng(seed)
        x = rng.random((n, 3)) * L
        x[:5] += L * np.array([1.0, -1.0, 0.0])        # periodic strays
        sets = [aosoa.create(schema, 4, 0) for _ in range(fabric.n_ranks)]
        sets[0].resize(n)
        sets[0].slice("x").copy_in(x)
        sets[0].slice("f").copy_in(rng.random((n, 3)))
        sets[0].slice("id").copy_in(np.arange(n, dtype=np.int64))
        decomp.migrate(fabric, sets)
        rec = {"L": np.float64(L), "dims": np.array(dims), "x": x,
               "width": np.float64(width)}
        rec["f_init"] = None
        for r, p in enumerate(sets):
            rec[f"mig_ids_{r}"] = p.slice("id").copy_out()
            rec[f"mig_x_{r}"] = p.slice("x").copy_out()
        plan = decomp.build_halo(fabric, sets, width)
        for r in range(fabric.n_ranks):
            rec[f"exp_index_{r}"] = plan.export_index[r]
            rec[f"exp_dest_{r}"] = plan.export_dest[r]
            rec[f"exp_shift_{r}"] = plan.export_shift[r]
            rec[f"imp_layout_{r}"] = np.array(plan.import_layout[r],
                                              np.int64).reshape(-1, 2)
        decomp.halo_gather(plan, sets)
        for r, p in enumerate(sets):
            rec[f"gat_x_{r}"] = p.slice("x").copy_out()
            rec[f"gat_id_{r}"] = p.slice("id").copy_out()
            rec[f"gat_ghosts_{r}"] = np.int64(p.ghosts)
            p.slice("f").copy_in(np.full((p.size, 3), 1.0) +
                                 np.arange(p.size)[:, None] * 1e-3)
        decomp.halo_scatter(plan, sets, ["f"])
        for r, p in enumerate(sets):
            rec[f"sca_f_{r}"] = p.slice("f").copy_out()
        del rec["f_init"]
        cases[name] = rec
    return cases


def save(name, cases):
    flat = {}
    for case, rec in cases.items():
        for k, v in rec.items():
            flat[f"{case}__{k}"] = np.asarray(v)
    np.savez_compressed(os.path.join(OUT, name), **flat)
    print("wrote", name, len(flat), "arrays")


def main():
    ref = load_reference()
    import particula_ref.neighbors  # noqa: F401
    save("neighbors.npz", neighbor_cases(ref))
    save("binning.npz", binning_cases(ref))
    save("decomp.npz", decomp_cases(ref))
    lj = {}
    lj.update(lj_case(ref, 8, 40, "c8"))
    lj.update(lj_case(ref, 16, 40, "c16"))
    np.savez_compressed(os.path.join(OUT, "lj.npz"), **lj)
    print("wrote lj.npz")
    np.savez_compressed(os.path.join(OUT, "md.npz"), **md_series(ref))
    print("wrote md.npz")


if __name__ == "__main__":
    main()
