"""Golden vectors for the Ewald real-space pass (ref longrange.py:47-72),
produced by running the REFERENCE itself (build container only):

    python tests/golden/make_ewald_golden.py

Cases: random neutral charges in a periodic cube with the reference's own
half list (neighbors.build_verlet(..., half_or_full="half"), as
longrange.spme does, longrange.py:142-146), and an ionic lattice with
jitter; alpha from the reference's default_alpha.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import OUT, load_reference  # noqa: E402


def main():
    load_reference()
    from particula_ref import longrange, neighbors
    from particula_ref.geometry import cube
    out = {}

    def add(name, x, q, L, r_cut):
        alpha = longrange.default_alpha(r_cut)
        vl = neighbors.build_verlet(x, cube(L), [True] * 3, r_cut, half_or_full="half")
        ii, jj = vl.pairs()
        e, f = longrange._real_space(x, q, L, alpha, r_cut, pairs=(ii, jj))
        e_all, f_all = longrange._real_space(x, q, L, alpha, r_cut)       # all pairs
        out.update({f"{name}_x": x, f"{name}_q": q, f"{name}_L": np.float64(L),
                    f"{name}_alpha": np.float64(alpha), f"{name}_rcut": np.float64(r_cut),
                    f"{name}_pi": ii.astype(np.int64), f"{name}_pj": jj.astype(np.int64),
                    f"{name}_energy": np.float64(e), f"{name}_forces": f,
                    f"{name}_energy_all": np.float64(e_all), f"{name}_forces_all": f_all})

    rng = np.random.default_rng(21)
    n = 400
    L = 9.0
    x = rng.random((n, 3)) * L
    q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    rng.shuffle(q)
    add("rand400", x, q, L, 3.5)
    # rock-salt lattice 6^3 sites, spacing 1.2, jittered
    m = 6
    g = np.stack(np.meshgrid(*[np.arange(m)] * 3, indexing="ij"), -1).reshape(-1, 3)
    x = (g + 0.15 * rng.standard_normal(g.shape)) * 1.2 % (m * 1.2)
    q = np.where(g.sum(1) % 2 == 0, 1.0, -1.0)
    add("nacl216", x, q, m * 1.2, 3.0)
    np.savez_compressed(os.path.join(OUT, "ewald.npz"), **out)
    print("wrote ewald.npz", {k: v.shape for k, v in out.items() if hasattr(v, "shape")})


if __name__ == "__main__":
    main()
