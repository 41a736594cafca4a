"""GPU Ewald real-space pass (pc_ewald_real_pairs) vs the reference's
_real_space (ref longrange.py:47-72) on golden vectors made by running the
reference (tests/golden/make_ewald_golden.py).  FP64 with CUDA's erfc/exp
(a few ulp per pair, not scipy's bits): energies to 1e-12 relative, forces to
1e-12 of the largest force component."""

import numpy as np
import pytest

from conftest import load_flat

pytestmark = pytest.mark.gpu

EW = load_flat("ewald.npz")
CASES = ["rand400", "nacl216"]


@pytest.fixture(scope="module")
def pc():
    import torch
    assert torch.cuda.is_available()
    import paper_2109_09056_b200 as pkg
    return pkg


def _g(name, k):
    return EW[f"{name}_{k}"]


def _close(e, f, e_ref, f_ref):
    assert abs(e - e_ref) <= 1e-12 * abs(e_ref)
    assert np.max(np.abs(f - f_ref)) <= 1e-12 * np.max(np.abs(f_ref))


@pytest.mark.parametrize("name", CASES)
def test_real_space_reference_pairs(pc, name):
    """Caller-given (i, j) pairs: the reference's own half list."""
    e, f = pc.longrange._real_space(_g(name, "x"), _g(name, "q"), float(_g(name, "L")),
                                    float(_g(name, "alpha")), float(_g(name, "rcut")),
                                    pairs=(_g(name, "pi"), _g(name, "pj")))
    _close(e, f, float(_g(name, "energy")), _g(name, "forces"))


@pytest.mark.parametrize("name", CASES)
def test_real_space_gpu_half_list(pc, name):
    """The GPU half list (what longrange.spme builds, longrange.py:142-146) and
    the all-pairs default: same pair set as the reference, same sums."""
    x, L, rc = _g(name, "x"), float(_g(name, "L")), float(_g(name, "rcut"))
    vl = pc.neighbors.build_verlet(x, pc.geometry.cube(L), [True] * 3, rc, half_or_full="half")
    i, j = vl.pairs()
    got = set(zip(i.tolist(), j.tolist()))
    assert got == set(zip(_g(name, "pi").tolist(), _g(name, "pj").tolist()))
    e, f = pc.longrange.real_space(x, _g(name, "q"), L, float(_g(name, "alpha")), rc,
                                   neighbor_list=vl)
    _close(e, f, float(_g(name, "energy_all")), _g(name, "forces_all"))
    e2, f2 = pc.longrange._real_space(x, _g(name, "q"), L, float(_g(name, "alpha")), rc)
    _close(e2, f2, float(_g(name, "energy_all")), _g(name, "forces_all"))


def test_real_space_errors(pc):
    x = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [1.0, 0.0, 0.0]])
    q = np.array([1.0, -1.0, 0.0])
    with pytest.raises(ValueError):
        pc.longrange._real_space(x, q, 4.0, 1.0, 1.5, pairs=(np.array([1]), np.array([2])))
    with pytest.raises(ValueError):
        pc.longrange._real_space(x, q, 4.0, -1.0, 1.5)
    e, f = pc.longrange._real_space(x[:2], q[:2], 4.0, 1.0, 1.5)
    assert e < 0 and f[0, 0] > 0 and f[1, 0] < 0 and np.allclose(f[0], -f[1])
