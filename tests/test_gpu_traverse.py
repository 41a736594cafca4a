"""Device neighbor traversal (include/particula_b200_traverse.cuh, SURVEY §8
f4): pair and three-body functors over the GPU Verlet list, Serial and Team
policies, vs numpy over the same list's entries in the reference's traversal
order (ref neighbors.py:137-154, restated by the host for_each_neighbor*)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pc():
    import torch
    assert torch.cuda.is_available()
    import paper_2109_09056_b200 as pkg
    return pkg


def _system(n=600, L=7.0, seed=8):
    rng = np.random.default_rng(seed)
    return rng.random((n, 3)) * L, L


def _mi(d, L):
    return d - L * np.round(d / L)


@pytest.mark.parametrize("team", [False, True])
def test_coordination(pc, team):
    x, L = _system()
    box = pc.geometry.cube(L)
    vl = pc.neighbors.build_verlet(x, box, [True] * 3, 1.6)
    got = pc.neighbors.coordination(vl, x, box, [True] * 3, 1.1, team=team)
    ref = np.zeros(x.shape[0])

    def kern(i, j):
        d = _mi(x[j] - x[i], L)
        if (d[0] * d[0] + d[2] * d[2]) + d[1] * d[1] < 1.1 * 1.1:
            ref[i] += 1

    pc.neighbors.for_each_neighbor(vl, (0, x.shape[0]), kern)
    assert np.array_equal(got, ref)
    part = pc.neighbors.coordination(vl, x, box, [True] * 3, 1.1, i_range=(100, 250), team=team)
    assert np.array_equal(part[100:250], ref[100:250])
    assert not part[:100].any() and not part[250:].any()


@pytest.mark.parametrize("team", [False, True])
def test_angle_sums(pc, team):
    x, L = _system(400, 6.0, 9)
    box = pc.geometry.cube(L)
    vl = pc.neighbors.build_verlet(x, box, [True] * 3, 1.5)
    got = pc.neighbors.angle_sums(vl, x, box, [True] * 3, team=team)
    ref = np.zeros(x.shape[0])
    ntrip = [0]

    def kern(i, j, k):
        u, w = _mi(x[j] - x[i], L), _mi(x[k] - x[i], L)
        ref[i] += u @ w / np.sqrt((u @ u) * (w @ w))
        ntrip[0] += 1

    pc.neighbors.for_each_neighbor2(vl, (0, x.shape[0]), kern)
    assert ntrip[0] == int((vl.counts * (vl.counts - 1) // 2).sum())
    assert np.max(np.abs(got - ref)) <= 1e-12 * max(1.0, np.abs(ref).max())
    half = pc.neighbors.build_verlet(x, box, [True] * 3, 1.5, half_or_full="half")
    with pytest.raises(ValueError):
        pc.neighbors.angle_sums(half, x, box, [True] * 3)


def test_team_long_rows(pc):
    """Rows longer than a warp (Team strides) and the pair unranking of
    for_each_neighbor2's Team policy on m(m-1)/2 > 32 pairs per row."""
    x, L = _system(1500, 6.0, 10)
    box = pc.geometry.cube(L)
    vl = pc.neighbors.build_verlet(x, box, [True] * 3, 1.9)
    assert vl.counts.max() > 40
    a = pc.neighbors.angle_sums(vl, x, box, [True] * 3, team=False)
    b = pc.neighbors.angle_sums(vl, x, box, [True] * 3, team=True)
    assert np.max(np.abs(a - b)) <= 1e-11 * max(1.0, np.abs(a).max())
    c = pc.neighbors.coordination(vl, x, box, [True] * 3, 10.0, team=True)
    assert np.array_equal(c, vl.counts.astype(np.float64))
