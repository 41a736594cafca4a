"""CPU-side checks of the C ABI boundary (no GPU needed):

* the shared library loads and exports every symbol include/particula_b200.h
  declares, and the ctypes binding covers all of them;
* the ctypes mirrors of pc_box / pc_grid / pc_lj match the C layout (gcc);
* the division-free min-image threshold reproduces the reference formula
  ``dx - L*round(dx/L)`` bit for bit (host emulation of pc_common.cuh).
"""

import ctypes
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "particula_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pc_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2109_09056_b200 import _lib
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    unbound = [n for n in names if n not in _lib.SIGNATURES]
    assert not unbound, unbound
    assert lib.pc_version() == 1


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_2109_09056_b200", "libparticula_b200.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def test_struct_layout_matches_header():
    from paper_2109_09056_b200 import _lib
    src = r"""
    #include <stdio.h>
    #include <stddef.h>
    #include "particula_b200.h"
    int main(void) {
      printf("%zu %zu %zu %zu %zu\n", sizeof(pc_box), offsetof(pc_box, length),
             offsetof(pc_box, mi_thresh), offsetof(pc_box, periodic), offsetof(pc_box, ndim));
      printf("%zu %zu %zu %zu %zu\n", sizeof(pc_grid), offsetof(pc_grid, width),
             offsetof(pc_grid, nc), offsetof(pc_grid, ncells), offsetof(pc_grid, ndim));
      printf("%zu %zu %zu\n", sizeof(pc_lj), offsetof(pc_lj, cutoff2), offsetof(pc_lj, overlap2));
      return 0;
    }
    """
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        exe = os.path.join(d, "t")
        open(c, "w").write(src)
        subprocess.check_call(["gcc", "-I", os.path.dirname(HEADER), c, "-o", exe])
        lines = subprocess.check_output([exe], text=True).split("\n")
    B, G, J = _lib.PcBox, _lib.PcGrid, _lib.PcLJ
    assert [int(v) for v in lines[0].split()] == [
        ctypes.sizeof(B), B.length.offset, B.mi_thresh.offset, B.periodic.offset, B.ndim.offset]
    assert [int(v) for v in lines[1].split()] == [
        ctypes.sizeof(G), G.width.offset, G.nc.offset, G.ncells.offset, G.ndim.offset]
    assert [int(v) for v in lines[2].split()] == [
        ctypes.sizeof(J), J.cutoff2.offset, J.overlap2.offset]


def _device_min_image(d, L, T):
    """numpy emulation of pc_common.cuh min_image for |d| < L."""
    a = np.abs(d)
    return np.where(a >= T, np.copysign(a - L, -d), d)


@pytest.mark.parametrize("L", [26.874, 107.4941, 214.9883, 4.0, 1.0, 3.0, 6.0,
                               2 * 107.49415, 0.1])
def test_min_image_threshold_bit_exact(L):
    from paper_2109_09056_b200 import _lib
    T = _lib.min_image_threshold(L)
    assert T / L > 0.5 and np.nextafter(T, 0) / L <= 0.5
    rng = np.random.default_rng(0)
    d = rng.uniform(-L, L, 200_000)
    # dense sampling around +-T and +-L/2 (ulp neighbourhoods)
    near = np.concatenate([T + np.arange(-64, 65) * np.spacing(T),
                           L / 2 + np.arange(-64, 65) * np.spacing(L / 2)])
    d = np.concatenate([d, near, -near, [0.0, -0.0]])
    d = d[np.abs(d) < L]
    ref = d - L * np.round(d / L)
    got = _device_min_image(d, L, T)
    assert np.array_equal(ref.view(np.int64), got.view(np.int64)) or \
        np.array_equal(ref, got)


def test_box_grid_packing():
    from paper_2109_09056_b200 import _lib
    b = _lib.make_box([0.0, -1.0], [2.0, 3.0], [True, False])
    assert b.ndim == 2 and b.periodic[0] == 1 and b.periodic[1] == 0
    assert b.mi_thresh[1] == np.inf and b.mi_thresh[2] == np.inf
    assert b.length[1] == 4.0
    g = _lib.make_grid([0.0], [1.0], [0.25], [4])
    assert (g.nc[0], g.nc[1], g.nc[2], g.ncells, g.ndim) == (4, 1, 1, 4, 1)


def test_python_call_sites_match_signatures():
    """Every call("pc_x", ...) in the package passes exactly the bound arity."""
    import ast
    from paper_2109_09056_b200 import _lib
    pkg = os.path.join(ROOT, "paper_2109_09056_b200")
    bad = []
    for fn in os.listdir(pkg):
        if not fn.endswith(".py"):
            continue
        tree = ast.parse(open(os.path.join(pkg, fn)).read())
        for node in ast.walk(tree):
            if isinstance(node, ast.Call) and getattr(node.func, "id", None) == "call" \
                    and node.args and isinstance(node.args[0], ast.Constant):
                name = node.args[0].value
                want = len(_lib.SIGNATURES[name][1])
                got = len(node.args) - 1
                if got != want:
                    bad.append((fn, node.lineno, name, got, want))
    assert not bad, bad
