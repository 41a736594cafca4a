"""Ewald real-space pass on the GPU (ref longrange.py:47-72, `_real_space`).

SURVEY §8(f3): the erfc-screened Coulomb pair sum that the reference's SPME
(longrange.spme, longrange.py:142-146) runs over a half Verlet list -- the only
consumer of ``build_verlet`` besides the MD driver.  The mesh part of SPME
(P2G, FFT, gather) is outside this package's scope.

``_real_space(positions, q, L, alpha, r_cut, pairs=None)`` keeps the
reference's signature and results: pairs = (i, j) arrays (a half list's
``pairs()``) or, when None, every pair within r_cut -- the reference
enumerates all i < j and selects r^2 < r_cut^2; here the GPU half list
(``build_verlet(..., "half")``) yields exactly that set.  Returns
(energy, forces) as numpy.  FP64 throughout (pc_ewald_real_pairs); erfc/exp
are CUDA's, so sums agree with the reference to ~1e-13 relative.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _kernels, _lib
from ._lib import call, ptr, stream
from .geometry import cube
from .neighbors import VerletList, build_verlet

__all__ = ["default_alpha", "real_space", "_real_space"]


def default_alpha(r_cut: float, target: float = 1e-8) -> float:
    """Splitting parameter with erfc(alpha * r_cut) <= target (ref longrange.py:36-39;
    host-side parameter choice, scipy as in the reference)."""
    from scipy.special import erfcinv
    return float(erfcinv(target)) / r_cut


def _pairs_device(pairs, n, dev):
    if isinstance(pairs, VerletList):
        counts, offsets, index = pairs.device_csr()
        m = int(index.numel())
        pi = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
        call("pc_csr_pairs", ptr(offsets), n, ptr(pi), stream())
        return pi[:m], index[:m].contiguous()
    ii, jj = pairs
    ii = torch.as_tensor(np.asarray(ii)).to(device=dev, dtype=torch.int32).contiguous()
    jj = torch.as_tensor(np.asarray(jj)).to(device=dev, dtype=torch.int32).contiguous()
    if ii.shape != jj.shape:
        raise ValueError("pairs must be two arrays of equal length")
    return ii, jj


def real_space(positions, q, box_length: float, alpha: float, r_cut: float,
               neighbor_list=None, pairs=None):
    """(energy, forces) of the real-space Ewald sum; ``neighbor_list`` a half
    VerletList (as longrange.spme passes), or explicit ``pairs``, or neither
    (all pairs within r_cut through the GPU half list)."""
    if alpha <= 0 or r_cut <= 0:
        raise ValueError("alpha and r_cut must be positive")
    x = _kernels.as_device(positions)
    if x.dim() != 2 or x.shape[1] != 3:
        raise ValueError("positions must be (n, 3)")
    n = int(x.shape[0])
    dev = x.device
    qd = _kernels.as_device(q).to(torch.float64).contiguous()
    if qd.numel() != n:
        raise ValueError("q must have one charge per particle")
    L = float(box_length)
    if neighbor_list is None and pairs is None:
        neighbor_list = build_verlet(x, cube(L), [True] * 3, r_cut, half_or_full="half")
    pi, pj = _pairs_device(neighbor_list if pairs is None else pairs, n, dev)
    m = int(pi.numel())
    f = torch.zeros((max(n, 1), 3), dtype=torch.float64, device=dev)
    nb = int(_lib.load().pc_ewald_real_blocks(m))
    epart = torch.zeros(max(nb, 1), dtype=torch.float64, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    box = _lib.make_box(np.zeros(3), np.full(3, L), np.ones(3, bool))
    call("pc_ewald_real_pairs", ptr(x.contiguous()), ptr(qd), ptr(pi), ptr(pj), m, box,
         float(alpha), float(r_cut), ptr(f), ptr(epart), ptr(flag), stream())
    if int(flag.item()) & _lib.FLAG_OVERLAP:
        raise ValueError("overlapping charges in real-space sum")
    energy = float(np.sum(epart[:nb].cpu().numpy())) if nb else 0.0
    return energy, f[:n].cpu().numpy()


def _real_space(positions, q, L, alpha, r_cut, pairs=None):
    """The reference's signature (longrange.py:47): pairs = (i, j) arrays or None."""
    return real_space(positions, q, L, alpha, r_cut, pairs=pairs)
