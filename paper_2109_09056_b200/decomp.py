"""Spatial domain decomposition -- drop-in for ``particula.decomp``.

``DomainFabric``/``decompose`` are host metadata (uniform Cartesian split,
row-major rank ids; ref decomp.py:21-70).  The particle exchanges
(``migrate``, ``build_halo``, ``halo_gather``, ``halo_scatter``) operate on
device-resident ParticleSets.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .geometry import Box


@dataclass(frozen=True)
class DomainFabric:
    global_box: Box
    rank_dims: np.ndarray
    periodic: np.ndarray

    def __post_init__(self):
        dims = np.atleast_1d(np.asarray(self.rank_dims, dtype=np.int64))
        per = np.atleast_1d(np.asarray(self.periodic, dtype=bool))
        if dims.shape[0] != self.global_box.ndim or per.shape[0] != self.global_box.ndim:
            raise ValueError("rank_dims/periodic must match box dimensionality")
        if np.any(dims < 1):
            raise ValueError("rank_dims must be >= 1 per axis")
        object.__setattr__(self, "rank_dims", dims)
        object.__setattr__(self, "periodic", per)

    @property
    def n_ranks(self) -> int:
        return int(np.prod(self.rank_dims))

    @property
    def block_lengths(self) -> np.ndarray:
        return self.global_box.lengths / self.rank_dims

    def coords_of(self, rank: int) -> np.ndarray:
        return np.array(np.unravel_index(rank, tuple(self.rank_dims)))

    def rank_of(self, coords) -> int:
        return int(np.ravel_multi_index(tuple(np.asarray(coords)), tuple(self.rank_dims)))

    def local_box(self, rank: int) -> Box:
        c = self.coords_of(rank)
        bl = self.block_lengths
        low = self.global_box.low + c * bl
        high = np.where(c == self.rank_dims - 1, self.global_box.high, low + bl)
        return Box(low, high)


def decompose(global_box: Box, rank_dims, periodic) -> DomainFabric:
    return DomainFabric(global_box, rank_dims, periodic)
