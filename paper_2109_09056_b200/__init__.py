"""paper_2109_09056_b200 -- B200-native short-range particle hot path.

Drop-in for the reference package ``particula`` (arXiv 2109.09056 proxy) on
its MD path: ``aosoa``, ``binning``, ``neighbors``, ``decomp``, ``md`` and
``geometry`` keep the reference's names and semantics; the arithmetic runs in
hand-written sm_100a kernels (``libparticula_b200.so``, C ABI in
include/particula_b200.h) called through ctypes.
"""

from . import _lib  # noqa: F401  (fails loudly if the library is missing)

_lib.load()

from . import aosoa, binning, decomp, geometry, longrange, md, neighbors  # noqa: E402

__all__ = ["aosoa", "binning", "decomp", "geometry", "longrange", "md", "neighbors"]
__version__ = "0.1.0"
