"""ctypes binding of libparticula_b200.so (the C ABI in include/particula_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (or ``make -C
paper_2109_09056_b200/csrc``).  There is no fallback: if the shared object or
a CUDA device is missing, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libparticula_b200.so")
# A/B builds (scripts/): PARTICULA_B200_LIB names another in-tree build of the same ABI
if os.environ.get("PARTICULA_B200_LIB"):
    LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)),
                            os.path.basename(os.environ["PARTICULA_B200_LIB"]))

PC_OK = 0
PC_ERR_VALUE = -1
PC_ERR_RUNTIME = -2
PC_ERR_OVERLAP = -3
PC_ERR_CUDA = -4
PC_ERR_CAPACITY = -5

PC_NBR_COUNT = 0
PC_NBR_CSR = 1
PC_NBR_ELL = 2

FLAG_OUTSIDE = 1
FLAG_OVERFLOW = 2
FLAG_OVERLAP = 4
FLAG_NONPERIODIC = 8
FLAG_STAGE = 16
PC_NBR_SELL = 3

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p


class PcBox(ctypes.Structure):
    _fields_ = [("low", c_dbl * 3), ("high", c_dbl * 3), ("length", c_dbl * 3),
                ("mi_thresh", c_dbl * 3), ("periodic", c_i32 * 3), ("ndim", c_i32)]


class PcGrid(ctypes.Structure):
    _fields_ = [("low", c_dbl * 3), ("high", c_dbl * 3), ("width", c_dbl * 3),
                ("nc", c_i32 * 3), ("ncells", c_i32), ("ndim", c_i32), ("pad", c_i32)]


class PcLJ(ctypes.Structure):
    _fields_ = [("epsilon", c_dbl), ("sigma", c_dbl), ("cutoff2", c_dbl),
                ("overlap2", c_dbl)]


# name -> (restype, argtypes); every symbol include/particula_b200.h declares
SIGNATURES = {
    "pc_last_error": (ctypes.c_char_p, []),
    "pc_version": (ctypes.c_int, []),
    "pc_launch_count": (c_i64, []),
    "pc_device_sync": (ctypes.c_int, [c_vp]),
    "pc_aosoa_permute": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, c_i32, c_i64, c_vp,
                                        c_i32, c_vp]),
    "pc_gather_rows": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, c_i32, c_vp]),
    "pc_bin_count": (ctypes.c_int, [c_vp, c_i64, c_i32, ctypes.POINTER(PcGrid), c_i32,
                                    c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pc_key_digits": (ctypes.c_int, [c_vp, c_vp, c_i64, c_i64, c_i32, c_i64, c_vp, c_vp,
                                     c_vp]),
    "pc_check_bijection": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp, c_vp]),
    "pc_scatter_rows": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, c_i32, c_vp]),
    "pc_aosoa_field": (ctypes.c_int, [c_vp, c_i64, c_i32, c_i64, c_i64, c_i32, c_vp, c_i32,
                                      c_vp]),
    "pc_csr_to_dense": (ctypes.c_int, [c_vp, c_i32, c_vp, c_i32, c_vp, c_vp]),
    "pc_scan_i32": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "pc_scan_i32_i64": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "pc_scan_tmp_bytes": (c_i64, [c_i64]),
    "pc_bin_place": (ctypes.c_int, [c_vp, c_i64, c_vp, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "pc_bin_place_unstable": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "pc_partition_chunks": (c_i64, [c_i64]),
    "pc_partition_hist": (ctypes.c_int, [c_vp, c_i64, c_i32, c_vp, c_vp]),
    "pc_partition_place": (ctypes.c_int, [c_vp, c_i64, c_i32, c_vp, c_vp, c_vp]),
    "pc_invert_order": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp]),
    "pc_nbr_build": (ctypes.c_int, [c_vp, c_i32, c_vp, ctypes.POINTER(PcGrid),
                                    ctypes.POINTER(PcBox), c_dbl, c_i32, c_i32, c_i32,
                                    c_vp, c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_vp,
                                    ctypes.POINTER(PcBox)]),
    "pc_sort_rows": (ctypes.c_int, [c_vp, c_i32, c_vp, c_vp]),
    "pc_nbr_build_sell": (ctypes.c_int, [c_vp, c_i32, c_vp, ctypes.POINTER(PcGrid),
                                         ctypes.POINTER(PcBox), c_dbl, c_i32, c_i32, c_vp,
                                         c_vp, c_vp, ctypes.POINTER(c_i32), c_vp, c_vp,
                                         ctypes.POINTER(PcBox), c_i32]),
    "pc_lj_force_sell_half": (ctypes.c_int, [c_vp, c_i32, c_vp, c_vp, c_i32,
                                             ctypes.POINTER(PcBox), ctypes.POINTER(PcLJ), c_dbl,
                                             c_vp, c_i64, c_vp, c_vp, c_vp]),
    "pc_domain_permute": (ctypes.c_int, [c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64,
                                         c_vp, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "pc_md_permute": (ctypes.c_int, [c_vp, c_i32, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_i64,
                                     c_vp, c_vp]),
    "pc_bin_count_planar": (ctypes.c_int, [c_vp, c_i64, c_i64, ctypes.POINTER(PcGrid), c_vp,
                                           c_vp, c_vp, c_vp]),
    "pc_pos_planar": (ctypes.c_int, [c_vp, c_i32, c_vp, c_i64, c_vp]),
    "pc_owner_of": (ctypes.c_int, [c_vp, c_i64, c_i32, ctypes.POINTER(PcGrid), c_vp, c_vp,
                                   c_vp]),
    "pc_owner_of_domain": (ctypes.c_int, [c_vp, c_i64, c_i32, ctypes.POINTER(PcGrid), c_vp, c_i32,
                                           c_vp, c_vp, c_vp]),
    "pc_check_nonperiodic": (ctypes.c_int, [c_vp, c_i64, c_i32, ctypes.POINTER(PcBox), c_vp,
                                            c_vp]),
    "pc_halo_plan": (ctypes.c_int, [c_vp, c_i64, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_i32,
                                    c_dbl, c_vp, c_vp, c_vp]),
    "pc_compact": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "pc_exact_sum": (ctypes.c_int, [c_vp, c_i64, c_i32, c_vp, c_vp, c_vp]),
    "pc_exact_finish": (ctypes.c_int, [c_vp, c_i32, c_vp, c_vp]),
    "pc_halo_force_pack": (ctypes.c_int, [c_vp, c_i64, c_vp, c_i64, c_vp, c_vp]),
    "pc_halo_force_add": (ctypes.c_int, [c_vp, c_i64, c_vp, c_i64, c_vp, c_vp]),
    "pc_halo_select_chunks": (c_i64, [c_i64]),
    "pc_halo_select_count": (ctypes.c_int, [c_vp, c_i64, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp,
                                            c_i32, c_dbl, c_vp, c_vp, c_vp, c_vp]),
    "pc_halo_select_place": (ctypes.c_int, [c_vp, c_i64, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp,
                                            c_i32, c_dbl, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pc_gather_shift": (ctypes.c_int, [c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_vp]),
    "pc_scatter_add": (ctypes.c_int, [c_vp, c_vp, c_i64, c_i32, c_vp, c_vp]),
    "pc_halo_pack": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_vp]),
    "pc_halo_pack_planar": (ctypes.c_int, [c_vp, c_i64, c_vp, c_i64, c_vp, c_vp]),
    "pc_tile_count": (c_i32, [ctypes.POINTER(PcGrid)]),
    "pc_tile_plan_ints": (c_i32, []),
    "pc_cell_zsort": (ctypes.c_int, [c_vp, c_i64, c_vp, c_i32, c_vp, c_vp, c_vp]),
    "pc_tile_stage_cap": (c_i32, []),
    "pc_tile_rows": (ctypes.c_int, [c_vp, ctypes.POINTER(PcGrid), c_vp, c_vp]),
    "pc_tile_rows_domain": (ctypes.c_int, [c_vp, ctypes.POINTER(PcGrid), c_vp, c_vp, c_vp]),
    "pc_tile_build": (ctypes.c_int, [c_vp, c_i64, c_vp, ctypes.POINTER(PcGrid),
                                     ctypes.POINTER(PcBox), c_dbl, c_i32, c_vp, c_vp, c_vp,
                                     c_vp, c_vp, c_vp, c_vp]),
    "pc_traverse_coordination": (ctypes.c_int, [c_vp, ctypes.POINTER(PcBox), c_vp, c_vp, c_i32,
                                                c_i32, c_i32, c_dbl, c_i32, c_vp, c_vp]),
    "pc_traverse_angle_sum": (ctypes.c_int, [c_vp, ctypes.POINTER(PcBox), c_vp, c_vp, c_i32,
                                             c_i32, c_i32, c_i32, c_vp, c_vp]),
    "pc_sell_sort_by_tag": (ctypes.c_int, [c_vp, c_i32, c_vp, c_vp, c_i32, c_vp, c_vp]),
    "pc_lj_force_sell_atoms": (ctypes.c_int, [c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_i32,
                                              ctypes.POINTER(PcBox), ctypes.POINTER(PcLJ), c_dbl,
                                              c_vp, c_i64, c_vp, c_i64, c_dbl, c_dbl, c_vp, c_vp,
                                              c_vp]),
    "pc_ewald_real_blocks": (c_i64, [c_i64]),
    "pc_csr_pairs": (ctypes.c_int, [c_vp, c_i32, c_vp, c_vp]),
    "pc_ewald_real_pairs": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, ctypes.POINTER(PcBox),
                                           c_dbl, c_dbl, c_vp, c_vp, c_vp, c_vp]),
    "pc_tile_build_domain": (ctypes.c_int, [c_vp, c_i64, c_vp, ctypes.POINTER(PcGrid),
                                            ctypes.POINTER(PcBox), c_dbl, c_i32, c_vp, c_vp,
                                            c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                            ctypes.POINTER(PcBox), c_vp, c_vp]),
    "pc_tile_build_ordered": (ctypes.c_int, [c_vp, c_i64, c_vp, ctypes.POINTER(PcGrid),
                                             ctypes.POINTER(PcBox), c_dbl, c_i32, c_vp, c_vp,
                                             c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                             ctypes.POINTER(PcBox), c_vp, c_vp, c_i32]),
    "pc_tile_force": (ctypes.c_int, [c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_i32,
                                     ctypes.POINTER(PcBox), ctypes.POINTER(PcLJ), c_dbl, c_vp,
                                     c_i64, c_vp, c_i64, c_dbl, c_dbl, c_vp, c_vp, c_vp, c_vp,
                                     c_dbl, c_dbl, c_vp, c_vp, c_vp, c_vp]),
    "pc_pos_from_planar": (ctypes.c_int, [c_vp, c_i64, c_i32, c_vp, c_vp]),
    "pc_tile_force_partials": (c_i32, [c_i32]),
    "pc_tile_order": (ctypes.c_int, [c_i32, c_vp, c_vp, c_vp, c_i32, c_i32, c_vp]),
    "pc_tile_decode": (ctypes.c_int, [c_i32, c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp,
                                      c_vp]),
    "pc_halo_unpack": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp]),
    "pc_lj_force_sell": (ctypes.c_int, [c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_i32,
                                        ctypes.POINTER(PcBox),
                                        ctypes.POINTER(PcLJ), c_dbl, c_vp, c_i64, c_vp, c_i64,
                                        c_dbl, c_dbl, c_vp, c_vp, c_vp]),
    "pc_lj_force": (ctypes.c_int, [c_vp, c_i32, c_vp, c_vp, c_vp, c_i64,
                                   ctypes.POINTER(PcBox), ctypes.POINTER(PcLJ), c_vp, c_i64,
                                   c_vp, c_vp, c_vp, c_i64, c_dbl, c_dbl, c_vp, c_vp, c_vp]),
    "pc_lj_force_blocks": (c_i32, [c_i32]),
    "pc_lj_force_sell_partials": (c_i32, [c_i32]),
    "pc_lj_force_half": (ctypes.c_int, [c_vp, c_i32, c_vp, c_vp, c_i64,
                                        ctypes.POINTER(PcBox), ctypes.POINTER(PcLJ), c_vp,
                                        c_i64, c_vp, c_vp, c_vp]),
    "pc_kick_drift_wrap": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_i64, c_i32, c_dbl,
                                          c_dbl, ctypes.POINTER(PcBox), c_vp, c_i64, c_vp]),
    "pc_kick": (ctypes.c_int, [c_vp, c_i64, c_vp, c_i64, c_i32, c_dbl, c_dbl, c_vp, c_vp]),
    "pc_reduce_partials": (ctypes.c_int, [c_vp, c_i32, c_vp, c_vp]),
    "pc_box_wrap": (ctypes.c_int, [c_vp, c_i64, c_i32, ctypes.POINTER(PcBox), c_vp]),
    "pc_box_min_image": (ctypes.c_int, [c_vp, c_i64, c_i32, ctypes.POINTER(PcBox), c_vp]),
    "pc_lj_pair": (ctypes.c_int, [c_vp, c_vp, c_i64, c_dbl, c_dbl, c_vp, c_vp, c_vp]),
    "pc_p2p_window_bytes": (ctypes.c_int, [c_i64, c_i32, c_i32, ctypes.POINTER(c_i64)]),
    "pc_p2p_window_alloc": (ctypes.c_int, [c_i64, c_i32, c_i32, ctypes.POINTER(c_vp), c_vp]),
    "pc_p2p_window_free": (ctypes.c_int, [c_vp]),
    "pc_p2p_handle_bytes": (c_i32, []),
    "pc_p2p_dest_bytes": (c_i32, []),
    "pc_p2p_open": (ctypes.c_int, [c_vp, ctypes.POINTER(c_vp)]),
    "pc_p2p_close": (ctypes.c_int, [c_vp]),
    "pc_p2p_put": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i64, c_i32, c_i64, c_i32, c_vp]),
    "pc_p2p_signal": (ctypes.c_int, [c_vp, c_i32, c_i64, c_i32, c_i64, c_vp]),
    "pc_p2p_pack_put": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp, c_i32, c_i64, c_i64, c_i32,
                                       c_vp]),
    "pc_p2p_wait": (ctypes.c_int, [c_vp, c_i64, c_vp, c_i32, c_i64, c_vp, c_i64, c_vp]),
}

_lib = None


def load():
    """Load the shared library (no GPU needed) and bind every signature."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()')")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str = ""):
    """Map a C-ABI status to the reference's exception classes."""
    if rc == PC_OK:
        return
    msg = load().pc_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == PC_ERR_VALUE:
        raise ValueError(text)
    if rc == PC_ERR_RUNTIME:
        raise RuntimeError(text)
    if rc == PC_ERR_OVERLAP:
        raise FloatingPointError(text)
    raise RuntimeError(f"CUDA failure ({rc}) {text}")


def call(name, *args):
    check(getattr(load(), name)(*args), name)


def device():
    """The CUDA device all compute runs on; raises without a GPU."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2109_09056_b200 needs a CUDA device (B200); "
                           "there is no CPU fallback")
    load()
    return torch.device("cuda", torch.cuda.current_device())


def stream():
    """The current CUDA stream of the current device as a raw handle (the
    C-ABI's `void* stream`).  torch's raw-stream query: ~10x cheaper than
    torch.cuda.current_stream() (a Stream object per call), which dominated
    the host time of the decomposed rebuild's ~150 kernel calls per rank."""
    import torch
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return ctypes.c_void_p(raw(torch._C._cuda_getDevice()))
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    """Raw device pointer of a torch tensor (None for None)."""
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def min_image_threshold(length: float) -> float:
    """Smallest d > 0 with fl(d/L) > 0.5, i.e. where round-half-even(d/L)
    becomes 1.  With it, d - L*round(d/L) == copysign(fl(|d| - L), -d) for
    T <= |d| < L and == d below T (see pc_common.cuh: min_image)."""
    L = float(length)
    d = np.float64(L * 0.5)
    while d / L <= 0.5:
        d = np.nextafter(d, np.inf)
    while np.nextafter(d, -np.inf) / L > 0.5:
        d = np.nextafter(d, -np.inf)
    return float(d)


def make_box(low, high, periodic) -> PcBox:
    low = np.asarray(low, np.float64)
    high = np.asarray(high, np.float64)
    per = np.asarray(periodic, bool)
    d = low.shape[0]
    if d > 3:
        raise ValueError("only 1-3 dimensional boxes are supported on the GPU path")
    b = PcBox()
    for a in range(3):
        if a < d:
            b.low[a], b.high[a] = low[a], high[a]
            b.length[a] = high[a] - low[a]
            b.periodic[a] = int(per[a])
            b.mi_thresh[a] = min_image_threshold(b.length[a]) if per[a] else np.inf
        else:   # padded axis: zero coordinate, non-periodic, one cell
            b.low[a], b.high[a], b.length[a] = 0.0, 1.0, 1.0
            b.periodic[a] = 0
            b.mi_thresh[a] = np.inf
    b.ndim = d
    return b


def make_grid(low, high, width, nc) -> PcGrid:
    low = np.asarray(low, np.float64)
    high = np.asarray(high, np.float64)
    d = low.shape[0]
    g = PcGrid()
    for a in range(3):
        if a < d:
            g.low[a], g.high[a], g.width[a], g.nc[a] = low[a], high[a], width[a], int(nc[a])
        else:
            g.low[a], g.high[a], g.width[a], g.nc[a] = 0.0, 1.0, 1.0, 1
    g.ncells = int(np.prod([g.nc[a] for a in range(3)]))
    g.ndim = d
    return g
