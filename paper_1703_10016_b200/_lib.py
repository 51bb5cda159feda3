"""ctypes binding of the C-ABI library ``libwqb200.so`` (include/wqb200.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).
There is no fallback: if it is missing, every GPU entry point raises
``DeviceError``.  PyTorch is used only for device memory and the current
CUDA stream; raw ``data_ptr()`` values cross the boundary.
"""

from __future__ import annotations

import ctypes
import os

from .errors import DeviceError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WQB200_LIB") or os.path.join(_HERE, "libwqb200.so")  # override: A/B tools only

c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p

WQ_FLAG_R_NONPOSITIVE = 1
WQ_TILE = 32
WQ_FTILE = 64
WQ_K1_TABLE, WQ_K1_OPEN, WQ_K1_CLOSED = 0, 1, 2


class WqSmooth(ctypes.Structure):
    _fields_ = [("n_rows", c_i64), ("nq", c_i64), ("wg", c_i64), ("closed", c_i64),
                ("k1_mode", c_i64), ("period", c_dbl), ("s", c_vp), ("fx", c_vp), ("fy", c_vp),
                ("J", c_vp), ("invp2", c_vp), ("g_start", c_vp), ("g_w", c_vp),
                ("near_k", c_i64), ("near_j2", c_vp)]


class WqLogpart(ctypes.Structure):
    _fields_ = [("n_rows", c_i64), ("n_fine", c_i64), ("da", c_i64), ("tu", c_i64),
                ("ws", c_i64), ("e_start", c_vp), ("U", c_vp), ("s_start", c_vp), ("s_w", c_vp)]


class WqPairs(ctypes.Structure):
    _fields_ = [("n_rows", c_i64), ("n_fine", c_i64), ("n_el", c_i64), ("n_gap", c_i64),
                ("da", c_i64), ("db", c_i64), ("closed", c_i64), ("wu", c_i64), ("wv", c_i64),
                ("u_el", c_vp), ("u_loc", c_vp), ("v_el", c_vp), ("v_loc", c_vp), ("u", c_vp),
                ("pu", c_i64), ("v", c_vp), ("m2", c_vp)]


# name -> argtypes (restype c_int unless noted)
_SIGS = {
    "wq_version": [],
    "wq_last_error": [],
    "wq_fp64_peak": [c_i64, c_int, c_vp, c_vp],
    "wq_ik1": [ctypes.POINTER(WqSmooth), c_i64, c_i64, c_i64, c_i64, c_vp, c_i64, c_int, c_i64,
               c_vp, c_vp],
    "wq_ik1_band": [ctypes.POINTER(WqSmooth), c_i64, c_i64, c_vp, c_i64, c_i64, c_vp, c_vp],
    "wq_pair_table": [c_i64, c_int, c_int, c_int, c_dbl, c_vp, c_vp, c_vp, c_int, c_vp, c_vp,
                      c_vp, c_vp],
    "wq_circ_tables": [c_i64, c_int, c_int, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp,
                       c_vp],
    "wq_ik2_circ": [ctypes.POINTER(WqLogpart), c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_vp,
                    c_i64, c_int, c_vp],
    "wq_theta_t": [ctypes.POINTER(WqPairs), c_vp, c_vp],
    "wq_theta_t_rows": [ctypes.POINTER(WqPairs), c_i64, c_i64, c_vp, c_i64, c_vp],
    "wq_dmat": [ctypes.POINTER(WqPairs), c_vp, c_vp],
    "wq_band_solve_cols": [c_i64, c_i64, c_vp, c_vp, c_i64, c_i64, c_vp],
    "wq_transpose": [c_vp, c_i64, c_i64, c_vp, c_vp],
    "wq_cyc_solve_cols": [c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp],
    "wq_gather_fs": [ctypes.POINTER(WqLogpart), c_dbl, c_vp, c_vp, c_vp],
    "wq_gather_yts": [ctypes.POINTER(WqLogpart), c_dbl, c_vp, c_vp, c_i64, c_vp],
    "wq_st_phi_sym": [ctypes.POINTER(WqLogpart), c_vp, c_vp, c_dbl, c_int, c_vp],
    "wq_add_st_phi": [ctypes.POINTER(WqLogpart), c_vp, c_i64, c_i64, c_vp, c_i64, c_int, c_vp],
    "wq_symmetrize": [c_vp, c_i64, c_dbl, c_vp],
    "wq_absmax_defect": [c_vp, c_i64, c_vp, c_vp],
    "wq_b1w": [ctypes.POINTER(WqSmooth), c_vp, c_vp, c_vp],
    "wq_ik1_sym": [ctypes.POINTER(WqSmooth), c_vp, c_i64, c_i64, c_vp, c_vp],
    "wq_zext": [c_i64, c_int, c_int, c_int, c_vp, c_vp, c_vp, c_vp],
    "wq_x2_pairs": [c_i64, c_int, c_int, c_int, c_int, c_int, c_int, c_vp, c_vp, c_vp, c_dbl,
                    c_dbl, c_vp, c_i64, c_vp],
    "wq_ik1_pairs": [ctypes.POINTER(WqSmooth), c_i64, c_i64, c_vp, c_i64, c_vp, c_vp],
    "wq_x2_pairs_range": [c_i64, c_int, c_int, c_int, c_int, c_int, c_int, c_vp, c_vp, c_vp, c_dbl,
                          c_dbl, c_i64, c_i64, c_vp, c_i64, c_vp],
    "wq_ik1_rows": [ctypes.POINTER(WqSmooth), c_i64, c_i64, c_vp, c_i64, c_vp, c_vp],
    "wq_x2_rows": [c_i64, c_int, c_int, c_int, c_int, c_int, c_int, c_vp, c_vp, c_vp, c_dbl, c_dbl,
                   c_i64, c_i64, c_vp, c_i64, c_vp],
    "wq_b2_inner": [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp],
    "wq_ik1_pair_list": [ctypes.POINTER(WqSmooth), c_vp, c_i64, c_vp, c_i64, c_vp, c_vp],
    "wq_x2_pair_list": [c_i64, c_int, c_int, c_int, c_int, c_int, c_int, c_vp, c_vp, c_vp, c_dbl,
                        c_dbl, c_vp, c_i64, c_vp, c_i64, c_vp],
    "wq_selftest_log": [c_i64, c_vp, c_vp, c_vp, c_vp],
    "wq_selftest_dmma": [c_vp, c_vp, c_vp, c_vp],
    "wq_gen_pair_blocks": [c_i64, c_i64, c_i64, c_int, c_int, c_int, c_int, c_dbl, c_vp, c_vp,
                           c_vp, c_vp, c_vp, c_vp, c_int, c_vp, c_vp, c_vp, c_vp, c_vp,
                           c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp],
    "wq_gen_gather_theta": [c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_int, c_int, c_int,
                            c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp],
    "wq_mirror_upper": [c_vp, c_i64, c_i64, c_vp],
    "wq_pack_pairs": [c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp],
    "wq_unpack_pairs": [c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp],
    "wq_mirror_lower": [c_vp, c_i64, c_i64, c_vp, c_vp, c_vp],
    "wq_gather_fs_rows": [ctypes.POINTER(WqLogpart), c_dbl, c_vp, c_vp, c_i64, c_i64, c_i64, c_vp],
    "wq_phi_s_rows": [ctypes.POINTER(WqLogpart), c_vp, c_i64, c_i64, c_vp, c_i64, c_int, c_vp],
    "wq_gen_gather_d": [c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_int, c_int, c_vp, c_vp, c_vp,
                        c_vp, c_vp],
    "wq_band_solve_seg": [c_i64, c_i64, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp],
    "wq_band_solve_win": [c_i64, c_i64, c_vp, c_vp, c_i64, c_i64, c_vp],
    "wq_gen_near_moments": [c_i64, c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_int, c_vp, c_vp, c_vp,
                            c_vp, c_vp, c_vp, c_vp],
    "wq_gen_moments_far": [c_i64, c_int, c_int, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                           c_vp, c_vp, c_vp],
    "wq_ystage": [c_i64, c_i64, c_i64, c_int, c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                  c_vp, c_vp, c_int, c_vp, c_int, c_vp, c_vp, c_vp, c_vp, c_int, c_vp, c_vp, c_vp,
                  c_i64, c_i64, c_vp, c_i64, c_i64, c_i64, c_int, c_vp, c_vp, c_vp, c_i64, c_vp],
    "wq_ystage_mma_prep": [c_i64, c_i64, c_i64, c_int, c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp,
                           c_vp, c_int, c_vp, c_vp, c_vp, c_int, c_vp, c_vp, c_vp, c_vp, c_vp,
                           c_vp, c_i64, c_vp],
    "wq_ystage_mma_tiles": [c_i64, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp],
    "wq_ystage_mma": [c_i64, c_i64, c_i64, c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                      c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64,
                      c_int, c_vp],
}

EXPORTED = tuple(_SIGS)

_lib = None


def load():
    """Load (once) and return the C-ABI library; raise DeviceError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(f"{LIB_PATH} is not built: run __graft_entry__.build() (nvcc sm_100a)")
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as exc:
        raise DeviceError(f"cannot load {LIB_PATH}: {exc}") from exc
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_char_p if name == "wq_last_error" else c_int
    _lib = lib
    return lib


def call(name, *args):
    """Invoke an entry point and raise DeviceError on a non-zero status."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.wq_last_error().decode(errors="replace")
        raise DeviceError(f"{name} failed ({rc}): {msg}")
    return rc


def ptr(t):
    """Raw device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def stream_handle(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)
