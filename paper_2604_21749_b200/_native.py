"""ctypes binding of ``libcurast_b200.so`` (include/curast.h).

The product path has no CPU fallback: if the library is missing or the GPU is
absent, ``lib()`` raises.  Build it with ``python -c "import __graft_entry__ as
g; g.build()"`` (nvcc, sm_100a).
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CURAST_LIB") or os.path.join(_HERE, "libcurast_b200.so")
ABI_VERSION = 3

POS_F64, POS_F32, POS_U16 = 0, 1, 2
IDX_U32, IDX_PACKED = 0, 1

C_Q2, C_Q3, C_S1, C_S2, C_S3 = 0, 1, 2, 10, 15
C_CLAIM1, C_CLAIM2, C_CLAIM3, C_EXACT, C_QX = 16, 17, 18, 19, 20
QX_RES = 128       # CURAST_QX_RES: fp64-queue slots a stage-1 warp reserves at a time
C_QXHOLES = 32     # fp64-queue slots reserved by a warp but left empty (tag -1)
COUNTER_SLOTS = 40
FILTER_FLOATS = 16
INST_BLOCK = 16          # CURAST_INST_BLOCK: instances per instanced work unit
QX_WORDS = 6
STEP_TRIS = 128          # CURAST_STEP_TRIS: triangles per warp step / index step
S1_CHUNK = 16 * STEP_TRIS      # curast_chunk_tris(0): flat stage-1 chunk

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_D = ctypes.c_double


class CurastFrame(ctypes.Structure):
    """Mirror of ``curast_frame_t`` (field order and types must match)."""

    _fields_ = [
        ("pos_format", _I32), ("idx_format", _I32),
        ("positions", _P), ("indices", _P),
        ("n_items", _I64), ("prefix", _P), ("item_mv", _P), ("item_mw", _P),
        ("item_vtx_off", _P), ("item_idx_off", _P), ("item_filter", _P),
        ("item_qgrid", _P), ("item_pack", _P),
        ("instanced", _I32), ("use_filter", _I32),
        ("n_groups", _I64), ("group_prefix", _P), ("group_item_off", _P),
        ("group_item_count", _P), ("group_items", _P),
        ("n_units", _I64), ("unit_index", _P), ("unit_lo", _P), ("unit_hi", _P),
        ("unit_chunk_prefix", _P), ("chunk_tris", _I64), ("flat_chunks", _I64),
        ("n_inst_units", _I64), ("inst_unit_index", _P), ("inst_unit_lo", _P),
        ("inst_unit_hi", _P), ("inst_unit_chunk_prefix", _P), ("inst_chunk_tris", _I64),
        ("p0", _D), ("p1", _D), ("near", _D), ("width", _I64), ("height", _I64),
        ("rot_t", _D * 9), ("cam", _D * 3), ("view_r2", _D * 3), ("view_t2", _D),
        ("tiny_cull", _I32), ("force_stage", _I32), ("s1_row_raster", _I32), ("reserved0", _I32),
        ("small_max", _I64), ("medium_max", _I64), ("tile_px", _I64),
        ("fb", _P), ("q2", _P), ("q2_cap", _I64), ("q3", _P), ("q3_cap", _I64),
        ("qx", _P), ("qx_cap", _I64), ("counters", _P),
    ]


class CurastDebug(ctypes.Structure):
    """Mirror of ``curast_debug_t``."""

    _fields_ = [
        ("fb", _P), ("width", _I64), ("height", _I64), ("mode", _I32),
        ("pos_format", _I32), ("idx_format", _I32), ("n_items", _I64), ("prefix", _P),
        ("item_vtx_off", _P), ("item_idx_off", _P), ("positions", _P), ("indices", _P),
        ("item_qgrid", _P), ("item_pack", _P), ("item_xform", _P), ("view", _D * 16),
        ("p0", _D), ("p1", _D), ("near", _D), ("small_max", _I64), ("medium_max", _I64),
        ("background", ctypes.c_uint8 * 4), ("out_rgba", _P), ("scratch", _P),
    ]


class CurastResolve(ctypes.Structure):
    """Mirror of ``curast_resolve_t``."""

    _fields_ = [
        ("fb", _P), ("width", _I64), ("height", _I64), ("n_items", _I64),
        ("prefix", _P), ("item_mw", _P), ("item_vtx_off", _P), ("item_idx_off", _P),
        ("pos_format", _I32), ("idx_format", _I32), ("positions", _P), ("indices", _P),
        ("item_qgrid", _P), ("item_pack", _P),
        ("item_mode", _P), ("item_color_off", _P), ("colors", _P), ("uvs", _P),
        ("item_tex", _P), ("tex_desc", _P), ("level_desc", _P), ("texels", _P),
        ("trilinear", _I32), ("headlight", _I32),
        ("background", ctypes.c_uint8 * 4), ("base_color", ctypes.c_uint8 * 4),
        ("p0", _D), ("p1", _D), ("cam", _D * 3), ("rot", _D * 9),
        ("out_rgba", _P), ("counters", _P), ("row0", _I64), ("rows", _I64),
    ]


class NativeError(RuntimeError):
    pass


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeError(
            f"{LIB_PATH} is missing: the CUDA extension has not been built "
            "(run __graft_entry__.build()); there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    L.curast_abi_version.restype = _I32
    L.curast_last_error.restype = ctypes.c_char_p
    L.curast_chunk_tris.restype = _I64
    L.curast_chunk_tris.argtypes = [_I32]
    L.curast_chunk_quantum.restype = _I64
    L.curast_chunk_quantum.argtypes = []
    for name in ("curast_frame_clear", "curast_stage1", "curast_stage2",
                 "curast_stage3", "curast_render"):
        fn = getattr(L, name)
        fn.restype = _I32
        fn.argtypes = [ctypes.POINTER(CurastFrame), _P]
    L.curast_filter_check.restype = _I32
    L.curast_filter_check.argtypes = [ctypes.POINTER(CurastFrame), _P, _P]
    L.curast_div_check.restype = _I32
    L.curast_div_check.argtypes = [_I64, ctypes.c_uint64, _I32, _P, _P]
    L.curast_fill_u64.restype = _I32
    L.curast_fill_u64.argtypes = [_P, _I64, ctypes.c_uint64, _P]
    L.curast_min_u64.restype = _I32
    L.curast_min_u64.argtypes = [_P, _P, _I64, _P]
    L.curast_resolve.restype = _I32
    L.curast_resolve.argtypes = [ctypes.POINTER(CurastResolve), _P]
    L.curast_debug_view.restype = _I32
    L.curast_debug_view.argtypes = [ctypes.POINTER(CurastDebug), _P]
    L.curast_downsample.restype = _I32
    L.curast_downsample.argtypes = [_P, _I64, _I64, _I32, _P, _P]
    if L.curast_abi_version() != ABI_VERSION:
        raise NativeError("libcurast_b200.so ABI version mismatch; rebuild it")
    _lib = L
    return L


EXPORTED_SYMBOLS = (
    "curast_abi_version", "curast_last_error", "curast_chunk_tris", "curast_chunk_quantum",
    "curast_frame_clear", "curast_stage1", "curast_stage2", "curast_stage3",
    "curast_render", "curast_fill_u64", "curast_min_u64", "curast_filter_check",
    "curast_div_check",
    "curast_resolve", "curast_downsample", "curast_debug_view",
)


def check(rc: int, what: str):
    if rc != 0:
        msg = lib().curast_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed ({rc}): {msg}")
