"""ORACLE HOST SIDE — TEST INFRASTRUCTURE ONLY.

Restates, in numpy, the reference's host frame setup and drives the C
restatement of its kernels (``oracle.c``).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline legs may import
this module; the product package never does.

Host setup must be bit-identical to the reference on the same machine, so the
numpy expressions below are the reference's own ones (same operands, same
``@`` products, same order):

* ``projection_vector``  — trirast/scenecore.py:119-127
* ``frustum_planes``     — trirast/scenecore.py:201-222
* ``_transformed_aabb``  — trirast/scenecore.py:225-230
* ``aabb_outside_plane`` — trirast/scenecore.py:233-237
* ``build_draw_list``    — trirast/scenecore.py:240-265
* ``build_context``      — trirast/pipeline.py:87-148
* ``render_reference``   — trirast/refraster.py:34-89 (sequential, unbounded)
* ``render_pipeline``    — trirast/pipeline.py:207-365 (threaded claim loop)
"""

from __future__ import annotations

import ctypes
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
CLEAR = np.uint64(0xFFFFFFFFFFFFFFFF)
MAX_TRIANGLE_ID = 1 << 36
_UNBOUNDED = 1 << 40

# ---------------------------------------------------------------------------
# C library

_lib = None


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        _lib = ctypes.CDLL(path)
        _declare(_lib)
    return _lib


def build():
    import subprocess
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_D = ctypes.c_double
_I32 = ctypes.c_int32


class OracleFrame(ctypes.Structure):
    _fields_ = [
        ("n_items", _I64), ("prefix", _P), ("item_mv", _P), ("item_mw", _P),
        ("item_vtx_off", _P), ("item_idx_off", _P), ("positions", _P), ("indices", _P),
        ("instanced", _I32), ("n_groups", _I64), ("group_prefix", _P),
        ("group_item_off", _P), ("group_item_count", _P), ("group_items", _P),
        ("p0", _D), ("p1", _D), ("near", _D), ("width", _I64), ("height", _I64),
        ("rot_t", _P), ("cam", _P), ("view_r2", _P), ("view_t2", _D),
        ("tiny_cull", _I32), ("force_stage", _I64), ("small_max", _I64),
        ("medium_max", _I64), ("tile_px", _I64), ("batch", _I64),
        ("s2_cap", _I64), ("s3_cap", _I64),
        ("work_begin", _I64), ("work_end", _I64),
    ]


def _declare(L):
    L.oracle_stage1_range.restype = _I64
    L.oracle_stage1_range.argtypes = [
        _I64, _I64, _P, _I64, _P, _P, _P, _P, _P, _D, _D, _I64, _I64, _D, _I32,
        _I64, _I64, _P, _P, _P, _I64, _I64, _P]
    L.oracle_stage1_instanced_range.restype = _I64
    L.oracle_stage1_instanced_range.argtypes = [
        _I64, _I64, _P, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _D, _D, _I64,
        _I64, _D, _I32, _I64, _I64, _P, _P, _P, _I64, _I64, _P]
    L.oracle_stage2_range.restype = _I64
    L.oracle_stage2_range.argtypes = [
        _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _D, _D, _I64, _I64, _D,
        _I64, _I64, _I64, _P, _P, _P, _P, _P, _I64, _I64, _P]
    L.oracle_stage3_range.restype = _I64
    L.oracle_stage3_range.argtypes = [
        _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _D,
        _D, _D, _I64, _I64, _D, _I64, _P, _P]
    L.oracle_clip_near.restype = _I32
    L.oracle_clip_near.argtypes = [_D] * 10 + [_P, _P, _P]
    L.oracle_render.restype = _I32
    L.oracle_render.argtypes = [ctypes.POINTER(OracleFrame), _I32, _P, _P, _P, _P]
    L.oracle_min_u64.restype = None
    L.oracle_min_u64.argtypes = [_P, _P, _I64]


def _ptr(a):
    return None if a is None else a.ctypes.data


# ---------------------------------------------------------------------------
# host setup (numpy, reference expressions)

def projection_vector(camera) -> np.ndarray:
    f = 1.0 / math.tan(camera.fovy / 2.0)
    return np.array([f / camera.aspect, f, -1.0], dtype=np.float64)


def frustum_planes(camera) -> np.ndarray:
    p = projection_vector(camera)
    view_planes = np.array([
        [0.0, 0.0, 1.0, camera.near],
        [p[0], 0.0, 1.0, 0.0],
        [-p[0], 0.0, 1.0, 0.0],
        [0.0, p[1], 1.0, 0.0],
        [0.0, -p[1], 1.0, 0.0],
    ])
    rot = camera.view_transform[:3, :3]
    trans = camera.view_transform[:3, 3]
    world = np.empty_like(view_planes)
    world[:, :3] = view_planes[:, :3] @ rot
    world[:, 3] = view_planes[:, :3] @ trans + view_planes[:, 3]
    return world


def _transformed_aabb(aabb, transform):
    corners = np.array([[aabb[i, 0], aabb[j, 1], aabb[k, 2], 1.0]
                        for i in (0, 1) for j in (0, 1) for k in (0, 1)])
    world = corners @ transform.T
    pts = world[:, :3]
    return np.stack([pts.min(axis=0), pts.max(axis=0)])


def _outside(aabb, plane) -> bool:
    corner = np.where(plane[:3] < 0.0, aabb[1], aabb[0])
    return float(plane[:3] @ corner + plane[3]) > 0.0


@dataclass
class OItem:
    mesh: object
    transform: np.ndarray
    first: int
    count: int
    node_index: int


@dataclass
class ODrawList:
    items: list
    prefix: np.ndarray      # uint64
    total: int


def build_draw_list(scene, camera) -> ODrawList:
    if not scene:
        raise ValueError("scene must not be empty")
    planes = frustum_planes(camera)
    items = []
    total = 0
    for node_index, node in enumerate(scene):
        for transform in node.transforms:
            transform = np.asarray(transform, dtype=np.float64)
            box = _transformed_aabb(np.asarray(node.mesh.aabb, dtype=np.float64), transform)
            if any(_outside(box, pl) for pl in planes):
                continue
            items.append(OItem(node.mesh, transform, total, node.mesh.triangle_count,
                               node_index))
            total += node.mesh.triangle_count
    if total >= MAX_TRIANGLE_ID:
        raise OverflowError("36-bit triangle ID space exceeded")
    prefix = np.zeros(len(items) + 1, dtype=np.uint64)
    for k, it in enumerate(items):
        prefix[k + 1] = prefix[k] + np.uint64(it.count)
    return ODrawList(items, prefix, total)


def mesh_positions_f64(mesh) -> np.ndarray:
    """Decoded positions (geomcodec.py:99-101 for quantized storage)."""
    pos = mesh.positions
    if isinstance(pos, np.ndarray):
        return np.ascontiguousarray(pos, dtype=np.float64)
    q = pos.coords.astype(np.float64)
    return np.ascontiguousarray(pos.grid_min + (q + 0.5) / 65536.0 * pos.grid_size)


def mesh_indices_u32(mesh) -> np.ndarray:
    """Decoded indices (geomcodec.py:56-62 for bit-packed storage)."""
    idx = mesh.indices
    if isinstance(idx, np.ndarray):
        return np.ascontiguousarray(idx, dtype=np.uint32)
    b = idx.bits_per_index
    bits = np.unpackbits(idx.data, count=idx.count * b, bitorder="little")
    bits = bits.reshape(idx.count, b).astype(np.uint64)
    weights = np.uint64(1) << np.arange(b, dtype=np.uint64)
    rel = (bits * weights).sum(axis=1, dtype=np.uint64)
    return (rel + np.uint64(idx.min_index)).astype(np.uint32)


@dataclass
class OContext:
    prefix: np.ndarray
    item_mv: np.ndarray
    item_mw: np.ndarray
    item_vtx_off: np.ndarray
    item_idx_off: np.ndarray
    positions: np.ndarray
    indices: np.ndarray
    group_prefix: np.ndarray
    group_item_off: np.ndarray
    group_item_count: np.ndarray
    group_items: np.ndarray
    max_instances: int
    keep: list = field(default_factory=list)


def build_context(dl: ODrawList, camera) -> OContext:
    items = dl.items
    n = len(items)
    view = np.asarray(camera.view_transform, dtype=np.float64)
    item_mv = np.empty((n, 3, 4))
    item_mw = np.empty((n, 3, 4))
    vtx_off = np.empty(n, dtype=np.int64)
    idx_off = np.empty(n, dtype=np.int64)
    seen = {}
    pos_chunks, idx_chunks = [], []
    nv = ni = 0
    for k, it in enumerate(items):
        item_mw[k] = it.transform[:3]
        item_mv[k] = (view @ it.transform)[:3]
        key = id(it.mesh)
        if key not in seen:
            pos = mesh_positions_f64(it.mesh)
            idx = mesh_indices_u32(it.mesh)
            seen[key] = (nv, ni)
            pos_chunks.append(pos)
            idx_chunks.append(idx)
            nv += len(pos)
            ni += len(idx)
        vtx_off[k], idx_off[k] = seen[key]
    counts, tris, flat = [], [], []
    k = 0
    max_inst = 1
    while k < n:
        node = items[k].node_index
        j = k
        while j < n and items[j].node_index == node:
            flat.append(j)
            j += 1
        counts.append(j - k)
        tris.append(items[k].count)
        max_inst = max(max_inst, j - k)
        k = j
    gp = np.zeros(len(counts) + 1, dtype=np.int64)
    np.cumsum(np.asarray(tris, dtype=np.int64), out=gp[1:])
    gcount = np.array(counts, dtype=np.int64)
    goff = np.zeros(len(counts), dtype=np.int64)
    if len(counts) > 1:
        np.cumsum(gcount[:-1], out=goff[1:])
    positions = (np.ascontiguousarray(np.concatenate(pos_chunks)) if pos_chunks
                 else np.zeros((0, 3)))
    indices = (np.ascontiguousarray(np.concatenate(idx_chunks)) if idx_chunks
               else np.zeros(0, dtype=np.uint32))
    return OContext(dl.prefix.astype(np.int64), item_mv, item_mw, vtx_off, idx_off,
                    positions, indices, gp, goff, gcount,
                    np.array(flat, dtype=np.int64), max_inst)


def camera_constants(camera):
    """Stage-3 constants (pipeline.py:339-343) and projection scalars."""
    p = projection_vector(camera)
    view = np.asarray(camera.view_transform, dtype=np.float64)
    return dict(
        p0=float(p[0]), p1=float(p[1]), near=float(camera.near),
        width=int(camera.internal_width), height=int(camera.internal_height),
        rot_t=np.ascontiguousarray(view[:3, :3].T),
        cam=np.ascontiguousarray(np.asarray(camera.position, dtype=np.float64)),
        view_r2=np.ascontiguousarray(view[2, :3]),
        view_t2=float(view[2, 3]))


# ---------------------------------------------------------------------------
# drivers

STAT_KEYS = ("rasterized", "forwarded", "culled_frustum", "culled_offscreen",
             "culled_tiny", "culled_backface", "culled_degenerate", "fragments")
S2_KEYS = ("direct", "tiled", "dropped", "fragments", "tiles")


def _stats_dict(raw):
    return {
        "stage1": {k: int(raw[i]) for i, k in enumerate(STAT_KEYS)},
        "stage2": {k: int(raw[8 + i]) for i, k in enumerate(S2_KEYS)},
        "stage3": {"entries": int(raw[13]), "fragments": int(raw[14])},
    }


def render_context(ctx: OContext, cc: dict, *, tiny_cull=True, force_stage=0,
                   small_max=128, medium_max=4096, tile_px=64, instanced=False,
                   workers=1, batch=256, s2_cap=None, s3_cap=None,
                   work_range=None):
    """Run the threaded C pipeline on a prebuilt context.

    Returns (words, stats, rc, needed, seconds).  rc 0 = ok, 2/3 = stage-2/3
    capacity overflow with ``needed`` the required size."""
    L = lib()
    total = int(ctx.prefix[-1])
    width, height = cc["width"], cc["height"]
    words = np.full(width * height, CLEAR, dtype=np.uint64)
    # the reference's render_reference queues are unbounded (refraster.py:
    # 51-70); here they are bounded so that per-worker allocations stay sane,
    # and an overflow is reported (rc 2/3), never silently truncated
    if s2_cap is None:
        s2_cap = max(1, min(total, 1 << 22))
    if s3_cap is None:
        tiles = (-(-width // tile_px)) * (-(-height // tile_px))
        s3_cap = max(1, min(s2_cap * tiles, 1 << 22))
    if work_range is None:
        work_range = (0, int(ctx.group_prefix[-1]) if instanced else total)
    f = OracleFrame()
    f.n_items = len(ctx.prefix) - 1
    f.prefix = _ptr(ctx.prefix)
    f.item_mv = _ptr(np.ascontiguousarray(ctx.item_mv))
    f.item_mw = _ptr(np.ascontiguousarray(ctx.item_mw))
    f.item_vtx_off = _ptr(ctx.item_vtx_off)
    f.item_idx_off = _ptr(ctx.item_idx_off)
    f.positions = _ptr(ctx.positions)
    f.indices = _ptr(ctx.indices)
    f.instanced = int(bool(instanced))
    f.n_groups = len(ctx.group_prefix) - 1
    f.group_prefix = _ptr(ctx.group_prefix)
    f.group_item_off = _ptr(ctx.group_item_off)
    f.group_item_count = _ptr(ctx.group_item_count)
    f.group_items = _ptr(ctx.group_items)
    f.p0, f.p1, f.near = cc["p0"], cc["p1"], cc["near"]
    f.width, f.height = width, height
    f.rot_t = _ptr(cc["rot_t"])
    f.cam = _ptr(cc["cam"])
    f.view_r2 = _ptr(cc["view_r2"])
    f.view_t2 = cc["view_t2"]
    f.tiny_cull = int(bool(tiny_cull))
    f.force_stage = int(force_stage)
    f.small_max = int(small_max)
    f.medium_max = int(medium_max)
    f.tile_px = int(tile_px)
    f.batch = int(batch)
    f.s2_cap = int(s2_cap)
    f.s3_cap = int(s3_cap)
    f.work_begin, f.work_end = int(work_range[0]), int(work_range[1])
    raw = np.zeros(16, dtype=np.int64)
    needed = np.zeros(1, dtype=np.int64)
    t0 = time.perf_counter()
    rc = L.oracle_render(ctypes.byref(f), int(workers), _ptr(words), _ptr(raw),
                         _ptr(needed), None)
    dt = time.perf_counter() - t0
    return words, _stats_dict(raw), int(rc), int(needed[0]), dt


def render_reference(scene, camera, *, honor_stages=True, instancing="off",
                     workers=1, **cfg):
    """Sequential oracle (refraster.py:34-89): unbounded queues.  With
    ``workers > 1`` runs the threaded pipeline instead (same words)."""
    dl = build_draw_list(scene, camera)
    cc = camera_constants(camera)
    if dl.total == 0:
        return (np.full(cc["width"] * cc["height"], CLEAR, dtype=np.uint64),
                None, dl)
    ctx = build_context(dl, camera)
    if not honor_stages:
        cfg["small_max"] = _UNBOUNDED
        cfg["medium_max"] = _UNBOUNDED
    instanced = instancing == "on" or (instancing == "auto" and ctx.max_instances >= 2)
    words, stats, rc, needed, _ = render_context(ctx, cc, instanced=instanced,
                                                 workers=workers, **cfg)
    if rc:
        raise RuntimeError(f"oracle capacity overflow in stage {rc}: {needed}")
    return words, stats, dl


def min_u64(out: np.ndarray, other: np.ndarray):
    lib().oracle_min_u64(_ptr(out), _ptr(np.ascontiguousarray(other)), out.size)
