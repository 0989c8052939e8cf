"""Drop-in ``render_frame`` / ``render_draw_list`` on the B200.

Same signatures, argument meaning, return types and errors as the
reference's ``trirast/pipeline.py:207-372``; the three stages run as sm_100a
kernels (libcurast_b200.so) on one CUDA stream with no host synchronisation
until the frame's counters are read back:

    clear VB -> stage 1 (+ fp64 fallback) -> stage 2 -> stage 3

Capacity contract (pipeline.py:281-285, 323-327): queues keep counting past
capacity and the host raises ``CapacityError`` with the required size.  The
reference's default capacities (config.py:32-42) are far larger than what is
worth allocating up front (64 x T stage-3 entries), so the device starts from
``DEVICE_Q*_INITIAL`` entries and, when a frame needs more but still fits the
capacity the reference would resolve, grows the queue and re-runs the frame
(the output is identical: the fragment multiset is the same).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .config import (DEVICE_Q2_INITIAL, DEVICE_Q3_INITIAL, DEVICE_QX_INITIAL, FrameStats, RasterConfig,
                     Stage1Stats, Stage2Stats, Stage3Stats)
from .device import PackedUpload, filter_rows, scene_geometry, workspace
from .scene import (CLEAR, CapacityError, DrawList, Framebuffer, build_draw_list,
                    projection_vector)

# resident stage-1 warps (<= 160 SMs x 32) x one reservation block each
QX_HOLE_SLACK = 160 * 32 * N.QX_RES

INST_BLOCK = N.INST_BLOCK

# CURAST_FILTER=0 disables the fp32 cull filter (every triangle fp64) — a
# debugging/verification switch, not a fallback.
_FILTER_DEFAULT = os.environ.get("CURAST_FILTER", "1") != "0"


@dataclass
class RenderContext:
    """Host-side flattened per-item arrays (pipeline.py:68-84)."""

    prefix: np.ndarray
    item_mv: np.ndarray
    item_mw: np.ndarray
    item_vtx_off: np.ndarray
    item_idx_off: np.ndarray
    meshes: list
    item_mesh: np.ndarray
    group_prefix: np.ndarray
    group_item_off: np.ndarray
    group_item_count: np.ndarray
    group_items: np.ndarray
    max_instances: int


def build_context(draw_list: DrawList, camera) -> RenderContext:
    """Per-item matrices with the reference's numpy expressions
    (pipeline.py:96-102) and the instancing groups (pipeline.py:114-135).
    Geometry is not concatenated on the host: meshes are uploaded once and
    concatenated on the device (device.SceneGeometry)."""
    items = draw_list.items
    n = len(items)
    view = camera.view_transform
    item_mv = np.empty((n, 3, 4))
    item_mw = np.empty((n, 3, 4))
    mesh_ids: dict = {}
    meshes = []
    item_mesh = np.empty(n, dtype=np.int64)
    for k, it in enumerate(items):
        item_mw[k] = it.instance_transform[:3]
        item_mv[k] = (view @ it.instance_transform)[:3]
        key = id(it.mesh)
        if key not in mesh_ids:
            mesh_ids[key] = len(meshes)
            meshes.append(it.mesh)
        item_mesh[k] = mesh_ids[key]
    counts, tris, flat = [], [], []
    k = 0
    max_inst = 1
    while k < n:
        node = items[k].node_index
        j = k
        while j < n and items[j].node_index == node:
            j += 1
        flat.extend(range(k, j))
        counts.append(j - k)
        tris.append(items[k].triangle_count)
        max_inst = max(max_inst, j - k)
        k = j
    gp = np.zeros(len(counts) + 1, dtype=np.int64)
    if counts:
        np.cumsum(np.asarray(tris, dtype=np.int64), out=gp[1:])
    gcount = np.asarray(counts, dtype=np.int64)
    goff = np.zeros(len(counts), dtype=np.int64)
    if len(counts) > 1:
        np.cumsum(gcount[:-1], out=goff[1:])
    return RenderContext(
        prefix=draw_list.prefix_sums.astype(np.int64), item_mv=item_mv, item_mw=item_mw,
        item_vtx_off=np.zeros(n, dtype=np.int64), item_idx_off=np.zeros(n, dtype=np.int64),
        meshes=meshes, item_mesh=item_mesh, group_prefix=gp, group_item_off=goff,
        group_item_count=gcount, group_items=np.asarray(flat, dtype=np.int64),
        max_instances=max_inst)


def adopt_context(ctx, draw_list: DrawList, camera) -> RenderContext:
    """Accept the reference's ``trirast.pipeline.RenderContext``
    (pipeline.py:68-84: flattened f64 ``positions`` / u32 ``indices`` with
    per-item ``item_vtx_off`` / ``item_idx_off``, ``prefix``, ``item_mv`` /
    ``item_mw``) as the ``ctx`` of ``render_draw_list``: its concatenated
    geometry becomes one device mesh addressed through the item offsets, and
    its matrices and prefix are used as given.  The instancing groups are
    rebuilt from the draw list (the reference builds them the same way,
    pipeline.py:114-135).  The flat mesh is cached on the context object."""
    if isinstance(ctx, RenderContext):
        return ctx
    for name in ("positions", "indices", "item_vtx_off", "item_idx_off", "item_mv", "prefix"):
        if not hasattr(ctx, name):
            raise TypeError(f"ctx has no '{name}': not a RenderContext of this package "
                            "or of the reference (trirast.pipeline.RenderContext)")
    own = build_context(draw_list, camera)
    cached = getattr(ctx, "_curast_flat_mesh", None)
    if cached is not None and cached[0] is ctx.positions and cached[1] is ctx.indices:
        flat = cached[2]
    else:
        from .scene import Mesh
        pos = np.ascontiguousarray(ctx.positions, dtype=np.float64).reshape(-1, 3)
        idx = np.ascontiguousarray(ctx.indices, dtype=np.uint32).ravel()
        aabb = (np.stack([pos.min(axis=0), pos.max(axis=0)]) if len(pos)
                else np.zeros((2, 3)))
        flat = Mesh(positions=pos, indices=idx, triangle_count=len(idx) // 3, aabb=aabb,
                    name="reference_context")
        try:
            object.__setattr__(ctx, "_curast_flat_mesh", (ctx.positions, ctx.indices, flat))
        except (AttributeError, TypeError):
            pass
    n = len(draw_list.items)
    own.meshes = [flat]
    own.item_mesh = np.zeros(n, dtype=np.int64)
    own.item_vtx_off = np.asarray(ctx.item_vtx_off, dtype=np.int64).reshape(n)
    own.item_idx_off = np.asarray(ctx.item_idx_off, dtype=np.int64).reshape(n)
    own.item_mv = np.ascontiguousarray(ctx.item_mv, dtype=np.float64).reshape(n, 3, 4)
    mw = getattr(ctx, "item_mw", None)
    if mw is not None:
        own.item_mw = np.ascontiguousarray(mw, dtype=np.float64).reshape(n, 3, 4)
    own.prefix = np.asarray(ctx.prefix, dtype=np.int64)
    return own


def work_space(draw_list: DrawList, cfg: RasterConfig) -> int:
    """Size of a frame's stage-1 work space: the unique triangles of the
    instancing groups for an instanced frame (pipeline.py:244), else the
    global triangle IDs.  Shards are ranges of this space."""
    n = len(draw_list.items)
    inst = cfg.instancing == "on"
    if cfg.instancing == "auto" and n >= 2:
        nodes = [it.node_index for it in draw_list.items]
        inst = any(a == b for a, b in zip(nodes, nodes[1:]))   # a node with >= 2 instances
    if not inst:
        return int(draw_list.total_triangles)
    tot, prev = 0, None
    for it in draw_list.items:
        if it.node_index != prev:
            tot += int(it.triangle_count)
            prev = it.node_index
    return tot


def shard_items(ctx: RenderContext, work_range, inst_kernel: bool) -> np.ndarray:
    """Boolean mask of the draw items a work range touches: the items whose
    global-ID range intersects it (flat work space), or every item of the
    instancing groups whose unique-triangle range intersects it (instanced
    work space, pipeline.py:244).  A sort-last rank uploads only these items'
    meshes (each GPU holds only its shard's geometry)."""
    lo, hi = int(work_range[0]), int(work_range[1])
    n = len(ctx.item_mesh)
    if not inst_kernel:
        s = ctx.prefix[:-1]
        e = ctx.prefix[1:]
        return (e > lo) & (s < hi) & (e > s)
    gs = ctx.group_prefix[:-1]
    ge = ctx.group_prefix[1:]
    gsel = (ge > lo) & (gs < hi) & (ge > gs)
    mask = np.zeros(n, dtype=bool)
    for g in np.nonzero(gsel)[0]:
        o = int(ctx.group_item_off[g])
        mask[ctx.group_items[o:o + int(ctx.group_item_count[g])]] = True
    return mask


def _span(starts: np.ndarray, counts: np.ndarray, begin: int, end: int) -> np.ndarray:
    """Triangles of each unit inside [begin, end) of the work space."""
    return np.maximum(np.minimum(starts + counts, end) - np.maximum(starts, begin), 0)


# work chunks per resident warp the chunk size aims for (load balance of the
# persistent stage-1 kernels: 148 SMs x 32 warps)
CHUNKS_PER_WARP = 4


def _target_chunks(device) -> int:
    try:
        sms = torch.cuda.get_device_properties(device).multi_processor_count
    except Exception:
        sms = 148
    return CHUNKS_PER_WARP * 32 * sms


def _choose_chunk(work: int, chunk_max: int, quantum: int, target: int) -> int:
    """Largest power-of-two multiple of ``quantum`` up to ``chunk_max`` that
    still splits ``work`` triangles into ``target`` chunks (streamed frames
    keep 2048-triangle chunks; small frames get more, smaller ones so every
    SM has work)."""
    c = chunk_max
    while c > quantum and work < target * c:
        c //= 2
    return max(quantum, c)


def _work_table(starts: np.ndarray, counts: np.ndarray, unit_ids: np.ndarray,
                begin: int, end: int, chunk: int):
    """Units (items or groups) intersected with [begin, end) of their global
    space, split into chunks of ``chunk`` triangles."""
    s = starts
    e = starts + counts
    lo = np.maximum(s, begin)
    hi = np.minimum(e, end)
    keep = hi > lo
    lo_l = (lo - s)[keep]
    hi_l = (hi - s)[keep]
    ids = unit_ids[keep]
    nch = (hi_l - lo_l + chunk - 1) // chunk
    cp = np.zeros(len(ids) + 1, dtype=np.int64)
    np.cumsum(nch, out=cp[1:])
    return ids.astype(np.int64), lo_l.astype(np.int64), hi_l.astype(np.int64), cp


def _instanced_kernel_preferred(geo) -> bool:
    """Instanced frames run the instanced stage-1 kernels (a unique
    triangle's vertices fetched once per block of 16 instances) unless
    CURAST_INSTANCED_KERNEL=0 selects the flat table over the items (same
    words and counters: instancing == flat, test_rasterpipe.py:186-203).
    Measured on config D (1M-triangle sphere x 998 instances): instanced
    3.69 ms vs flat 4.05 ms stage 1 (profiles/r02_configs.jsonl)."""
    return os.environ.get("CURAST_INSTANCED_KERNEL", "1") != "0"


class PreparedFrame:
    """A frame whose descriptors are resident on the device; ``launch()``
    enqueues clear + stages 1-3 without synchronising (CUDA-graph capturable
    once the queues are large enough)."""

    def __init__(self, draw_list: DrawList, camera, cfg: RasterConfig,
                 ctx: RenderContext | None = None, *, device=None,
                 work_range=None, use_filter=None, fresh_fb=True):
        _lib = N.lib()
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = device
        self.cfg = cfg
        self.camera = camera
        self.draw_list = draw_list
        self.width = camera.internal_width
        self.height = camera.internal_height
        self.total = int(draw_list.total_triangles)
        self.n_items = len(draw_list.items)
        if ctx is None:
            ctx = build_context(draw_list, camera)
        ctx = adopt_context(ctx, draw_list, camera)
        self.ctx = ctx
        self.instanced = (cfg.instancing == "on"
                          or (cfg.instancing == "auto" and ctx.max_instances >= 2))
        if use_filter is None:
            use_filter = _FILTER_DEFAULT
        self.use_filter = bool(use_filter) and cfg.force_stage < 2
        n = self.n_items
        # geometry: every mesh of the draw list for a full frame; only the
        # meshes of the items the work range touches for a shard
        if work_range is None:
            need = np.ones(n, dtype=bool)
        else:
            inst_space = self.instanced
            need = shard_items(ctx, work_range, inst_space)
        used = np.unique(ctx.item_mesh[need]) if n else np.zeros(0, np.int64)
        self.mesh_ids = used
        slot = {int(m): k for k, m in enumerate(used)}
        self.geo = scene_geometry([ctx.meshes[int(m)] for m in used], device)
        geo = self.geo
        self.s2_cap = cfg.resolved_stage2_capacity(self.total)
        self.s3_cap = cfg.resolved_stage3_capacity(self.total)
        ws = workspace(device)
        self.ws = ws
        self.fb = ws.framebuffer(self.width * self.height, fresh_fb)

        gslot = [slot.get(int(m), -1) if need[k] else -1 for k, m in enumerate(ctx.item_mesh)]
        vtx_off = np.asarray([geo.vtx_off[g] if g >= 0 else 0 for g in gslot], dtype=np.int64)
        vtx_off += ctx.item_vtx_off
        idx_off = np.asarray([geo.idx_off[g] if g >= 0 else 0 for g in gslot], dtype=np.int64)
        idx_off += ctx.item_idx_off
        p = projection_vector(camera)
        p0, p1 = float(p[0]), float(p[1])
        self.p0, self.p1 = p0, p1
        pos_bound = (np.stack([geo.meshes[g].pos_bound if g >= 0 else np.zeros(3)
                               for g in gslot]) if n else np.zeros((0, 3)))
        qgrid = (np.stack([geo.meshes[g].qgrid if g >= 0 else np.zeros(6) for g in gslot])
                 if n else np.zeros((0, 6)))
        pack = np.asarray([geo.meshes[g].pack if g >= 0 else (0, 32) for g in gslot],
                          dtype=np.int64).reshape(n, 2)
        filt = filter_rows(ctx.item_mv.reshape(n, 12), pos_bound, p0, p1, self.width,
                           self.height, float(camera.near), geo.pos_format)

        # Stage-1 kernel for instanced frames: the instanced one (a unique
        # triangle fetched once, tested under every instance) or, with
        # CURAST_INSTANCED_KERNEL=0, the flat one over the items (same words
        # and counters); sharded frames keep the instanced work space, whose
        # work ranges count unique triangles (pipeline.py:244).
        self.inst_kernel = self.instanced and (
            work_range is not None or _instanced_kernel_preferred(geo))
        if work_range is None:
            work_range = (0, int(ctx.group_prefix[-1]) if self.inst_kernel else self.total)
        self.work_range = (int(work_range[0]), int(work_range[1]))
        chunk_max = int(_lib.curast_chunk_tris(0))
        ichunk_max = int(_lib.curast_chunk_tris(1))
        quantum = int(_lib.curast_chunk_quantum())
        target = _target_chunks(device)
        lo_w, hi_w = self.work_range
        if self.inst_kernel:
            # work space = unique triangles of the node groups (pipeline.py:244);
            # single-instance groups stream through the flat kernel
            ng = len(ctx.group_item_count)
            starts = ctx.group_prefix[:-1]
            tris = np.diff(ctx.group_prefix)
            single = ctx.group_item_count == 1
            first_item = ctx.group_items[ctx.group_item_off] if ng else np.zeros(0, np.int64)
            # multi-instance groups: one unit per block of CURAST_INST_BLOCK
            # instances (unit id = group | first_instance << 32)
            multi = np.nonzero(~single)[0]
            nkb = -(-ctx.group_item_count[multi] // INST_BLOCK)
            rep_g = np.repeat(multi, nkb)
            kb = np.concatenate([np.arange(k) for k in nkb]) if len(nkb) else np.zeros(0, np.int64)
            ids = rep_g.astype(np.int64) | ((kb.astype(np.int64) * INST_BLOCK) << 32)
            ninst = np.minimum(ctx.group_item_count[rep_g] - kb * INST_BLOCK, INST_BLOCK)
            span_s = _span(starts[single], tris[single], lo_w, hi_w)
            span_m = _span(starts[rep_g], tris[rep_g], lo_w, hi_w)
            chunk = _choose_chunk(int(span_s.sum()), chunk_max, quantum, target)
            # an instanced unit costs its triangles x its instances
            ichunk = _choose_chunk(int((span_m * ninst).sum()) // INST_BLOCK, ichunk_max,
                                   quantum, target)
            u = _work_table(starts[single], tris[single], first_item[single],
                            *self.work_range, chunk)
            v = _work_table(starts[rep_g], tris[rep_g], ids, *self.work_range, ichunk)
        else:
            counts = np.diff(ctx.prefix)
            chunk = _choose_chunk(int(_span(ctx.prefix[:-1], counts, lo_w, hi_w).sum()),
                                  chunk_max, quantum, target)
            ichunk = ichunk_max
            u = _work_table(ctx.prefix[:-1], counts, np.arange(n), *self.work_range, chunk)
            v = (np.zeros(0, np.int64),) * 3 + (np.zeros(1, np.int64),)
        self.chunk, self.ichunk = chunk, ichunk
        self.unit_index, self.unit_lo, self.unit_hi, self.unit_cp = u
        self.iunit_index, self.iunit_lo, self.iunit_hi, self.iunit_cp = v

        up = PackedUpload()
        k_prefix = up.add(ctx.prefix)
        k_mv = up.add(ctx.item_mv.reshape(-1))
        k_mw = up.add(ctx.item_mw.reshape(-1))
        k_vo = up.add(vtx_off)
        k_io = up.add(idx_off)
        k_f = up.add(filt.reshape(-1))
        k_q = up.add(qgrid.reshape(-1).astype(np.float64))
        k_pk = up.add(pack.reshape(-1))
        k_gp = up.add(ctx.group_prefix)
        k_go = up.add(ctx.group_item_off)
        k_gc = up.add(ctx.group_item_count)
        k_gi = up.add(ctx.group_items)
        k_ui = up.add(self.unit_index)
        k_ul = up.add(self.unit_lo)
        k_uh = up.add(self.unit_hi)
        k_uc = up.add(self.unit_cp)
        k_vi = up.add(self.iunit_index)
        k_vl = up.add(self.iunit_lo)
        k_vh = up.add(self.iunit_hi)
        k_vc = up.add(self.iunit_cp)
        up.upload(device)
        self.upload = up
        self.h2d_bytes = up.nbytes

        f = N.CurastFrame()
        f.pos_format = geo.pos_format
        f.idx_format = geo.idx_format
        f.positions = geo.positions.data_ptr()
        f.indices = geo.indices.data_ptr()
        f.n_items = n
        f.prefix = up.ptr(k_prefix)
        f.item_mv = up.ptr(k_mv)
        f.item_mw = up.ptr(k_mw)
        f.item_vtx_off = up.ptr(k_vo)
        f.item_idx_off = up.ptr(k_io)
        f.item_filter = up.ptr(k_f)
        f.item_qgrid = up.ptr(k_q)
        f.item_pack = up.ptr(k_pk)
        f.instanced = int(self.inst_kernel)
        f.use_filter = int(self.use_filter)
        f.n_groups = len(ctx.group_item_count)
        f.group_prefix = up.ptr(k_gp)
        f.group_item_off = up.ptr(k_go)
        f.group_item_count = up.ptr(k_gc)
        f.group_items = up.ptr(k_gi)
        f.n_units = len(self.unit_index)
        f.unit_index = up.ptr(k_ui)
        f.unit_lo = up.ptr(k_ul)
        f.unit_hi = up.ptr(k_uh)
        f.unit_chunk_prefix = up.ptr(k_uc)
        f.chunk_tris = self.chunk
        f.flat_chunks = int(self.unit_cp[-1])
        f.n_inst_units = len(self.iunit_index)
        f.inst_unit_index = up.ptr(k_vi)
        f.inst_unit_lo = up.ptr(k_vl)
        f.inst_unit_hi = up.ptr(k_vh)
        f.inst_unit_chunk_prefix = up.ptr(k_vc)
        f.inst_chunk_tris = self.ichunk
        f.p0, f.p1, f.near = p0, p1, float(camera.near)
        f.width, f.height = self.width, self.height
        view = np.asarray(camera.view_transform, dtype=np.float64)
        rot_t = np.ascontiguousarray(view[:3, :3].T).reshape(-1)
        for i in range(9):
            f.rot_t[i] = float(rot_t[i])
        for i in range(3):
            f.cam[i] = float(np.asarray(camera.position, dtype=np.float64)[i])
            f.view_r2[i] = float(view[2, i])
        f.view_t2 = float(view[2, 3])
        f.tiny_cull = int(bool(cfg.tiny_cull))
        f.force_stage = int(cfg.force_stage)
        f.s1_row_raster = 0
        f.small_max = int(cfg.small_max_px)
        f.medium_max = int(cfg.medium_max_px)
        f.tile_px = int(cfg.tile_px)
        f.fb = self.fb.data_ptr()
        f.counters = ws.counters.data_ptr()
        self.frame = f
        if len(self.iunit_index):
            k0 = self.iunit_index >> 32
            gc = ctx.group_item_count[self.iunit_index & 0xFFFFFFFF]
            per_unit = np.minimum(gc - k0, INST_BLOCK)
        else:
            per_unit = np.zeros(0, np.int64)
        # entries <= triangles; per-warp reservations (CURAST_QX_RES) add
        # holes: < 1 step per block of >= 129 used slots, plus each warp's
        # final rest
        flat = int((self.unit_hi - self.unit_lo).sum())
        self.qx_need_max = int(2 * flat + ((self.iunit_hi - self.iunit_lo) * per_unit).sum()
                               + QX_HOLE_SLACK)
        self._size_queues(DEVICE_Q2_INITIAL, DEVICE_Q3_INITIAL)

    def _size_queues(self, want2: int, want3: int, wantx: int = 0):
        ws = self.ws
        ax = min(max(1, self.qx_need_max), max(wantx, min(DEVICE_QX_INITIAL, self.qx_need_max),
                                                ws.qx_alloc))
        ws.ensure_qx(ax)
        ws.ensure_q2(min(self.s2_cap, max(want2, ws.q2_alloc)))
        ws.ensure_q3(min(self.s3_cap, max(want3, ws.q3_alloc)))
        self._bind_queues()

    def _bind_queues(self):
        """Point the frame at the workspace's current queues.  The queues are
        shared per device and grow-only: another frame may have replaced them
        since this one was sized, so ``launch`` re-binds, and the frame keeps
        references to the tensors its pointers (and any captured graph) use
        so that memory is never handed back to the allocator under them."""
        ws = self.ws
        self._queues = (ws.qx, ws.q2, ws.q3)
        self.qx_alloc = ws.qx_alloc
        self.frame.qx = ws.qx.data_ptr()
        self.frame.qx_cap = self.qx_alloc
        self.q2_alloc = max(0, min(self.s2_cap, ws.q2_alloc))
        self.q3_alloc = max(0, min(self.s3_cap, ws.q3_alloc))
        self.frame.q2 = ws.q2.data_ptr()
        self.frame.q2_cap = self.q2_alloc
        self.frame.q3 = ws.q3.data_ptr()
        self.frame.q3_cap = self.q3_alloc

    def _queues_current(self) -> bool:
        ws = self.ws
        q = self._queues
        return q[0] is ws.qx and q[1] is ws.q2 and q[2] is ws.q3

    def refresh(self, new_framebuffer: bool = True):
        """Reuse this prepared frame for another call with the same inputs:
        re-upload the per-frame descriptors (one pinned H2D copy, as every
        frame does) and, for a caller that keeps the previous frame's words,
        bind a new visibility buffer.  The host-side setup (filter rows,
        work table, packing) is not redone."""
        up = self.upload
        up.dev.copy_(up.host, non_blocking=True)
        if new_framebuffer:
            self.fb = self.ws.framebuffer(self.width * self.height, True)
            self.frame.fb = self.fb.data_ptr()

    def launch(self, stream=None, events=None):
        """Enqueue clear + stages 1-3 on ``stream`` (default: torch's current)."""
        L = N.lib()
        st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        if not self._queues_current():
            ws = self.ws
            if ws.qx is None or ws.q2 is None or ws.q3 is None:
                self._size_queues(self.q2_alloc, self.q3_alloc, self.qx_alloc)
            else:
                self._bind_queues()
        fp = ctypes.byref(self.frame)
        if events:
            events[0].record()
        N.check(L.curast_frame_clear(fp, st), "frame_clear")
        if events:
            events[1].record()
        N.check(L.curast_stage1(fp, st), "stage1")
        if events:
            events[2].record()
        N.check(L.curast_stage2(fp, st), "stage2")
        if events:
            events[3].record()
        N.check(L.curast_stage3(fp, st), "stage3")
        if events:
            events[4].record()

    def capture(self):
        """Capture clear + stages 1-3 into a CUDA graph (torch.cuda.CUDAGraph)
        for repeated frames of the same draw list: one graph launch per frame
        instead of five kernel launches through ctypes.  Run the frame once
        first (``run()``) so the device queues are sized; replay with
        ``graph.replay()`` and read the counters as after ``launch``.  The
        graph keeps this frame's device pointers (the frame keeps those
        buffers alive): re-capture after a queue grew (``stale_graph``)."""
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            self.launch(stream=s)                 # warm the launch path outside capture
        torch.cuda.current_stream(self.device).wait_stream(s)
        torch.cuda.synchronize(self.device)
        with torch.cuda.graph(g):
            self.launch()
        self._graph_queues = self._queues
        return g

    @property
    def stale_graph(self) -> bool:
        """True when the queues moved since ``capture()`` (the graph still
        writes into this frame's previous, still-referenced buffers)."""
        return getattr(self, "_graph_queues", None) is not self._queues

    def _choose_row_raster(self, c) -> None:
        """Frames whose stage-1 triangles average at least one fragment
        (larger triangles: config C 1.3, A4) let the fp64 pass rasterize wide
        bboxes row-parallel (curast.h s1_row_raster); dense frames (B 0.5,
        D 0.3) keep the per-thread loop, which the extra per-entry check would
        slow by ~2%.  Same words and counters either way; applies from the
        next launch (re-capture a graph taken before)."""
        rast, frags = int(c[N.C_S1 + 0]), int(c[N.C_S1 + 7])
        self.frame.s1_row_raster = int(rast > 0 and frags >= rast)

    def read_counters(self) -> np.ndarray:
        ws = self.ws
        ws.counters_host.copy_(ws.counters, non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        return ws.counters_host.numpy().copy()

    def run(self, timed=True) -> tuple[np.ndarray, list]:
        """Run until the queues were large enough; returns (counters,
        per-stage seconds).  Raises CapacityError like the reference."""
        while True:
            events = [torch.cuda.Event(enable_timing=True) for _ in range(5)] if timed else None
            self.launch(events=events)
            c = self.read_counters()
            nx = int(c[N.C_QX])
            if nx > self.qx_alloc:
                # reserved slots vary a little run to run: leave headroom
                self._size_queues(self.q2_alloc, self.q3_alloc, nx + nx // 32 + QX_HOLE_SLACK // 4)
                continue
            n2, n3 = int(c[N.C_Q2]), int(c[N.C_Q3])
            if n2 > self.s2_cap:
                raise CapacityError(
                    f"stage-2 queue overflow: {n2} entries forwarded, "
                    f"capacity {self.s2_cap}; raise stage2_capacity to at least {n2}")
            if n2 > self.q2_alloc:
                self._size_queues(n2, self.q3_alloc, self.qx_alloc)
                continue
            if n3 > self.s3_cap:
                raise CapacityError(
                    f"stage-3 queue overflow: {n3} tile entries, capacity "
                    f"{self.s3_cap}; raise stage3_capacity to at least {n3}")
            if n3 > self.q3_alloc:
                self._size_queues(self.q2_alloc, n3, self.qx_alloc)
                continue
            secs = [0.0] * 4
            if timed:
                secs = [events[i].elapsed_time(events[i + 1]) * 1e-3 for i in range(4)]
            self._choose_row_raster(c)
            return c, secs

    def stats(self, c: np.ndarray, secs) -> FrameStats:
        s1 = c[N.C_S1:N.C_S1 + 8]
        s2 = c[N.C_S2:N.C_S2 + 5]
        st = FrameStats(total_triangles=self.total, items=self.n_items,
                        instanced=self.instanced)
        st.stage1 = Stage1Stats(rasterized=int(s1[0]), forwarded=int(s1[1]),
                                culled_frustum=int(s1[2]), culled_offscreen=int(s1[3]),
                                culled_tiny=int(s1[4]), culled_backface=int(s1[5]),
                                culled_degenerate=int(s1[6]), fragments=int(s1[7]))
        st.stage2 = Stage2Stats(direct=int(s2[0]), tiled=int(s2[1]), dropped=int(s2[2]),
                                tiles=int(s2[4]), fragments=int(s2[3]))
        st.stage3 = Stage3Stats(entries=int(c[N.C_Q3]), fragments=int(c[N.C_S3]))
        st.merge_s, st.stage1_s, st.stage2_s, st.stage3_s = secs
        st.exact_fallbacks = int(c[N.C_QX]) - int(c[N.C_QXHOLES]) + int(c[N.C_EXACT])
        return st


_FRAME_CACHE_MAX = 4
_frame_cache: dict = {}


def _camera_key(camera):
    return (np.asarray(camera.position, dtype=np.float64).tobytes(),
            np.asarray(camera.view_transform, dtype=np.float64).tobytes(),
            float(camera.fovy), float(camera.aspect), float(camera.near),
            int(camera.internal_width), int(camera.internal_height))


def _cfg_key(cfg):
    return (cfg.small_max_px, cfg.medium_max_px, cfg.tile_px, cfg.stage2_capacity,
            cfg.stage3_capacity, bool(cfg.tiny_cull), cfg.force_stage, cfg.instancing)


def _cached_frame(draw_list, camera, cfg, ctx, use_filter, work_range):
    """A PreparedFrame for these inputs, reused across calls.  Entries hold
    the draw list / context objects they were built from and match them by
    identity (plus the item count and triangle total); the camera and the
    config by value; the geometry by ``scene_geometry``'s identity check, so
    re-assigned mesh arrays rebuild the frame.  At most 4 frames are kept."""
    device = torch.device("cuda", torch.cuda.current_device())
    key = (id(draw_list), id(ctx), _camera_key(camera), _cfg_key(cfg), use_filter,
           None if work_range is None else (int(work_range[0]), int(work_range[1])), str(device))
    ent = _frame_cache.get(key)
    if ent is not None:
        pf = ent
        if (pf.draw_list is draw_list and (ctx is None or pf.ctx_arg is ctx)
                and len(draw_list.items) == pf.n_items
                and int(draw_list.total_triangles) == pf.total
                and pf.geo is scene_geometry([pf.ctx.meshes[int(m)] for m in pf.mesh_ids],
                                             device)):
            pf.refresh(new_framebuffer=True)
            return pf
        _frame_cache.pop(key, None)
    pf = PreparedFrame(draw_list, camera, cfg, ctx, device=device, use_filter=use_filter,
                       work_range=work_range)
    pf.ctx_arg = ctx
    if len(_frame_cache) >= _FRAME_CACHE_MAX:
        _frame_cache.pop(next(iter(_frame_cache)))
    _frame_cache[key] = pf
    return pf


def render_draw_list(draw_list: DrawList, camera, cfg: RasterConfig | None = None,
                     ctx: RenderContext | None = None, *, use_filter=None,
                     work_range=None) -> tuple[Framebuffer, FrameStats]:
    """Run the three stages over a prebuilt draw list (pipeline.py:207-365).

    ``ctx`` may be this package's RenderContext or the reference's
    (``trirast.pipeline.RenderContext``, see ``adopt_context``).  Repeated
    calls with the same draw list, camera and config reuse the prepared
    frame (descriptors re-uploaded, host setup skipped).  The returned
    Framebuffer keeps its words in HBM (``device_words``); ``.words``
    downloads them as the reference's host ``np.uint64`` array."""
    cfg = cfg or RasterConfig()
    width, height = camera.internal_width, camera.internal_height
    total = draw_list.total_triangles
    if total == 0:
        st = FrameStats(total_triangles=0, items=len(draw_list.items))
        return Framebuffer(width, height), st
    frame = _cached_frame(draw_list, camera, cfg, ctx, use_filter, work_range)
    c, secs = frame.run()
    return Framebuffer(width, height, device_words=frame.fb), frame.stats(c, secs)


def render_frame(scene, camera, cfg: RasterConfig | None = None
                 ) -> tuple[Framebuffer, FrameStats]:
    """Frustum-cull, assemble the draw list, run all three stages
    (pipeline.py:368-372)."""
    return render_draw_list(build_draw_list(scene, camera), camera, cfg)


# ---------------------------------------------------------------------------
# classification mirror (pipeline.py:379-418) — host debug helper

STAGE1 = 1
STAGE2_DIRECT = 2
STAGE3_TILED = 3


def clip_triangle_near_plane(view_verts, near: float) -> np.ndarray:
    """Sutherland-Hodgman against z = -near (kernels.py:257-281)."""
    v = np.asarray(view_verts, dtype=np.float64)
    out = []
    for i in range(3):
        j = (i + 1) % 3
        da = -v[i, 2] - near
        db = -v[j, 2] - near
        if da >= 0.0:
            out.append(v[i].copy())
        if (da >= 0.0) != (db >= 0.0):
            u = da / (da - db)
            out.append(v[i] + u * (v[j] - v[i]))
    return np.asarray(out, dtype=np.float64).reshape(-1, 3)


def classify_route(view_verts, camera, cfg: RasterConfig | None = None):
    cfg = cfg or RasterConfig()
    v = np.asarray(view_verts, dtype=np.float64)
    width, height = camera.internal_width, camera.internal_height
    p = projection_vector(camera)
    depths = -v[:, 2]
    if np.all(depths < camera.near):
        return None, 0
    near_cross = bool(np.any(depths < camera.near))
    poly = clip_triangle_near_plane(v, camera.near) if near_cross else v
    if len(poly) == 0:
        return None, 0
    d = np.maximum(-poly[:, 2], camera.near)
    px = (poly[:, 0] * p[0] / d + 1.0) * 0.5 * width
    py = (1.0 - poly[:, 1] * p[1] / d) * 0.5 * height
    ix0 = max(int(np.floor(px.min())), 0)
    ix1 = min(int(np.ceil(px.max())), width)
    iy0 = max(int(np.floor(py.min())), 0)
    iy1 = min(int(np.ceil(py.max())), height)
    if ix0 >= ix1 or iy0 >= iy1:
        return None, 0
    area = (ix1 - ix0) * (iy1 - iy0)
    if near_cross or area >= cfg.medium_max_px:
        return STAGE3_TILED, area
    if area >= cfg.small_max_px:
        return STAGE2_DIRECT, area
    return STAGE1, area
