"""GPU resolve pass: visibility buffer -> shaded RGBA8 (resolvepass.py:297-407).

``resolve_frame(framebuffer, draw_list, camera, shading)`` has the
reference's signature and returns ``(image[h, w, 4] uint8, ResolveStats)``;
``resolve_frame_device`` keeps the image in HBM (torch uint8 tensor) for
callers that composite, downsample or display on the GPU.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .config import ShadingConfig
from .device import PackedUpload, scene_geometry
from .pipeline import build_context
from .scene import projection_vector

MODE_FLAT, MODE_VCOLOR, MODE_TEX = 0, 1, 2


@dataclass
class ResolveStats:
    shaded: int = 0
    background: int = 0
    degenerate: int = 0


def _item_mode(mesh, mode: str) -> int:
    """Shading mode per mesh (resolvepass.py:350-378)."""
    has_tex = getattr(mesh, "uvs", None) is not None and getattr(mesh, "texture", None) is not None
    has_col = getattr(mesh, "vertex_colors", None) is not None
    if mode == "auto":
        mode = "textured" if has_tex else ("vertexColor" if has_col else "flat")
    if mode == "textured" and has_tex:
        return MODE_TEX
    if mode == "vertexColor" and has_col:
        return MODE_VCOLOR
    return MODE_FLAT


class _Attributes:
    """Per-vertex colours / UVs and mip chains of a geometry, on the device."""

    def __init__(self, meshes, geo, device):
        nv = sum(m.vertex_count for m in geo.meshes)
        colors = np.zeros((max(nv, 1), 4), dtype=np.uint8)
        uvs = np.zeros((max(nv, 1), 2), dtype=np.float64)
        tex_ids = []
        levels = []
        tex_desc = []
        blobs = []
        off = 0
        textures = {}
        for m, voff, dm in zip(meshes, geo.vtx_off, geo.meshes):
            n = dm.vertex_count
            if getattr(m, "vertex_colors", None) is not None:
                colors[voff:voff + n] = np.asarray(m.vertex_colors, dtype=np.uint8).reshape(n, 4)
            if getattr(m, "uvs", None) is not None:
                uvs[voff:voff + n] = np.asarray(m.uvs, dtype=np.float64).reshape(n, 2)
            tex = getattr(m, "texture", None)
            if tex is not None and id(tex) not in textures:
                textures[id(tex)] = len(tex_desc)
                tex_desc.append((len(tex.levels), len(levels)))
                for lv in tex.levels:
                    lv = np.ascontiguousarray(lv, dtype=np.uint8)
                    levels.append((lv.shape[1], lv.shape[0], off))
                    blobs.append(lv.reshape(-1))
                    off += lv.size
            tex_ids.append(textures[id(tex)] if tex is not None else -1)
        self.mesh_tex = tex_ids
        self.colors = torch.from_numpy(colors).to(device)
        self.uvs = torch.from_numpy(uvs).to(device)
        texels = np.concatenate(blobs) if blobs else np.zeros(4, dtype=np.uint8)
        self.texels = torch.from_numpy(texels).to(device)
        self.tex_desc = torch.from_numpy(np.asarray(tex_desc or [(0, 0)], dtype=np.int64)).to(device)
        self.level_desc = torch.from_numpy(np.asarray(levels or [(1, 1, 0)], dtype=np.int64)).to(device)


_attr_cache: dict = {}


def _attributes(meshes, geo, device):
    key = (id(geo), tuple((id(getattr(m, "vertex_colors", None)), id(getattr(m, "uvs", None)),
                           id(getattr(m, "texture", None))) for m in meshes))
    a = _attr_cache.get(key)
    if a is None:
        if len(_attr_cache) > 8:
            _attr_cache.clear()
        a = _Attributes(meshes, geo, device)
        _attr_cache[key] = a
    return a


class _DeviceResolveStats(ResolveStats):
    """ResolveStats whose counters stay on the device until first read, so
    resolve_frame_device does not synchronise the host."""

    def __init__(self, counters):
        object.__setattr__(self, "_c", counters)
        object.__setattr__(self, "_v", None)

    def _vals(self):
        if self._v is None:
            object.__setattr__(self, "_v", [int(x) for x in self._c.cpu().tolist()[:3]])
        return self._v

    shaded = property(lambda self: self._vals()[0])
    background = property(lambda self: self._vals()[1])
    degenerate = property(lambda self: self._vals()[2])

    def __repr__(self):
        return (f"ResolveStats(shaded={self.shaded}, background={self.background}, "
                f"degenerate={self.degenerate})")


class PreparedResolve:
    """The resolve descriptors of one (draw list, camera, shading) resident on
    the device: built and uploaded once, reused by every resolve of frames
    of that draw list (the per-call work is one kernel launch)."""

    def __init__(self, draw_list, camera, shading, device):
        ctx = build_context(draw_list, camera)
        geo = scene_geometry(ctx.meshes, device)
        attrs = _attributes(ctx.meshes, geo, device)
        self.draw_list, self.geo, self.attrs = draw_list, geo, attrs
        n = len(draw_list.items)
        modes = np.asarray([_item_mode(ctx.meshes[i], shading.mode) for i in ctx.item_mesh],
                           dtype=np.int32)
        up = PackedUpload()
        kp = up.add(ctx.prefix)
        kmw = up.add(ctx.item_mw.reshape(-1))
        kvo = up.add(np.asarray([geo.vtx_off[i] for i in ctx.item_mesh], dtype=np.int64))
        kio = up.add(np.asarray([geo.idx_off[i] for i in ctx.item_mesh], dtype=np.int64))
        kq = up.add(np.stack([geo.meshes[i].qgrid for i in ctx.item_mesh]).reshape(-1))
        kpk = up.add(np.asarray([geo.meshes[i].pack for i in ctx.item_mesh],
                                dtype=np.int64).reshape(-1))
        kmo = up.add(modes)
        kco = up.add(np.asarray([geo.vtx_off[i] for i in ctx.item_mesh], dtype=np.int64))
        ktx = up.add(np.asarray([attrs.mesh_tex[i] for i in ctx.item_mesh], dtype=np.int64))
        up.upload(device)
        self.upload = up
        r = N.CurastResolve()
        r.n_items = n
        r.prefix, r.item_mw = up.ptr(kp), up.ptr(kmw)
        r.item_vtx_off, r.item_idx_off = up.ptr(kvo), up.ptr(kio)
        r.pos_format, r.idx_format = geo.pos_format, geo.idx_format
        r.positions, r.indices = geo.positions.data_ptr(), geo.indices.data_ptr()
        r.item_qgrid, r.item_pack = up.ptr(kq), up.ptr(kpk)
        r.item_mode, r.item_color_off = up.ptr(kmo), up.ptr(kco)
        r.colors, r.uvs = attrs.colors.data_ptr(), attrs.uvs.data_ptr()
        r.item_tex, r.tex_desc = up.ptr(ktx), attrs.tex_desc.data_ptr()
        r.level_desc, r.texels = attrs.level_desc.data_ptr(), attrs.texels.data_ptr()
        r.trilinear = int(shading.mip_filter == "trilinear")
        r.headlight = int(bool(shading.headlight))
        for i in range(4):
            r.background[i] = int(shading.background[i])
            r.base_color[i] = int(shading.base_color[i])
        p = projection_vector(camera)
        r.p0, r.p1 = float(p[0]), float(p[1])
        pos = np.asarray(camera.position, dtype=np.float64)
        rot = np.asarray(camera.view_transform, dtype=np.float64)[:3, :3].reshape(-1)
        for i in range(3):
            r.cam[i] = float(pos[i])
        for i in range(9):
            r.rot[i] = float(rot[i])
        self.r = r
        self.meshes = ctx.meshes

    def current(self, device) -> bool:
        return scene_geometry(self.meshes, device) is self.geo

    def launch(self, words, w, h, out, counters, row0, nrows, stream=None):
        r = self.r
        r.fb = words.data_ptr()
        r.width, r.height = w, h
        r.out_rgba = out.data_ptr()
        r.counters = counters.data_ptr()
        r.row0, r.rows = row0, nrows
        st = (stream or torch.cuda.current_stream()).cuda_stream
        N.check(N.lib().curast_resolve(ctypes.byref(r), st), "resolve")


_resolve_cache: dict = {}


def _shading_key(s):
    return (s.mode, tuple(s.background), tuple(s.base_color), s.mip_filter, bool(s.headlight))


def prepared_resolve(draw_list, camera, shading, device) -> PreparedResolve:
    """Cached PreparedResolve (by draw-list identity, camera and shading
    values; at most 4 kept; rebuilt when the scene geometry changed)."""
    from .pipeline import _camera_key
    key = (id(draw_list), _camera_key(camera), _shading_key(shading), str(device))
    pr = _resolve_cache.get(key)
    if pr is not None and pr.draw_list is draw_list and pr.current(device):
        return pr
    if len(_resolve_cache) >= 4:
        _resolve_cache.pop(next(iter(_resolve_cache)))
    pr = PreparedResolve(draw_list, camera, shading, device)
    _resolve_cache[key] = pr
    return pr


def resolve_frame_device(framebuffer, draw_list, camera, shading: ShadingConfig | None = None,
                         *, rows=None, stripe_words=None):
    """Shade every pixel on the GPU; returns (uint8 CUDA tensor [h, w, 4],
    ResolveStats).  ``rows=(row0, n)`` shades image rows [row0, row0 + n)
    only (a sort-last stripe) from ``stripe_words`` (int64 CUDA tensor of
    n*w words; default: the framebuffer's rows) into an [n, w, 4] image.
    Nothing synchronises the host: the stats read their device counters on
    first access; the descriptors are prepared once per draw list / camera /
    shading (prepared_resolve)."""
    shading = shading or ShadingConfig()
    device = torch.device("cuda", torch.cuda.current_device())
    w, h = framebuffer.width, framebuffer.height
    if stripe_words is not None:
        words = stripe_words
    else:
        words = framebuffer.device_words if hasattr(framebuffer, "device_words") else \
            torch.from_numpy(np.asarray(framebuffer.words).view(np.int64).copy()).to(device)
    row0, nrows = (0, h) if rows is None else (int(rows[0]), int(rows[1]))
    if stripe_words is None and rows is not None:
        words = words[row0 * w:(row0 + nrows) * w]
    out = torch.empty((nrows, w, 4), dtype=torch.uint8, device=device)
    if draw_list.total_triangles == 0 or len(draw_list.items) == 0:
        out[:] = torch.tensor(shading.background, dtype=torch.uint8, device=device)
        return out, ResolveStats(background=w * nrows)
    counters = torch.zeros(4, dtype=torch.int64, device=device)
    pr = prepared_resolve(draw_list, camera, shading, device)
    pr.launch(words, w, h, out, counters, row0, nrows)
    return out, _DeviceResolveStats(counters)


def resolve_frame(framebuffer, draw_list, camera, shading: ShadingConfig | None = None):
    """Drop-in for resolvepass.resolve_frame: host RGBA8 image + stats."""
    img, st = resolve_frame_device(framebuffer, draw_list, camera, shading)
    return img.cpu().numpy(), st


def downsample_device(image: torch.Tensor, factor: int) -> torch.Tensor:
    if factor == 1:
        return image
    h, w = image.shape[:2]
    if h % factor or w % factor:
        raise ValueError("internal resolution must be a multiple of the factor")
    out = torch.empty((h // factor, w // factor, 4), dtype=torch.uint8, device=image.device)
    N.check(N.lib().curast_downsample(image.data_ptr(), w, h, factor, out.data_ptr(),
                                      torch.cuda.current_stream().cuda_stream), "downsample")
    return out


def downsample(image, factor: int):
    """Box-average factor x factor blocks, floor rounding (resolvepass.py:398-407).
    Accepts a host array (returns host) or a CUDA tensor (returns CUDA)."""
    if factor == 1:
        return image
    if isinstance(image, torch.Tensor):
        return downsample_device(image.contiguous(), factor)
    img = np.asarray(image, dtype=np.uint8)
    h, w = img.shape[:2]
    if h % factor or w % factor:
        raise ValueError("internal resolution must be a multiple of the factor")
    dev = torch.from_numpy(np.ascontiguousarray(img)).cuda()
    return downsample_device(dev, factor).cpu().numpy()


_DEBUG_MODES = {"depth": 0, "stageID": 1, "bboxSize": 2, "meshID": 3}


def debug_view_device(framebuffer, draw_list, camera, mode: str, cfg=None,
                      background=(40, 40, 44, 255)) -> torch.Tensor:
    """Diagnostic views of the visibility buffer on the GPU
    (resolvepass.py:417-490): 'depth' (log-scaled grey), 'stageID' (the stage
    whose classification the winning triangle satisfies), 'bboxSize'
    (green / yellow / red by the bbox-size thresholds), 'meshID'.  Returns a
    uint8 CUDA tensor [h, w, 4]."""
    from .config import RasterConfig
    if mode not in _DEBUG_MODES:
        raise ValueError(f"unknown debug view mode {mode!r}")
    cfg = cfg or RasterConfig()
    L = N.lib()
    device = torch.device("cuda", torch.cuda.current_device())
    w, h = framebuffer.width, framebuffer.height
    words = framebuffer.device_words
    out = torch.empty((h, w, 4), dtype=torch.uint8, device=device)
    if draw_list.total_triangles == 0 or len(draw_list.items) == 0:
        out[:] = torch.tensor(background, dtype=torch.uint8, device=device)
        return out
    ctx = build_context(draw_list, camera)
    geo = scene_geometry(ctx.meshes, device)
    xform = np.stack([np.asarray(it.instance_transform, dtype=np.float64).reshape(4, 4)
                      for it in draw_list.items])
    up = PackedUpload()
    kp = up.add(ctx.prefix)
    kvo = up.add(np.asarray([geo.vtx_off[i] for i in ctx.item_mesh], dtype=np.int64))
    kio = up.add(np.asarray([geo.idx_off[i] for i in ctx.item_mesh], dtype=np.int64))
    kq = up.add(np.stack([geo.meshes[i].qgrid for i in ctx.item_mesh]).reshape(-1))
    kpk = up.add(np.asarray([geo.meshes[i].pack for i in ctx.item_mesh], dtype=np.int64).reshape(-1))
    kx = up.add(xform.reshape(-1))
    up.upload(device)
    scratch = torch.zeros(2, dtype=torch.int32, device=device)
    d = N.CurastDebug()
    d.fb = words.data_ptr()
    d.width, d.height, d.mode = w, h, _DEBUG_MODES[mode]
    d.pos_format, d.idx_format = geo.pos_format, geo.idx_format
    d.n_items = len(draw_list.items)
    d.prefix, d.item_vtx_off, d.item_idx_off = up.ptr(kp), up.ptr(kvo), up.ptr(kio)
    d.positions, d.indices = geo.positions.data_ptr(), geo.indices.data_ptr()
    d.item_qgrid, d.item_pack, d.item_xform = up.ptr(kq), up.ptr(kpk), up.ptr(kx)
    view = np.asarray(camera.view_transform, dtype=np.float64).reshape(-1)
    for i in range(16):
        d.view[i] = float(view[i])
    p = projection_vector(camera)
    d.p0, d.p1, d.near = float(p[0]), float(p[1]), float(camera.near)
    d.small_max, d.medium_max = int(cfg.small_max_px), int(cfg.medium_max_px)
    for i in range(4):
        d.background[i] = int(background[i])
    d.out_rgba = out.data_ptr()
    d.scratch = scratch.data_ptr()
    N.check(L.curast_debug_view(ctypes.byref(d), torch.cuda.current_stream().cuda_stream),
            "debug_view")
    return out


def debug_view(framebuffer, draw_list, camera, mode: str, cfg=None,
               background=(40, 40, 44, 255)) -> np.ndarray:
    """Drop-in for resolvepass.debug_view: host RGBA8 image [h, w, 4]."""
    return debug_view_device(framebuffer, draw_list, camera, mode, cfg, background).cpu().numpy()
