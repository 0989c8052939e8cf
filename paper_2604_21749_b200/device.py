"""HBM residency of scene geometry and per-frame descriptors.

Layout in HBM (per GPU):

* geometry (uploaded once per mesh, cached on the mesh object's identity):
  - positions: ``float32[V,4]`` (x, y, z, 0) when every coordinate is
    exactly representable in float32 (16 B/vertex: one 128-bit gather per
    vertex, the roofline layout);
    ``float64[V,3]`` otherwise (the reference's ctx.positions);
    ``uint16[V,4]`` (x, y, z, 0) for ``QuantizedPositions`` (decoded
    in-register).
  - indices: ``uint32[3T]``, or the bit-packed stream of a
    ``PackedIndexBuffer`` as little-endian 32-bit words (decoded in-register).
* per-frame descriptors (one pinned H2D copy per frame): global-ID prefix,
  object->view / object->world 3x4 float64 matrices from numpy (exactly the
  reference's ``(view @ T)[:3]``, pipeline.py:101-102), the fp32 filter rows
  with their error bounds, instancing groups and the stage-1 work table.
* workspace (grow-only, reused across frames): visibility buffer
  ``uint64[W*H]`` (66 MB at 4K, L2-resident), stage-2/3 queues, counters.
"""

from __future__ import annotations

import math
import os

import numpy as np
import torch

from . import _native as N
from .codec import is_packed_indices, is_quantized_positions

U = 2.0 ** -24
# |X' - X| <= E_FACTOR * u * S per position format (S = sum |coeff * pos|):
# coefficient rounding (1u) + the 3-FMA chain (3u) for exact f32 positions,
# + 1u for f64 positions rounded to f32, + 3u for the u16 grid decode; the
# factors below keep >= 1.2x margin over those sums.
E_FACTOR = {N.POS_F32: 6.0, N.POS_F64: 7.0, N.POS_U16: 10.0}


def _to_device(a: np.ndarray, device) -> torch.Tensor:
    """Host array -> device tensor without a host copy; read-only inputs
    (e.g. TRIMESH1 payloads viewing the file buffer) are only read."""
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)
        return torch.from_numpy(a).to(device)


def _pad4(p3: torch.Tensor) -> torch.Tensor:
    """(V, 3) -> (V, 4) with a zero pad column, on p3's device."""
    p4 = torch.zeros((p3.shape[0], 4), dtype=p3.dtype, device=p3.device)
    p4[:, :3] = p3
    return p4


def _require_cuda():
    if not torch.cuda.is_available():
        raise N.NativeError("no CUDA device: the B200 path has no CPU fallback")


# --------------------------------------------------------------- geometry
class DeviceMesh:
    """One mesh resident on the GPU in its storage format."""

    def __init__(self, mesh, device):
        pos = mesh.positions
        idx = mesh.indices
        self.triangle_count = int(mesh.triangle_count)
        self.device = device
        if hasattr(mesh, "generate") and getattr(mesh, "compressed", False):
            # generated in HBM, stored compressed (config E at 2 GPUs)
            coords, qgrid, words, pack = mesh.generate_compressed(device)
            self.pos_format = N.POS_U16
            self.positions = coords
            self.vertex_count = int(coords.shape[0])
            self.qgrid = qgrid
            self.pos_bound = np.abs(qgrid[:3]) + np.abs(qgrid[3:])
            self.idx_format = N.IDX_PACKED
            self.indices = words
            self.pack = pack
            return
        if hasattr(mesh, "generate"):
            # generated in HBM (generators.DeviceGeneratedMesh, config E):
            # float32-exact by construction, no host copy
            p4, i32 = mesh.generate(device)
            self.pos_format = N.POS_F32
            self.positions = p4
            self.vertex_count = int(p4.shape[0])
            self.qgrid = np.zeros(6)
            self.pos_bound = p4[:, :3].abs().amax(dim=0).double().cpu().numpy()
            self.idx_format = N.IDX_U32
            self.indices = i32
            self.pack = (0, 32)
            return
        if is_quantized_positions(pos):
            self.pos_format = N.POS_U16
            # u16[V][4] (x, y, z, 0): one 64-bit load per vertex in-kernel
            c3 = np.asarray(pos.coords, dtype=np.uint16).reshape(-1, 3)
            coords = np.zeros((len(c3), 4), dtype=np.uint16)
            coords[:, :3] = c3
            self.qgrid = np.concatenate([np.asarray(pos.grid_min, dtype=np.float64),
                                         np.asarray(pos.grid_size, dtype=np.float64)])
            gmin = np.abs(self.qgrid[:3])
            self.pos_bound = gmin + np.abs(self.qgrid[3:])
            self.positions = _to_device(coords.view(np.int16), device)
            self.vertex_count = len(coords)
            self._host_f64 = None
        elif isinstance(pos, np.ndarray) and pos.dtype == np.float32:
            # stored f32 (e.g. a TRIMESH1 payload): exact by construction;
            # uploaded as is, padded to float4 on the device
            d32 = _to_device(np.ascontiguousarray(pos.reshape(-1, 3)), device)
            self.vertex_count = int(d32.shape[0])
            self.qgrid = np.zeros(6)
            self.pos_bound = (d32.abs().amax(dim=0).double().cpu().numpy() if self.vertex_count
                              else np.zeros(3))
            self.pos_format = N.POS_F32
            self.positions = _pad4(d32)
        else:
            # f64 positions: uploaded once, the f32-exactness check and the
            # float4 packing run on the device (one host pass fewer per array)
            p64 = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
            d64 = _to_device(p64, device)
            self.vertex_count = len(p64)
            self.qgrid = np.zeros(6)
            self.pos_bound = (d64.abs().amax(dim=0).cpu().numpy() if len(p64) else np.zeros(3))
            d32 = d64.float()
            if torch.equal(d32.double(), d64):
                # float4 per vertex: a stage-1 vertex gather is one 128-bit
                # load; the pad word is never read as data
                self.pos_format = N.POS_F32
                self.positions = _pad4(d32)
                del d64
            else:
                self.pos_format = N.POS_F64
                self.positions = d64
        if is_packed_indices(idx):
            self.idx_format = N.IDX_PACKED
            data = np.asarray(idx.data, dtype=np.uint8)
            nwords = (len(data) + 3) // 4 + 2
            buf = np.zeros(nwords * 4, dtype=np.uint8)
            buf[:len(data)] = data
            self.indices = torch.from_numpy(buf.view(np.int32)).to(device)
            self.pack = (int(idx.min_index), int(idx.bits_per_index))
        else:
            i32 = np.ascontiguousarray(idx, dtype=np.uint32).ravel()
            self.idx_format = N.IDX_U32
            self.indices = _to_device(i32.view(np.int32), device)
            self.pack = (0, 32)

    def positions_as(self, fmt):
        """Positions converted on the device to a wider common format."""
        if fmt == self.pos_format:
            return self.positions
        if fmt == N.POS_F64:
            if self.pos_format == N.POS_F32:
                return self.positions[:, :3].double()
            q = self.positions[:, :3].to(torch.int32) & 0xFFFF
            q = q.double()
            g = torch.from_numpy(self.qgrid).to(self.device)
            # grid_min + (q + 0.5) / 65536.0 * grid_size  (geomcodec.py:101)
            return g[:3] + (q + 0.5) / 65536.0 * g[3:]
        raise ValueError("unsupported position conversion")

    def indices_u32(self):
        if self.idx_format == N.IDX_U32:
            return self.indices
        mn, b = self.pack
        n = 3 * self.triangle_count
        e = torch.arange(n, device=self.device, dtype=torch.int64)
        bit = e * b
        w = self.indices.to(torch.int64) & 0xFFFFFFFF
        lo = w[bit >> 5]
        hi = w[(bit >> 5) + 1]
        win = lo | (hi << 32)
        rel = (win >> (bit & 31)) & ((1 << b) - 1) if b < 63 else win
        return (rel + mn).to(torch.int64).to(torch.int32)


_CACHE_ATTR = "_curast_device_copies"


def device_mesh(mesh, device) -> DeviceMesh:
    """Upload (once) and return the device copy of a mesh.

    The copy is cached ON the mesh object (it dies with the mesh; an id-keyed
    global table could hand a freed mesh's geometry to a new mesh that reuses
    its id).  The entry holds the positions/indices objects it was built from
    and is reused only while the mesh still holds those same objects, so
    assigning new arrays re-uploads; in-place edits of the arrays are not
    detected (assign a new array instead)."""
    key = str(device)
    cache = getattr(mesh, _CACHE_ATTR, None)
    if cache is not None:
        ent = cache.get(key)
        if (ent is not None and ent[0] is mesh.positions and ent[1] is mesh.indices
                and ent[2] == int(mesh.triangle_count)):
            return ent[3]
    dm = DeviceMesh(mesh, device)
    try:
        if cache is None:
            cache = {}
            object.__setattr__(mesh, _CACHE_ATTR, cache)
        cache[key] = (mesh.positions, mesh.indices, int(mesh.triangle_count), dm)
    except (AttributeError, TypeError):
        pass                                    # slotted/frozen mesh: no cache
    return dm


class _MeshSlice:
    """A generated mesh's place in a streamed SceneGeometry: the DeviceMesh
    metadata the host needs (formats, bounds, codec parameters) and views of
    its slice of the concatenated buffers."""

    def __init__(self, dm, positions, indices):
        for k in ("pos_format", "vertex_count", "triangle_count", "qgrid", "pos_bound",
                  "idx_format", "pack", "device"):
            setattr(self, k, getattr(dm, k))
        self.positions = positions
        self.indices = indices


def _packed_words(mesh) -> int:
    """int32 words of generators.DeviceGeneratedMesh.generate_compressed."""
    V = mesh.vertex_count()
    b = max(1, int(V - 1).bit_length())
    return (3 * int(mesh.triangle_count) * b + 31) // 32 + 1 + 2


class SceneGeometry:
    """Concatenation of the draw list's unique meshes in one device format,
    in first-appearance order (pipeline.py:103-111)."""

    def __init__(self, meshes: list, device):
        if (len(meshes) > 1 and all(hasattr(m, "generate") for m in meshes)
                and len({bool(getattr(m, "compressed", False)) for m in meshes}) == 1):
            self._streamed(meshes, device)
            return
        dms = [device_mesh(m, device) for m in meshes]
        self.meshes = dms
        pfs = {d.pos_format for d in dms}
        ifs = {d.idx_format for d in dms}
        if pfs == {N.POS_F32}:
            self.pos_format = N.POS_F32
        elif pfs == {N.POS_U16}:
            self.pos_format = N.POS_U16
        else:
            self.pos_format = N.POS_F64
        self.idx_format = N.IDX_PACKED if ifs == {N.IDX_PACKED} else N.IDX_U32
        self.vtx_off = []
        self.idx_off = []
        pos_parts, idx_parts = [], []
        nv = ni = 0
        for d in dms:
            self.vtx_off.append(nv)
            self.idx_off.append(ni)
            p = d.positions_as(self.pos_format)
            pos_parts.append(p.reshape(-1))
            ix = d.indices if self.idx_format == N.IDX_PACKED else d.indices_u32()
            ix = ix.reshape(-1)
            if self.idx_format == N.IDX_U32 and ix.numel() % 4:
                # keep every mesh's stream 16-byte aligned (128-bit index loads)
                ix = torch.cat([ix, ix.new_zeros(4 - ix.numel() % 4)])
            idx_parts.append(ix)
            nv += d.vertex_count
            ni += ix.numel()
        if len(dms) == 1:
            self.positions = pos_parts[0]
            self.indices = idx_parts[0]
        else:
            self.positions = torch.cat(pos_parts)
            self.indices = torch.cat(idx_parts)
        self.keepalive = dms

    def _streamed(self, meshes: list, device):
        """Generated meshes (config E) go straight into preallocated
        concatenated buffers, one at a time: peak memory is the scene plus
        one mesh, instead of every mesh's own copy plus the concatenation
        (which did not fit a 4-GPU shard of E, ~89 GB per GPU)."""
        comp = bool(getattr(meshes[0], "compressed", False))
        nvs = [int(m.vertex_count()) for m in meshes]
        if comp:
            nis = [_packed_words(m) for m in meshes]
            self.positions = torch.empty((sum(nvs), 4), dtype=torch.int16, device=device)
            self.pos_format, self.idx_format = N.POS_U16, N.IDX_PACKED
        else:
            nis = [-(-3 * int(m.triangle_count) // 4) * 4 for m in meshes]
            self.positions = torch.empty((sum(nvs), 4), dtype=torch.float32, device=device)
            self.pos_format, self.idx_format = N.POS_F32, N.IDX_U32
        self.indices = torch.zeros(sum(nis), dtype=torch.int32, device=device)
        self.vtx_off, self.idx_off, self.meshes = [], [], []
        nv = ni = 0
        for m, v, i in zip(meshes, nvs, nis):
            dm = DeviceMesh(m, device)               # transient, not cached on the mesh
            pv = self.positions[nv:nv + v]
            pv.copy_(dm.positions.reshape(v, 4))
            ix = dm.indices.reshape(-1)
            iv = self.indices[ni:ni + i]
            iv[:ix.numel()].copy_(ix)
            self.vtx_off.append(nv)
            self.idx_off.append(ni)
            self.meshes.append(_MeshSlice(dm, pv, iv))
            del dm, ix
            nv += v
            ni += i
        self.positions = self.positions.reshape(-1)
        self.keepalive = []


_scene_cache: dict = {}


def scene_geometry(meshes: list, device) -> SceneGeometry:
    """Cached concatenation for a draw list's unique meshes.  Entries hold the
    mesh/positions/indices objects they were built from (so their ids cannot
    be reused by new objects while the entry lives) and are matched by
    identity; at most 8 scenes are kept."""
    objs = tuple((m, m.positions, m.indices) for m in meshes)
    key = (tuple(id(o) for t in objs for o in t), str(device))
    ent = _scene_cache.get(key)
    if ent is not None and all(a is b for ta, tb in zip(ent[0], objs) for a, b in zip(ta, tb)):
        return ent[1]
    if len(_scene_cache) >= 8:
        _scene_cache.pop(next(iter(_scene_cache)))
    sg = SceneGeometry(meshes, device)
    _scene_cache[key] = (objs, sg)
    return sg


def drop_device_copies(meshes=()) -> None:
    """Forget cached device geometry (all scenes, and the given meshes' own
    uploads) so the next frame re-uploads."""
    _scene_cache.clear()
    for m in meshes:
        try:
            delattr(m, _CACHE_ATTR)
        except AttributeError:
            pass


# --------------------------------------------------------- filter constants
def filter_rows(item_mv: np.ndarray, pos_bound: np.ndarray, p0: float, p1: float,
                width: int, height: int, near: float, pos_format: int = N.POS_F64) -> np.ndarray:
    """fp32 filter block per item (curast.h CURAST_FILTER_FLOATS).

    X = px*d = A*vx + B*d, Y = py*d = Dh*d - C*vy, d = -vz with
    A = W/2*p0, B = W/2, C = H/2*p1, Dh = H/2 (kernels.py:78-96 rearranged).
    Error bounds E = E_FACTOR[pos_format] * u * sum |term| over the item's position box
    (6 / 7 / 10 u for f32 / f64 / u16 positions, see E_FACTOR)."""
    n = len(item_mv)
    m = item_mv.reshape(n, 3, 4)
    A = 0.5 * width * p0
    B = 0.5 * width
    C = 0.5 * height * p1
    Dh = 0.5 * height
    X = A * m[:, 0, :] - B * m[:, 2, :]
    Y = -C * m[:, 1, :] - Dh * m[:, 2, :]
    Dd = -m[:, 2, :]
    P = np.concatenate([pos_bound, np.ones((n, 1))], axis=1)   # (n, 4)
    SX = ((np.abs(A * m[:, 0, :]) + np.abs(B * m[:, 2, :])) * P).sum(axis=1)
    SY = ((np.abs(C * m[:, 1, :]) + np.abs(Dh * m[:, 2, :])) * P).sum(axis=1)
    SD = (np.abs(m[:, 2, :]) * P).sum(axis=1)
    ef = E_FACTOR[pos_format]
    exy = ef * U * np.maximum(SX, SY) * (1 + 2.0 ** -20) + 1e-30
    ed = ef * U * SD * (1 + 2.0 ** -20) + 1e-30
    near_hi = np.maximum(near + 2.0 * ed + 2.0 ** -40 * SD, 4.0 * ed)
    out = np.zeros((n, N.FILTER_FLOATS), dtype=np.float32)
    # (X, Y) rows interleaved: X0 Y0 X1 Y1 X2 Y2 X3 Y3 (filter.cuh: one
    # 128-bit load gives two FFMA2-ready (X, Y) coefficient pairs)
    out[:, 0:8:2] = X
    out[:, 1:8:2] = Y
    out[:, 8:12] = Dd
    out[:, 12] = _f32_up(exy)
    out[:, 13] = _f32_up(ed)
    out[:, 14] = _f32_up(near_hi)
    bad = ~np.all(np.isfinite(out), axis=1)
    if bad.any():
        # non-finite rows never decide anything: near_hi = +inf forces fp64
        out[bad, 14] = np.inf
    return out


def _f32_up(x: np.ndarray) -> np.ndarray:
    f = np.asarray(x, dtype=np.float64).astype(np.float32)
    lo = f.astype(np.float64) < x
    f[lo] = np.nextafter(f[lo], np.float32(np.inf))
    return f


# ------------------------------------------------------------- workspace
class Workspace:
    """Grow-only device buffers reused across frames (no allocation on the
    frame path once warm)."""

    def __init__(self, device):
        self.device = device
        self.fb = None
        self.npix = 0
        self.q2 = None
        self.q2_alloc = 0
        self.q3 = None
        self.q3_alloc = 0
        self.qx = None
        self.qx_alloc = 0
        self.counters = torch.zeros(N.COUNTER_SLOTS, dtype=torch.int64, device=device)
        self.counters_host = torch.zeros(N.COUNTER_SLOTS, dtype=torch.int64).pin_memory()

    def framebuffer(self, npix: int, fresh: bool):
        """Visibility buffer for a frame.  ``fresh`` returns a new tensor (the
        caller keeps it, e.g. in a returned Framebuffer)."""
        if fresh:
            return torch.empty(npix, dtype=torch.int64, device=self.device)
        if self.fb is None or self.npix != npix:
            self.fb = torch.empty(npix, dtype=torch.int64, device=self.device)
            self.npix = npix
        return self.fb

    def ensure_q2(self, n: int):
        n = max(1, int(n))
        if n > self.q2_alloc:
            self.q2 = torch.empty(2 * n, dtype=torch.int64, device=self.device)
            self.q2_alloc = n
        return self.q2

    def ensure_qx(self, n: int):
        n = max(1, int(n))
        if n > self.qx_alloc:
            self.qx = torch.empty(N.QX_WORDS * n, dtype=torch.int64, device=self.device)
            self.qx_alloc = n
        return self.qx

    def ensure_q3(self, n: int):
        n = max(1, int(n))
        if n > self.q3_alloc:
            self.q3 = torch.empty(4 * n, dtype=torch.int64, device=self.device)
            self.q3_alloc = n
        return self.q3


_workspaces: dict = {}


def workspace(device) -> Workspace:
    key = str(device)
    ws = _workspaces.get(key)
    if ws is None:
        ws = Workspace(device)
        _workspaces[key] = ws
    return ws


class PackedUpload:
    """Packs many small host arrays into one pinned buffer and one H2D copy;
    returns device tensors viewing it."""

    def __init__(self):
        self.parts = []

    def add(self, arr: np.ndarray) -> int:
        arr = np.ascontiguousarray(arr)
        self.parts.append(arr)
        return len(self.parts) - 1

    def upload(self, device, stream=None):
        offs = []
        total = 0
        for a in self.parts:
            total = (total + 255) & ~255
            offs.append(total)
            total += a.nbytes
        total = max(total, 256)
        host = torch.empty(total, dtype=torch.uint8).pin_memory()
        hn = host.numpy()
        for a, o in zip(self.parts, offs):
            hn[o:o + a.nbytes] = a.view(np.uint8).reshape(-1)
        dev = torch.empty(total, dtype=torch.uint8, device=device)
        dev.copy_(host, non_blocking=True)
        self.host = host          # keep pinned source alive until the copy ran
        self.dev = dev
        self.offsets = offs
        return dev

    def ptr(self, k: int) -> int:
        return self.dev.data_ptr() + self.offsets[k]

    @property
    def nbytes(self) -> int:
        return int(self.dev.numel())
