"""TRIMESH1 native mesh files (geomcodec.py:262-362) straight to the device.

The reference's binary format, read and written byte-for-byte:

    header  <8sQQIB3x>  magic "TRIMESH1", vertex count, triangle count,
                        flags, bits per packed index
    positions           QUANTIZED: grid_min f32[3], grid_size f32[3],
                                   coords u16[V][3]
                        else       f32[V][3]
    indices             PACKED:    min_index u32, ceil(3T*bits/8) stream bytes
                        else       u32[3T]
    uvs                 f32[V][2]            (FLAG_UVS)
    vertex colours      u8[V][4]             (FLAG_VERTEX_COLORS)

``load_mesh`` returns a ``Mesh`` whose payloads are the stored arrays
themselves (numpy views over one read of the file): u16 coordinates and the
bit-packed stream stay compressed — the stage kernels decode them in
registers (codec.py) — and raw f32 positions stay f32 (the exact device
format).  With ``device=...`` the payloads are uploaded once, as stored, and
cached on the mesh (device.device_mesh); nothing is decoded on the host.
Errors follow the reference: ``ParseError`` naming the file, the truncated
part and its byte offset.
"""

from __future__ import annotations

import struct

import numpy as np

from .codec import PackedIndexBuffer, QuantizedPositions
from .scene import Mesh

MAGIC = b"TRIMESH1"
FLAG_QUANTIZED_POSITIONS = 1 << 0
FLAG_PACKED_INDICES = 1 << 1
FLAG_UVS = 1 << 2
FLAG_VERTEX_COLORS = 1 << 3

_HEADER = struct.Struct("<8sQQIB3x")


class ParseError(RuntimeError):
    """Malformed mesh input (geomcodec.py:27-28)."""


def _is_quantized(p) -> bool:
    return isinstance(p, QuantizedPositions) or (hasattr(p, "grid_min") and hasattr(p, "coords"))


def _is_packed(i) -> bool:
    return isinstance(i, PackedIndexBuffer) or (hasattr(i, "bits_per_index") and hasattr(i, "data"))


def save_mesh(path, mesh: Mesh) -> None:
    """Write ``mesh`` in TRIMESH1 (geomcodec.py:268-300), keeping whichever
    compressed or raw payloads it carries."""
    quantized = _is_quantized(mesh.positions)
    packed = _is_packed(mesh.indices)
    flags = ((FLAG_QUANTIZED_POSITIONS if quantized else 0)
             | (FLAG_PACKED_INDICES if packed else 0)
             | (FLAG_UVS if mesh.uvs is not None else 0)
             | (FLAG_VERTEX_COLORS if mesh.vertex_colors is not None else 0))
    bits = int(mesh.indices.bits_per_index) if packed else 0
    nverts = (len(mesh.positions.coords) if quantized
              else len(np.asarray(mesh.positions).reshape(-1, 3)))
    parts = [_HEADER.pack(MAGIC, nverts, int(mesh.triangle_count), flags, bits)]
    if quantized:
        parts.append(np.asarray(mesh.positions.grid_min).astype("<f4").tobytes())
        parts.append(np.asarray(mesh.positions.grid_size).astype("<f4").tobytes())
        parts.append(np.asarray(mesh.positions.coords).astype("<u2").tobytes())
    else:
        parts.append(np.asarray(mesh.positions).astype("<f4").tobytes())
    if packed:
        parts.append(struct.pack("<I", int(mesh.indices.min_index)))
        parts.append(np.asarray(mesh.indices.data, dtype=np.uint8).tobytes())
    else:
        parts.append(np.asarray(mesh.indices).astype("<u4").tobytes())
    if mesh.uvs is not None:
        parts.append(np.asarray(mesh.uvs).astype("<f4").tobytes())
    if mesh.vertex_colors is not None:
        parts.append(np.asarray(mesh.vertex_colors, dtype=np.uint8).tobytes())
    with open(path, "wb") as fh:
        fh.write(b"".join(parts))


def load_mesh(path, device=None) -> Mesh:
    """Read a TRIMESH1 file (geomcodec.py:303-347).  Payloads stay as
    stored; with ``device`` they are uploaded without host decode."""
    path = str(path)
    with open(path, "rb") as fh:
        data = fh.read()
    mesh = _parse(memoryview(data), path)
    if device is not None:
        from .device import device_mesh
        device_mesh(mesh, device)
    return mesh


def _parse(data, name: str) -> Mesh:
    size = len(data)
    if size < _HEADER.size:
        raise ParseError(f"{name}: truncated header at offset {size}")
    magic, nverts, ntris, flags, bits = _HEADER.unpack_from(data, 0)
    if magic != MAGIC:
        raise ParseError(f"{name}: bad magic {bytes(magic)!r} at offset 0")
    off = _HEADER.size

    def take(n, what, dtype):
        nonlocal off
        if off + n > size:
            raise ParseError(f"{name}: truncated {what} at offset {off}")
        arr = np.frombuffer(data, dtype=dtype, count=n // np.dtype(dtype).itemsize, offset=off)
        off += n
        return arr

    if flags & FLAG_QUANTIZED_POSITIONS:
        grid = take(24, "grid bounds", "<f4").astype(np.float64)
        coords = take(6 * nverts, "positions", "<u2").reshape(nverts, 3)
        positions = QuantizedPositions(grid_min=grid[:3], grid_size=grid[3:], coords=coords)
        aabb = np.stack([positions.grid_min, positions.grid_min + positions.grid_size])
    else:
        positions = take(12 * nverts, "positions", "<f4").reshape(nverts, 3)
        aabb = (np.stack([positions.min(axis=0), positions.max(axis=0)]).astype(np.float64)
                if nverts else np.zeros((2, 3)))
    if flags & FLAG_PACKED_INDICES:
        (min_index,) = struct.unpack("<I", bytes(take(4, "index header", np.uint8)))
        count = 3 * ntris
        nbytes = (count * bits + 7) // 8
        indices = PackedIndexBuffer(min_index=min_index, bits_per_index=bits, count=count,
                                    data=take(nbytes, "indices", np.uint8))
    else:
        indices = take(12 * ntris, "indices", "<u4")
    uvs = None
    if flags & FLAG_UVS:
        uvs = take(8 * nverts, "uvs", "<f4").reshape(nverts, 2).astype(np.float64)
    vertex_colors = None
    if flags & FLAG_VERTEX_COLORS:
        vertex_colors = take(4 * nverts, "vertex colors", np.uint8).reshape(nverts, 4)
    return Mesh(positions=positions, indices=indices, triangle_count=int(ntris), aabb=aabb,
                uvs=uvs, vertex_colors=vertex_colors, name=name)
