"""Compressed geometry formats consumed in-register by the stage kernels.

Formats are the reference's (trirast/geomcodec.py:31-126):

* ``PackedIndexBuffer`` — indices rebased to ``min_index`` and bit-packed at
  ``bits_per_index`` = bit_length(span) bits (min 1), little-endian bit order
  inside bytes, no per-element alignment (geomcodec.py:31-84).
* ``QuantizedPositions`` — u16 cell index per axis on the mesh box grid,
  decoded as ``grid_min + (q + 0.5) / 65536.0 * grid_size`` in float64, in
  that order (geomcodec.py:87-120).

The GPU never receives decoded arrays for these meshes: the u16 coordinates
and the bit stream are uploaded as stored and decoded inside the kernels.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class PackedIndexBuffer:
    min_index: int
    bits_per_index: int
    count: int
    data: np.ndarray           # uint8 bit stream

    def decode(self, i: int) -> int:
        if not 0 <= i < self.count:
            raise IndexError(f"element {i} out of range [0, {self.count})")
        b = self.bits_per_index
        bit = i * b
        lo = bit >> 3
        nbytes = (b + (bit & 7) + 7) >> 3
        chunk = int.from_bytes(self.data[lo:lo + nbytes].tobytes(), "little")
        return self.min_index + ((chunk >> (bit & 7)) & ((1 << b) - 1))

    def decode_all(self) -> np.ndarray:
        b = self.bits_per_index
        bits = np.unpackbits(self.data, count=self.count * b, bitorder="little")
        bits = bits.reshape(self.count, b).astype(np.uint64)
        rel = (bits << np.arange(b, dtype=np.uint64)).sum(axis=1, dtype=np.uint64)
        return (rel + np.uint64(self.min_index)).astype(np.uint32)


def compress_indices(indices) -> PackedIndexBuffer:
    """Same bit stream as geomcodec.compress_indices (geomcodec.py:65-84),
    built word-wise so 10^8-element buffers fit in memory: element i occupies
    bits [i*b, i*b + b) of the little-endian 32-bit word stream, and since the
    fields never overlap, OR-ing them equals summing them."""
    idx = np.asarray(indices, dtype=np.uint32).ravel()
    if idx.size == 0:
        raise ValueError("indices must be non-empty")
    lo = int(idx.min())
    span = int(idx.max()) - lo
    b = max(1, span.bit_length())
    n = idx.size
    nbytes = (n * b + 7) // 8
    nwords = (n * b + 31) // 32 + 1
    words = np.zeros(nwords, dtype=np.uint64)
    step = 1 << 24
    for s in range(0, n, step):
        rel = idx[s:s + step].astype(np.uint64) - np.uint64(lo)
        bit = (np.arange(s, s + rel.size, dtype=np.uint64) * np.uint64(b))
        w = (bit >> np.uint64(5)).astype(np.int64)
        sh = bit & np.uint64(31)
        full = rel << sh                                   # < 2^63
        words += np.bincount(w, weights=(full & np.uint64(0xFFFFFFFF)).astype(np.float64),
                             minlength=nwords).astype(np.uint64)
        words += np.bincount(w + 1, weights=(full >> np.uint64(32)).astype(np.float64),
                             minlength=nwords).astype(np.uint64)
    data = words.astype(np.uint32).view(np.uint8)[:nbytes].copy()
    return PackedIndexBuffer(min_index=lo, bits_per_index=b, count=n, data=data)


@dataclass
class QuantizedPositions:
    grid_min: np.ndarray       # (3,) float64
    grid_size: np.ndarray      # (3,) float64, > 0
    coords: np.ndarray         # (n, 3) uint16

    @property
    def count(self) -> int:
        return len(self.coords)

    def dequantize_all(self) -> np.ndarray:
        q = self.coords.astype(np.float64)
        return self.grid_min + (q + 0.5) / 65536.0 * self.grid_size


def quantize_positions(positions, aabb) -> QuantizedPositions:
    pos = np.asarray(positions, dtype=np.float64)
    box = np.asarray(aabb, dtype=np.float64)
    gmin = box[0].copy()
    size = box[1] - box[0]
    if np.any(pos < box[0]) or np.any(pos > box[1]):
        raise ValueError("position outside the quantization bounding box")
    size = np.where(size > 0.0, size, 1.0)
    q = np.floor(65536.0 * (pos - gmin) / size)
    return QuantizedPositions(grid_min=gmin, grid_size=size,
                              coords=np.clip(q, 0, 65535).astype(np.uint16))


def is_packed_indices(obj) -> bool:
    return (not isinstance(obj, np.ndarray) and hasattr(obj, "bits_per_index")
            and hasattr(obj, "data"))


def is_quantized_positions(obj) -> bool:
    return (not isinstance(obj, np.ndarray) and hasattr(obj, "grid_min")
            and hasattr(obj, "coords"))
