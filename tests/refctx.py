"""A stand-in for the reference's ``trirast.pipeline.RenderContext``
(pipeline.py:68-84) built from a golden fixture's stored context arrays —
the object a reference caller passes as ``render_draw_list(..., ctx=)``."""

from dataclasses import dataclass

import numpy as np


@dataclass
class TrirastRenderContext:
    prefix: np.ndarray
    item_mv: np.ndarray
    item_mw: np.ndarray
    item_vtx_off: np.ndarray
    item_idx_off: np.ndarray
    positions: np.ndarray
    indices: np.ndarray
    group_prefix: np.ndarray | None = None
    group_item_off: np.ndarray | None = None
    group_item_count: np.ndarray | None = None
    group_items: np.ndarray | None = None
    max_instances: int = 1


def from_golden(g) -> TrirastRenderContext:
    return TrirastRenderContext(
        prefix=np.asarray(g["prefix"], dtype=np.int64),
        item_mv=np.asarray(g["item_mv"], dtype=np.float64),
        item_mw=np.asarray(g["item_mw"], dtype=np.float64),
        item_vtx_off=np.asarray(g["item_vtx_off"], dtype=np.int64),
        item_idx_off=np.asarray(g["item_idx_off"], dtype=np.int64),
        positions=np.asarray(g["ctx_positions"], dtype=np.float64),
        indices=np.asarray(g["ctx_indices"], dtype=np.uint32),
        group_prefix=np.asarray(g["group_prefix"], dtype=np.int64),
        group_item_off=np.asarray(g["group_item_off"], dtype=np.int64),
        group_item_count=np.asarray(g["group_item_count"], dtype=np.int64),
        group_items=np.asarray(g["group_items"], dtype=np.int64),
        max_instances=int(g["max_instances"]))
