"""Fixture -> oracle context helpers (test infrastructure)."""

import numpy as np

from oracle import host as oh


def oracle_ctx(g):
    return oh.OContext(
        prefix=g["prefix"].astype(np.int64), item_mv=g["item_mv"], item_mw=g["item_mw"],
        item_vtx_off=g["item_vtx_off"], item_idx_off=g["item_idx_off"],
        positions=np.ascontiguousarray(g["ctx_positions"]),
        indices=np.ascontiguousarray(g["ctx_indices"]),
        group_prefix=g["group_prefix"], group_item_off=g["group_item_off"],
        group_item_count=g["group_item_count"], group_items=g["group_items"],
        max_instances=int(g["max_instances"]))


def camera_consts(g, camera):
    cc = oh.camera_constants(camera)
    p = g["p"]
    cc["p0"], cc["p1"] = float(p[0]), float(p[1])
    return cc


def cfg_kwargs(cfg, honor_stages=True):
    kw = dict(tiny_cull=cfg.tiny_cull, force_stage=cfg.force_stage,
              small_max=cfg.small_max_px, medium_max=cfg.medium_max_px,
              tile_px=cfg.tile_px)
    if not honor_stages:
        kw["small_max"] = 1 << 40
        kw["medium_max"] = 1 << 40
    return kw
