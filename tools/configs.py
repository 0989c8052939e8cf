"""Per-config measurements for DESIGN.md / profiles (not the driver bench).

    python tools/configs.py [A B C D Bq Dq] [--check]

For each SURVEY §8(d) config: frame time (CUDA events, mean of K frames after
warm-up, geometry resident), triangles/s, stage split, stage counters, and —
with --check — bit-exactness against the oracle on this host (slow for D).
Bq / Dq: the same scenes with QuantizedPositions + PackedIndexBuffer meshes
(decoded in-register).  One JSON line per config.
"""

import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2604_21749_b200 as cr  # noqa: E402
from paper_2604_21749_b200 import generators as gen  # noqa: E402
from paper_2604_21749_b200.pipeline import PreparedFrame  # noqa: E402
from scenes import compress_scene  # noqa: E402


def build(name):
    if name == "A":
        return gen.config_a()
    if name == "B":
        return gen.config_b()
    if name == "C":
        return gen.config_c()
    if name == "D":
        return gen.config_d()
    if name == "Bq":
        s, c = gen.config_b()
        return compress_scene(s), c
    if name == "Dq":
        s, c = gen.config_d()
        return compress_scene(s), c
    if name == "E200":
        # config E scaled to one GPU: 200 of its 4,750 displaced grids (800M
        # triangles, generated in HBM)
        return gen.config_e(n_meshes=200, on_device=True)
    if name == "A4":
        s, c = gen.config_a()
        return s, cr.Camera(position=c.position, view_transform=c.view_transform, fovy=c.fovy,
                            aspect=c.aspect, near=c.near, image_width=c.image_width,
                            image_height=c.image_height, supersampling=4)
    raise ValueError(name)


def algorithmic_bytes(pf):
    """12 B per unique triangle (u32 indices) + 12 B per unique
    vertex (f32 xyz); compressed: ceil(3 T bits / 8) + 6 B per vertex."""
    from paper_2604_21749_b200 import _native as N
    b = 0
    for m in pf.geo.meshes:
        T, V = m.triangle_count, m.vertex_count
        if m.idx_format == N.IDX_PACKED:
            b += -(-3 * T * m.pack[1] // 8)
        else:
            b += 12 * T
        b += 6 * V if m.pos_format == N.POS_U16 else 12 * V
    return b


def measure(name, steps=20, check=False):
    scene, cam = build(name)
    dl = cr.build_draw_list(scene, cam)
    cfg = cr.RasterConfig()
    pf = PreparedFrame(dl, cam, cfg, fresh_fb=False)
    c, _ = pf.run()
    st = pf.stats(c, [0, 0, 0, 0])
    for _ in range(3):
        pf.launch()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(steps)]
    for k in range(steps):
        pf.launch(events=evs[k])
    torch.cuda.synchronize()
    stage = np.mean([[e[i].elapsed_time(e[i + 1]) for i in range(4)] for e in evs], axis=0)
    frame_ms = float(np.mean([e[0].elapsed_time(e[4]) for e in evs]))
    geo = pf.geo
    geo_bytes = int(geo.positions.numel() * geo.positions.element_size()
                    + geo.indices.numel() * geo.indices.element_size())
    out = {
        "config": name, "triangles": dl.total_triangles, "items": len(dl.items),
        "instanced": pf.instanced, "width": cam.internal_width, "height": cam.internal_height,
        "frame_ms": frame_ms, "tri_per_s": dl.total_triangles / (frame_ms * 1e-3),
        "stage_ms": {"clear": stage[0], "stage1": stage[1], "stage2": stage[2], "stage3": stage[3]},
        "geometry_bytes_resident": geo_bytes,
        "stage1_algorithmic_bytes": algorithmic_bytes(pf),
        "stage1_hbm_frac": algorithmic_bytes(pf) / (stage[1] * 1e-3) / 1e9 / 6536.4,
        "pos_format": int(geo.pos_format), "idx_format": int(geo.idx_format),
        "stats": {"s1": vars(st.stage1), "s2": vars(st.stage2), "s3": vars(st.stage3),
                  "exact_fallbacks": st.exact_fallbacks},
    }
    if check:
        from oracle import host as oh
        t0 = time.time()
        words = torch.empty_like(pf.fb)
        words.copy_(pf.fb)
        ref, rst, _ = oh.render_reference(scene, cam, workers=len(os.sched_getaffinity(0)),
                                          s2_cap=1 << 22, s3_cap=1 << 22)
        got = words.cpu().numpy().view(np.uint64)
        out["bit_exact_vs_oracle"] = bool(np.array_equal(got, ref))
        out["oracle_s"] = time.time() - t0
    return out


if __name__ == "__main__":
    names = [a for a in sys.argv[1:] if not a.startswith("--")] or ["A", "B", "C", "D"]
    check = "--check" in sys.argv
    for n in names:
        print(json.dumps(measure(n, check=check)), flush=True)
