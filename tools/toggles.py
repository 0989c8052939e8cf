"""Bench toggles in the spirit of the reference's `bench` command
(cli.py:106-223: tinyCull on/off, instancing on/off, superSampling 1/2/4),
reproducing the directions of the paper's toggle tables on the B200.

    python tools/toggles.py [--frames N] [--out profiles/rNN_toggles.jsonl]

Per row: stage 1/2/3 device ms (CUDA events, mean over N frames after
warm-up), resolve ms (GPU resolve + downsample of the supersampled image),
fragments and stage-1 culls.  Timing-only toggles (tinyCull, instancing) must
leave the visibility buffer unchanged: the sha256 of the words is checked per
scene, as the reference's bench does.
"""

import argparse
import hashlib
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2604_21749_b200 as cr  # noqa: E402
from paper_2604_21749_b200 import generators as gen  # noqa: E402
from paper_2604_21749_b200.pipeline import PreparedFrame  # noqa: E402
from paper_2604_21749_b200.resolve import downsample_device, resolve_frame_device  # noqa: E402
from paper_2604_21749_b200.scene import Camera  # noqa: E402


def run_row(scene_name, label, scene, cam, cfg, frames):
    dl = cr.build_draw_list(scene, cam)
    pf = PreparedFrame(dl, cam, cfg)
    for _ in range(3):
        c, secs = pf.run()
    acc = np.zeros(4)
    for _ in range(frames):
        c, secs = pf.run()
        acc += np.asarray(secs)
    st = pf.stats(c, secs)
    fb = cr.Framebuffer(pf.width, pf.height, device_words=pf.fb)
    digest = hashlib.sha256(fb.words.tobytes()).hexdigest()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    resolve_frame_device(fb, dl, cam)
    ev0.record()
    for _ in range(frames):
        img, _ = resolve_frame_device(fb, dl, cam)
        downsample_device(img, cam.supersampling)
    ev1.record()
    torch.cuda.synchronize()
    s1 = st.stage1
    culls = (s1.culled_frustum + s1.culled_offscreen + s1.culled_tiny + s1.culled_backface
             + s1.culled_degenerate)
    ms = acc / frames * 1e3
    return {"scene": scene_name, "config": label, "visibleTriangles": int(dl.total_triangles),
            "stage1Ms": ms[1], "stage2Ms": ms[2], "stage3Ms": ms[3], "clearMs": ms[0],
            "resolveMs": ev0.elapsed_time(ev1) / frames,
            "totalMs": float(ms.sum()) + ev0.elapsed_time(ev1) / frames,
            "fragments": int(st.fragments), "culled": int(culls), "sha256": digest[:16]}


def with_ss(cam, ss):
    return Camera(position=cam.position, view_transform=cam.view_transform, fovy=cam.fovy,
                  aspect=cam.aspect, near=cam.near, image_width=cam.image_width,
                  image_height=cam.image_height, supersampling=ss)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=20)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rows = []
    base = cr.RasterConfig()
    on = cr.RasterConfig(**{**base.__dict__, "tiny_cull": True})
    off = cr.RasterConfig(**{**base.__dict__, "tiny_cull": False})
    for name, (scene, cam) in (("A", gen.config_a()), ("C", gen.config_c())):
        r = [run_row(name, "tinyCull=on", scene, cam, on, args.frames),
             run_row(name, "tinyCull=off", scene, cam, off, args.frames)]
        assert r[0]["sha256"] == r[1]["sha256"], "tiny cull changed the image"
        rows += r
        # supersampling changes the image (not timing-only), 1080p/4K internal
        for ss in (1, 2, 4):
            c2 = with_ss(cam, ss)
            if c2.internal_width * c2.internal_height > 3840 * 2160 * 4:
                continue
            rows.append(run_row(name, f"superSampling={ss}", scene, c2, base, args.frames))
    scene, cam = gen.config_d()
    r = [run_row("D", f"instancing={m}", scene, cam,
                 cr.RasterConfig(**{**base.__dict__, "instancing": m}), max(3, args.frames // 4))
         for m in ("on", "off")]
    assert r[0]["sha256"] == r[1]["sha256"], "instancing changed the image"
    rows += r
    cols = ["scene", "config", "visibleTriangles", "stage1Ms", "stage2Ms", "stage3Ms",
            "resolveMs", "totalMs", "fragments", "culled"]
    print("  ".join(cols))
    for row in rows:
        print("  ".join(f"{row[c]:.3f}" if isinstance(row[c], float) else str(row[c]) for c in cols))
    if args.out:
        with open(args.out, "w") as fh:
            for row in rows:
                fh.write(json.dumps(row) + "\n")


if __name__ == "__main__":
    main()
