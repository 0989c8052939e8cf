"""Per-frame benchmark protocol of the reference's ``trirast bench``
(cli.py:115-223) on the GPU path.

    python -m paper_2604_21749_b200.benchcli A --toggle superSampling --frames 60 \\
        --output rows.csv

Same rows, warm-up, guard and columns as the reference:

* rows: the base configuration, or the rows of one toggle — ``tinyCull``
  (on / off), ``instancing`` (on / off), ``workers`` (1 / 2 / 4 / 8: accepted
  for parity; the GPU path ignores the worker count, cli.py:121-124),
  ``superSampling`` (1 / 2 / 4) (cli.py:115-141);
* per row 5 warm-up frames, then the SHA-256 of the visibility words: every
  timing-only row must reproduce the first row's hash, else the run fails
  (cli.py:160-170);
* ``frames`` (default 60, cli.py:396) frames of render_draw_list +
  resolve_frame + downsample; columns stage1Ms / stage2Ms / stage3Ms (CUDA
  events around each stage), resolveMs (CUDA events around resolve +
  downsample: device time only, the host setup is prepared once),
  totalMs (wall clock of the whole frame, host included, as the reference),
  fragments and stage-1 culls — the mean over the frames;
* a table on stdout and optionally the same rows as CSV.

Scenes are the SURVEY §8(d) configs by name (A, B, C, D, E) — the
reference's JSON scene files are host tooling, out of scope.
"""

from __future__ import annotations

import argparse
import csv
import hashlib
import sys
import time

COLS = ["scene", "config", "visibleTriangles", "stage1Ms", "stage2Ms", "stage3Ms",
        "resolveMs", "totalMs", "fragments", "culled"]
TOGGLES = ("tinyCull", "workers", "instancing", "superSampling")


def bench_rows(camera, cfg, toggle=None):
    """(label, camera, cfg, timing_only) rows of a toggle (cli.py:115-141)."""
    from .config import RasterConfig
    from .scene import Camera
    if toggle is None:
        return [("base", camera, cfg, True)]
    if toggle == "tinyCull":
        return [("tinyCull=on", camera, RasterConfig(**{**cfg.__dict__, "tiny_cull": True}), True),
                ("tinyCull=off", camera, RasterConfig(**{**cfg.__dict__, "tiny_cull": False}), True)]
    if toggle == "workers":
        return [(f"workers={n}", camera, RasterConfig(**{**cfg.__dict__, "workers": n}), True)
                for n in (1, 2, 4, 8)]
    if toggle == "instancing":
        return [(f"instancing={m}", camera, RasterConfig(**{**cfg.__dict__, "instancing": m}), True)
                for m in ("on", "off")]
    if toggle == "superSampling":
        rows = []
        for ss in (1, 2, 4):
            cam = Camera(position=camera.position, view_transform=camera.view_transform,
                         fovy=camera.fovy, aspect=camera.aspect, near=camera.near,
                         image_width=camera.image_width, image_height=camera.image_height,
                         supersampling=ss)
            rows.append((f"superSampling={ss}", cam, cfg, False))
        return rows
    raise ValueError(f"unknown toggle {toggle!r} (one of {', '.join(TOGGLES)})")


class FramebufferHashError(RuntimeError):
    """A timing-only toggle changed the visibility buffer (cli.py:163-170)."""


def bench(scene, camera, cfg=None, shading=None, *, toggle=None, frames=60, scene_name="scene"):
    """Run the protocol; returns the report rows (dicts keyed by COLS)."""
    import torch

    from .config import RasterConfig, ShadingConfig
    from .pipeline import render_draw_list
    from .resolve import downsample_device, resolve_frame_device
    from .scene import build_draw_list
    cfg = cfg or RasterConfig()
    shading = shading or ShadingConfig()
    reports, timing_hash = [], None
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for label, cam, row_cfg, timing_only in bench_rows(camera, cfg, toggle):
        draw_list = build_draw_list(scene, cam)
        for _ in range(5):                       # warm-up (geometry upload, preparation)
            fb, stats = render_draw_list(draw_list, cam, row_cfg)
            img, _ = resolve_frame_device(fb, draw_list, cam, shading)
            downsample_device(img, cam.supersampling)
        digest = hashlib.sha256(fb.words.tobytes()).hexdigest()
        if timing_only:
            timing_hash = timing_hash or digest
            if digest != timing_hash:
                raise FramebufferHashError(
                    f"framebuffer hash changed under timing-only toggle {label!r}")
        sums = dict(stage1=0.0, stage2=0.0, stage3=0.0, resolve=0.0, total=0.0)
        for _ in range(frames):
            t0 = time.perf_counter()
            fb, stats = render_draw_list(draw_list, cam, row_cfg)
            ev[0].record()
            img, _ = resolve_frame_device(fb, draw_list, cam, shading)
            downsample_device(img, cam.supersampling)
            ev[1].record()
            ev[1].synchronize()
            sums["total"] += time.perf_counter() - t0
            sums["stage1"] += stats.stage1_s
            sums["stage2"] += stats.stage2_s
            sums["stage3"] += stats.stage3_s
            sums["resolve"] += ev[0].elapsed_time(ev[1]) * 1e-3
        s1 = stats.stage1
        reports.append({
            "scene": scene_name, "config": label,
            "visibleTriangles": int(draw_list.total_triangles),
            "stage1Ms": 1e3 * sums["stage1"] / frames, "stage2Ms": 1e3 * sums["stage2"] / frames,
            "stage3Ms": 1e3 * sums["stage3"] / frames, "resolveMs": 1e3 * sums["resolve"] / frames,
            "totalMs": 1e3 * sums["total"] / frames,
            "fragments": int(stats.fragments),
            "culled": int(s1.culled_frustum + s1.culled_offscreen + s1.culled_tiny
                          + s1.culled_backface + s1.culled_degenerate),
        })
    return reports


def format_table(reports) -> str:
    fmt = {float: "{:.3f}".format, int: "{:d}".format}
    table = [[fmt.get(type(r[c]), str)(r[c]) for c in COLS] for r in reports]
    widths = [max(len(c), *(len(row[i]) for row in table)) for i, c in enumerate(COLS)]
    lines = ["  ".join(c.ljust(w) for c, w in zip(COLS, widths))]
    lines += ["  ".join(v.rjust(w) for v, w in zip(row, widths)) for row in table]
    return "\n".join(lines)


def write_csv(reports, path):
    with open(path, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=COLS)
        w.writeheader()
        w.writerows(reports)


def scene_by_name(name: str):
    from . import generators as gen
    table = {"A": gen.config_a, "B": gen.config_b, "C": gen.config_c, "D": gen.config_d,
             "E": lambda: gen.config_e(n_meshes=64, on_device=True)}
    if name not in table:
        raise ValueError(f"unknown scene {name!r} (A, B, C, D, E)")
    return table[name]()


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="benchcli", description=__doc__.splitlines()[0])
    ap.add_argument("scene", help="SURVEY config name: A, B, C, D or E (64 meshes)")
    ap.add_argument("--toggle", choices=TOGGLES)
    ap.add_argument("--frames", type=int, default=60)
    ap.add_argument("--output", help="CSV file for the rows")
    args = ap.parse_args(argv)
    scene, cam = scene_by_name(args.scene)
    try:
        reports = bench(scene, cam, toggle=args.toggle, frames=args.frames,
                        scene_name=args.scene)
    except FramebufferHashError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    print(format_table(reports))
    if args.output:
        write_csv(reports, args.output)
        print(f"wrote {args.output}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
