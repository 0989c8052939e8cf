"""Render one SURVEY config a few times through the default path (for ncu
captures: ``ncu -k regex:... python tools/frame_once.py C``).

    python tools/frame_once.py <A|B|C|D|Bq|Dq|A4> [frames]

A4 = config A at supersampling 4 (7680x4320 internal, ~5.5 M fragments):
the fragment-heavy case for the visibility-buffer atomicMin."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import paper_2604_21749_b200 as cr  # noqa: E402
from paper_2604_21749_b200 import generators as gen  # noqa: E402
from paper_2604_21749_b200.pipeline import PreparedFrame  # noqa: E402


def scene_for(name):
    if name == "A4":
        scene, cam = gen.config_a()
        cam = cr.Camera(position=cam.position, view_transform=cam.view_transform, fovy=cam.fovy,
                        aspect=cam.aspect, near=cam.near, image_width=cam.image_width,
                        image_height=cam.image_height, supersampling=4)
        return scene, cam
    from configs import build
    return build(name)


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "C"
    frames = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    scene, cam = scene_for(name)
    dl = cr.build_draw_list(scene, cam)
    pf = PreparedFrame(dl, cam, cr.RasterConfig(), fresh_fb=False)
    c, _ = pf.run()
    for _ in range(frames):
        pf.launch()
    torch.cuda.synchronize()
    st = pf.stats(pf.read_counters(), [0.0] * 4)
    print(name, st.summary().splitlines()[1:3])
