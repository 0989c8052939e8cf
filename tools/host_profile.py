"""cProfile of the public per-frame call (render_draw_list + words) on
config B: where the host part of the end-to-end frame goes."""
import cProfile
import os
import pstats
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_21749_b200 as cr  # noqa: E402
from paper_2604_21749_b200 import generators as gen  # noqa: E402

scene, cam = gen.config_b(n=int(sys.argv[1]) if len(sys.argv) > 1 else 7071)
dl = cr.build_draw_list(scene, cam)
cfg = cr.RasterConfig()
for _ in range(5):
    fb, st = cr.render_draw_list(dl, cam, cfg)
    w = fb.words
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    fb, st = cr.render_draw_list(dl, cam, cfg)
    w = fb.words
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
