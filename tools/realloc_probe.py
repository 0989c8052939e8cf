"""Does the filter's slow mode follow the vertex array's allocation?  Times
k_s1_lean_flat (CUPTI) for the same frame after re-allocating the device
positions / indices several times within one process."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_21749_b200 as cr  # noqa: E402
from paper_2604_21749_b200 import generators as gen  # noqa: E402
from paper_2604_21749_b200.pipeline import PreparedFrame  # noqa: E402


def lean_us(pf):
    for _ in range(3):
        pf.run()
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            pf.launch()
        torch.cuda.synchronize()
    v = [e.device_time_total for e in prof.events()
         if e.device_type == torch.autograd.DeviceType.CUDA and "lean" in e.name]
    return round(sum(v) / max(1, len(v)), 1)


scene, cam = gen.config_b()
dl = cr.build_draw_list(scene, cam)
pf = PreparedFrame(dl, cam, cr.RasterConfig())
res = [("initial", lean_us(pf))]
keep = []
for k in range(4):
    g = pf.geo
    keep.append(g.positions)
    g.positions = g.positions.clone()          # new allocation, same contents
    pf.frame.positions = g.positions.data_ptr()
    res.append((f"pos{k}", lean_us(pf)))
for k in range(2):
    g = pf.geo
    keep.append(g.indices)
    g.indices = g.indices.clone()
    pf.frame.indices = g.indices.data_ptr()
    res.append((f"idx{k}", lean_us(pf)))
print(json.dumps(res))
