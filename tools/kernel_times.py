"""Per-kernel device times of config-B frames via torch.profiler (CUPTI
activity records, no kernel serialisation), plus the frame time — used to
study process-to-process variance of the stage-1 kernels."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_21749_b200 as cr  # noqa: E402
from paper_2604_21749_b200 import generators as gen  # noqa: E402
from paper_2604_21749_b200.pipeline import PreparedFrame  # noqa: E402

scene, cam = gen.config_b()
dl = cr.build_draw_list(scene, cam)
pf = PreparedFrame(dl, cam, cr.RasterConfig())
for _ in range(5):
    pf.run()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        pf.launch()
    torch.cuda.synchronize()
times = {}
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        times.setdefault(e.name[:40], []).append(e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total)
out = {k: round(sum(v) / len(v), 1) for k, v in times.items()}
fb_ptr = pf.fb.data_ptr()
c = pf.read_counters()
from paper_2604_21749_b200 import _native as N  # noqa: E402
print(json.dumps({"us": out, "qx_slots": int(c[N.C_QX]), "qx_holes": int(c[N.C_QXHOLES]), "fb": hex(fb_ptr), "pos": hex(pf.geo.positions.data_ptr()),
                  "idx": hex(pf.geo.indices.data_ptr())}))
