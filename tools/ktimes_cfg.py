"""Per-kernel device times of one config under RasterConfig overrides:
python tools/ktimes_cfg.py <config> key=value ..."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import paper_2604_21749_b200 as cr  # noqa: E402
from paper_2604_21749_b200.pipeline import PreparedFrame  # noqa: E402
from frame_once import scene_for  # noqa: E402

name = sys.argv[1]
kw = {k: int(v) for k, v in (a.split("=") for a in sys.argv[2:])}
scene, cam = scene_for(name)
dl = cr.build_draw_list(scene, cam)
pf = PreparedFrame(dl, cam, cr.RasterConfig(**kw), fresh_fb=False)
c, _ = pf.run()
st = pf.stats(pf.read_counters(), [0] * 4)
for _ in range(3):
    pf.launch()
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(10):
        pf.launch()
    torch.cuda.synchronize()
ker = {ev.key[:40]: round(ev.device_time_total / max(1, ev.count) / 1000.0, 4)
       for ev in prof.key_averages() if ev.device_time_total > 0}
print(json.dumps({"config": name, "cfg": kw, "s1": [st.stage1.rasterized, st.stage1.forwarded,
                  st.stage1.fragments], "kernels_ms": ker}))
