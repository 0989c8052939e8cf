"""Per-frame stage-1 time of config B over a long run (CUDA events), with
NVML SM / memory clocks, power and temperatures sampled every 10 frames:
finds the filter's slow phases.  python tools/phase_trace.py [frames]"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import paper_2604_21749_b200 as cr  # noqa: E402
from paper_2604_21749_b200.pipeline import PreparedFrame  # noqa: E402
from frame_once import scene_for  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 600
import pynvml  # noqa: E402
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
scene, cam = scene_for("B")
dl = cr.build_draw_list(scene, cam)
pf = PreparedFrame(dl, cam, cr.RasterConfig(), fresh_fb=False)
pf.run()
t0 = time.time()
rows = []
for k in range(T):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    pf.launch(events=ev)
    if k % 10 == 0:
        torch.cuda.synchronize()
        s = {"sm": pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
             "mem": pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
             "pw": pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
             "t": pynvml.nvmlDeviceGetTemperature(h, pynvml.NVML_TEMPERATURE_GPU)}
    else:
        s = None
    rows.append((ev, s, time.time() - t0))
torch.cuda.synchronize()
out = []
for k, (ev, s, t) in enumerate(rows):
    out.append({"k": k, "t": round(t, 3), "s1": round(ev[1].elapsed_time(ev[2]), 4), **(s or {})})
s1 = np.array([o["s1"] for o in out])
print(json.dumps({"n": T, "median": float(np.median(s1)), "p10": float(np.percentile(s1, 10)),
                  "p90": float(np.percentile(s1, 90)), "slow_frac": float(np.mean(s1 > 0.70))}))
for o in out:
    print(json.dumps(o))
