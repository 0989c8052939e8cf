"""Is the config-B stage-1 time bimodal per allocation?  In one process:
per trial, fresh workspace buffers (counters, queues, VB) behind a spacer
allocation of random size (and, every other trial, re-uploaded geometry);
median stage-1 ms over K frames, with the buffers' device addresses.

    python tools/bimodal.py [trials] [K] [config]
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import paper_2604_21749_b200 as cr  # noqa: E402
from paper_2604_21749_b200 import device as dv  # noqa: E402
from paper_2604_21749_b200.pipeline import PreparedFrame  # noqa: E402
from frame_once import scene_for  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 8
K = int(sys.argv[2]) if len(sys.argv) > 2 else 15
name = sys.argv[3] if len(sys.argv) > 3 else "B"
scene, cam = scene_for(name)
dl = cr.build_draw_list(scene, cam)
meshes = list({id(it.mesh): it.mesh for it in dl.items}.values())
rng = np.random.default_rng(1)
keep = []
for t in range(T):
    if t % 2 == 1:
        dv.drop_device_copies(meshes)
    dv._workspaces.clear()
    keep.append(torch.empty(int(rng.integers(1, 64)) << 20, dtype=torch.uint8, device="cuda"))
    pf = PreparedFrame(dl, cam, cr.RasterConfig(), fresh_fb=False)
    pf.run()
    for _ in range(3):
        pf.launch()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(K)]
    for k in range(K):
        pf.launch(events=evs[k])
    torch.cuda.synchronize()
    s1 = float(np.median([e[1].elapsed_time(e[2]) for e in evs]))
    ws = pf.ws
    g = dv.scene_geometry(meshes, torch.device("cuda")).meshes[0]
    print(json.dumps({"trial": t, "reupload": t % 2 == 1, "stage1_ms": round(s1, 4),
                      "counters": hex(ws.counters.data_ptr()), "qx": hex(ws.qx.data_ptr()),
                      "fb": hex(pf.fb.data_ptr()), "pos": hex(g.positions.data_ptr()),
                      "idx": hex(g.indices.data_ptr())}), flush=True)
