"""Frame time through the launch path vs one CUDA-graph replay per frame
(PreparedFrame.capture), configs A and B, CUDA events over 50 frames."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_21749_b200 as cr  # noqa: E402
from paper_2604_21749_b200 import generators as gen  # noqa: E402
from paper_2604_21749_b200.pipeline import PreparedFrame  # noqa: E402


def timed(fn, k=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


for name, (scene, cam) in (("A", gen.config_a()), ("C", gen.config_c()), ("B", gen.config_b())):
    dl = cr.build_draw_list(scene, cam)
    pf = PreparedFrame(dl, cam, cr.RasterConfig())
    pf.run()
    t_launch = timed(pf.launch)
    g = pf.capture()
    t_graph = timed(g.replay)
    print(json.dumps({"config": name, "launch_ms": round(t_launch, 4), "graph_ms": round(t_graph, 4)}))
