"""Per-process spread of the config-B stage-1 time: P child processes, each
timing K frames (CUDA events) and then 5 frames under torch.profiler for
per-kernel device times, with the SM / memory clocks (NVML) at that point.

    python tools/bimodal_procs.py [P] [K]
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(K):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import numpy as np
    import torch
    import paper_2604_21749_b200 as cr
    from paper_2604_21749_b200.pipeline import PreparedFrame
    from frame_once import scene_for
    scene, cam = scene_for("B")
    dl = cr.build_draw_list(scene, cam)
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
    clocks = {}
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        clocks = {"sm": pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                  "mem": pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM)}
    except Exception as e:  # noqa: BLE001
        clocks = {"err": str(e)[:80]}
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(5):
            pf.launch()
        torch.cuda.synchronize()
    ker = {}
    for ev in prof.key_averages():
        if "k_s1" in ev.key:
            ker[ev.key[:40]] = round(ev.device_time_total / max(1, ev.count) / 1000.0, 4)
    print(json.dumps({"stage1_ms": round(s1, 4), "kernels_ms": ker, "clocks": clocks,
                      "fb": hex(pf.fb.data_ptr()), "qx": hex(pf.ws.qx.data_ptr())}), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child(int(sys.argv[2]))
        sys.exit(0)
    P = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    for p in range(P):
        r = subprocess.run([sys.executable, __file__, "--child", str(K)], capture_output=True,
                           text=True)
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        print(line[-1] if line else json.dumps({"err": r.stderr[-300:]}), flush=True)
