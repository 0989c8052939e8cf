"""Where the time of one public render_draw_list + Framebuffer.words call
goes (config B), and the resolve pass at 4K.  Prints one JSON line."""

import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2604_21749_b200 as cr  # noqa: E402
from paper_2604_21749_b200 import generators as gen  # noqa: E402
from paper_2604_21749_b200.pipeline import PreparedFrame, build_context  # noqa: E402
from paper_2604_21749_b200.resolve import downsample_device, resolve_frame_device  # noqa: E402


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3, out


def main():
    scene, cam = gen.config_b()
    dl = cr.build_draw_list(scene, cam)
    cfg = cr.RasterConfig()
    res = {}
    res["build_context_ms"], ctx = t(lambda: build_context(dl, cam))
    res["prepare_ms"], pf = t(lambda: PreparedFrame(dl, cam, cfg, ctx))
    res["run_ms"], _ = t(lambda: pf.run(timed=False))
    res["render_draw_list_ms"], fbst = t(lambda: cr.render_draw_list(dl, cam, cfg))
    fb = fbst[0]

    def rd():
        f2 = cr.Framebuffer(fb.width, fb.height, device_words=fb.device_words)
        return f2.words
    res["words_d2h_ms"], _ = t(rd)
    res["e2e_ms"], _ = t(lambda: cr.render_draw_list(dl, cam, cfg)[0].words)
    # resolve pass (flat shading) + 2x downsample on the 4K frame
    res["resolve_ms"], img = t(lambda: resolve_frame_device(fb, dl, cam)[0])
    res["downsample2_ms"], _ = t(lambda: downsample_device(img, 2))
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(10):
        resolve_frame_device(fb, dl, cam)
    ev1.record()
    torch.cuda.synchronize()
    res["resolve_device_ms_incl_host"] = ev0.elapsed_time(ev1) / 10
    print(json.dumps(res))


if __name__ == "__main__":
    main()
