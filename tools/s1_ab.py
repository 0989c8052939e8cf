"""A/B of stage-1 routes / builds on one config: per variant, in its own
process, stage-1 / frame ms over K frames (CUDA events, geometry resident),
the frame's counters, and whether the words equal the first variant's.
A variant is "default" or comma-free env assignments joined by '+', e.g.
CURAST_ILV=1 or CURAST_LIB=/path/to/libcurast_b200.so (an A/B build).

    python tools/s1_ab.py B default:CURAST_INSTANCED_KERNEL=0 [K] [rounds]
"""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(config, K):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import numpy as np
    import torch
    import paper_2604_21749_b200 as cr
    from paper_2604_21749_b200.pipeline import PreparedFrame
    from frame_once import scene_for
    if os.environ.get("AB_CHUNK"):                       # override the host's chunk choice
        import paper_2604_21749_b200.pipeline as _pl
        _c = int(os.environ["AB_CHUNK"])
        _pl._choose_chunk = lambda work, cmax, q, target: _c
    scene, cam = scene_for(config)
    dl = cr.build_draw_list(scene, cam)
    pf = PreparedFrame(dl, cam, cr.RasterConfig(), fresh_fb=False)
    c, _ = pf.run()
    if os.environ.get("AB_ROW_RASTER") is not None:      # override the host's choice
        pf.frame.s1_row_raster = int(os.environ["AB_ROW_RASTER"])
    for _ in range(3):
        pf.launch()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(K)]
    for k in range(K):
        pf.launch(events=evs[k])
    torch.cuda.synchronize()
    st = np.median([[e[i].elapsed_time(e[i + 1]) for i in range(4)] for e in evs], axis=0)
    fr = float(np.median([e[0].elapsed_time(e[4]) for e in evs]))
    c = pf.read_counters()
    h = hashlib.sha256(pf.fb.cpu().numpy().tobytes()).hexdigest()[:16]
    from scenes import stats_vector_from_frame
    sv = stats_vector_from_frame(pf.stats(c, [0] * 4)).tolist()
    print(json.dumps({"frame_ms": fr, "stage1_ms": float(st[1]), "stage2_ms": float(st[2]),
                      "stage3_ms": float(st[3]), "words": h, "stats": sv}))


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(sys.argv[2], int(sys.argv[3]))
        sys.exit(0)
    config = sys.argv[1]
    modes = sys.argv[2].split(":")
    K = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    ref = None
    for r in range(rounds):
        for m in modes:
            env = dict(os.environ)
            if m != "default":
                env.update(kv.split("=", 1) for kv in m.split("+"))
            out = subprocess.run([sys.executable, __file__, "--child", config, str(K)], env=env,
                                 capture_output=True, text=True)
            if out.returncode:
                print(json.dumps({"mode": m, "error": out.stderr[-800:]}), flush=True)
                continue
            d = json.loads(out.stdout.strip().splitlines()[-1])
            if ref is None:
                ref = (d["words"], d["stats"])
            d["same_words"] = d["words"] == ref[0]
            d["same_stats"] = d["stats"] == ref[1]
            d.update(mode=m, config=config, round=r)
            print(json.dumps(d), flush=True)
