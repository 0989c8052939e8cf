"""Resolve + downsample device time (CUDA events, median of K) on SURVEY
configs; A/B of builds through CURAST_LIB in separate processes.

    python tools/resolve_ab.py B,A,A4 lib1.so:lib2.so [K]
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(configs, K):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import numpy as np
    import torch
    import paper_2604_21749_b200 as cr
    from paper_2604_21749_b200.resolve import downsample_device, resolve_frame_device
    from frame_once import scene_for
    out = {}
    for c in configs:
        scene, cam = scene_for(c)
        dl = cr.build_draw_list(scene, cam)
        fb, _ = cr.render_draw_list(dl, cam)
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
        for k in range(K + 3):
            e = ev[k - 3] if k >= 3 else None
            if e:
                e[0].record()
            img, st = resolve_frame_device(fb, dl, cam)
            if e:
                e[1].record()
            small = downsample_device(img, cam.supersampling)
            if e:
                e[2].record()
        torch.cuda.synchronize()
        r = float(np.median([e[0].elapsed_time(e[1]) for e in ev]))
        d = float(np.median([e[1].elapsed_time(e[2]) for e in ev]))
        import hashlib
        out[c] = {"resolve_ms": r, "downsample_ms": d, "shaded": st.shaded,
                  "img": hashlib.sha256(small.cpu().numpy().tobytes()).hexdigest()[:12]}
    print(json.dumps(out))


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(sys.argv[2].split(","), int(sys.argv[3]))
        sys.exit(0)
    K = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    for lib in sys.argv[2].split(":"):
        env = dict(os.environ)
        if lib != "default":
            env["CURAST_LIB"] = lib
        r = subprocess.run([sys.executable, __file__, "--child", sys.argv[1], str(K)], env=env,
                           capture_output=True, text=True)
        print(json.dumps({"lib": lib, "out": r.stdout.strip()[-2000:], "err": r.stderr[-500:] if r.returncode else ""}), flush=True)
