"""One frame + 3 resolves of a SURVEY config (ncu target): python tools/resolve_once.py B"""
import sys, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests"); sys.path.insert(0, "tools")
import paper_2604_21749_b200 as cr
from paper_2604_21749_b200.resolve import resolve_frame_device, downsample_device
from frame_once import scene_for
scene, cam = scene_for(sys.argv[1])
dl = cr.build_draw_list(scene, cam)
fb, st = cr.render_draw_list(dl, cam)
for _ in range(3):
    img, rs = resolve_frame_device(fb, dl, cam)
    downsample_device(img, cam.supersampling)
torch.cuda.synchronize()
print(rs)
