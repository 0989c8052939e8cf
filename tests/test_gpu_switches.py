"""Every stage-1 route the host can select renders bit-exact frames: the
streamed flat filter (k_s1_v2), the instanced kernel (k_s1i_v2, default for
instanced frames) or the flat table for them (CURAST_INSTANCED_KERNEL=0),
and the no-filter route (CURAST_FILTER=0: every triangle through the fp64 pass) —
golden fixtures, random scenes and a grid against the stored reference words
/ the oracle.  The routes are chosen on the host when a frame is prepared, so
each runs in its own process."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, %(root)r); sys.path.insert(0, %(tests)r)
from oracle import host as oh
from paper_2604_21749_b200 import RasterConfig, render_frame, render_draw_list, build_draw_list
from paper_2604_21749_b200 import generators as gen
from scenes import golden_names, load_golden, golden_scene, golden_camera, golden_cfg, random_scene
bad = []
for name in [n for n in golden_names() if n != "classifier_unstaged"][::3]:
    g = load_golden(name)
    if int(g["total"]) == 0:
        continue
    fb, _ = render_frame(golden_scene(g), golden_camera(g), golden_cfg(g))
    if not np.array_equal(fb.words, g["ref_words"]):
        bad.append(name)
rng = np.random.default_rng(5)
for k in range(25):
    scene, cam = random_scene(rng)
    fb, _ = render_frame(scene, cam, RasterConfig())
    if not np.array_equal(fb.words, oh.render_reference(scene, cam)[0]):
        bad.append("random%%d" %% k)
scene, cam = gen.config_b(n=700)
fb, _ = render_frame(scene, cam, RasterConfig())
if not np.array_equal(fb.words, oh.render_reference(scene, cam, workers=8)[0]):
    bad.append("grid700")
scene = gen.make_lantern_grid(6, 5, tris_per_mesh=20000, spacing=1.8, f32=True)
cam = gen.Camera.look_at((0.0, 9.0, 13.0), (0.0, 0.0, 0.0), width=640, height=480)
fb, _ = render_frame(scene, cam, RasterConfig())
if not np.array_equal(fb.words, oh.render_reference(scene, cam, workers=8)[0]):
    bad.append("lanterns")
print("BAD", bad)
sys.exit(1 if bad else 0)
"""


@pytest.mark.parametrize("env", [
    {},
    {"CURAST_INSTANCED_KERNEL": "1"},
    {"CURAST_INSTANCED_KERNEL": "0"},
    {"CURAST_FILTER": "0"},
], ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()) or "default")
def test_route_is_bit_exact(env):
    script = SCRIPT % {"root": ROOT, "tests": os.path.join(ROOT, "tests")}
    r = subprocess.run([sys.executable, "-c", script], env={**os.environ, **env},
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
