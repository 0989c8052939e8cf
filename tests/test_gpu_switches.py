"""Every stage-1 experiment switch (read once at library load, so each runs in
a subprocess) renders bit-exact frames: golden fixtures, random scenes, an
instanced scene and the compressed sphere against the stored reference
words / the oracle."""

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
print("BAD", bad)
sys.exit(1 if bad else 0)
"""


@pytest.mark.parametrize("env", [
    {"CURAST_PROVE": "1"},
    {"CURAST_S1": "leanT"},
    {"CURAST_S1": "leanI"},
    {"CURAST_S1": "nomesh", "CURAST_MESHLETS": "1"},
    {"CURAST_MESHLETS": "1"},
    {"CURAST_SLICES": "2"},
    {"CURAST_S1": "cull"},
    {"CURAST_S1": "split"},
    {"CURAST_XMINB": "8"},
    {"CURAST_INSTANCED_KERNEL": "1"},
    {"CURAST_S1": "strip"},
    {"CURAST_S1": "plain"},
    {"CURAST_S1": "pfi"},
    {"CURAST_S1": "die"},
    {"CURAST_S1": "fused", "CURAST_XMINB": "4"},
], ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_switch_is_bit_exact(env):
    script = SCRIPT % {"root": ROOT, "tests": os.path.join(ROOT, "tests")}
    r = subprocess.run([sys.executable, "-c", script], env={**os.environ, **env},
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("env", [{"CURAST_ILV": "1"}, {"CURAST_ILV": "0"}],
                         ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_index_step_layout_is_bit_exact(env):
    test_switch_is_bit_exact(env)
