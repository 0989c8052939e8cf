"""GPU debug views (resolve.debug_view, k_debug_view) against the reference's
resolvepass.debug_view images of golden scenes (make_golden.py debug).
meshID / stageID / bboxSize are categorical and must match exactly; depth
greys are log-scaled in fp64 (CUDA log vs libm: within 1 level)."""

import os

import numpy as np
import pytest

from paper_2604_21749_b200 import build_draw_list, render_frame
from paper_2604_21749_b200.resolve import debug_view
from scenes import GOLDEN, golden_camera, golden_cfg, golden_scene, load_golden

pytestmark = pytest.mark.gpu

D = np.load(os.path.join(GOLDEN, "debug_views.npz"))
NAMES = sorted({k.split("__")[0] for k in D.files})


@pytest.mark.parametrize("name", NAMES)
def test_debug_views_match_reference(name):
    g = load_golden(name)
    scene, cam, cfg = golden_scene(g), golden_camera(g), golden_cfg(g)
    fb, _ = render_frame(scene, cam, cfg)
    dl = build_draw_list(scene, cam)
    for mode in ("meshID", "stageID", "bboxSize"):
        img = debug_view(fb, dl, cam, mode, cfg)
        want = D[f"{name}__{mode}"]
        assert img.shape == want.shape
        assert np.array_equal(img, want), (mode, int((img != want).any(axis=2).sum()))
    img = debug_view(fb, dl, cam, "depth", cfg).astype(np.int16)
    want = D[f"{name}__depth"].astype(np.int16)
    assert np.abs(img - want).max() <= 1
    assert (img != want).any(axis=2).mean() < 1e-3


def test_unknown_mode_raises():
    g = load_golden("classifier")
    scene, cam = golden_scene(g), golden_camera(g)
    fb, _ = render_frame(scene, cam)
    with pytest.raises(ValueError, match="unknown debug view mode"):
        debug_view(fb, build_draw_list(scene, cam), cam, "normals")
