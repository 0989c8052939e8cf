"""The meshlet stage-1 kernel (k_s1_mesh, CURAST_MESHLETS=1) against the
oracle: golden fixtures, random scenes, meshlets over the u8 vertex limit
(RAW half-meshlet batches) and sharded work ranges that split meshlets."""

import numpy as np
import pytest

from oracle import host as oh
from paper_2604_21749_b200 import RasterConfig, build_draw_list, render_draw_list, render_frame
from paper_2604_21749_b200 import device as dv
from paper_2604_21749_b200 import generators as gen
from paper_2604_21749_b200.scene import Camera, SceneNode
from scenes import (golden_camera, golden_cfg, golden_names, golden_scene, load_golden,
                    mesh_from_soup, random_scene, stats_vector_from_frame)

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _meshlets_on(monkeypatch):
    monkeypatch.setenv("CURAST_MESHLETS", "1")
    dv.drop_device_copies()
    yield
    dv.drop_device_copies()


def _check(scene, cam, cfg=None, work_range=None):
    cfg = cfg or RasterConfig()
    dl = build_draw_list(scene, cam)
    fb, st = render_draw_list(dl, cam, cfg)
    ref, _, _ = oh.render_reference(scene, cam)
    assert np.array_equal(fb.words, ref)
    return dl, st


def test_meshlets_built_and_used():
    scene, cam = gen.config_a()
    dl = build_draw_list(scene, cam)
    geo = dv.scene_geometry([dl.items[0].mesh], __import__("torch").device("cuda"))
    assert geo.ml_voff is not None and geo.ml_voff.numel() > 1
    fb, _ = render_draw_list(dl, cam, RasterConfig())
    ref, _, _ = oh.render_reference(scene, cam, workers=8)
    assert np.array_equal(fb.words, ref)


@pytest.mark.parametrize("name", [n for n in golden_names() if n != "classifier_unstaged"][:24])
def test_golden_through_meshlets(name):
    g = load_golden(name)
    if int(g["total"]) == 0:
        pytest.skip("empty")
    fb, st = render_frame(golden_scene(g, compressed=False), golden_camera(g), golden_cfg(g))
    assert np.array_equal(fb.words, g["ref_words"])


def test_random_scenes_through_meshlets():
    rng = np.random.default_rng(7)
    for _ in range(40):
        scene, cam = random_scene(rng)
        fb, _ = render_frame(scene, cam, RasterConfig())
        ref, _, _ = oh.render_reference(scene, cam)
        assert np.array_equal(fb.words, ref)


def test_overflow_meshlets_use_raw_batches():
    """A triangle soup with scattered indices: every meshlet lists > 256
    vertices, so the kernel runs the RAW half-meshlet path."""
    rng = np.random.default_rng(3)
    cam = Camera.look_at((0.0, 0.0, 3.0), (0.0, 0.0, 0.0), width=320, height=240)
    V = 3000
    pos = rng.uniform(-1.0, 1.0, size=(V, 3)).astype(np.float32).astype(np.float64)
    pos[:, 2] *= 0.2
    idx = rng.integers(0, V, size=3 * 2000).astype(np.uint32)
    mesh = mesh_from_soup(pos, idx)
    voff, _, _ = dv.build_meshlets(__import__("torch").from_numpy(idx.view(np.int32)),
                                   mesh.triangle_count)
    assert int((voff[1:] - voff[:-1]).min()) > 256
    _check([SceneNode(mesh=mesh, transforms=[np.eye(4)])], cam)


def test_sharded_ranges_split_meshlets():
    scene, cam = gen.config_a()
    dl = build_draw_list(scene, cam)
    ref, _, _ = oh.render_reference(scene, cam, workers=8)
    T = dl.total_triangles
    cuts = [0, 1000, 1000 + 126 * 37 + 5, T // 2 + 3, T]
    acc = np.full(ref.shape, np.iinfo(np.uint64).max, dtype=np.uint64)
    for a, b in zip(cuts[:-1], cuts[1:]):
        fb, _ = render_draw_list(dl, cam, RasterConfig(), work_range=(a, b))
        acc = np.minimum(acc, fb.words)
    assert np.array_equal(acc, ref)
