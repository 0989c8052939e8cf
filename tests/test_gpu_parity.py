"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden outputs and the C oracle, bit-exact on visibility words and stats."""

import os

import numpy as np
import pytest

from oracle import host as oh
from paper_2604_21749_b200 import (CLEAR, Camera, CapacityError, RasterConfig, SceneNode,
                                   build_draw_list, render_draw_list, render_frame)
from paper_2604_21749_b200 import generators as gen
from paper_2604_21749_b200.pipeline import PreparedFrame, build_context
from scenes import (STAT_ORDER, golden_camera, golden_cfg, golden_names, golden_scene,
                    identity_camera, load_golden, mesh_from_soup, pixel_triangle_scene,
                    random_scene, stats_vector_from_frame, stats_vector_from_oracle)

pytestmark = pytest.mark.gpu

NAMES = [n for n in golden_names() if n != "classifier_unstaged"]


def _render_with_golden_ctx(g, cfg, compressed=True, use_filter=None):
    scene = golden_scene(g, compressed=compressed)
    cam = golden_camera(g)
    dl = build_draw_list(scene, cam)
    assert np.array_equal(dl.prefix_sums.astype(np.int64), g["prefix"])
    ctx = build_context(dl, cam)
    ctx.item_mv = np.ascontiguousarray(g["item_mv"])      # the reference's own matrices
    return render_draw_list(dl, cam, cfg, ctx=ctx, use_filter=use_filter)


@pytest.mark.parametrize("use_filter", [True, False])
@pytest.mark.parametrize("name", NAMES)
def test_golden_words_and_stats(name, use_filter):
    g = load_golden(name)
    if int(g["total"]) == 0:
        pytest.skip("empty")
    cfg = golden_cfg(g)
    fb, st = _render_with_golden_ctx(g, cfg, use_filter=use_filter)
    words = fb.words
    diff = np.nonzero(words != g["ref_words"])[0]
    assert diff.size == 0, f"{name}: {diff.size} differing words, first {diff[:8]}"
    got = stats_vector_from_frame(st)
    want = g["stats"][:15]
    bad = [(STAT_ORDER[i], int(got[i]), int(want[i])) for i in range(15) if got[i] != want[i]]
    assert not bad, bad
    assert st.instanced == bool(g["stats"][15])


def test_compressed_geometry_decoded_in_kernel():
    g = load_golden("compressed_sphere")
    fb_c, st_c = _render_with_golden_ctx(g, RasterConfig(), compressed=True)
    fb_u, st_u = _render_with_golden_ctx(g, RasterConfig(), compressed=False)
    assert np.array_equal(fb_c.words, g["ref_words"])
    assert np.array_equal(fb_u.words, g["ref_words"])


def test_random_scenes_seed2024_vs_oracle():
    """Criterion 1 (test_acceptance.py:49-69): 200 random scenes, GPU vs the
    sequential oracle run on this host."""
    rng = np.random.default_rng(2024)
    mism = []
    for k in range(200):
        scene, cam = random_scene(rng)
        ref, _, dl = oh.render_reference(scene, cam)
        fb, st = render_frame(scene, cam, RasterConfig())
        if not np.array_equal(fb.words, ref):
            mism.append(k)
    assert not mism, mism


def _bbox_scene(xs, ys, cam):
    return pixel_triangle_scene([(0.25, 0.25), (xs - 0.25, 0.25), (0.25, ys - 0.25)],
                                [2.0] * 3, cam)


def test_capacity_errors_report_requirement():
    cam = identity_camera(width=256, height=128)
    scene = _bbox_scene(64, 64, cam)
    m = scene[0].mesh
    m.positions = np.tile(m.positions, (3, 1))
    m.indices = np.arange(9, dtype=np.uint32)
    m.triangle_count = 3
    with pytest.raises(CapacityError, match="at least 3"):
        render_frame(scene, cam, RasterConfig(stage2_capacity=1))
    scene = _bbox_scene(130, 70, cam)
    with pytest.raises(CapacityError, match="at least 6"):
        render_frame(scene, cam, RasterConfig(stage3_capacity=2))


def test_queue_autogrow_keeps_output(monkeypatch):
    """Device queues start small and grow when a frame needs more than
    allocated but less than the reference capacity."""
    from paper_2604_21749_b200 import device as dv
    cam = identity_camera(width=256, height=128)
    scene = _bbox_scene(130, 70, cam)
    ref, _, _ = oh.render_reference(scene, cam)
    ws = dv.workspace(__import__("torch").device("cuda", 0))
    ws.q3 = None
    ws.q3_alloc = 0
    monkeypatch.setattr("paper_2604_21749_b200.pipeline.DEVICE_Q3_INITIAL", 1)
    fb, st = render_frame(scene, cam, RasterConfig())
    assert st.stage2.tiles == 6
    assert np.array_equal(fb.words, ref)


@pytest.mark.parametrize("inst_kernel", ["0", "1"])
def test_tiny_cull_and_instancing_toggles_bit_identical(inst_kernel, monkeypatch):
    """Both stage-1 routes of an instanced frame (the instanced kernel and
    the flat table over the items, pipeline._instanced_kernel_preferred)."""
    monkeypatch.setenv("CURAST_INSTANCED_KERNEL", inst_kernel)
    mesh = gen.make_tessellated_quad(300)
    cam = Camera.look_at((0.0, 0.0, 3.2), (0.0, 0.0, 0.0), width=96, height=96)
    scene = [SceneNode(mesh=mesh, transforms=[np.eye(4)])]
    fb_on, st_on = render_frame(scene, cam, RasterConfig(tiny_cull=True))
    fb_off, st_off = render_frame(scene, cam, RasterConfig(tiny_cull=False))
    assert st_on.stage1.culled_tiny / st_on.total_triangles >= 0.30
    assert np.array_equal(fb_on.words, fb_off.words)
    scene = gen.make_lantern_grid(10, 10, tris_per_mesh=10 ** 4, spacing=1.8)
    cam = Camera.look_at((0.0, 14.0, 20.0), (0.0, 0.0, 0.0), width=320, height=240)
    fi, si = render_frame(scene, cam, RasterConfig(instancing="on"))
    ff, sf = render_frame(scene, cam, RasterConfig(instancing="off"))
    assert si.instanced and not sf.instanced
    assert np.array_equal(fi.words, ff.words)
    ref, rst, _ = oh.render_reference(scene, cam)
    assert np.array_equal(fi.words, ref)
    assert np.array_equal(stats_vector_from_frame(si), stats_vector_from_oracle(rst))


def test_depth_winner_and_tie_break():
    cam = identity_camera()
    pix = [(30.25, 30.25), (40.75, 30.25), (30.25, 40.75)]
    scene = pixel_triangle_scene(pix, [2.0, 2.0, 2.0], cam)
    dup = SceneNode(mesh=mesh_from_soup(scene[0].mesh.positions.copy()), transforms=[np.eye(4)])
    scene.append(dup)
    fb, _ = render_frame(scene, cam, RasterConfig())
    covered = fb.words[fb.words != CLEAR]
    assert covered.size and ((covered & np.uint64(0xFFFFFFFFF)) == 0).all()


def _oracle_threads():
    return max(1, min(32, len(os.sched_getaffinity(0))))


def test_config_a_sphere_1m_1080p_bit_exact():
    scene, cam = gen.config_a()
    fb, st = render_frame(scene, cam, RasterConfig())
    ref, rst, _ = oh.render_reference(scene, cam, workers=_oracle_threads())
    assert np.array_equal(fb.words, ref)
    assert np.array_equal(stats_vector_from_frame(st), stats_vector_from_oracle(rst))
    assert st.stage1.forwarded == 0


def test_config_c_mixed_sizes_bit_exact():
    scene, cam = gen.config_c()
    fb, st = render_frame(scene, cam, RasterConfig())
    ref, rst, _ = oh.render_reference(scene, cam, workers=_oracle_threads(),
                                      s3_cap=1 << 22)
    assert np.array_equal(fb.words, ref)
    assert np.array_equal(stats_vector_from_frame(st), stats_vector_from_oracle(rst))
    assert st.stage2.direct > 0 and st.stage2.tiled > 0 and st.stage3.fragments > 0


@pytest.mark.slow
def test_config_b_grid_100m_4k_bit_exact_and_filter_sound():
    scene, cam = gen.config_b()
    dl = build_draw_list(scene, cam)
    fb, st = render_draw_list(dl, cam, RasterConfig())
    words = fb.words.copy()
    ref, rst, _ = oh.render_reference(scene, cam, workers=_oracle_threads(), s2_cap=1 << 20,
                                      s3_cap=1 << 20)
    assert np.array_equal(words, ref)
    assert np.array_equal(stats_vector_from_frame(st), stats_vector_from_oracle(rst))
    # exact-only path gives the same words
    fb2, st2 = render_draw_list(dl, cam, RasterConfig(), use_filter=False)
    assert np.array_equal(fb2.words, ref)
    assert st2.exact_fallbacks == dl.total_triangles


def test_filter_bound_never_violated():
    """Every vertex's fp32 projection lies within the filter's error bound of
    the exact fp64 value (curast_filter_check), on scenes with wide depth and
    magnitude ranges."""
    import ctypes
    import torch
    from paper_2604_21749_b200 import _native as N
    scenes = [gen.config_a(), gen.config_b(n=1500)]
    rng = np.random.default_rng(5)
    for _ in range(20):
        scenes.append(random_scene(rng))
    for scene, cam in scenes:
        dl = build_draw_list(scene, cam)
        if dl.total_triangles == 0:
            continue
        pf = PreparedFrame(dl, cam, RasterConfig())
        out = torch.zeros(3, dtype=torch.int64, device="cuda")
        N.check(N.lib().curast_filter_check(ctypes.byref(pf.frame), out.data_ptr(),
                                            torch.cuda.current_stream().cuda_stream), "check")
        checked, bad, worst = (int(v) for v in out.cpu())
        assert bad == 0, (checked, bad, worst / 1e6)
        assert worst < 1_000_000


def test_cuda_graph_replay_is_identical():
    """PreparedFrame.capture(): the frame as one CUDA graph gives the same
    words and counters as the launch path, frame after frame."""
    import torch
    scene, cam = gen.config_a()
    dl = build_draw_list(scene, cam)
    pf = PreparedFrame(dl, cam, RasterConfig())
    c0, _ = pf.run()
    w0 = pf.fb.clone()
    g = pf.capture()
    for _ in range(3):
        g.replay()
        c = pf.read_counters()
        assert np.array_equal(c[:16], c0[:16])
        assert torch.equal(pf.fb, w0)


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_div_shared_equals_ieee_division(mode):
    """exact.cuh div_recip / div_shared (one reciprocal refinement shared by
    the divisions by the same vertex depth) against __ddiv_rn / __drcp_rn on
    10^8 hashed operand pairs per mode: every fast-path quotient and
    reciprocal is bit-identical; the rest take the __ddiv_rn fallback."""
    import torch
    from paper_2604_21749_b200 import _native as N
    out = torch.zeros(4, dtype=torch.int64, device="cuda")
    for seed in (1, 2):
        N.check(N.lib().curast_div_check(50_000_000, seed * 7919 + mode, mode, out.data_ptr(),
                                         torch.cuda.current_stream().cuda_stream), "div_check")
    checked, bad, slow, rbad = (int(v) for v in out.cpu())
    assert checked >= 99_000_000
    assert bad == 0 and rbad == 0, (checked, bad, slow, rbad)
    if mode == 1:
        assert slow == 0          # the rasterizer's magnitudes never leave the fast path


def _vs_oracle(scene, cam, cfg=None):
    cfg = cfg or RasterConfig()
    dl = build_draw_list(scene, cam)
    fb, st = render_draw_list(dl, cam, cfg)
    ref, rst, _ = oh.render_reference(scene, cam, tiny_cull=cfg.tiny_cull,
                                      force_stage=cfg.force_stage)
    assert np.array_equal(fb.words, ref)
    if rst is not None:
        assert np.array_equal(stats_vector_from_frame(st), stats_vector_from_oracle(rst))
    return fb, st


def test_edge_cases_empty_behind_degenerate_tiny_frames():
    """Edge cases of kernels.py:49-157 through the GPU path: a scene whose
    every triangle is behind the camera (all CULL_FRUSTUM after the draw
    list keeps the node), collinear (degenerate) and zero-area triangles,
    1x1 / 3x2 / 1x64 frames, a frame with no surviving item (CLEAR, empty
    stats), and single-triangle meshes at unaligned index offsets."""
    cam = identity_camera(width=64, height=48)
    # every vertex behind the camera; the node's box straddles the near
    # plane so the draw list keeps it
    p = np.array([[0, 0, 1.0], [0.1, 0, 1.0], [0, 0.1, 1.0],
                  [-1, -1, -5.0], [1, -1, -5.0], [0, 1, 0.5]], dtype=np.float64)
    m = mesh_from_soup(p)
    _vs_oracle([SceneNode(mesh=m, transforms=[np.eye(4)])], cam)
    # degenerate: collinear and repeated vertices, in front of the camera
    pix = [(10.25, 10.25), (20.25, 20.25), (30.25, 30.25)]
    deg = pixel_triangle_scene(pix, [2.0, 2.0, 2.0], cam)
    pix2 = [(5.5, 5.5), (5.5, 5.5), (9.5, 7.5)]
    deg += pixel_triangle_scene(pix2, [3.0, 3.0, 3.0], cam)
    fb, st = _vs_oracle(deg, cam)
    assert st.stage1.culled_degenerate + st.stage1.culled_offscreen + st.stage1.culled_tiny > 0
    # tiny frames
    rng = np.random.default_rng(9)
    for w, h in ((1, 1), (3, 2), (1, 64)):
        scene, _ = random_scene(rng)
        c = Camera.look_at((0.0, 0.0, 6.0), (0.0, 0.0, 0.0), width=w, height=h)
        dl = build_draw_list(scene, c)
        if dl.total_triangles:
            _vs_oracle(scene, c)
    # nothing survives the draw-list cull: a CLEAR frame
    c = Camera.look_at((0.0, 0.0, 6.0), (0.0, 0.0, 12.0), width=32, height=16)
    scene = [SceneNode(mesh=m, transforms=[np.eye(4)])]
    dl = build_draw_list(scene, c)
    fb, st = render_draw_list(dl, c)
    assert dl.total_triangles == 0 and (fb.words == CLEAR).all() and st.fragments == 0


@pytest.mark.parametrize("force", [2, 3])
def test_abi_filter_flag_ignored_when_forcing_stages(force):
    """force_stage >= 2 forwards every triangle before the frustum and tiny
    tests (kernels.py:73-76), so the fp32 cull filter must not decide: a C-ABI
    caller that leaves frame.use_filter = 1 still gets the reference's words
    and counters (the library drops the filter itself)."""
    from paper_2604_21749_b200.pipeline import PreparedFrame
    rng = np.random.default_rng(11 + force)
    for _ in range(3):
        scene, cam = random_scene(rng)
        cfg = RasterConfig(force_stage=force)
        dl = build_draw_list(scene, cam)
        pf = PreparedFrame(dl, cam, cfg)
        pf.frame.use_filter = 1
        c, secs = pf.run()
        ref, rst, _ = oh.render_reference(scene, cam, force_stage=force)
        assert np.array_equal(pf.fb.cpu().numpy().view(np.uint64), ref)
        if rst is not None:
            assert np.array_equal(stats_vector_from_frame(pf.stats(c, secs)),
                                  stats_vector_from_oracle(rst))


@pytest.mark.parametrize("force,compressed", [(0, False), (1, False), (0, True), (1, True)])
def test_row_parallel_stage1_raster_matches_oracle(force, compressed):
    """frame.s1_row_raster = 1: the fp64 pass hands stage-1 bboxes of >= 16
    pixels / 2 rows to its warp (one row per lane, the row's serial s/t
    stepping kept, kernels.py:140-157).  Random scenes and, with force_stage 1
    (every triangle rasterized in stage 1, so large bboxes overflow the four
    per-warp slots into the thread's own loop), the same words and counters
    as the oracle."""
    from paper_2604_21749_b200 import _native as N
    from paper_2604_21749_b200.pipeline import PreparedFrame
    rng = np.random.default_rng(21 + force)
    cases = [random_scene(rng) for _ in range(4)]
    cases.append(gen.config_c(width=640, height=360))
    if compressed:
        # u16 grid positions + packed indices: the fp64 pass's u16 queue entries
        from scenes import compress_scene
        cases = [(compress_scene(sc), cam) for sc, cam in cases]
    for scene, cam in cases:
        cfg = RasterConfig(force_stage=force)
        dl = build_draw_list(scene, cam)
        pf = PreparedFrame(dl, cam, cfg)
        pf.frame.s1_row_raster = 1
        pf.launch()
        c = pf.read_counters()
        if int(c[N.C_QX]) > pf.qx_alloc or int(c[0]) > pf.q2_alloc or int(c[1]) > pf.q3_alloc:
            pf.run()                      # sized the queues (resets the flag)
            pf.frame.s1_row_raster = 1
            pf.launch()
            c = pf.read_counters()
        ref, rst, _ = oh.render_reference(scene, cam, force_stage=force)
        assert np.array_equal(pf.fb.cpu().numpy().view(np.uint64), ref)
        if rst is not None:
            assert np.array_equal(stats_vector_from_frame(pf.stats(c, [0.0] * 4)),
                                  stats_vector_from_oracle(rst))

