"""GPU parity on the SURVEY §8(d) configs the round-1 suite only checked in
scratch runs (D, Bq, Dq: words AND FrameStats against the C oracle), on
partial work ranges through the default stage-1 kernels (the sort-last
shards, cut at unaligned and chunk-straddling offsets), and on the
reference's own RenderContext passed as ``ctx=`` (pipeline.py:68-84).

Reference behaviour matched: bit-identity of the visibility buffer across
worker counts and work splits (test_acceptance.py:49-69) and the min-merge
of per-worker buffers (pipeline.py:151-204)."""

import os

import numpy as np
import pytest
import torch

from oracle import host as oh
from paper_2604_21749_b200 import (Camera, RasterConfig, SceneNode, build_draw_list,
                                   render_draw_list)
from paper_2604_21749_b200 import generators as gen
from paper_2604_21749_b200.distributed import shard_range
from paper_2604_21749_b200.pipeline import PreparedFrame
from scenes import (STAT_ORDER, compress_scene, golden_camera, golden_cfg, golden_names,
                    golden_scene, load_golden, stats_vector_from_frame,
                    stats_vector_from_oracle)

pytestmark = pytest.mark.gpu


def _threads():
    return max(1, min(32, len(os.sched_getaffinity(0))))


def _assert_same(words, st_vec, ref, ref_vec, what):
    diff = np.nonzero(words != ref)[0]
    assert diff.size == 0, f"{what}: {diff.size} differing words, first {diff[:8]}"
    bad = [(STAT_ORDER[i], int(st_vec[i]), int(ref_vec[i])) for i in range(15)
           if st_vec[i] != ref_vec[i]]
    assert not bad, (what, bad)


def _full_frame_vs_oracle(scene, cam, what, instancing="auto"):
    cfg = RasterConfig(instancing=instancing)
    dl = build_draw_list(scene, cam)
    fb, st = render_draw_list(dl, cam, cfg)
    words = fb.words.copy()
    odl = oh.build_draw_list(scene, cam)
    octx = oh.build_context(odl, cam)
    inst = instancing == "on" or (instancing == "auto" and octx.max_instances >= 2)
    ref, rst, rc, _, _ = oh.render_context(octx, oh.camera_constants(cam), instanced=inst,
                                           workers=_threads(), batch=4096,
                                           s2_cap=1 << 22, s3_cap=1 << 22)
    assert rc == 0
    _assert_same(words, stats_vector_from_frame(st), ref, stats_vector_from_oracle(rst), what)
    return st


@pytest.mark.slow
def test_config_d_instanced_1b_bit_exact_words_and_stats():
    scene, cam = gen.config_d()
    st = _full_frame_vs_oracle(scene, cam, "D")
    assert st.instanced and st.total_triangles == 997_698_604


@pytest.mark.slow
def test_config_bq_compressed_100m_bit_exact_words_and_stats():
    scene, cam = gen.config_b()
    _full_frame_vs_oracle(compress_scene(scene), cam, "Bq")


@pytest.mark.slow
def test_config_dq_compressed_instanced_bit_exact_words_and_stats():
    scene, cam = gen.config_d()
    st = _full_frame_vs_oracle(compress_scene(scene), cam, "Dq")
    assert st.instanced


def _pieces_vs_oracle(scene, cam, cuts, instanced):
    """Render the work-space pieces [cuts[k], cuts[k+1]) separately through
    PreparedFrame(work_range=...), compare each with the oracle on the same
    range (words + stats), min-compose them and compare with the full frame."""
    cfg = RasterConfig(instancing="on" if instanced else "off")
    dl = build_draw_list(scene, cam)
    odl = oh.build_draw_list(scene, cam)
    octx = oh.build_context(odl, cam)
    cc = oh.camera_constants(cam)
    full, fst, rc, _, _ = oh.render_context(octx, cc, instanced=instanced, workers=_threads(),
                                            s2_cap=1 << 22, s3_cap=1 << 22)
    assert rc == 0
    comp = None
    tot = np.zeros(15, dtype=np.int64)
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        pf = PreparedFrame(dl, cam, cfg, work_range=(lo, hi))
        assert pf.inst_kernel == instanced
        c, _ = pf.run()
        words = pf.fb.cpu().numpy().view(np.uint64).copy()
        sv = stats_vector_from_frame(pf.stats(c, [0.0] * 4))
        ref, rst, rc, _, _ = oh.render_context(octx, cc, instanced=instanced,
                                               workers=_threads(), work_range=(lo, hi),
                                               s2_cap=1 << 22, s3_cap=1 << 22)
        assert rc == 0
        _assert_same(words, sv, ref, stats_vector_from_oracle(rst), f"range [{lo}, {hi})")
        comp = words if comp is None else np.minimum(comp, words)
        tot += sv
    assert np.array_equal(comp, full)
    assert np.array_equal(tot, stats_vector_from_oracle(fst))


def test_flat_work_ranges_unaligned_and_chunk_straddling():
    """k_s1_lean_flat on shard ranges whose first triangle is not 16-byte
    aligned in the index stream (the vec == false branch) and whose cuts
    fall inside 2016-triangle chunks, 126-triangle steps and lanes."""
    scene, cam = gen.config_b(n=900, width=1280, height=720)
    T = build_draw_list(scene, cam).total_triangles
    cuts = [0, 126 * 37 + 5, T // 2 + 3, T // 2 + 2016 + 1, T - 7, T]
    _pieces_vs_oracle(scene, cam, cuts, instanced=False)


def test_flat_work_ranges_over_many_items():
    """Cuts inside and at the ends of items of a multi-item flat frame."""
    scene, cam = gen.config_c(width=1280, height=720)
    T = build_draw_list(scene, cam).total_triangles
    cuts = sorted({0, 1, 2017, T // 3 + 1, T // 2, T - 4033, T})
    _pieces_vs_oracle(scene, cam, cuts, instanced=False)


def test_instanced_work_ranges_start_mid_group():
    """The instanced stage-1 kernel on unique-triangle ranges starting and
    ending inside node groups (pipeline.py:244: the instanced work space)."""
    scene = gen.make_lantern_grid(6, 5, tris_per_mesh=20_000, spacing=1.8)
    extra = gen.make_sphere(*gen.sphere_dims_for(3000), radius=0.9)
    T = np.eye(4)
    T[:3, 3] = (0.5, 2.0, 3.0)
    scene = scene + [SceneNode(mesh=extra, transforms=[T])]
    cam = Camera.look_at((0.0, 9.0, 13.0), (0.0, 0.0, 0.0), width=640, height=480)
    dl = build_draw_list(scene, cam)
    from paper_2604_21749_b200.pipeline import build_context
    ctx = build_context(dl, cam)
    U = int(ctx.group_prefix[-1])
    g1 = int(ctx.group_prefix[1])
    cuts = sorted({0, 33, g1 // 2 + 1, g1 + 31, U - 5, U})
    _pieces_vs_oracle(scene, cam, cuts, instanced=True)


def test_shard_ranges_cover_a_frame_at_world_4():
    """The exact partition render_sharded uses (shard_range) at world 4."""
    scene, cam = gen.config_b(n=700, width=960, height=540)
    T = build_draw_list(scene, cam).total_triangles
    cuts = [shard_range(T, 4, r)[0] for r in range(4)] + [T]
    _pieces_vs_oracle(scene, cam, cuts, instanced=False)


@pytest.mark.parametrize("name", ["lantern_on", "lantern_off", "classifier", "random2024_003",
                                  "random2024_025", "tiny_on", "quad48_ss2"])
def test_reference_render_context_as_ctx(name):
    """render_draw_list(ctx=<the reference's RenderContext>): its flattened
    positions / indices and item offsets (unaligned index offsets included)
    render the reference's words and stats."""
    from refctx import from_golden
    g = load_golden(name)
    if int(g["total"]) == 0:
        pytest.skip("empty")
    scene = golden_scene(g, compressed=False)
    cam = golden_camera(g)
    dl = build_draw_list(scene, cam)
    fb, st = render_draw_list(dl, cam, golden_cfg(g), ctx=from_golden(g))
    _assert_same(fb.words, stats_vector_from_frame(st), g["ref_words"], g["stats"][:15], name)


def test_repeated_calls_reuse_the_prepared_frame():
    """The e2e path: a second render_draw_list call with the same inputs
    reuses the prepared frame (descriptors re-uploaded) and returns a new,
    independent framebuffer with the same words."""
    from paper_2604_21749_b200 import pipeline as P
    scene, cam = gen.config_a()
    dl = build_draw_list(scene, cam)
    fb1, st1 = render_draw_list(dl, cam)
    n = len(P._frame_cache)
    fb2, st2 = render_draw_list(dl, cam)
    assert len(P._frame_cache) == n
    assert fb1.device_words.data_ptr() != fb2.device_words.data_ptr()
    assert np.array_equal(fb1.words, fb2.words)
    assert np.array_equal(stats_vector_from_frame(st1), stats_vector_from_frame(st2))
    # a different camera is a different frame
    cam2 = Camera.look_at((0.0, 0.2, 3.0), (0.0, 0.0, 0.0), width=1920, height=1080)
    fb3, _ = render_draw_list(dl, cam2)
    ref, _, _ = oh.render_reference(scene, cam2, workers=_threads())
    assert np.array_equal(fb3.words, ref)


def test_framebuffer_host_edits_reach_the_device_views():
    """A forged host word (test_resolvepass.py:218 edits fb.words in place)
    is what resolve / debug_view read afterwards."""
    from paper_2604_21749_b200 import pack_fragment
    scene, cam = gen.config_a()
    dl = build_draw_list(scene, cam)
    fb, _ = render_draw_list(dl, cam)
    w = fb.words
    w[5] = pack_fragment(1.0, (1 << 36) - 2)
    dev = fb.device_words.cpu().numpy().view(np.uint64)
    assert dev[5] == w[5]
    assert np.array_equal(dev, w)


def test_config_e_device_generated_equals_host_and_oracle():
    """Config E's meshes generated in HBM (f32 and compressed) are the host
    generator's meshes bit for bit: frames rendered from both are identical,
    and the f32 one equals the oracle."""
    from scenes import compress_scene
    scene_h, cam = gen.config_e(n_meshes=5, n=150, width=960, height=540)
    scene_d, _ = gen.config_e(n_meshes=5, n=150, width=960, height=540, on_device=True)
    scene_c, _ = gen.config_e(n_meshes=5, n=150, width=960, height=540, on_device=True,
                              compressed=True)
    fh, sh = render_draw_list(build_draw_list(scene_h, cam), cam)
    fd, sd = render_draw_list(build_draw_list(scene_d, cam), cam)
    fc, sc = render_draw_list(build_draw_list(scene_c, cam), cam)
    fq, sq = render_draw_list(build_draw_list(compress_scene(scene_h), cam), cam)
    assert np.array_equal(fh.words, fd.words)
    assert np.array_equal(fc.words, fq.words)
    assert np.array_equal(stats_vector_from_frame(sc), stats_vector_from_frame(sq))
    ref, rst, _ = oh.render_reference(scene_h, cam, workers=_threads())
    assert np.array_equal(fh.words, ref)
    refq, _, _ = oh.render_reference(compress_scene(scene_h), cam, workers=_threads())
    assert np.array_equal(fc.words, refq)
