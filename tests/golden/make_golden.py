"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
The reference package is copied to /tmp (numba's cache=True writes next to
the sources; /root/reference is read-only) and imported from there.  Each
fixture stores the reference's kernel inputs exactly as the reference built
them (prefix sums, object->view / object->world matrices, flattened
positions/indices, camera constants) together with its outputs (visibility
words of ``render_reference`` and ``render_frame``, FrameStats), so tests on
other hosts do not depend on numpy/BLAS rounding there.

Nothing on the GPU box runs this script; only its .npz outputs travel.
"""

from __future__ import annotations

import hashlib
import math
import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg"
TMP = "/tmp/curast_golden_ref"


def _import_reference():
    if not os.path.exists(TMP):
        shutil.copytree(REF_SRC, TMP)
    sys.path.insert(0, os.path.join(TMP, "src"))
    sys.path.insert(0, os.path.join(TMP, "tests"))
    import trirast  # noqa: F401
    import conftest  # noqa: F401
    return trirast, conftest


def _case_arrays(name, scene, camera, cfg_kwargs, trirast, honor_stages=True,
                 compressed=False):
    from trirast.config import RasterConfig
    from trirast.pipeline import build_context, render_frame
    from trirast.refraster import OracleConfig, render_reference
    from trirast.scenecore import build_draw_list, projection_vector

    cfg = RasterConfig(workers=1, **cfg_kwargs)
    dl = build_draw_list(scene, camera)
    out = {}
    out["name"] = np.array(name)
    out["cfg_json"] = np.array(repr(sorted(cfg_kwargs.items())))
    out["honor_stages"] = np.array(bool(honor_stages))
    # scene description (decoded geometry + compressed payloads)
    out["n_nodes"] = np.array(len(scene))
    for i, node in enumerate(scene):
        m = node.mesh
        out[f"node{i}_positions"] = m.positions_f64()
        out[f"node{i}_indices"] = m.indices_u32()
        out[f"node{i}_aabb"] = np.asarray(m.aabb, dtype=np.float64)
        out[f"node{i}_tricount"] = np.array(m.triangle_count)
        out[f"node{i}_transforms"] = np.stack(node.transforms)
        if not isinstance(m.positions, np.ndarray):
            out[f"node{i}_q_coords"] = m.positions.coords
            out[f"node{i}_q_grid"] = np.concatenate([m.positions.grid_min, m.positions.grid_size])
        if not isinstance(m.indices, np.ndarray):
            out[f"node{i}_p_data"] = m.indices.data
            out[f"node{i}_p_meta"] = np.array([m.indices.min_index, m.indices.bits_per_index,
                                               m.indices.count], dtype=np.int64)
        if m.vertex_colors is not None:
            out[f"node{i}_colors"] = m.vertex_colors
    out["cam_position"] = camera.position
    out["cam_view"] = camera.view_transform
    out["cam_scalars"] = np.array([camera.fovy, camera.aspect, camera.near])
    out["cam_ints"] = np.array([camera.image_width, camera.image_height,
                                camera.supersampling], dtype=np.int64)
    # reference kernel inputs
    out["prefix"] = dl.prefix_sums.astype(np.int64)
    out["total"] = np.array(dl.total_triangles)
    if dl.total_triangles:
        ctx = build_context(dl, camera)
        out["item_mv"] = ctx.item_mv
        out["item_mw"] = ctx.item_mw
        out["item_vtx_off"] = ctx.item_vtx_off
        out["item_idx_off"] = ctx.item_idx_off
        out["ctx_positions"] = ctx.positions
        out["ctx_indices"] = ctx.indices
        out["group_prefix"] = ctx.group_prefix
        out["group_item_off"] = ctx.group_item_off
        out["group_item_count"] = ctx.group_item_count
        out["group_items"] = ctx.group_items
        out["max_instances"] = np.array(ctx.max_instances)
    out["p"] = projection_vector(camera)
    # reference outputs
    ref = render_reference(scene, camera, OracleConfig(raster=cfg, honor_stages=honor_stages))
    out["ref_words"] = ref.words
    if honor_stages:
        fb, st = render_frame(scene, camera, cfg)
        assert np.array_equal(fb.words, ref.words), name
        s = st
        out["stats"] = np.array([
            s.stage1.rasterized, s.stage1.forwarded, s.stage1.culled_frustum,
            s.stage1.culled_offscreen, s.stage1.culled_tiny, s.stage1.culled_backface,
            s.stage1.culled_degenerate, s.stage1.fragments,
            s.stage2.direct, s.stage2.tiled, s.stage2.dropped, s.stage2.fragments,
            s.stage2.tiles, s.stage3.entries, s.stage3.fragments, int(s.instanced)],
            dtype=np.int64)
    out["words_sha256"] = np.array(hashlib.sha256(ref.words.tobytes()).hexdigest())
    return out


def main():
    trirast, conftest = _import_reference()
    from trirast import geomcodec as gc
    from trirast.scenecore import Camera, SceneNode
    from trirast.scenedesc import (make_classifier_scene, make_lantern_grid, make_sphere,
                                   make_tessellated_quad, sphere_dims_for)

    cases = {}
    # criterion-1 random scenes (test_acceptance.py:49-69), seed 2024: keep the
    # first 40 (geometry stored; scenes up to 10^4 triangles)
    rng = np.random.default_rng(2024)
    for k in range(40):
        scene, camera = conftest.random_scene(rng)
        cases[f"random2024_{k:03d}"] = _case_arrays(f"random2024_{k:03d}", scene, camera, {},
                                                    trirast)
    # classifier scene (scenedesc.py:278-300)
    scene, camera = make_classifier_scene()
    cases["classifier"] = _case_arrays("classifier", scene, camera, {}, trirast)
    for fs in (1, 2, 3):
        cases[f"classifier_force{fs}"] = _case_arrays(f"classifier_force{fs}", scene, camera,
                                                      {"force_stage": fs}, trirast)
    cases["classifier_unstaged"] = _case_arrays("classifier_unstaged", scene, camera, {},
                                                trirast, honor_stages=False)
    # routing thresholds (test_rasterpipe.py:20-49)
    cam = conftest.identity_camera(width=256, height=128)
    for xs, ys in [(8, 8), (127, 1), (8, 16), (65, 63), (64, 64), (130, 70)]:
        pixels = [(0.25, 0.25), (xs - 0.25, 0.25), (0.25, ys - 0.25)]
        sc = conftest.pixel_triangle_scene(pixels, [2.0] * 3, cam)
        cases[f"route_{xs}x{ys}"] = _case_arrays(f"route_{xs}x{ys}", sc, cam, {}, trirast)
    # tiny cull on/off on a dense quad (test_acceptance.py:182-210)
    mesh = make_tessellated_quad(120)
    cam = Camera.look_at((0.0, 0.0, 3.2), (0.0, 0.0, 0.0), width=96, height=96)
    sc = [SceneNode(mesh=mesh, transforms=[np.eye(4)])]
    cases["tiny_on"] = _case_arrays("tiny_on", sc, cam, {"tiny_cull": True}, trirast)
    cases["tiny_off"] = _case_arrays("tiny_off", sc, cam, {"tiny_cull": False}, trirast)
    # instancing (test_acceptance.py:213-235), smaller mesh
    sc = make_lantern_grid(6, 6, tris_per_mesh=2000, spacing=1.8)
    cam = Camera.look_at((0.0, 14.0, 20.0), (0.0, 0.0, 0.0), width=320, height=240)
    cases["lantern_on"] = _case_arrays("lantern_on", sc, cam, {"instancing": "on"}, trirast)
    cases["lantern_off"] = _case_arrays("lantern_off", sc, cam, {"instancing": "off"}, trirast)
    # supersampled quad (test_acceptance.py:315-336 scene)
    mesh = make_tessellated_quad(48)
    cam = Camera.look_at((0, 0, 1.4), (0, 0, 0), width=160, height=120, supersampling=2)
    cases["quad48_ss2"] = _case_arrays("quad48_ss2", [SceneNode(mesh=mesh, transforms=[np.eye(4)])],
                                       cam, {}, trirast)
    # compressed geometry rendered through the reference (no reference test
    # renders one)
    sph = make_sphere(*sphere_dims_for(3000), radius=0.8)
    qpos = gc.quantize_positions(sph.positions_f64(), sph.aabb)
    pidx = gc.compress_indices(sph.indices_u32())
    from trirast.scenecore import Mesh
    cm = Mesh(positions=qpos, indices=pidx, triangle_count=sph.triangle_count, aabb=sph.aabb)
    cam = Camera.look_at((0.3, 0.4, 2.2), (0.0, 0.0, 0.0), width=200, height=150)
    cases["compressed_sphere"] = _case_arrays("compressed_sphere",
                                              [SceneNode(mesh=cm, transforms=[np.eye(4)])],
                                              cam, {}, trirast)
    # a medium sphere with f64 positions (non f32-representable)
    sph = make_sphere(*sphere_dims_for(20000))
    cam = Camera.look_at((0.0, 0.0, 3.0), (0.0, 0.0, 0.0), width=320, height=240)
    cases["sphere20k"] = _case_arrays("sphere20k", [SceneNode(mesh=sph, transforms=[np.eye(4)])],
                                      cam, {}, trirast)

    os.makedirs(HERE, exist_ok=True)
    for name, arrs in cases.items():
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrs)

    # generator identity: hashes of the reference generators' arrays
    gen = {}
    for rings, segs in [(4, 5), (30, 31), (sphere_dims_for(20000))]:
        m = make_sphere(rings, segs)
        gen[f"sphere_{rings}_{segs}_pos"] = m.positions_f64()
        gen[f"sphere_{rings}_{segs}_idx"] = m.indices_u32()
        gen[f"sphere_{rings}_{segs}_col"] = m.vertex_colors
    for n in (1, 7, 37):
        m = make_tessellated_quad(n)
        gen[f"quad_{n}_pos"] = m.positions_f64()
        gen[f"quad_{n}_idx"] = m.indices_u32()
        gen[f"quad_{n}_uv"] = m.uvs
    gen["sphere_dims"] = np.array([sphere_dims_for(t) for t in (10, 2000, 10 ** 6, 10 ** 8)])
    np.savez_compressed(os.path.join(HERE, "generators.npz"), **gen)

    # pack_fragment golden words (test_scenecore.py:20-22)
    from trirast.scenecore import pack_fragment
    rngp = np.random.default_rng(7)
    depths = np.exp(rngp.uniform(np.log(1e-6), np.log(1e30), 2000))
    ids = rngp.integers(0, 1 << 36, 2000)
    words = np.array([pack_fragment(float(d), int(i)) for d, i in zip(depths, ids)],
                     dtype=np.uint64)
    np.savez_compressed(os.path.join(HERE, "packing.npz"), depths=depths, ids=ids, words=words)
    print("wrote", len(cases), "fixtures")


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def main_resolve():
    """Resolve-pass fixtures: reference resolve_frame / downsample outputs."""
    trirast, conftest = _import_reference()
    from trirast.config import RasterConfig, ShadingConfig
    from trirast.pipeline import render_frame
    from trirast.resolvepass import downsample, resolve_frame
    from trirast.scenecore import Camera, SceneNode, build_draw_list
    from trirast.scenedesc import (make_checker_texture, make_sphere, make_tessellated_quad,
                                   sphere_dims_for, make_classifier_scene)

    def save(name, scene, cam, shadings):
        fb, _ = render_frame(scene, cam, RasterConfig(workers=1))
        dl = build_draw_list(scene, cam)
        out = {"words": fb.words, "cam_position": cam.position, "cam_view": cam.view_transform,
               "cam_scalars": np.array([cam.fovy, cam.aspect, cam.near]),
               "cam_ints": np.array([cam.image_width, cam.image_height, cam.supersampling]),
               "n_nodes": np.array(len(scene))}
        for i, node in enumerate(scene):
            m = node.mesh
            out[f"node{i}_positions"] = m.positions_f64()
            out[f"node{i}_indices"] = m.indices_u32()
            out[f"node{i}_aabb"] = m.aabb
            out[f"node{i}_tricount"] = np.array(m.triangle_count)
            out[f"node{i}_transforms"] = np.stack(node.transforms)
            if m.vertex_colors is not None:
                out[f"node{i}_colors"] = m.vertex_colors
            if m.uvs is not None:
                out[f"node{i}_uvs"] = m.uvs
            if m.texture is not None:
                out[f"node{i}_nlevels"] = np.array(len(m.texture.levels))
                for k, lv in enumerate(m.texture.levels):
                    out[f"node{i}_level{k}"] = lv
        for k, sh in enumerate(shadings):
            img, st = resolve_frame(fb, dl, cam, sh)
            out[f"shading{k}"] = np.array(repr((sh.mode, sh.headlight, tuple(sh.background),
                                                sh.mip_filter, tuple(sh.base_color))))
            out[f"image{k}"] = img
            out[f"rstats{k}"] = np.array([st.shaded, st.background, st.degenerate])
            if cam.supersampling > 1:
                out[f"down{k}"] = downsample(img, cam.supersampling)
        np.savez_compressed(os.path.join(HERE, f"resolve_{name}.npz"), **out)

    sph = make_sphere(*sphere_dims_for(20000))
    cam = Camera.look_at((0.0, 0.0, 3.0), (0.0, 0.0, 0.0), width=320, height=240)
    save("sphere", [SceneNode(mesh=sph, transforms=[np.eye(4)])], cam,
         [ShadingConfig(), ShadingConfig(headlight=True), ShadingConfig(mode="flat")])
    scene, cam = make_classifier_scene()
    save("classifier", scene, cam, [ShadingConfig(), ShadingConfig(headlight=True)])
    quad = make_tessellated_quad(48)
    quad.texture = make_checker_texture()
    cam = Camera.look_at((0.3, -0.2, 1.4), (0, 0, 0), width=160, height=120, supersampling=2)
    save("textured", [SceneNode(mesh=quad, transforms=[np.eye(4)])], cam,
         [ShadingConfig(), ShadingConfig(mip_filter="trilinear", headlight=True)])
    cam = Camera.look_at((0.0, 0.0, 4.5), (0, 0, 0), width=160, height=120, supersampling=4)
    save("textured_far", [SceneNode(mesh=quad, transforms=[np.eye(4)])], cam,
         [ShadingConfig(mip_filter="trilinear"), ShadingConfig()])
    print("wrote resolve fixtures")


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "resolve":
    main_resolve()


def main_trimesh():
    """TRIMESH1 fixtures written by the reference's save_mesh (raw, quantized +
    packed, with uvs and colours) plus what its load_mesh_asset returns."""
    trirast, conftest = _import_reference()
    from trirast.geomcodec import compress_indices, load_mesh_asset, quantize_positions, save_mesh
    from trirast.scenecore import Mesh as RMesh
    from trirast.scenedesc import make_sphere, make_tessellated_quad
    out = {}
    sph = make_sphere(12, 16, radius=0.8)
    quad = make_tessellated_quad(6)
    q_pos = quantize_positions(sph.positions_f64(), sph.aabb)
    p_idx = compress_indices(sph.indices_u32())
    cases = {
        "raw": sph,
        "compressed": RMesh(positions=q_pos, indices=p_idx, triangle_count=sph.triangle_count,
                            aabb=sph.aabb, vertex_colors=sph.vertex_colors, name="c"),
        "uvquad": quad,
    }
    for name, mesh in cases.items():
        path = os.path.join(HERE, f"mesh_{name}.trimesh")
        save_mesh(path, mesh)
        m = load_mesh_asset(path)
        out[f"{name}_positions"] = m.positions_f64()
        out[f"{name}_indices"] = m.indices_u32()
        out[f"{name}_aabb"] = np.asarray(m.aabb, dtype=np.float64)
        out[f"{name}_ntris"] = np.int64(m.triangle_count)
        if m.uvs is not None:
            out[f"{name}_uvs"] = np.asarray(m.uvs)
        if m.vertex_colors is not None:
            out[f"{name}_colors"] = np.asarray(m.vertex_colors)
    np.savez_compressed(os.path.join(HERE, "trimesh.npz"), **out)
    print("wrote trimesh fixtures")


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "trimesh":
    main_trimesh()


def main_debug():
    """debug_view fixtures: the reference's four diagnostic views of a few
    golden scenes (rebuilt from the stored arrays with the reference's own
    types, rendered by the reference)."""
    trirast, conftest = _import_reference()
    from trirast.config import RasterConfig
    from trirast.geomcodec import PackedIndexBuffer, QuantizedPositions
    from trirast.pipeline import render_frame
    from trirast.resolvepass import debug_view
    from trirast.scenecore import Camera, Mesh, SceneNode, build_draw_list
    import ast
    out = {}
    for name in ("classifier", "lantern_off", "compressed_sphere", "tiny_on", "quad48_ss2",
                 "random2024_000", "random2024_003", "route_130x70"):
        g = np.load(os.path.join(HERE, f"{name}.npz"))
        nodes = []
        for i in range(int(g["n_nodes"])):
            pos, idx = g[f"node{i}_positions"], g[f"node{i}_indices"]
            if f"node{i}_q_coords" in g:
                grid = g[f"node{i}_q_grid"]
                pos = QuantizedPositions(grid_min=grid[:3].copy(), grid_size=grid[3:].copy(),
                                         coords=g[f"node{i}_q_coords"])
            if f"node{i}_p_data" in g:
                mn, b, cnt = (int(v) for v in g[f"node{i}_p_meta"])
                idx = PackedIndexBuffer(min_index=mn, bits_per_index=b, count=cnt,
                                        data=g[f"node{i}_p_data"])
            mesh = Mesh(positions=pos, indices=idx, triangle_count=int(g[f"node{i}_tricount"]),
                        aabb=g[f"node{i}_aabb"])
            nodes.append(SceneNode(mesh=mesh, transforms=list(g[f"node{i}_transforms"])))
        fovy, aspect, near = (float(v) for v in g["cam_scalars"])
        w, h, ss = (int(v) for v in g["cam_ints"])
        cam = Camera(position=g["cam_position"], view_transform=g["cam_view"], fovy=fovy,
                     aspect=aspect, near=near, image_width=w, image_height=h, supersampling=ss)
        cfg = RasterConfig(**dict(ast.literal_eval(str(g["cfg_json"]))))
        fb, _ = render_frame(nodes, cam, cfg)
        assert np.array_equal(fb.words, g["ref_words"]) or np.array_equal(fb.words, g["frame_words"])
        dl = build_draw_list(nodes, cam)
        for mode in ("depth", "stageID", "bboxSize", "meshID"):
            out[f"{name}__{mode}"] = debug_view(fb, dl, cam, mode, cfg)
    np.savez_compressed(os.path.join(HERE, "debug_views.npz"), **out)
    print("wrote debug fixtures", len(out))


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "debug":
    main_debug()
