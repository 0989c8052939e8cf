"""CPU tests: host logic, generators, packing, C-ABI exports (no GPU)."""

import ctypes
import math
import os
import re

import numpy as np
import pytest

from paper_2604_21749_b200 import (CLEAR, Camera, CapacityError, MAX_TRIANGLE_ID,
                                   RasterConfig, SceneNode, build_draw_list, pack_fragment,
                                   unpack_fragment)
from paper_2604_21749_b200 import _native as N
from paper_2604_21749_b200 import codec
from paper_2604_21749_b200.generators import (grid_indices, make_sphere,
                                              make_tessellated_quad, sphere_dims_for)
from paper_2604_21749_b200.pipeline import _work_table, build_context, classify_route
from oracle import host as oh
from scenes import (ROOT, golden_camera, golden_names, golden_scene, load_golden,
                    mesh_from_soup, random_scene, view_point_for_pixel, identity_camera)


def test_pack_fragment_golden_words():
    assert pack_fragment(1.0, 7) == np.uint64(0x7F00000000000007)
    assert pack_fragment(1.0, 0) == np.uint64(0x7F00000000000000)
    g = np.load(os.path.join(ROOT, "tests", "golden", "packing.npz"))
    got = np.array([pack_fragment(float(d), int(i)) for d, i in zip(g["depths"], g["ids"])],
                   dtype=np.uint64)
    assert np.array_equal(got, g["words"])
    d28, d, tid = unpack_fragment(got[0])
    assert tid == int(g["ids"][0])
    with pytest.raises(ValueError):
        unpack_fragment(CLEAR)
    with pytest.raises(ValueError):
        pack_fragment(-1.0, 0)
    with pytest.raises(ValueError):
        pack_fragment(1.0, MAX_TRIANGLE_ID)


def test_generators_identical_to_reference():
    g = np.load(os.path.join(ROOT, "tests", "golden", "generators.npz"))
    for key in g.files:
        if key.startswith("sphere_") and key.endswith("_pos"):
            _, r, s, _ = key.split("_")
            m = make_sphere(int(r), int(s))
            assert np.array_equal(m.positions, g[key]), key
            assert np.array_equal(m.indices, g[key.replace("_pos", "_idx")]), key
            assert np.array_equal(m.vertex_colors, g[key.replace("_pos", "_col")]), key
        if key.startswith("quad_") and key.endswith("_pos"):
            n = int(key.split("_")[1])
            m = make_tessellated_quad(n)
            assert np.array_equal(m.positions, g[key]), key
            assert np.array_equal(m.indices, g[key.replace("_pos", "_idx")]), key
            assert np.array_equal(m.uvs, g[key.replace("_pos", "_uv")]), key
    dims = np.array([sphere_dims_for(t) for t in (10, 2000, 10 ** 6, 10 ** 8)])
    assert np.array_equal(dims, g["sphere_dims"])


def test_random_scene_matches_reference_generator():
    rng = np.random.default_rng(2024)
    for k in range(40):
        scene, cam = random_scene(rng)
        gd = load_golden(f"random2024_{k:03d}")
        assert int(gd["n_nodes"]) == len(scene)
        for i, node in enumerate(scene):
            assert np.array_equal(node.mesh.positions, gd[f"node{i}_positions"])
            assert np.array_equal(np.stack(node.transforms), gd[f"node{i}_transforms"])
        assert np.array_equal(cam.view_transform, gd["cam_view"])


@pytest.mark.parametrize("name", golden_names("random2024_0")[:10] + ["lantern_on", "classifier"])
def test_product_draw_list_matches_reference(name):
    g = load_golden(name)
    scene = golden_scene(g)
    cam = golden_camera(g)
    dl = build_draw_list(scene, cam)
    assert np.array_equal(dl.prefix_sums.astype(np.int64), g["prefix"])
    if dl.total_triangles:
        ctx = build_context(dl, cam)
        assert np.array_equal(ctx.item_mw, g["item_mw"])
        np.testing.assert_allclose(ctx.item_mv, g["item_mv"], rtol=1e-14, atol=1e-14)
        assert np.array_equal(ctx.group_prefix, g["group_prefix"])
        assert np.array_equal(ctx.group_items, g["group_items"])
        assert ctx.max_instances == int(g["max_instances"])


def test_draw_list_capacity_error():
    mesh = mesh_from_soup([(0, 0, -2.0), (1, 0, -2.0), (0, 1, -2.0)])
    mesh.triangle_count = MAX_TRIANGLE_ID
    with pytest.raises(CapacityError):
        build_draw_list([SceneNode(mesh=mesh, transforms=[np.eye(4)])], identity_camera())
    with pytest.raises(ValueError):
        build_draw_list([], identity_camera())


def test_codec_roundtrip():
    rng = np.random.default_rng(11)
    idx = rng.integers(2500, 3001, 500, dtype=np.uint32)
    idx[0], idx[1] = 2500, 3000
    p = codec.compress_indices(idx)
    assert p.bits_per_index == 9
    assert np.array_equal(p.decode_all(), idx)
    assert all(p.decode(i) == idx[i] for i in range(0, 500, 37))
    for _ in range(200):
        bits = int(rng.integers(1, 33))
        lo = int(rng.integers(0, 2 ** 31))
        span = min(2 ** bits - 1, 2 ** 32 - 1 - lo)
        buf = rng.integers(lo, lo + span + 1, int(rng.integers(1, 40)), dtype=np.int64).astype(np.uint32)
        assert np.array_equal(codec.compress_indices(buf).decode_all(), buf)
    aabb = np.array([[-7.0, 3.0, -1.0], [9.0, 3.5, 200.0]])
    pts = rng.uniform(aabb[0], aabb[1], (1000, 3))
    q = codec.quantize_positions(pts, aabb)
    assert (np.abs(q.dequantize_all() - pts) <= (aabb[1] - aabb[0]) / 131072.0 + 1e-12).all()
    # oracle host decode agrees with the product codec
    m = mesh_from_soup(pts[:9])
    m.positions = q
    assert np.array_equal(oh.mesh_positions_f64(m), q.dequantize_all())


def test_work_table_covers_range_exactly():
    starts = np.array([0, 10, 10, 25], dtype=np.int64)
    counts = np.array([10, 0, 15, 7], dtype=np.int64)
    ids, lo, hi, cp = _work_table(starts, counts, np.arange(4), 5, 30, 4)
    covered = []
    for u in range(len(ids)):
        covered += list(range(starts[ids[u]] + lo[u], starts[ids[u]] + hi[u]))
        assert cp[u + 1] - cp[u] == -(-(hi[u] - lo[u]) // 4)
    assert covered == list(range(5, 30))


def test_grid_indices_layout():
    m = make_tessellated_quad(3)
    assert np.array_equal(grid_indices(3), m.indices)


def test_classify_route_mirror():
    cam = identity_camera(width=256, height=128)
    for xs, ys, want in [(8, 8, 1), (16, 16, 2), (64, 64, 3)]:
        pts = [view_point_for_pixel(0.25, 0.25, 2.0, cam),
               view_point_for_pixel(xs - 0.25, 0.25, 2.0, cam),
               view_point_for_pixel(0.25, ys - 0.25, 2.0, cam)]
        assert classify_route(np.asarray(pts), cam)[0] == want


def _header_functions():
    text = open(os.path.join(ROOT, "include", "curast.h")).read()
    return sorted(set(re.findall(r"\b(curast_[a-z0-9_]+)\s*\(", text)))


def test_c_abi_library_exports_every_header_symbol():
    path = N.LIB_PATH
    if not os.path.exists(path):
        pytest.skip("library not built")
    lib = ctypes.CDLL(path)
    names = _header_functions()
    assert "curast_stage1" in names and "curast_resolve" in names
    for name in names:
        assert hasattr(lib, name), name
    assert set(N.EXPORTED_SYMBOLS) == set(names)
    assert lib.curast_abi_version() == N.ABI_VERSION


@pytest.mark.parametrize("cname,pyname", [("curast_frame_t", "CurastFrame"),
                                           ("curast_resolve_t", "CurastResolve"),
                                           ("curast_debug_t", "CurastDebug")])
def test_struct_layout_matches_header(tmp_path, cname, pyname):
    """Compile a probe against include/curast.h and compare every field
    offset and the struct size with the ctypes mirror."""
    import subprocess
    cls = getattr(N, pyname)
    fields = [f[0] for f in cls._fields_]
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "curast.h"',
             "int main(void){",
             f'printf("size %zu\\n", sizeof({cname}));']
    for fn in fields:
        lines.append(f'printf("{fn} %zu\\n", offsetof({cname}, {fn}));')
    lines.append("return 0;}")
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    got = dict(l.split() for l in out.strip().splitlines())
    assert int(got["size"]) == ctypes.sizeof(cls)
    for fn in fields:
        assert int(got[fn]) == getattr(cls, fn).offset, fn


def test_compress_indices_matches_reference_bitstream():
    g = load_golden("compressed_sphere")
    mn, b, cnt = (int(v) for v in g["node0_p_meta"])
    p = codec.compress_indices(g["node0_indices"])
    assert (p.min_index, p.bits_per_index, p.count) == (mn, b, cnt)
    assert np.array_equal(p.data, g["node0_p_data"])
    rng = np.random.default_rng(3)
    for _ in range(50):
        bits = int(rng.integers(1, 33))
        lo = int(rng.integers(0, 2 ** 31))
        span = min(2 ** bits - 1, 2 ** 32 - 1 - lo)
        buf = rng.integers(lo, lo + span + 1, int(rng.integers(1, 300)), dtype=np.int64).astype(np.uint32)
        ref = np.packbits(((buf.astype(np.uint64)[:, None] - np.uint64(buf.min()))
                           >> np.arange(max(1, int(buf.max() - buf.min()).bit_length()),
                                        dtype=np.uint64) & np.uint64(1)).astype(np.uint8).ravel(),
                          bitorder="little")
        assert np.array_equal(codec.compress_indices(buf).data, ref)


def test_device_copy_cache_is_identity_checked():
    """Device geometry is cached on the mesh and matched by object identity:
    a new mesh never inherits a freed mesh's upload (ids get reused), and
    assigning new arrays re-uploads (device.py device_mesh/scene_geometry)."""
    import gc

    import torch

    from paper_2604_21749_b200 import device as dv
    from paper_2604_21749_b200.generators import make_sphere
    cpu = torch.device("cpu")
    m = make_sphere(4, 6)
    m.positions = np.asarray(m.positions, np.float32).astype(np.float64)   # f32-exact
    a = dv.device_mesh(m, cpu)
    assert dv.device_mesh(m, cpu) is a
    assert a.pos_format == N.POS_F32 and tuple(a.positions.shape) == (m.vertex_count(), 4)
    assert torch.all(a.positions[:, 3] == 0)
    sg = dv.scene_geometry([m], cpu)
    assert dv.scene_geometry([m], cpu) is sg
    m.positions = np.array(m.positions, copy=True) * 2.0
    b = dv.device_mesh(m, cpu)
    assert b is not a
    assert np.array_equal(b.positions[:, :3].numpy(), np.asarray(m.positions, np.float32))
    assert dv.scene_geometry([m], cpu) is not sg

    for k in range(20):
        mk = make_sphere(4 + k % 3, 6)
        d = dv.scene_geometry([mk], cpu)
        assert d.meshes[0].vertex_count == mk.vertex_count()
        del mk, d
        gc.collect()
    dv.drop_device_copies([m])
    assert dv.device_mesh(m, cpu) is not b


def test_chunk_size_balances_small_frames():
    """pipeline._choose_chunk: 2048-triangle chunks for streamed frames, down
    to 128 so a small frame still gives every resident warp several chunks."""
    from paper_2604_21749_b200.pipeline import _choose_chunk
    target = 4 * 32 * 148
    assert _choose_chunk(99_998_082, 2048, 128, target) == 2048
    assert _choose_chunk(999_698, 2048, 128, target) == 128
    assert _choose_chunk(10_078_880, 2048, 128, target) == 512
    assert _choose_chunk(0, 2048, 128, target) == 128
    for w in (1, 10 ** 5, 3 * 10 ** 6, 10 ** 9):
        c = _choose_chunk(w, 2048, 128, target)
        assert c % 128 == 0 and 128 <= c <= 2048


def _grazing_transforms(rng, cam, n):
    """Instance transforms whose boxes touch or nearly touch frustum planes:
    random rotations / scales, translated so the box's extreme corner lands
    on a plane (plus tiny offsets of a few ulps either way)."""
    from paper_2604_21749_b200.scene import frustum_planes, transformed_aabb
    planes = frustum_planes(cam)
    aabb = np.array([[-0.5, -0.5, -0.5], [0.5, 0.5, 0.5]])
    out = []
    for k in range(n):
        q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
        T = np.eye(4)
        T[:3, :3] = q * rng.uniform(0.1, 2.0)
        T[:3, 3] = rng.uniform(-8, 8, size=3) + np.array([0, 0, -10.0])
        if k % 2 == 0:
            pl = planes[rng.integers(0, len(planes))]
            box = transformed_aabb(aabb, T)
            c = np.where(pl[:3] < 0.0, box[1], box[0])
            v = float(pl[:3] @ c + pl[3])
            n3 = pl[:3] / np.dot(pl[:3], pl[:3])
            T[:3, 3] -= v * n3                        # corner onto the plane
            T[:3, 3] += n3 * rng.choice([0.0, 1e-15, -1e-15, 1e-12, -1e-12])
        out.append(T)
    return out


def test_batched_cull_matches_per_instance_path():
    """build_draw_list's batched, certified cull (scene._node_visibility)
    gives the reference's items, order and prefix sums (scenecore.py:240-265,
    restated per instance in oracle/host.py), including boxes that graze the
    frustum planes."""
    from paper_2604_21749_b200.scene import Mesh, SceneNode
    rng = np.random.default_rng(11)
    cam = Camera.look_at((0.0, 0.0, 2.0), (0.0, 0.0, -10.0), width=640, height=480)
    mesh = Mesh(positions=np.zeros((3, 3)), indices=np.array([0, 1, 2], dtype=np.uint32),
                triangle_count=1, aabb=np.array([[-0.5, -0.5, -0.5], [0.5, 0.5, 0.5]]))
    scene = [SceneNode(mesh=mesh, transforms=_grazing_transforms(rng, cam, 400)),
             SceneNode(mesh=mesh, transforms=_grazing_transforms(rng, cam, 5)),
             SceneNode(mesh=mesh, transforms=_grazing_transforms(rng, cam, 1000))]
    dl = build_draw_list(scene, cam)
    ref = oh.build_draw_list(scene, cam)
    assert len(dl.items) == len(ref.items)
    for a, b in zip(dl.items, ref.items):
        assert a.node_index == b.node_index
        assert np.array_equal(np.asarray(a.instance_transform), b.transform)
    assert np.array_equal(dl.prefix_sums, ref.prefix)
    assert 0 < len(dl.items) < 1405


# --------------------------------------------------------------------------
# drop-in context and shard-local geometry (CPU: host logic only)

def test_reference_render_context_is_adopted():
    """render_draw_list(ctx=<trirast RenderContext>): the reference's flat
    positions / indices become one mesh addressed through its item offsets,
    and its matrices and prefix are used as given (pipeline.py:68-84)."""
    from refctx import from_golden
    from paper_2604_21749_b200.pipeline import adopt_context
    for name in ("lantern_on", "random2024_005", "classifier"):
        g = load_golden(name)
        scene = golden_scene(g, compressed=False)
        cam = golden_camera(g)
        dl = build_draw_list(scene, cam)
        ref = from_golden(g)
        ctx = adopt_context(ref, dl, cam)
        assert len(ctx.meshes) == 1
        m = ctx.meshes[0]
        assert np.array_equal(m.positions, g["ctx_positions"])
        assert np.array_equal(m.indices, g["ctx_indices"])
        assert np.array_equal(ctx.item_vtx_off, g["item_vtx_off"])
        assert np.array_equal(ctx.item_idx_off, g["item_idx_off"])
        assert np.array_equal(ctx.item_mv, g["item_mv"])
        assert np.array_equal(ctx.prefix, g["prefix"])
        assert np.array_equal(ctx.group_prefix, g["group_prefix"])
        assert np.array_equal(ctx.group_items, g["group_items"])
        assert (ctx.item_mesh == 0).all()
        # cached on the context object: the same flat mesh next time
        assert adopt_context(ref, dl, cam).meshes[0] is m
    with pytest.raises(TypeError, match="RenderContext"):
        adopt_context(object(), dl, cam)


def test_shard_items_select_only_the_ranks_geometry():
    """A rank's work range touches only its items: PreparedFrame uploads
    only those items' meshes (each GPU holds its shard)."""
    from paper_2604_21749_b200.distributed import shard_range
    from paper_2604_21749_b200.pipeline import build_context, shard_items
    from paper_2604_21749_b200 import generators as gen
    # 6 distinct meshes, one node each (flat work space)
    nodes = []
    for k in range(6):
        m = gen.make_tessellated_quad(4 + k)
        T = np.eye(4)
        T[0, 3] = 1.5 * k - 4.0
        nodes.append(SceneNode(mesh=m, transforms=[T]))
    cam = Camera.look_at((0.0, 0.0, 9.0), (0.0, 0.0, 0.0), width=320, height=120)
    dl = build_draw_list(nodes, cam)
    ctx = build_context(dl, cam)
    assert len(ctx.meshes) == 6
    total = dl.total_triangles
    seen = np.zeros(6, dtype=int)
    for world in (2, 3):
        for r in range(world):
            lo, hi = shard_range(total, world, r)
            mask = shard_items(ctx, (lo, hi), False)
            s, e = ctx.prefix[:-1], ctx.prefix[1:]
            want = (e > lo) & (s < hi)
            assert np.array_equal(mask, want)
            used = np.unique(ctx.item_mesh[mask])
            assert len(used) < 6                         # never the whole scene
            seen[used] += 1
    assert (seen > 0).all()
    # instanced work space: whole groups (all instances of a node)
    lg = gen.make_lantern_grid(3, 2, tris_per_mesh=200, spacing=1.8)
    extra = SceneNode(mesh=gen.make_tessellated_quad(10), transforms=[np.eye(4)])
    cam = Camera.look_at((0.0, 6.0, 9.0), (0.0, 0.0, 0.0), width=160, height=120)
    dl = build_draw_list(lg + [extra], cam)
    ctx = build_context(dl, cam)
    g0 = int(ctx.group_prefix[1])
    m0 = shard_items(ctx, (0, g0), True)
    assert m0.sum() == ctx.group_item_count[0]
    assert len(np.unique(ctx.item_mesh[m0])) == 1
    m1 = shard_items(ctx, (g0, int(ctx.group_prefix[-1])), True)
    assert not (m0 & m1).any() and (m0 | m1).all()


def test_benchcli_rows_mirror_the_reference_toggles(tmp_path):
    """benchcli.bench_rows = cli.py:115-141: labels, configs, timing-only."""
    from paper_2604_21749_b200 import benchcli
    cam = Camera.look_at((0.0, 0.0, 3.0), (0.0, 0.0, 0.0), width=64, height=48)
    cfg = RasterConfig()
    assert [r[0] for r in benchcli.bench_rows(cam, cfg)] == ["base"]
    rows = benchcli.bench_rows(cam, cfg, "tinyCull")
    assert [(r[0], r[2].tiny_cull, r[3]) for r in rows] == [("tinyCull=on", True, True),
                                                          ("tinyCull=off", False, True)]
    rows = benchcli.bench_rows(cam, cfg, "workers")
    assert [r[2].workers for r in rows] == [1, 2, 4, 8] and all(r[3] for r in rows)
    rows = benchcli.bench_rows(cam, cfg, "instancing")
    assert [r[2].instancing for r in rows] == ["on", "off"]
    rows = benchcli.bench_rows(cam, cfg, "superSampling")
    assert [(r[1].supersampling, r[1].internal_width, r[3]) for r in rows] == [
        (1, 64, False), (2, 128, False), (4, 256, False)]
    with pytest.raises(ValueError):
        benchcli.bench_rows(cam, cfg, "nope")
    rep = [{c: (1.5 if c.endswith("Ms") else (3 if c in ("visibleTriangles", "fragments", "culled")
                                               else "x")) for c in benchcli.COLS}]
    out = tmp_path / "rows.csv"
    benchcli.write_csv(rep, out)
    assert out.read_text().splitlines()[0] == ",".join(benchcli.COLS)
    assert "stage1Ms" in benchcli.format_table(rep).splitlines()[0]


def test_row_raster_choice_follows_fragments_per_triangle():
    """PreparedFrame._choose_row_raster: the fp64 pass's row-parallel raster
    (curast.h s1_row_raster) only for frames averaging >= 1 stage-1 fragment
    per rasterized triangle — config C (604,610 / 462,315) and A4 on, the
    dense configs B (4,666,508 / 9,331,200) and D (0.32) off, empty frames off."""
    import types
    from paper_2604_21749_b200 import _native as N
    from paper_2604_21749_b200.pipeline import PreparedFrame

    def choose(rast, frags):
        c = np.zeros(N.COUNTER_SLOTS, dtype=np.int64)
        c[N.C_S1 + 0], c[N.C_S1 + 7] = rast, frags
        pf = types.SimpleNamespace(frame=N.CurastFrame())
        PreparedFrame._choose_row_raster(pf, c)
        return pf.frame.s1_row_raster

    assert choose(462_315, 604_610) == 1
    assert choose(9_331_200, 4_666_508) == 0
    assert choose(7_097_009, 2_276_079) == 0
    assert choose(0, 0) == 0


def test_c_abi_rejects_invalid_frames_before_any_launch():
    """The C ABI validates a frame on the host and returns CURAST_E_INVALID
    with a message before touching the device (no GPU needed): resolution
    limits, tile size, filter without rows, stage-1 work tables, chunk sizes,
    the fp64 queue and the 2^22-item limit of the queue tags."""
    import ctypes
    from paper_2604_21749_b200 import _native as N
    L = N.lib()
    dummy = ctypes.c_void_p(0x1000)        # never dereferenced on these paths

    def base():
        f = N.CurastFrame()
        f.fb = dummy
        f.counters = dummy
        f.width, f.height, f.tile_px = 64, 48, 64
        f.n_units = 1
        f.unit_chunk_prefix = dummy
        f.unit_index = dummy
        f.chunk_tris = 128
        f.qx = dummy
        f.qx_cap = 1024
        f.n_items = 1
        return f

    def err(f, fn=L.curast_stage1):
        rc = fn(ctypes.byref(f), None)
        return rc, L.curast_last_error().decode()

    cases = [
        (dict(width=1 << 16, height=1 << 15), "resolution"),
        (dict(tile_px=0), "tile_px"),
        (dict(tile_px=5000), "tile_px"),
        (dict(use_filter=1), "item_filter"),
        (dict(unit_chunk_prefix=None), "work table"),
        (dict(chunk_tris=100), "chunk_tris"),
        (dict(chunk_tris=4096), "chunk_tris"),
        (dict(qx=None), "fp64 queue"),
        (dict(qx_cap=1 << 32), "2^32"),
        (dict(n_items=1 << 22), "2^22"),
    ]
    for fields, needle in cases:
        f = base()
        for k, v in fields.items():
            setattr(f, k, v)
        rc, msg = err(f)
        assert rc == -1, (fields, rc, msg)
        assert needle in msg, (fields, msg)
    f = base()
    f.fb = None
    assert err(f, L.curast_frame_clear)[0] == -1
