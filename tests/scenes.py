"""Seeded test scenes.

``random_scene`` reproduces the reference test suite's scene generator call
for call (pkg/tests/conftest.py:61-116: same RNG draws in the same order) so
that a seed names the same scene here and in the reference; identity is
checked against the reference's own output stored in tests/golden/.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2604_21749_b200 import codec  # noqa: E402
from paper_2604_21749_b200.generators import (make_lantern_grid, make_sphere,  # noqa: E402
                                              make_tessellated_quad, mesh_from_arrays,
                                              sphere_dims_for)
from paper_2604_21749_b200.scene import Camera, Mesh, SceneNode, projection_vector  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")


def mesh_from_soup(positions, indices=None, name="soup") -> Mesh:
    positions = np.asarray(positions, dtype=np.float64).reshape(-1, 3)
    if indices is None:
        indices = np.arange(len(positions), dtype=np.uint32)
    indices = np.asarray(indices, dtype=np.uint32).ravel()
    aabb = np.stack([positions.min(axis=0), positions.max(axis=0)])
    return Mesh(positions=positions, indices=indices, triangle_count=len(indices) // 3,
                aabb=aabb, name=name)


def identity_camera(width=128, height=96, fovy=math.radians(60.0), near=0.1,
                    supersampling=1) -> Camera:
    return Camera(position=np.zeros(3), view_transform=np.eye(4), fovy=fovy,
                  aspect=width / height, near=near, image_width=width,
                  image_height=height, supersampling=supersampling)


def view_point_for_pixel(px, py, depth, camera) -> np.ndarray:
    p = projection_vector(camera)
    w, h = camera.internal_width, camera.internal_height
    ndc_x = 2.0 * px / w - 1.0
    ndc_y = 1.0 - 2.0 * py / h
    return np.array([ndc_x * depth / p[0], ndc_y * depth / p[1], -depth])


def pixel_triangle_scene(pixels, depths, camera, extra=()):
    pts = [view_point_for_pixel(px, py, d, camera) for (px, py), d in zip(pixels, depths)]
    verts = list(pts) + [np.asarray(v, dtype=np.float64) for v in extra]
    return [SceneNode(mesh=mesh_from_soup(verts), transforms=[np.eye(4)])]


def _soup(rng, count, lo, hi, size_lo, size_hi):
    centers = rng.uniform(lo, hi, size=(count, 3))
    sizes = np.exp(rng.uniform(np.log(size_lo), np.log(size_hi), size=(count, 1, 1)))
    offsets = rng.normal(size=(count, 3, 3)) * sizes
    return (centers[:, None, :] + offsets).reshape(-1, 3)


def random_scene(rng):
    """Log-uniform 1..10^4 triangles, mixed sizes, >=10% near-plane crossers,
    30% chance of an instanced node, random 96x64 camera."""
    cam_pos = rng.uniform(-4.0, 4.0, 3)
    cam_pos += np.sign(cam_pos) * 1.5
    target = rng.uniform(-1.0, 1.0, 3)
    near = float(rng.uniform(0.05, 0.4))
    camera = Camera.look_at(cam_pos, target, width=96, height=64, near=near,
                            fovy=float(rng.uniform(0.6, 1.8)))
    total = max(1, int(round(10.0 ** rng.uniform(0.0, 4.0))))
    n_near = max(1, -(-total // 10))
    n_large = min(int(rng.integers(0, 6)), total)
    n_medium = min(int(rng.integers(0, 30)), total)
    n_small = max(0, total - n_near - n_large - n_medium)
    radius = max(1.0, float(np.linalg.norm(cam_pos - target)))
    parts = []
    if n_small:
        parts.append(_soup(rng, n_small, target - radius, target + radius,
                           0.004 * radius, 0.06 * radius))
    if n_medium:
        parts.append(_soup(rng, n_medium, target - radius, target + radius,
                           0.1 * radius, 0.35 * radius))
    if n_large:
        parts.append(_soup(rng, n_large, target - 0.3 * radius, target + 0.3 * radius,
                           0.8 * radius, 2.0 * radius))
    if n_near:
        centers = cam_pos + rng.normal(size=(n_near, 3)) * 0.2
        offsets = rng.normal(size=(n_near, 3, 3)) * rng.uniform(0.5, 2.0, size=(n_near, 1, 1))
        parts.append((centers[:, None, :] + offsets).reshape(-1, 3))
    nodes = [SceneNode(mesh=mesh_from_soup(np.concatenate(parts)), transforms=[np.eye(4)])]
    if rng.random() < 0.3:
        inst = _soup(rng, int(rng.integers(1, 20)), target - 0.5 * radius,
                     target + 0.5 * radius, 0.01 * radius, 0.2 * radius)
        transforms = []
        for _ in range(int(rng.integers(2, 5))):
            m = np.eye(4)
            m[:3, 3] = rng.uniform(-0.5, 0.5, 3) * radius
            transforms.append(m)
        nodes.append(SceneNode(mesh=mesh_from_soup(inst, name="inst"), transforms=transforms))
    return nodes, camera


def default_camera(width=640, height=480, supersampling=1):
    return Camera.look_at((0.0, 0.0, 5.0), (0.0, 0.0, 0.0), width=width, height=height,
                          supersampling=supersampling)


def classifier_scene():
    """Triangles straddling the 128 / 4096 px thresholds plus a near-plane
    crosser (the reference's make_classifier_scene layout)."""
    camera = default_camera()
    quads = [(0.08, -1.6, 1.2), (0.08, -1.3, 1.2), (0.5, 0.0, 1.4), (0.55, 0.8, 1.2),
             (2.2, 0.0, -0.6), (2.6, -0.9, -1.0)]
    pos, tris = [], []
    for size, cx, cy in quads:
        b = len(pos)
        h = size / 2.0
        pos += [(cx - h, cy - h, 0.0), (cx + h, cy - h, 0.0), (cx - h, cy + h, 0.0),
                (cx + h, cy + h, 0.0)]
        tris.append((b, b + 2, b + 1))
        tris.append((b + 1, b + 2, b + 3))
    b = len(pos)
    pos += [(-0.2, -0.2, 5.5), (0.2, -0.2, 5.5), (0.0, 0.2, 3.0)]
    tris.append((b, b + 2, b + 1))
    mesh = mesh_from_arrays(pos, tris, name="classifier")
    return [SceneNode(mesh=mesh, transforms=[np.eye(4)])], camera


def sphere_mesh(tris, radius=1.0, f32=False):
    return make_sphere(*sphere_dims_for(tris), radius=radius, f32=f32)


# ------------------------------------------------------------ golden loading
def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False))


def golden_names(prefix=""):
    return sorted(f[:-4] for f in os.listdir(GOLDEN)
                  if f.endswith(".npz") and f.startswith(prefix)
                  and f not in ("generators.npz", "packing.npz", "trimesh.npz", "debug_views.npz")
                  and not f.startswith("resolve_"))


def golden_scene(g, compressed=True):
    """Rebuild the fixture's scene with this package's types."""
    nodes = []
    for i in range(int(g["n_nodes"])):
        pos = g[f"node{i}_positions"]
        idx = g[f"node{i}_indices"]
        if compressed and f"node{i}_q_coords" in g:
            grid = g[f"node{i}_q_grid"]
            pos = codec.QuantizedPositions(grid_min=grid[:3].copy(), grid_size=grid[3:].copy(),
                                           coords=g[f"node{i}_q_coords"])
        if compressed and f"node{i}_p_data" in g:
            mn, b, cnt = (int(v) for v in g[f"node{i}_p_meta"])
            idx = codec.PackedIndexBuffer(min_index=mn, bits_per_index=b, count=cnt,
                                          data=g[f"node{i}_p_data"])
        mesh = Mesh(positions=pos, indices=idx, triangle_count=int(g[f"node{i}_tricount"]),
                    aabb=g[f"node{i}_aabb"],
                    vertex_colors=g.get(f"node{i}_colors"))
        nodes.append(SceneNode(mesh=mesh, transforms=list(g[f"node{i}_transforms"])))
    return nodes


def golden_camera(g):
    fovy, aspect, near = (float(v) for v in g["cam_scalars"])
    w, h, ss = (int(v) for v in g["cam_ints"])
    return Camera(position=g["cam_position"], view_transform=g["cam_view"], fovy=fovy,
                  aspect=aspect, near=near, image_width=w, image_height=h, supersampling=ss)


def golden_cfg(g):
    import ast
    kw = dict(ast.literal_eval(str(g["cfg_json"])))
    from paper_2604_21749_b200.config import RasterConfig
    return RasterConfig(**kw)


STAT_ORDER = ("s1.rasterized", "s1.forwarded", "s1.culled_frustum", "s1.culled_offscreen",
              "s1.culled_tiny", "s1.culled_backface", "s1.culled_degenerate",
              "s1.fragments", "s2.direct", "s2.tiled", "s2.dropped", "s2.fragments",
              "s2.tiles", "s3.entries", "s3.fragments")


def stats_vector_from_oracle(st):
    s1, s2, s3 = st["stage1"], st["stage2"], st["stage3"]
    return np.array([s1["rasterized"], s1["forwarded"], s1["culled_frustum"],
                     s1["culled_offscreen"], s1["culled_tiny"], s1["culled_backface"],
                     s1["culled_degenerate"], s1["fragments"], s2["direct"], s2["tiled"],
                     s2["dropped"], s2["fragments"], s2["tiles"], s3["entries"],
                     s3["fragments"]], dtype=np.int64)


def stats_vector_from_frame(st):
    s1, s2, s3 = st.stage1, st.stage2, st.stage3
    return np.array([s1.rasterized, s1.forwarded, s1.culled_frustum, s1.culled_offscreen,
                     s1.culled_tiny, s1.culled_backface, s1.culled_degenerate, s1.fragments,
                     s2.direct, s2.tiled, s2.dropped, s2.fragments, s2.tiles, s3.entries,
                     s3.fragments], dtype=np.int64)


def compress_scene(scene):
    """The same scene with QuantizedPositions + PackedIndexBuffer meshes
    (geomcodec.py:65-120 encoders), decoded in-register on the GPU and on
    the host by the oracle (configs Bq / Dq)."""
    from paper_2604_21749_b200 import codec
    out = []
    for node in scene:
        m = node.mesh
        q = codec.quantize_positions(m.positions, m.aabb)
        p = codec.compress_indices(m.indices)
        cm = Mesh(positions=q, indices=p, triangle_count=m.triangle_count, aabb=m.aabb,
                  vertex_colors=m.vertex_colors, name=m.name + "_q")
        out.append(SceneNode(mesh=cm, transforms=node.transforms))
    return out
