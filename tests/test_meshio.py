"""TRIMESH1 files (meshio.py) against fixtures written and read back by the
reference's own save_mesh / load_mesh_asset (tests/golden/make_golden.py
trimesh), plus round trips and the reference's error behaviour."""

import os

import numpy as np
import pytest

from paper_2604_21749_b200 import RasterConfig, render_frame
from paper_2604_21749_b200 import meshio
from paper_2604_21749_b200.codec import is_packed_indices, is_quantized_positions
from paper_2604_21749_b200.scene import Camera, SceneNode
from oracle import host as oh
from scenes import GOLDEN

G = np.load(os.path.join(GOLDEN, "trimesh.npz"))
NAMES = ("raw", "compressed", "uvquad")


@pytest.mark.parametrize("name", NAMES)
def test_reference_files_load_identically(name):
    m = meshio.load_mesh(os.path.join(GOLDEN, f"mesh_{name}.trimesh"))
    assert m.triangle_count == int(G[f"{name}_ntris"])
    assert np.array_equal(m.positions_f64(), G[f"{name}_positions"])
    assert np.array_equal(m.indices_u32(), G[f"{name}_indices"])
    assert np.array_equal(np.asarray(m.aabb, np.float64), G[f"{name}_aabb"])
    if f"{name}_uvs" in G:
        assert np.array_equal(m.uvs, G[f"{name}_uvs"])
    if f"{name}_colors" in G:
        assert np.array_equal(m.vertex_colors, G[f"{name}_colors"])
    if name == "compressed":
        # payloads stay compressed: no host decode on load
        assert is_quantized_positions(m.positions) and is_packed_indices(m.indices)
    else:
        assert m.positions.dtype == np.float32


@pytest.mark.parametrize("name", NAMES)
def test_save_round_trip_is_byte_identical(name, tmp_path):
    src = os.path.join(GOLDEN, f"mesh_{name}.trimesh")
    m = meshio.load_mesh(src)
    dst = tmp_path / "out.trimesh"
    meshio.save_mesh(dst, m)
    assert open(src, "rb").read() == open(dst, "rb").read()


def test_parse_errors_name_the_offset(tmp_path):
    data = open(os.path.join(GOLDEN, "mesh_compressed.trimesh"), "rb").read()
    p = tmp_path / "t.trimesh"
    p.write_bytes(data[:10])
    with pytest.raises(meshio.ParseError, match="truncated header at offset 10"):
        meshio.load_mesh(p)
    p.write_bytes(b"XXXXXXXX" + data[8:])
    with pytest.raises(meshio.ParseError, match="bad magic"):
        meshio.load_mesh(p)
    p.write_bytes(data[:32 + 24 + 10])
    with pytest.raises(meshio.ParseError, match="truncated positions at offset 56"):
        meshio.load_mesh(p)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_loaded_meshes_render_bit_exact(name):
    import torch
    m = meshio.load_mesh(os.path.join(GOLDEN, f"mesh_{name}.trimesh"), device=torch.device("cuda"))
    cam = Camera.look_at((0.3, 0.4, 2.2), (0.0, 0.0, 0.0), width=160, height=120)
    scene = [SceneNode(mesh=m, transforms=[np.eye(4)])]
    fb, _ = render_frame(scene, cam, RasterConfig())
    ref, _, _ = oh.render_reference(scene, cam)
    assert np.array_equal(fb.words, ref)
    assert int((fb.words != np.iinfo(np.uint64).max).sum()) > 100
