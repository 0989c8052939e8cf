"""Vectorised synthetic geometry of the named benchmark shapes.

Outputs are element-for-element identical to the reference generators
(trirast/scenedesc.py:197-316), which build vertex/triangle lists in Python
loops and cannot reach 10^8 triangles; identity is checked in
tests/test_generators.py against the reference's own outputs
(tests/golden/generators.npz).  Trigonometry is evaluated with ``math`` on the
distinct angles only (numpy's SIMD sin/cos may round differently).

``f32=True`` rounds positions to float32 (the SURVEY §8(d) configs feed the
same rounded positions to the GPU path and to the CPU oracle).
"""

from __future__ import annotations

import math

import numpy as np

from .scene import Camera, Mesh, SceneNode


def mesh_from_arrays(positions, indices, uvs=None, colors=None, name="") -> Mesh:
    positions = np.asarray(positions, dtype=np.float64)
    indices = np.asarray(indices, dtype=np.uint32).ravel()
    aabb = np.stack([positions.min(axis=0), positions.max(axis=0)])
    return Mesh(positions=positions, indices=indices,
                triangle_count=len(indices) // 3, aabb=aabb,
                uvs=None if uvs is None else np.asarray(uvs, dtype=np.float64),
                vertex_colors=None if colors is None else np.asarray(colors, dtype=np.uint8),
                name=name)


def _round_f32(mesh: Mesh) -> Mesh:
    p = np.asarray(mesh.positions, dtype=np.float64).astype(np.float32).astype(np.float64)
    mesh.positions = p
    mesh.aabb = np.stack([p.min(axis=0), p.max(axis=0)])
    mesh._positions_cache = None
    return mesh


def grid_indices(n: int) -> np.ndarray:
    """Triangles (a,c,b),(b,c,d) per cell, row-major (scenedesc.py:207-214)."""
    j, i = np.meshgrid(np.arange(n, dtype=np.int64), np.arange(n, dtype=np.int64),
                       indexing="ij")
    a = (j * (n + 1) + i).ravel()
    b = a + 1
    c = a + n + 1
    d = c + 1
    tris = np.empty((a.size, 2, 3), dtype=np.uint32)
    tris[:, 0, 0] = a
    tris[:, 0, 1] = c
    tris[:, 0, 2] = b
    tris[:, 1, 0] = b
    tris[:, 1, 1] = c
    tris[:, 1, 2] = d
    return tris.reshape(-1)


def make_tessellated_quad(n: int, *, f32: bool = False, with_uvs: bool = True) -> Mesh:
    """Unit quad in the XY plane as an n x n grid, 2n^2 triangles, front faces
    toward +z (scenedesc.py:197-215)."""
    if n < 1:
        raise ValueError("tessellation factor must be >= 1")
    axis = np.linspace(-0.5, 0.5, n + 1)
    xs, ys = np.meshgrid(axis, axis)
    pos = np.stack([xs.ravel(), ys.ravel(), np.zeros((n + 1) ** 2)], axis=1)
    uvs = np.stack([xs.ravel() + 0.5, ys.ravel() + 0.5], axis=1) if with_uvs else None
    mesh = mesh_from_arrays(pos, grid_indices(n), uvs=uvs, name=f"quad{n}")
    return _round_f32(mesh) if f32 else mesh


def make_sphere(rings: int, segments: int, radius: float = 1.0, name: str = "sphere",
                *, f32: bool = False) -> Mesh:
    """UV sphere with normal-encoding vertex colours (scenedesc.py:218-245)."""
    if rings < 2 or segments < 3:
        raise ValueError("need rings >= 2 and segments >= 3")
    st = np.array([math.sin(math.pi * r / rings) for r in range(rings + 1)])
    ct = np.array([math.cos(math.pi * r / rings) for r in range(rings + 1)])
    sp = np.array([math.sin(2.0 * math.pi * s / segments) for s in range(segments)])
    cp = np.array([math.cos(2.0 * math.pi * s / segments) for s in range(segments)])
    rs = radius * st
    verts = np.empty((rings + 1, segments, 3))
    verts[:, :, 0] = rs[:, None] * cp[None, :]
    verts[:, :, 1] = (radius * ct)[:, None]
    verts[:, :, 2] = rs[:, None] * sp[None, :]
    verts = verts.reshape(-1, 3)
    colors = np.clip((verts / radius * 0.5 + 0.5) * 255, 0, 255)
    colors = np.concatenate([colors, np.full((len(verts), 1), 255)], axis=1)
    r = np.arange(rings, dtype=np.int64)[:, None]
    s = np.arange(segments, dtype=np.int64)[None, :]
    a = r * segments + s
    b = r * segments + (s + 1) % segments
    c = a + segments
    d = b + segments
    t1 = np.stack(np.broadcast_arrays(a, b, c), axis=-1)      # (rings, segs, 3)
    t2 = np.stack(np.broadcast_arrays(b, d, c), axis=-1)
    both = np.stack([t1, t2], axis=2)                         # (rings, segs, 2, 3)
    keep = np.ones((rings, segments, 2), dtype=bool)
    keep[0, :, 0] = False
    keep[rings - 1, :, 1] = False
    tris = both[keep]
    mesh = mesh_from_arrays(verts, tris, colors=colors, name=name)
    return _round_f32(mesh) if f32 else mesh


def sphere_dims_for(tris: int) -> tuple[int, int]:
    """rings/segments for roughly ``tris`` triangles (scenedesc.py:248-252)."""
    segments = max(3, int(round(math.sqrt(tris / 2.0))))
    rings = max(2, int(round(tris / (2.0 * segments))) + 1)
    return rings, segments


def make_lantern_grid(count_x: int, count_y: int, tris_per_mesh: int = 2000,
                      spacing: float = 2.0, *, f32: bool = False) -> list:
    """Grid of instances of one sphere mesh (scenedesc.py:303-316)."""
    rings, segments = sphere_dims_for(tris_per_mesh)
    mesh = make_sphere(rings, segments, radius=0.7, name="lantern", f32=f32)
    transforms = []
    for iy in range(count_y):
        for ix in range(count_x):
            m = np.eye(4)
            m[0, 3] = (ix - (count_x - 1) / 2.0) * spacing
            m[2, 3] = (iy - (count_y - 1) / 2.0) * spacing
            transforms.append(m)
    return [SceneNode(mesh=mesh, transforms=transforms)]


# ---------------------------------------------------------------- configs
def config_a(f32: bool = True):
    """A: 1M tessellated sphere @1920x1080."""
    mesh = make_sphere(*sphere_dims_for(1_000_000), f32=f32)
    cam = Camera.look_at((0.0, 0.0, 3.0), (0.0, 0.0, 0.0), width=1920, height=1080)
    return [SceneNode(mesh=mesh, transforms=[np.eye(4)])], cam


def config_b(n: int = 7071, f32: bool = True, width: int = 3840, height: int = 2160):
    """B: dense grid (make_tessellated_quad layout), n=7071 -> 99,998,082
    pixel-sized triangles, camera framing the quad's vertical extent
    @3840x2160."""
    mesh = make_tessellated_quad(n, f32=f32, with_uvs=False)
    dist = 0.5 / math.tan(math.radians(30.0))
    cam = Camera.look_at((0.0, 0.0, dist), (0.0, 0.0, 0.0), width=width, height=height)
    return [SceneNode(mesh=mesh, transforms=[np.eye(4)])], cam


def config_c(f32: bool = True, width: int = 3840, height: int = 2160):
    """C: mixed-size scene (far micro-grid, near-crossing ground plane, 40
    medium spheres) exercising stages 2 and 3."""
    grid = make_tessellated_quad(2236, f32=f32, with_uvs=False)
    gt = np.eye(4)
    gt[:3, :3] *= 8.0
    gt[:3, 3] = (0.0, 1.0, -30.0)
    ground = make_tessellated_quad(8, f32=f32, with_uvs=False)
    rt = np.eye(4)
    # quad lies in XY; rotate to the XZ plane facing +y, scale to 200x200
    rt[:3, :3] = np.array([[200.0, 0.0, 0.0], [0.0, 0.0, 200.0], [0.0, -200.0, 0.0]])
    rt[:3, 3] = (0.0, -1.0, 0.0)
    sph = make_sphere(*sphere_dims_for(2000), radius=0.6, f32=f32)
    rng = np.random.default_rng(1)
    sts = []
    for c in rng.uniform([-6.0, -0.5, -14.0], [6.0, 3.0, -4.0], size=(40, 3)):
        m = np.eye(4)
        m[:3, 3] = c
        sts.append(m)
    scene = [SceneNode(mesh=grid, transforms=[gt]), SceneNode(mesh=ground, transforms=[rt]),
             SceneNode(mesh=sph, transforms=sts)]
    cam = Camera.look_at((0.0, 0.5, 2.0), (0.0, 0.3, -10.0), width=width, height=height)
    return scene, cam


def config_d(f32: bool = True, tris_per_mesh: int = 1_000_000, width: int = 3840,
             height: int = 2160):
    """D: 1M-triangle sphere x 1000 instances (40 x 25 lantern grid)."""
    scene = make_lantern_grid(40, 25, tris_per_mesh=tris_per_mesh, spacing=2.0, f32=f32)
    cam = Camera.look_at((0.0, 32.0, 45.0), (0.0, 0.0, 0.0), width=width, height=height)
    return scene, cam


# --------------------------------------------------------------------- config E
# Zorah-scale synthetic scene: distinct displaced grids
# of n x n cells, tiled edge to edge into one terrain-like surface and seen
# from above.  Each mesh's heights come from an integer hash of (column, row,
# seed), so every coordinate is exactly representable in float32 and the host
# (numpy) and device (torch) generators produce the same bits.
E_DISPLACEMENT = 2.0 ** -20          # height step: |z| <= 512 steps ~ 4.9e-4


def _e_heights(i, j, seed, xp):
    """z of grid vertex (column i, row j) of mesh ``seed`` (int64 arrays of
    numpy or torch): a 32-bit integer hash, 10 bits of it, centred."""
    h = (i * 73856093) ^ (j * 19349663) ^ (seed * 83492791 + 0x9E3779B9)
    h = h & 0xFFFFFFFF
    h = (h ^ (h >> 15)) * 0x2C1B3C6D & 0xFFFFFFFF
    h = (h ^ (h >> 12)) * 0x297A2D39 & 0xFFFFFFFF
    h = h ^ (h >> 15)
    v = ((h >> 8) & 0x3FF) - 512
    return v


def _e_axis(n: int) -> np.ndarray:
    """Vertex coordinates along one axis, float32-rounded (the make_tessellated_quad axis)."""
    return np.linspace(-0.5, 0.5, n + 1).astype(np.float32)


E_AABB_Z = (-512 * E_DISPLACEMENT, 511 * E_DISPLACEMENT)


def displaced_grid(n: int, seed: int) -> Mesh:
    """Host-generated mesh ``seed`` of config E (float32-exact float64
    positions, grid_indices topology)."""
    ax = _e_axis(n).astype(np.float64)
    j, i = np.meshgrid(np.arange(n + 1, dtype=np.int64), np.arange(n + 1, dtype=np.int64),
                       indexing="ij")
    z = _e_heights(i.ravel(), j.ravel(), np.int64(seed), np) * E_DISPLACEMENT
    pos = np.stack([ax[i.ravel()], ax[j.ravel()], z.astype(np.float64)], axis=1)
    aabb = np.array([[-0.5, -0.5, E_AABB_Z[0]], [0.5, 0.5, E_AABB_Z[1]]])
    return Mesh(positions=pos, indices=grid_indices(n), triangle_count=2 * n * n, aabb=aabb,
                name=f"egrid{seed}")


class DeviceGeneratedMesh(Mesh):
    """A config-E mesh whose geometry is generated on the GPU when it is
    first made resident (device.device_mesh): no host copy of the positions
    or indices ever exists, so a rank materialises only its shard's meshes
    (SURVEY §7.3 hard part 5).  The bits equal ``displaced_grid(n, seed)``."""

    def __init__(self, n: int, seed: int, compressed: bool = False):
        super().__init__(positions=("egrid", n, seed, compressed),
                         indices=("egrid", n, seed, compressed), triangle_count=2 * n * n,
                         aabb=np.array([[-0.5, -0.5, E_AABB_Z[0]], [0.5, 0.5, E_AABB_Z[1]]]),
                         name=f"egrid{seed}")
        self.grid_n = n
        self.seed = seed
        self.compressed = compressed

    def vertex_count(self) -> int:
        return (self.grid_n + 1) ** 2

    def generate(self, device):
        """(positions float32[V, 4] CUDA, indices int32[3T] CUDA)."""
        import torch
        n = self.grid_n
        ax = torch.from_numpy(_e_axis(n)).to(device)
        k = torch.arange((n + 1) ** 2, device=device, dtype=torch.int64)
        i, j = k % (n + 1), k // (n + 1)
        z = _e_heights(i, j, int(self.seed), torch).to(torch.float32) * E_DISPLACEMENT
        pos = torch.zeros(((n + 1) ** 2, 4), dtype=torch.float32, device=device)
        pos[:, 0] = ax[i]
        pos[:, 1] = ax[j]
        pos[:, 2] = z
        c = torch.arange(n * n, device=device, dtype=torch.int64)
        a = (c // n) * (n + 1) + c % n
        b, cc = a + 1, a + n + 1
        d = cc + 1
        tri = torch.stack([a, cc, b, b, cc, d], dim=1).reshape(-1).to(torch.int32)
        return pos, tri

    def generate_compressed(self, device):
        """The same mesh stored as codec.quantize_positions + compress_indices
        would store it (u16 grid coordinates on the mesh box, indices bit-packed
        at bit_length(V - 1) bits), built in HBM: (coords int16[V, 4] (x, y, z,
        0), qgrid float64[6] (grid_min, grid_size), packed int32 words,
        (min_index, bits))."""
        import torch
        pos, tri = self.generate(device)
        box = torch.from_numpy(np.asarray(self.aabb, dtype=np.float64)).to(device)
        gmin = box[0]
        size = box[1] - box[0]
        size = torch.where(size > 0.0, size, torch.ones_like(size))
        q = torch.floor(65536.0 * (pos[:, :3].double() - gmin) / size).clamp_(0, 65535)
        coords = torch.zeros((pos.shape[0], 4), dtype=torch.int32, device=device)
        coords[:, :3] = q.to(torch.int32)
        coords = coords.to(torch.int16)                      # u16 bit patterns
        V = pos.shape[0]
        b = max(1, int(V - 1).bit_length())
        n = tri.numel()
        nwords = (n * b + 31) // 32 + 1
        words = torch.zeros(nwords + 2, dtype=torch.int64, device=device)
        rel = tri.to(torch.int64)
        bit = torch.arange(n, device=device, dtype=torch.int64) * b
        w, sh = bit >> 5, bit & 31
        full = rel << sh                                     # < 2^63: fields never overlap
        words.index_add_(0, w, full & 0xFFFFFFFF)
        words.index_add_(0, w + 1, full >> 32)
        packed = words & 0xFFFFFFFF                          # the u32 words, as int32 bits
        packed = torch.where(packed >= 2 ** 31, packed - 2 ** 32, packed).to(torch.int32)
        qgrid = np.concatenate([np.asarray(self.aabb[0], dtype=np.float64),
                                (size.cpu().numpy())])
        return coords, qgrid, packed, (0, b)


def config_e(n_meshes: int = 4750, n: int = 1414, seed: int = 0, width: int = 3840,
             height: int = 2160, on_device: bool = False, compressed: bool = False):
    """E: ~19B unique triangles (4,750 distinct displaced n=1414 grids of
    3,998,792 triangles = 18.99B), tiled edge to edge, overview camera
    @3840x2160.  ``on_device`` makes each mesh a
    DeviceGeneratedMesh (generated in HBM when a rank first needs it);
    otherwise the meshes are host arrays (small instances, oracle-checkable)."""
    cols = max(1, int(math.ceil(math.sqrt(n_meshes * width / height))))
    rows = -(-n_meshes // cols)
    scene = []
    for k in range(n_meshes):
        c, r = k % cols, k // cols
        T = np.eye(4)
        T[0, 3] = c - (cols - 1) / 2.0
        T[1, 3] = r - (rows - 1) / 2.0
        mesh = (DeviceGeneratedMesh(n, seed + k, compressed) if on_device
                else displaced_grid(n, seed + k))
        scene.append(SceneNode(mesh=mesh, transforms=[T]))
    half = max(rows / 2.0, cols / 2.0 * height / width) * 1.02
    dist = half / math.tan(math.radians(30.0))
    cam = Camera.look_at((0.0, 0.0, dist), (0.0, 0.0, 0.0), width=width, height=height)
    return scene, cam
