"""B200-native (sm_100a) CuRast 3-stage visibility-buffer rasterizer.

Drop-in for the reference package's rasterization path (``trirast``):
``render_frame`` / ``render_draw_list`` with the same arguments, return types,
64-bit visibility-word format and errors, running as hand-written CUDA kernels
behind a C ABI (include/curast.h).
"""

from .config import (FrameStats, RasterConfig, ShadingConfig, Stage1Stats,
                     Stage2Stats, Stage3Stats)
from .scene import (CLEAR, MAX_TRIANGLE_ID, TRIANGLE_ID_MASK, Camera, CapacityError,
                    DrawItem, DrawList, Framebuffer, Mesh, SceneNode,
                    build_draw_list, pack_fragment, projection_vector,
                    unpack_fragment)
from .pipeline import (PreparedFrame, build_context, classify_route,
                       clip_triangle_near_plane, render_draw_list, render_frame)
from .meshio import ParseError, load_mesh, save_mesh
from .resolve import debug_view, downsample, resolve_frame

__version__ = "0.1.0"

__all__ = [
    "CLEAR", "Camera", "CapacityError", "DrawItem", "DrawList", "Framebuffer",
    "FrameStats", "MAX_TRIANGLE_ID", "Mesh", "ParseError", "PreparedFrame", "RasterConfig",
    "SceneNode", "ShadingConfig", "Stage1Stats", "Stage2Stats", "Stage3Stats",
    "TRIANGLE_ID_MASK", "build_context", "build_draw_list", "classify_route",
    "clip_triangle_near_plane", "debug_view", "downsample", "load_mesh", "pack_fragment", "projection_vector",
    "render_draw_list", "render_frame", "resolve_frame", "save_mesh", "unpack_fragment",
]
