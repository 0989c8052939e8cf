"""Sort-last multi-GPU rendering.

One process per GPU.  Every rank builds the same host draw list (same prefix
sums, hence the same global triangle IDs), rasterizes the contiguous global-ID
range ``shard_range(total, world, rank)`` (or a unique-triangle range of the
instancing groups) into its own full-resolution visibility buffer, and the
buffers are composited with an unsigned 64-bit minimum:

* on GPUs: ``ncclAllReduce`` / ``ncclReduce`` / ``ncclReduceScatter`` with
  ``ncclUint64`` + ``ncclMin`` through libcurast_nccl.so (the communicator is
  bootstrapped by broadcasting an ncclUniqueId over torch.distributed);
* on CPU process groups (gloo, used by the tests): ``all_reduce(MIN)`` on the
  words with the sign bit flipped, which maps unsigned order onto signed order
  (CLEAR = all ones must stay the largest value; a plain int64 min would make
  it -1 and let it win).

The composite is bit-identical to a 1-GPU frame: min is associative and
commutative and every fragment carries its global ID.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch
import torch.distributed as dist

from . import _native as N

SIGN = -0x8000000000000000
_HERE = os.path.dirname(os.path.abspath(__file__))
NCCL_LIB = os.path.join(_HERE, "libcurast_nccl.so")


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, disjoint, covering split of [0, total) (rank-major)."""
    base, rem = divmod(int(total), int(world))
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def composite_min_u64_(words: torch.Tensor, group=None) -> torch.Tensor:
    """In-place unsigned-min all-reduce of int64-viewed u64 words through
    torch.distributed (any backend that supports MIN on int64)."""
    words ^= SIGN
    dist.all_reduce(words, op=dist.ReduceOp.MIN, group=group)
    words ^= SIGN
    return words


_nccl = None


def nccl_lib():
    global _nccl
    if _nccl is None:
        if not os.path.exists(NCCL_LIB):
            raise N.NativeError(f"{NCCL_LIB} missing (run __graft_entry__.build())")
        L = ctypes.CDLL(NCCL_LIB)
        P, I64, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        L.curast_nccl_last_error.restype = ctypes.c_char_p
        L.curast_nccl_unique_id.argtypes = [ctypes.c_char_p]
        L.curast_nccl_init.argtypes = [ctypes.POINTER(P), ctypes.c_char_p, I32, I32]
        L.curast_nccl_destroy.argtypes = [P]
        L.curast_nccl_allreduce_min_u64.argtypes = [P, P, I64, P]
        L.curast_nccl_reduce_min_u64.argtypes = [P, P, P, I64, I32, P]
        L.curast_nccl_reduce_scatter_min_u64.argtypes = [P, P, P, I64, P]
        for fn in ("curast_nccl_unique_id", "curast_nccl_init", "curast_nccl_destroy",
                   "curast_nccl_allreduce_min_u64", "curast_nccl_reduce_min_u64",
                   "curast_nccl_reduce_scatter_min_u64"):
            getattr(L, fn).restype = I32
        _nccl = L
    return _nccl


def _ncheck(rc, what):
    if rc != 0:
        raise N.NativeError(f"{what}: {nccl_lib().curast_nccl_last_error().decode()}")


def _group_key(group):
    """Cache key of a process group (None = the default group)."""
    return "default" if group is None else id(group)


def _group_src(group) -> int:
    """Global rank of the group's rank 0 (broadcast sources are global ranks)."""
    if group is None:
        return 0
    return dist.get_global_rank(group, 0)


class NcclComm:
    """A raw NCCL communicator over the ranks of ``group`` (default: the
    default process group).  The ncclUniqueId is broadcast from the group's
    first rank; ``close()`` destroys the communicator."""

    def __init__(self, group=None):
        L = nccl_lib()
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        buf = ctypes.create_string_buffer(128)
        if self.rank == 0:
            _ncheck(L.curast_nccl_unique_id(buf), "ncclGetUniqueId")
        obj = [bytes(buf.raw)]
        dist.broadcast_object_list(obj, src=_group_src(group), group=group)
        self.comm = ctypes.c_void_p()
        _ncheck(L.curast_nccl_init(ctypes.byref(self.comm), obj[0], self.world, self.rank),
                "ncclCommInitRank")

    def allreduce_min(self, words: torch.Tensor, stream=None):
        st = (stream or torch.cuda.current_stream()).cuda_stream
        _ncheck(nccl_lib().curast_nccl_allreduce_min_u64(self.comm, words.data_ptr(),
                                                         words.numel(), st), "allreduce")

    def reduce_min(self, words: torch.Tensor, out: torch.Tensor, root=0, stream=None):
        st = (stream or torch.cuda.current_stream()).cuda_stream
        _ncheck(nccl_lib().curast_nccl_reduce_min_u64(self.comm, words.data_ptr(), out.data_ptr(),
                                                      words.numel(), root, st), "reduce")

    def reduce_scatter_min(self, words: torch.Tensor, stripe: torch.Tensor, stream=None):
        st = (stream or torch.cuda.current_stream()).cuda_stream
        _ncheck(nccl_lib().curast_nccl_reduce_scatter_min_u64(
            self.comm, words.data_ptr(), stripe.data_ptr(), stripe.numel(), st), "reduce_scatter")

    def close(self):
        if self.comm:
            nccl_lib().curast_nccl_destroy(self.comm)
            self.comm = None


_comms: dict = {}


def group_comm(group=None) -> NcclComm:
    """The cached NCCL communicator of ``group`` (created on first use, one
    per group for the life of the process; ``close_comms()`` releases them).
    A communicator per frame would leak one ncclComm and its buffers per
    call."""
    key = _group_key(group)
    c = _comms.get(key)
    if c is None or c.comm is None:
        c = NcclComm(group)
        _comms[key] = c
    return c


def close_comms() -> None:
    """Destroy every cached communicator (call before destroy_process_group)."""
    for c in _comms.values():
        c.close()
    _comms.clear()


def _use_nccl(words: torch.Tensor, group) -> bool:
    return (words.is_cuda and dist.get_backend(group) == "nccl"
            and os.path.exists(NCCL_LIB))


def _min_on_host(words: torch.Tensor, group) -> None:
    """Unsigned-min all-reduce through a CPU process group (gloo): CUDA
    words are staged through host memory."""
    if words.is_cuda:
        host = words.cpu()
        composite_min_u64_(host, group)
        words.copy_(host)
    else:
        composite_min_u64_(words, group)


class Compositor:
    """Per-frame composite of a rank's visibility buffer (int64 tensor) over
    the ranks of ``group``: NCCL (ncclUint64 / ncclMin, cached communicator)
    for CUDA words on an NCCL group, else the sign-flipped MIN all-reduce of
    the group's backend (gloo, through host memory)."""

    def __init__(self, words: torch.Tensor, world: int | None = None, group=None):
        self.words = words
        self.group = group
        self.world = dist.get_world_size(group) if world is None else int(world)
        self.launches_per_call = 1
        if _use_nccl(words, group):
            self.comm = group_comm(group)
        else:
            self.comm = None
            self.launches_per_call = 3

    def allreduce_min(self):
        if self.comm is not None:
            self.comm.allreduce_min(self.words)
        else:
            _min_on_host(self.words, self.group)

    def reduce_scatter_min(self, rank: int | None = None):
        """Composite into stripes: this rank receives the unsigned-min of all
        ranks' words over its 1/world slice (self.stripe); the full VB exists
        once, distributed — the input of the striped resolve."""
        if rank is None:
            rank = dist.get_rank(self.group)
        n = self.words.numel()
        per = -(-n // self.world)
        if not hasattr(self, "stripe"):
            self.stripe = torch.empty(per, dtype=torch.int64, device=self.words.device)
            self._padded = (self.words if per * self.world == n else
                            torch.full((per * self.world,), -1, dtype=torch.int64,
                                       device=self.words.device))
        if self._padded is not self.words:
            self._padded[:n].copy_(self.words)
        if self.comm is not None:
            self.comm.reduce_scatter_min(self._padded, self.stripe)
        else:
            full = self._padded.clone()
            _min_on_host(full, self.group)
            self.stripe.copy_(full[rank * per:(rank + 1) * per])
        return self.stripe


def render_sharded(draw_list, camera, cfg=None, *, group=None):
    """Sort-last frame on the calling rank's GPU: rasterize this rank's
    global-ID shard, composite over all ranks of ``group``; every rank
    returns the full composite Framebuffer and its shard's FrameStats (sum
    them for totals).  Only the meshes of this rank's shard are uploaded
    (``PreparedFrame(work_range=...)``)."""
    from .config import RasterConfig
    from .pipeline import _cached_frame, work_space
    from .scene import Framebuffer
    cfg = cfg or RasterConfig()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = shard_range(work_space(draw_list, cfg), world, rank)
    pf = _cached_frame(draw_list, camera, cfg, None, None, (lo, hi))
    c, secs = pf.run()
    st = pf.stats(c, secs)
    if world > 1:
        Compositor(pf.fb, world, group).allreduce_min()
    return Framebuffer(camera.internal_width, camera.internal_height, device_words=pf.fb), st


def stripe_rows(height: int, world: int, rank: int) -> tuple[int, int, int]:
    """(first row, rows, rows per stripe) of ``rank``'s resolve stripe: equal
    stripes of ceil(H / world) rows (NCCL reduce-scatter needs equal
    counts; the tail is padded with CLEAR rows)."""
    per = -(-int(height) // int(world))
    r0 = int(rank) * per
    return r0, max(0, min(per, int(height) - r0)), per


def render_sharded_resolved(draw_list, camera, cfg=None, shading=None, *, root=0, group=None):
    """Sort-last frame with a striped resolve: rasterize this
    rank's shard, reduce-scatter the visibility buffers by unsigned min so
    each rank owns a stripe of rows, shade the stripe
    (resolve_frame_device(rows=...)), gather the RGBA8 stripes on ``root``.
    Returns (image [H, W, 4] uint8 CUDA tensor on root / None elsewhere,
    this rank's FrameStats, this rank's ResolveStats)."""
    from .config import RasterConfig, ShadingConfig
    from .pipeline import PreparedFrame, build_context
    from .resolve import resolve_frame_device
    from .scene import Framebuffer
    cfg = cfg or RasterConfig()
    shading = shading or ShadingConfig()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    ctx = build_context(draw_list, camera)
    instanced = (cfg.instancing == "on"
                 or (cfg.instancing == "auto" and ctx.max_instances >= 2))
    space = int(ctx.group_prefix[-1]) if instanced else int(draw_list.total_triangles)
    lo, hi = shard_range(space, world, rank)
    pf = PreparedFrame(draw_list, camera, cfg, ctx, work_range=(lo, hi))
    c, secs = pf.run()
    st = pf.stats(c, secs)
    W, H = camera.internal_width, camera.internal_height
    r0, n, per = stripe_rows(H, world, rank)
    words = pf.fb
    if per * world * W > words.numel():                    # pad with CLEAR rows
        words = torch.cat([words, words.new_full((per * world * W - words.numel(),), -1)])
    stripe = torch.empty(per * W, dtype=torch.int64, device=words.device)
    if world > 1 and _use_nccl(words, group):
        group_comm(group).reduce_scatter_min(words, stripe)
    else:
        full = words.clone()
        if world > 1:
            _min_on_host(full, group)
        stripe.copy_(full[rank * per * W:(rank + 1) * per * W])
    fb = Framebuffer(W, H, device_words=pf.fb)
    img, rst = resolve_frame_device(fb, draw_list, camera, shading, rows=(r0, n),
                                    stripe_words=stripe[:n * W])
    part = torch.zeros((per, W, 4), dtype=torch.uint8, device=img.device)
    part[:n] = img
    if world > 1 and _use_nccl(part, group):
        parts = [torch.empty_like(part) for _ in range(world)]
        dist.all_gather(parts, part, group=group)
    elif world > 1:
        hp = part.cpu()
        hparts = [torch.empty_like(hp) for _ in range(world)]
        dist.all_gather(hparts, hp, group=group)
        parts = [p.to(part.device) for p in hparts]
    else:
        parts = [part]
    image = torch.cat(parts)[:H] if rank == root else None
    return image, st, rst
