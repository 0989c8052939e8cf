"""Sort-last multi-rank path on CPU (gloo, world_size 2): every rank renders
its global-ID shard (the same partition the GPUs use), the visibility
buffers are composited with the unsigned-min all-reduce of
paper_2604_21749_b200.distributed, and the result must equal the 1-rank
frame bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_21749_b200.distributed import composite_min_u64_, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scenes():
    from scenes import random_scene, classifier_scene
    from paper_2604_21749_b200.generators import make_lantern_grid
    from paper_2604_21749_b200.scene import Camera
    out = [classifier_scene()]
    rng = np.random.default_rng(77)
    for _ in range(4):
        out.append(random_scene(rng))
    lg = make_lantern_grid(4, 3, tris_per_mesh=800, spacing=1.8)
    out.append((lg, Camera.look_at((0.0, 6.0, 9.0), (0.0, 0.0, 0.0), width=160, height=120)))
    return out


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import host as oh
    try:
        for k, (scene, cam) in enumerate(_scenes()):
            dl = oh.build_draw_list(scene, cam)
            cc = oh.camera_constants(cam)
            ctx = oh.build_context(dl, cam)
            for instanced in (False, True):
                space = int(ctx.group_prefix[-1]) if instanced else dl.total
                lo, hi = shard_range(space, world, rank)
                words, st, rc, _, _ = oh.render_context(ctx, cc, instanced=instanced,
                                                        work_range=(lo, hi))
                assert rc == 0
                t = torch.from_numpy(words.view(np.int64).copy())
                composite_min_u64_(t)
                n1 = torch.tensor([st["stage1"]["rasterized"], st["stage1"]["culled_tiny"],
                                   st["stage3"]["fragments"]], dtype=torch.int64)
                dist.all_reduce(n1)
                if rank == 0:
                    results[(k, instanced)] = (t.numpy().view(np.uint64).copy(), n1.numpy())
    finally:
        dist.destroy_process_group()


def test_shard_range_partitions():
    for total in (0, 1, 7, 100, 99998082):
        for world in (1, 2, 3, 8):
            parts = [shard_range(total, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == total
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c and a <= b


def test_two_rank_sort_last_composite_equals_single_rank():
    from oracle import host as oh
    mgr = mp.Manager()
    results = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, results), nprocs=2, join=True)
    for k, (scene, cam) in enumerate(_scenes()):
        ref, rst, _ = oh.render_reference(scene, cam)
        for instanced in (False, True):
            words, n1 = results[(k, instanced)]
            assert np.array_equal(words, ref), (k, instanced)
            if rst is not None:
                assert n1[0] == rst["stage1"]["rasterized"]
                assert n1[1] == rst["stage1"]["culled_tiny"]
                assert n1[2] == rst["stage3"]["fragments"]


def test_sign_flip_min_is_unsigned_min():
    """CLEAR (all ones) must stay the maximum: a plain int64 MIN would see -1."""
    a = np.array([0xFFFFFFFFFFFFFFFF, 5, 0x8000000000000001, 0x7F00000000000007], dtype=np.uint64)
    b = np.array([3, 0xFFFFFFFFFFFFFFFF, 0x7FFFFFFFFFFFFFFF, 0x7F00000000000008], dtype=np.uint64)
    t = torch.from_numpy(a.view(np.int64).copy())
    t ^= -0x8000000000000000
    u = torch.from_numpy(b.view(np.int64).copy())
    u ^= -0x8000000000000000
    m = torch.minimum(t, u) ^ -0x8000000000000000
    assert np.array_equal(m.numpy().view(np.uint64), np.minimum(a, b))


def test_stripe_rows_cover_the_image_once():
    from paper_2604_21749_b200.distributed import stripe_rows
    for H in (1, 7, 120, 1080, 2160):
        for world in (1, 2, 3, 4, 8):
            rows = []
            for r in range(world):
                r0, n, per = stripe_rows(H, world, r)
                assert per * world >= H and n <= per
                rows += list(range(r0, r0 + n))
            assert rows == list(range(H))


def _rs_worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_21749_b200.distributed import Compositor
    try:
        rng = np.random.default_rng(100 + rank)
        n = 1001                                   # not a multiple of the world size
        w = rng.integers(0, 2 ** 63, size=n, dtype=np.int64)
        w[::7] = -1                                # CLEAR words (all ones)
        w[::11] = np.int64(-2 ** 63)               # top bit set: unsigned order != signed
        t = torch.from_numpy(w.copy())
        stripe = Compositor(t, world).reduce_scatter_min(rank).clone()
        allw = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(allw, t)
        parts = [torch.empty_like(stripe) for _ in range(world)]
        dist.all_gather(parts, stripe)
        if rank == 0:
            results["words"] = np.stack([a.numpy() for a in allw])
            results["stripes"] = torch.cat(parts).numpy()
    finally:
        dist.destroy_process_group()


def test_reduce_scatter_stripes_are_the_unsigned_min():
    """Compositor.reduce_scatter_min (the bench's sort-last composite): the
    concatenated stripes equal the elementwise unsigned min of all ranks'
    words, CLEAR-padded to equal stripes."""
    world = 2
    results = mp.Manager().dict()
    mp.spawn(_rs_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    words = results["words"].view(np.uint64)
    want = words.min(axis=0)
    got = results["stripes"].view(np.uint64)
    assert np.array_equal(got[:len(want)], want)
    assert np.all(got[len(want):] == np.uint64(2 ** 64 - 1))
