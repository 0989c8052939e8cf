"""Sort-last path on the GPU with a 1-rank NCCL group (this run has one GPU):
exercises libcurast_nccl.so (ncclAllReduce / ncclReduce / ncclReduceScatter on
ncclUint64 + ncclMin) and render_sharded end to end.  The multi-rank partition
and composite are covered with gloo on CPU in test_multirank.py."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_group():
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0,
                            world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def test_nccl_u64_min_collectives(nccl_group):
    from paper_2604_21749_b200.distributed import NcclComm
    comm = NcclComm()
    a = np.array([0xFFFFFFFFFFFFFFFF, 7, 0x8000000000000000, 3], dtype=np.uint64)
    t = torch.from_numpy(a.view(np.int64).copy()).cuda()
    comm.allreduce_min(t)
    out = torch.empty_like(t)
    comm.reduce_min(t, out, root=0)
    stripe = torch.empty_like(t)
    comm.reduce_scatter_min(t, stripe)
    torch.cuda.synchronize()
    assert np.array_equal(t.cpu().numpy().view(np.uint64), a)
    assert np.array_equal(out.cpu().numpy().view(np.uint64), a)
    assert np.array_equal(stripe.cpu().numpy().view(np.uint64), a)
    comm.close()


def test_render_sharded_equals_render_frame(nccl_group):
    import paper_2604_21749_b200 as cr
    from paper_2604_21749_b200.distributed import render_sharded
    from scenes import random_scene
    rng = np.random.default_rng(11)
    for _ in range(5):
        scene, cam = random_scene(rng)
        dl = cr.build_draw_list(scene, cam)
        if dl.total_triangles == 0:
            continue
        fb1, _ = cr.render_frame(scene, cam, cr.RasterConfig())
        fb2, _ = render_sharded(dl, cam, cr.RasterConfig())
        assert np.array_equal(fb1.words, fb2.words)


def test_render_sharded_resolved_equals_single_gpu(nccl_group):
    import paper_2604_21749_b200 as cr
    from paper_2604_21749_b200 import generators as gen
    from paper_2604_21749_b200.distributed import render_sharded_resolved
    from paper_2604_21749_b200.resolve import resolve_frame_device
    scene, cam = gen.config_a()
    dl = cr.build_draw_list(scene, cam)
    img, st, rst = render_sharded_resolved(dl, cam, group=nccl_group)
    fb, _ = cr.render_draw_list(dl, cam)
    ref, _ = resolve_frame_device(fb, dl, cam)
    assert img is not None and torch.equal(img, ref)
