"""Sort-last at world size 2 through the CUDA product path.

Two processes share cuda:0 (this run has one GPU) and a gloo process group.
Each rank rasterizes its global-ID shard with the default kernels, the
composite is the unsigned-min all-reduce (gloo branch of Compositor, words
staged through host memory), and the result must equal the 1-GPU frame bit
for bit — for ``render_sharded`` and for the striped
``render_sharded_resolved``.  The ranks' kernels never wait on each other:
the only exchange is the host-side collective after each rank's frame.
Reference: pipeline.py:151-204 (claim split + min-merge),
test_acceptance.py:49-69 (bit-identity across worker splits)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scenes():
    import paper_2604_21749_b200 as cr
    from paper_2604_21749_b200 import generators as gen
    from scenes import classifier_scene
    out = [("classifier",) + classifier_scene()]
    out.append(("C",) + gen.config_c(width=960, height=540))
    out.append(("grid",) + gen.config_b(n=800, width=1280, height=720))
    lg = gen.make_lantern_grid(5, 4, tris_per_mesh=20_000, spacing=1.8)
    out.append(("lanterns", lg, cr.Camera.look_at((0.0, 8.0, 12.0), (0.0, 0.0, 0.0),
                                                   width=640, height=480)))
    return out


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for p in (root, os.path.join(root, "tests")):
        if p not in sys.path:
            sys.path.insert(0, p)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2604_21749_b200 as cr
    from paper_2604_21749_b200.distributed import render_sharded, render_sharded_resolved
    try:
        for name, scene, cam in _scenes():
            dl = cr.build_draw_list(scene, cam)
            fb, st = render_sharded(dl, cam, cr.RasterConfig())
            words = fb.words.copy()
            mesh_ids = None
            img, _, _ = render_sharded_resolved(dl, cam, cr.RasterConfig())
            n1 = torch.tensor([st.stage1.rasterized, st.stage1.culled_tiny,
                               st.stage1.fragments, st.stage3.fragments], dtype=torch.int64)
            dist.all_reduce(n1)
            if rank == 0:
                results[name] = (words, n1.numpy(), img.cpu().numpy())
    finally:
        dist.destroy_process_group()


def test_world2_render_sharded_equals_single_gpu_frame():
    import paper_2604_21749_b200 as cr
    from paper_2604_21749_b200.resolve import resolve_frame_device
    results = mp.Manager().dict()
    mp.spawn(_worker, args=(2, _port(), results), nprocs=2, join=True)
    for name, scene, cam in _scenes():
        dl = cr.build_draw_list(scene, cam)
        fb, st = cr.render_draw_list(dl, cam, cr.RasterConfig())
        words, n1, img = results[name]
        assert np.array_equal(words, fb.words), name
        assert n1[0] == st.stage1.rasterized and n1[1] == st.stage1.culled_tiny, name
        assert n1[2] == st.stage1.fragments and n1[3] == st.stage3.fragments, name
        ref, _ = resolve_frame_device(fb, dl, cam)
        assert np.array_equal(img, ref.cpu().numpy()), name


def _geo_worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for p in (root, os.path.join(root, "tests")):
        if p not in sys.path:
            sys.path.insert(0, p)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2604_21749_b200 as cr
    from paper_2604_21749_b200 import generators as gen
    from paper_2604_21749_b200.distributed import render_sharded, shard_range
    from paper_2604_21749_b200.pipeline import PreparedFrame, build_context
    try:
        scene, cam = gen.config_e(n_meshes=6, n=120, width=640, height=360)
        dl = cr.build_draw_list(scene, cam)
        ctx = build_context(dl, cam)
        lo, hi = shard_range(dl.total_triangles, world, rank)
        pf = PreparedFrame(dl, cam, cr.RasterConfig(), ctx, work_range=(lo, hi))
        fb, st = render_sharded(dl, cam, cr.RasterConfig())
        if rank == 0:
            results["words"] = fb.words.copy()
        results[f"meshes{rank}"] = [int(m) for m in pf.mesh_ids]
        results["n_meshes"] = len(ctx.meshes)
    finally:
        dist.destroy_process_group()


def test_world2_config_e_scaled_down_shard_local_geometry():
    """A scaled-down config E (distinct displaced grids):
    each rank uploads only its shard's meshes, and the composite equals the
    1-GPU frame."""
    import paper_2604_21749_b200 as cr
    from paper_2604_21749_b200 import generators as gen
    results = mp.Manager().dict()
    mp.spawn(_geo_worker, args=(2, _port(), results), nprocs=2, join=True)
    scene, cam = gen.config_e(n_meshes=6, n=120, width=640, height=360)
    fb, _ = cr.render_frame(scene, cam, cr.RasterConfig())
    assert np.array_equal(results["words"], fb.words)
    m0, m1 = set(results["meshes0"]), set(results["meshes1"])
    assert len(m0) < results["n_meshes"] and len(m1) < results["n_meshes"]
    assert len(m0 & m1) <= 1                    # a mesh cut by the shard boundary


@pytest.mark.parametrize("mode", ["B", "strong"])
def test_bench_world2_harness_runs(mode):
    """bench.py under torchrun at N=2 (both ranks on cuda:0 through the
    CURAST_BENCH_SHARED_GPU=1 harness self-test switch, gloo composite): the
    sort-last shards, the composite, the max-over-ranks timing and the one
    JSON line of rank 0.  Not a scaling measurement."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CURAST_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--mode", mode, "--grid-n", "600", "--profile"]
    r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 3 and d["value"] > 0
    assert d["scaling"] == ("weak" if mode == "B" else "strong")
    tri = 2 * 600 * 600
    assert d["config"]["triangles"] == (2 * tri if mode == "B" else tri)
