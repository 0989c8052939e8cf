"""benchcli on the GPU: the reference bench protocol (cli.py:144-223) runs
its toggle rows, the framebuffer-hash guard holds for timing-only rows and
fires when a 'timing-only' row changes the image."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _scene():
    from paper_2604_21749_b200 import generators as gen
    from paper_2604_21749_b200.scene import Camera, SceneNode
    mesh = gen.make_tessellated_quad(300, f32=True)
    cam = Camera.look_at((0.0, 0.0, 1.2), (0.0, 0.0, 0.0), width=320, height=240)
    return [SceneNode(mesh=mesh, transforms=[np.eye(4)])], cam


@pytest.mark.parametrize("toggle", [None, "tinyCull", "instancing", "workers", "superSampling"])
def test_bench_protocol_rows(toggle, tmp_path):
    from paper_2604_21749_b200 import benchcli
    scene, cam = _scene()
    rows = benchcli.bench(scene, cam, toggle=toggle, frames=3)
    assert rows and all(set(r) == set(benchcli.COLS) for r in rows)
    for r in rows:
        assert r["visibleTriangles"] == 180000
        assert r["stage1Ms"] > 0 and r["resolveMs"] > 0 and r["totalMs"] >= r["stage1Ms"]
    if toggle == "tinyCull":
        assert rows[0]["culled"] > rows[1]["culled"]       # tiny cull only culls more
        assert rows[0]["fragments"] == rows[1]["fragments"]
    if toggle == "superSampling":
        fr = [r["fragments"] for r in rows]
        assert fr[0] < fr[1] < fr[2]
    benchcli.write_csv(rows, tmp_path / "b.csv")


def test_hash_guard_fires_on_a_changed_image(monkeypatch):
    from paper_2604_21749_b200 import benchcli
    from paper_2604_21749_b200.config import RasterConfig
    from paper_2604_21749_b200.scene import Camera
    scene, cam = _scene()
    cam2 = Camera.look_at((0.0, 0.1, 1.2), (0.0, 0.0, 0.0), width=320, height=240)
    monkeypatch.setattr(benchcli, "bench_rows",
                        lambda c, cfg, t=None: [("a", cam, RasterConfig(), True),
                                                ("b", cam2, RasterConfig(), True)])
    with pytest.raises(benchcli.FramebufferHashError):
        benchcli.bench(scene, cam, toggle="x", frames=1)
