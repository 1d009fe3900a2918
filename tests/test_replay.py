"""replay (io/pipeline.hpp:27-72, pipeline.cpp:46-168) — the caller of the hot path.

GPU: the device replay of in-memory frames equals the reference's replay logic
(integrate every frame, fold the pending changed blocks into the ESDF every
update_every frames and after the last one) restated over the reference's own
integrate_depth / update_esdf (oracle/_ref); timings record the ESDF exactly on
the derive frames; the reference's argument errors.  CPU: the timing CSV format.
"""
import numpy as np
import pytest

from paper_2311_00626_b200 import _abi as A
from tests.helpers import camera_frames, layers_identical


def _ref_replay(ref, frames, cam, cfg):
    """pipeline.cpp:54-148 (TSDF source, no color / mesh) over the reference calls."""
    T, E = ref.layer(A.LAYER_TSDF, cfg.voxel_size), ref.layer(A.LAYER_ESDF, cfg.voxel_size)
    pending = np.zeros((0, 3), np.int32)
    derived = []
    for k, (pose, d) in enumerate(frames):
        ch = ref.integrate_camera(T, d, pose, cam, cfg.integrator)
        pending = np.unique(np.concatenate([pending, ch]), axis=0)
        last = k + 1 == len(frames)
        if ((k + 1) % cfg.update_every == 0 or last) and len(pending):
            ref.update_esdf(E, T, pending, cfg.esdf)
            pending = np.zeros((0, 3), np.int32)
            derived.append(k)
    return T, E, derived


@pytest.mark.gpu
@pytest.mark.parametrize("update_every", [1, 3, 4])
def test_replay_matches_reference_pipeline(vx, ref, update_every):
    cam, frames = camera_frames("room", 320, 240, 7, 16)
    cfg = vx.make_replay_config(0.04)
    cfg.update_every = update_every
    assert cfg.integrator.truncation == pytest.approx(0.16) and cfg.esdf.site_threshold == pytest.approx(0.04)
    T, E, timings = vx.replay(frames, cam, cfg)
    To, Eo, derived = _ref_replay(ref, frames, cam, cfg)
    assert layers_identical(*T.export(), *ref.export(To))
    assert layers_identical(*E.export(), *ref.export(Eo))
    assert list(timings["frame"]) == list(range(len(frames)))
    assert list(np.nonzero(timings["esdf_ms"] > 0)[0]) == derived
    assert np.all(timings["tsdf_ms"] > 0)
    assert list(np.nonzero(timings["mesh_ms"] > 0)[0]) == derived


@pytest.mark.gpu
def test_replay_with_color_and_mesh_matches_reference_pipeline(vx, ref):
    """derive_layers with update_mesh(..., cake.color) and per-frame
    integrate_color (pipeline.cpp:71-86, 111-117)."""
    from tests.test_mesh import _same_mesh
    cam, frames = camera_frames("room", 320, 240, 5, 16)
    frames = [(T, d, ref.render_color("room", T, cam)) for T, d in frames]
    cfg = vx.make_replay_config(0.04)
    cfg.update_every = 2
    cfg.with_color = 1
    cake, timings = vx.replay_cake(frames, cam, cfg)
    To, Eo = ref.layer(A.LAYER_TSDF, 0.04), ref.layer(A.LAYER_ESDF, 0.04)
    Co, Mo = ref.layer(A.LAYER_COLOR, 0.04), ref.mesh_layer(0.04)
    pending = np.zeros((0, 3), np.int32)
    derived = []
    for k, (pose, d, rgb) in enumerate(frames):
        pending = np.unique(np.concatenate([pending, ref.integrate_camera(To, d, pose, cam, cfg.integrator)]),
                            axis=0)
        ref.integrate_color(Co, rgb, d, pose, cam, To, cfg.integrator)
        if ((k + 1) % 2 == 0 or k + 1 == len(frames)) and len(pending):
            ref.update_esdf(Eo, To, pending, cfg.esdf)
            ref.update_mesh(Mo, To, pending, cfg.mesh.min_weight, Co)
            pending = np.zeros((0, 3), np.int32)
            derived.append(k)
    assert layers_identical(*cake["source"].export(), *ref.export(To))
    assert layers_identical(*cake["esdf"].export(), *ref.export(Eo))
    assert layers_identical(*cake["color"].export(), *ref.export(Co))
    assert _same_mesh(cake["mesh"], Mo)
    assert list(np.nonzero(timings["mesh_ms"] > 0)[0]) == derived
    assert np.all(timings["color_ms"] > 0)


@pytest.mark.gpu
def test_replay_argument_errors(vx):
    cam, frames = camera_frames("room", 160, 120, 1, 8)
    cfg = vx.make_replay_config(0.05)
    with pytest.raises(vx.InvalidArgumentError, match="no frames"):
        vx.replay([], cam, cfg)
    cfg.update_every = 0
    with pytest.raises(vx.InvalidArgumentError, match="update_every"):
        vx.replay(frames, cam, cfg)
    cfg.update_every = 1
    cfg.with_color = 1
    cfg.use_occupancy = 1
    with pytest.raises(vx.InvalidArgumentError, match="color needs a camera"):
        vx.replay(frames, cam, cfg)


def test_timing_csv_format(tmp_path):
    from paper_2311_00626_b200 import voxmap
    t = np.zeros(2, A.FRAME_TIMING_DTYPE)
    t["frame"] = [0, 1]
    t["tsdf_ms"] = [1.23456, 2.0]
    t["esdf_ms"] = [0.0, 0.5]
    p = tmp_path / "t.csv"
    voxmap.write_timing_csv(t, str(p))
    assert p.read_text() == ("frame,tsdf_ms,color_ms,esdf_ms,mesh_ms\n"
                             "0,1.235,0.000,0.000,0.000\n1,2.000,0.000,0.500,0.000\n")
