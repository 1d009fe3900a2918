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
    assert np.all(timings["tsdf_ms"] > 0) and np.all(timings["mesh_ms"] == 0)


@pytest.mark.gpu
def test_replay_argument_errors(vx):
    cam, frames = camera_frames("room", 160, 120, 1, 8)
    cfg = vx.make_replay_config(0.05)
    with pytest.raises(vx.InvalidArgumentError, match="no frames"):
        vx.replay([], cam, cfg)
    cfg.update_every = 0
    with pytest.raises(vx.InvalidArgumentError, match="update_every"):
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
