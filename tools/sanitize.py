"""Small workload over every device entry point, for compute-sanitizer runs:

  compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize.py

camera + LiDAR TSDF integration, the ESDF update and its phases, occupancy,
color + meshing, queries, the fused frame step, replay and the in-process
sharded ESDF, each checked against the C oracle where it is cheap.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2311_00626_b200 as vx  # noqa: E402
from oracle.bindings import PortOracle  # noqa: E402
from paper_2311_00626_b200 import _abi as A  # noqa: E402
from tests.helpers import camera_frames, lidar_frames  # noqa: E402

port = PortOracle()
cam, seq = camera_frames("sphere_in_box", 96, 72, 2, 8)
icfg = A.default_integrator_config(truncation=0.2)
ecfg = A.default_esdf_config(site_threshold=0.05)
T, E = vx.TsdfLayer(0.05), vx.EsdfLayer(0.05)
To, Eo = port.layer(A.LAYER_TSDF, 0.05), port.layer(A.LAYER_ESDF, 0.05)
for pose, d in seq:
    a = vx.integrate_depth(T, d, pose, cam, icfg)
    assert np.array_equal(a, port.integrate_camera(To, d, pose, cam, icfg))
    assert np.array_equal(vx.update_esdf(E, T, a, ecfg), port.update_esdf(Eo, To, a, ecfg))
st = vx.EsdfUpdateState()
vx.mark_sites(E, T, T.sorted_indices()[:8], ecfg, st)
vx.clear_invalid(E, ecfg, st)
vx.lower_esdf(E, st, ecfg)
vx.query_batch(E, np.random.default_rng(0).uniform(0, 1, (64, 3)), True)
li, lseq = lidar_frames("sphere_in_box", 90, 8, 1, 8)
L = vx.TsdfLayer(0.05)
vx.integrate_depth(L, lseq[0][1], lseq[0][0], li, icfg)
O, EO = vx.OccupancyLayer(0.05), vx.EsdfLayer(0.05)
vx.update_esdf(EO, O, vx.integrate_depth(O, seq[0][1], seq[0][0], cam, icfg), ecfg)
Cl, M = vx.ColorLayer(0.05), vx.MeshLayer(0.05)
rgb = np.full((72, 96, 3), 100, np.uint8)
vx.integrate_color(Cl, rgb, seq[1][1], seq[1][0], cam, T, icfg)
vx.update_mesh(M, T, T.sorted_indices(), color=Cl)
cfg = vx.make_replay_config(0.05)
cfg.update_every = 2
vx.replay(seq, cam, cfg)
print("sanitize workload done")
