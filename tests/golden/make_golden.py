"""Generates tests/golden/golden.json from the REFERENCE's own code.

Runs in the build container only (needs oracle/_ref, i.e. the reference's
sources compiled by oracle/Makefile from /root/reference).  Inputs are the
reference's own scenes / trajectories / renderer (via oracle/_ref), so the
fixtures pin the reference's outputs, not ours.  Each case records the
changed-block lists and SHA-256 digests of the sorted layer bytes.

    python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.bindings import RefOracle  # noqa: E402
from paper_2311_00626_b200 import _abi as A  # noqa: E402


def digest(keys, vox):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(keys).tobytes())
    h.update(np.ascontiguousarray(vox).tobytes())
    return h.hexdigest()


def pose_list(p):
    return [list(p.R), list(p.t)]


def camera_case(ref, scene, w, h, vs, frames, orbit, icfg, ecfg=None):
    cam = A.default_camera(w, h)
    T = ref.layer(A.LAYER_TSDF, vs)
    E = ref.layer(A.LAYER_ESDF, vs) if ecfg else None
    out = {"scene": scene, "width": w, "height": h, "voxel_size": vs, "frames": frames,
           "orbit": orbit, "icfg": {f: getattr(icfg, f) for f, _ in icfg._fields_},
           "steps": []}
    if ecfg:
        out["ecfg"] = {f: getattr(ecfg, f) for f, _ in ecfg._fields_}
    for k in range(frames):
        p = ref.orbit_pose(scene, k, orbit)
        d = ref.render_camera(scene, p, cam)
        ch = ref.integrate_camera(T, d, p, cam, icfg)
        step = {"pose": pose_list(p), "depth_sha256": hashlib.sha256(d.tobytes()).hexdigest(),
                "changed": ch.tolist(), "tsdf_sha256": digest(*T.export())}
        if ecfg:
            ech = ref.update_esdf(E, T, ch, ecfg)
            step["esdf_changed"] = ech.tolist()
            step["esdf_sha256"] = digest(*E.export())
        out["steps"].append(step)
    return out


def lidar_case(ref, scene, na, ne, vs, frames, orbit, icfg):
    li = A.default_lidar(na, ne)
    T = ref.layer(A.LAYER_TSDF, vs)
    out = {"scene": scene, "na": na, "ne": ne, "voxel_size": vs, "frames": frames, "orbit": orbit,
           "icfg": {f: getattr(icfg, f) for f, _ in icfg._fields_}, "steps": []}
    for k in range(frames):
        p = ref.orbit_pose(scene, k, orbit, lidar=True)
        d = ref.render_lidar(scene, p, li)
        ch = ref.integrate_lidar(T, d, p, li, icfg)
        keys, vox = T.export()
        out["steps"].append({"pose": pose_list(p), "depth_sha256": hashlib.sha256(d.tobytes()).hexdigest(),
                             "changed": ch.tolist(), "tsdf_sha256": digest(keys, vox),
                             "observed_sha256": hashlib.sha256(
                                 np.ascontiguousarray(vox["weight"] > 0).tobytes()).hexdigest()})
    return out


def main():
    ref = RefOracle()
    g = {"generator": "tests/golden/make_golden.py (reference sources via oracle/_ref)"}
    g["camera_nearest_sphere_in_box"] = camera_case(
        ref, "sphere_in_box", 160, 120, 0.05, 3, 8, A.default_integrator_config(truncation=0.2),
        A.default_esdf_config(site_threshold=0.05))
    g["camera_linear_sphere_in_box"] = camera_case(
        ref, "sphere_in_box", 160, 120, 0.05, 3, 8,
        A.default_integrator_config(truncation=0.2, camera_sample=A.SAMPLE_LINEAR))
    g["camera_room_2cm"] = camera_case(
        ref, "room", 320, 240, 0.02, 2, 100, A.default_integrator_config(truncation=0.08),
        A.default_esdf_config(site_threshold=0.02, max_distance=2.0))
    g["lidar_inverse_square_sphere_in_box"] = lidar_case(
        ref, "sphere_in_box", 180, 16, 0.05, 3, 8,
        A.default_integrator_config(truncation=0.2, weighting=A.WEIGHT_INVERSE_SQUARE))
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as f:
        json.dump(g, f, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
