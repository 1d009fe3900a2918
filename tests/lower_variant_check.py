"""Runs camera frames + a dense volume through update_esdf and checks them
bit-for-bit against the oracle; used by test_gpu_lower_variants.py under each
lowering kernel selection (VXM_LOWER_XROUND / VXM_LOWER_DATAFLOW)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2311_00626_b200 as vx  # noqa: E402
from oracle.bindings import PortOracle  # noqa: E402
from paper_2311_00626_b200 import _abi as A  # noqa: E402
from paper_2311_00626_b200 import synth  # noqa: E402
from tests.helpers import camera_frames, layers_identical  # noqa: E402


def main():
    port = PortOracle()
    cam, seq = camera_frames("room", 320, 240, 4, 16)
    icfg = A.default_integrator_config(truncation=0.16)
    ecfg = A.default_esdf_config(site_threshold=0.04, max_distance=1.0)
    T, E = vx.TsdfLayer(0.04), vx.EsdfLayer(0.04)
    To, Eo = port.layer(A.LAYER_TSDF, 0.04), port.layer(A.LAYER_ESDF, 0.04)
    for pose, d in seq:
        a = vx.integrate_depth(T, d, pose, cam, icfg)
        b = port.integrate_camera(To, d, pose, cam, icfg)
        assert np.array_equal(a, b)
        assert np.array_equal(vx.update_esdf(E, T, a, ecfg), port.update_esdf(Eo, To, b, ecfg))
    assert layers_identical(*E.export(), *port.export(Eo))
    keys, vox = synth.sphere_world(64, 0.02, 0.08)
    cfg = A.default_esdf_config(site_threshold=0.02, max_distance=2.0)
    T2, E2 = vx.TsdfLayer(0.02), vx.EsdfLayer(0.02)
    T2.write_blocks(keys, vox)
    To2, Eo2 = port.layer(A.LAYER_TSDF, 0.02), port.layer(A.LAYER_ESDF, 0.02)
    port.write_blocks(To2, keys, vox)
    assert np.array_equal(vx.update_esdf(E2, T2, keys, cfg), port.update_esdf(Eo2, To2, keys, cfg))
    assert layers_identical(*E2.export(), *port.export(Eo2))
    print("ok")


if __name__ == "__main__":
    main()
