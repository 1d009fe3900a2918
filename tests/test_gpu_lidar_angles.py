"""The LiDAR projection's angles on the device (vxm_atan2, integrate.cu)
against the host libm the reference uses (lidar.hpp:43-55: atan2 for the
azimuth, acos(z/|p|) for the polar angle): within 2 ulp, exact on the axes and
at the +-pi seam."""
import numpy as np
import pytest

import paper_2311_00626_b200 as vx

pytestmark = pytest.mark.gpu


def _points():
    rng = np.random.default_rng(11)
    n = 400_000
    ang = rng.uniform(-np.pi, np.pi, n)
    rad = 10 ** rng.uniform(-2, 2.5, n)
    el = rng.uniform(-0.7, 0.7, n)
    p = np.stack([rad * np.cos(ang) * np.cos(el), rad * np.sin(ang) * np.cos(el), rad * np.sin(el)], 1)
    edge = [(1.0, 0.0, 0.1), (-1.0, 0.0, 0.1), (-1.0, -0.0, 0.1), (0.0, 1.0, 0.1), (0.0, -1.0, 0.1),
            (-3.0, 1e-12, 0.0), (-3.0, -1e-12, 0.0), (2.0, 1e-300, 1.0), (1e-9, 5.0, 0.2),
            (0.0, 0.0, 2.0), (0.0, 0.0, -2.0)]
    # just either side of the table's nodes k pi / 512 and of the +-pi seam
    k = rng.integers(-512, 513, 2000)
    t = k * np.pi / 512 + rng.choice([-1, 1], 2000) * 10 ** rng.uniform(-15, -6, 2000)
    t = np.clip(t, -np.pi, np.pi)
    near = np.stack([5 * np.cos(t), 5 * np.sin(t), np.zeros_like(t)], 1)
    return np.concatenate([p, np.array(edge), near])


def test_lidar_angles_match_libm():
    p = _points()
    az, po = vx.diag_lidar_angles(p)
    ref_az = np.arctan2(p[:, 1], p[:, 0])
    ulp = np.spacing(np.abs(ref_az)).clip(min=np.finfo(float).tiny)
    err = np.abs(az - ref_az) / ulp
    assert err.max() <= 2.0, (err.max(), p[err.argmax()])
    zero_y = p[:, 1] == 0
    assert np.array_equal(np.signbit(az[zero_y]), np.signbit(ref_az[zero_y]))
    assert np.array_equal(az[zero_y], ref_az[zero_y])
    r = np.sqrt(p[:, 0] ** 2 + (p[:, 1] ** 2 + p[:, 2] ** 2))
    ref_po = np.arccos(np.clip(p[:, 2] / r, -1.0, 1.0))
    fan = np.abs(p[:, 2] / r) < 0.9  # acos of the rounded ratio is well conditioned there
    e_po = np.abs(po[fan] - ref_po[fan]) / np.spacing(ref_po[fan])
    assert e_po.max() <= 4.0, e_po.max()
    assert np.abs(po - ref_po).max() < 1e-7  # everywhere (only ever compared against the beam fan)
