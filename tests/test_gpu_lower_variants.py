"""Every lowering kernel the library may select is bit-identical to the
oracle: the cross-round kernel (k_lower_xr, the default for every map; both
its 2- and 3-CTA-per-SM instantiations, VXM_XR_WIDE), the
barrier-per-round dataflow kernel (k_lower3, VXM_LOWER_XROUND=0/1) and its phased form
(grid barrier before every border axis), plain launches instead of
programmatic dependent launch (VXM_NO_PDL), and the cross-round kernel's
precomputed round-1 pair lists forced on small maps (VXM_XR_R1_COMPACT_MIN=0; they
exist only in the 3-CTA instantiation, so VXM_XR_WIDE=2 with it).  The selection is process-wide, so
each variant runs tests/lower_variant_check.py in its own process."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [{"VXM_LOWER_XROUND": "2"}, {"VXM_LOWER_XROUND": "0"},
                                 {"VXM_LOWER_XROUND": "0", "VXM_LOWER_DATAFLOW": "0"},
                                 {"VXM_XR_WIDE": "2"}, {"VXM_XR_WIDE": "0"}, {"VXM_NO_PDL": "1"},
                                 {"VXM_XR_R1_COMPACT_MIN": "0"}, {"VXM_XR_R1_COMPACT_MIN": "0", "VXM_XR_WIDE": "2"}])
def test_lowering_variant_bitwise(env):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "lower_variant_check.py")],
                       env={**os.environ, **env}, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr
