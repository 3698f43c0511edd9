"""Full-scale device runs against the reference control plane (B200).

The bench configs at their real geometry (C3: 145 GiB arena, C5: 117 GiB) on the
device must make every decision the reference Driver makes on the same workload
(shrunk geometry, identical tokens per page): per step the live sessions, trains,
commits and emitted tokens are equal and the byte columns equal after rescaling;
the device K-scan equals the host reduce on every step.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("name,steps", [("c3", 60), ("c5", 80)])
def test_full_scale_control_plane_matches_reference(name, steps):
    out = subprocess.run([sys.executable, "scripts/scale_control_parity.py", name, str(steps)],
                         cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert f"{steps} steps identical" in out.stdout
