"""T4: compute-sanitizer (memcheck, racecheck, synccheck) over every kernel on
small inputs (scripts/sanitize_case.py)."""
import os
import shutil
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer(tool):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not found")
    cmd = [SAN, "--tool", tool, "--error-exitcode", "99", sys.executable,
           os.path.join(ROOT, "scripts", "sanitize_case.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    out = r.stdout + r.stderr
    if r.returncode == 86 and "closed" in out:  # the pool's wrapper refuses the tool (no run happened)
        pytest.skip("compute-sanitizer is closed on this GPU pool: " + out.strip().splitlines()[-1][:200])
    assert r.returncode == 0, out[-4000:]
    assert "sanitize case OK" in out
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-2000:]
