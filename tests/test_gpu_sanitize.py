"""compute-sanitizer as part of the GPU suite ("racecheck /
memcheck in CI"): the stored-Heaviside kernel 1 and zst4 (interior and face
tiles) and the linked-slab push path under memcheck and racecheck must report
no errors.  The full sweep over every kernel variant is tools/sanitize.sh
(profiles/r02_sanitize/)."""
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = Path(__file__).resolve().parents[1]
SANITIZER = "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck"])
def test_sanitizer_clean(tool):
    if not Path(SANITIZER).exists() and shutil.which("compute-sanitizer") is None:
        pytest.skip("compute-sanitizer not available")
    r = subprocess.run([SANITIZER, "--tool", tool, "--error-exitcode", "9", sys.executable,
                        str(ROOT / "tools" / "sanitize_case.py"), "--quick"], capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-3000:]
    assert "ok quick" in out
    assert ("ERROR SUMMARY: 0 errors" in out) or ("0 hazards displayed (0 errors" in out), out[-2000:]
