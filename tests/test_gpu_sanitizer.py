"""compute-sanitizer over a small end-to-end case (tools/sanitize_case.py): memcheck,
racecheck (shared-memory hazards: K5's per-warp survivor lists, K6's warp-private staging),
initcheck and synccheck (the look-back scans spin on flags).  Each tool must report
0 errors; the summaries are written to gpurun_out/sanitizer_<tool>.log."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sanitizer():
    for c in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if c and os.path.exists(c):
            return c
    pytest.fail("compute-sanitizer not found")


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "initcheck", "synccheck"])
def test_compute_sanitizer(tool):
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "3", "--target-processes", "all"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    cmd += [sys.executable, os.path.join(ROOT, "tools", "sanitize_case.py")]
    env = dict(os.environ, PYTORCH_NO_CUDA_MEMORY_CACHING="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, env=env, cwd=ROOT)
    out = r.stdout + r.stderr
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"sanitizer_{tool}.log"), "w") as f:
        f.write(out)
    summary = [ln for ln in out.splitlines() if "ERROR SUMMARY" in ln or "RACECHECK SUMMARY" in ln]
    print(tool, summary)
    assert "sanitize case ok" in out, out[-3000:]
    assert r.returncode == 0, out[-3000:]
    assert summary and all(" 0 errors" in s or " 0 hazards" in s for s in summary), summary
