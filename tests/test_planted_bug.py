"""The parity harness can fail: a build with a planted off-by-one in the window closure
(-DMAYURA_PLANT_BUG: t_m - t_1 < delta instead of <= delta; csrc/comine.cu
window_end_of) must turn the GPU parity tests red (SPEC.md:572 asks for exactly this check),
while the same tests pass on the real library (the rest of the -m gpu suite)."""
import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_planted_window_bug_turns_parity_red():
    sys.path.insert(0, ROOT)
    import __graft_entry__
    lib = __graft_entry__._builder().build(variant="planted", defines=["MAYURA_PLANT_BUG"])
    env = dict(os.environ, MAYURA_LIB_PATH=lib)
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-m", "gpu",
           os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-k", "hand_examples or fuzz_groups or C1"]
    out = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=1800)
    assert out.returncode != 0, "the planted bug went unnoticed:\n" + out.stdout[-2000:]
    assert "failed" in out.stdout and "AssertionError" in out.stdout + out.stderr, out.stdout[-2000:]
