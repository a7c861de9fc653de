"""GPU: the REFERENCE's own test files, unchanged, with `render_forward` / `render_backward` bound to this path.

SURVEY Appendix B lists the reference tests "worth running through the adapter unchanged": tests/test_raster.py,
tests/test_grad.py, tests/test_shade.py (the joint shader + feature fit) and tests/test_optim.py (`fit`).  The build
hook copies those files next to the installed reference (git-ignored baseline/_ref/_reference_tests, it travels to
the GPU box); `refgpu_plugin` rebinds the two entry points before the test modules import them.  Everything the
tests compare against -- `oracle_render`, `draw_pixel`, `backward_pixel`, `fd_gradient`, `compute_bounds`,
`_bin_tiles`, the fit loop's bookkeeping -- remains the reference's own float64 code.

All but six of the suite's 165 tests pass as written (74 of the 80 in the four files named above).  The six assert float64 round-off (1e-12, 1e-6 absolute) or difference a
float32 forward pass with float64 step sizes; this path computes the blend in float32 by design (north_star: 1e-5
relative forward, 1e-4 gradients), and the same properties are checked at those tolerances in test_gpu_parity.py /
test_gpu_round2.py (finite differences with Richardson steps sized for float32).
"""
import os
import re
import subprocess
import sys

import pytest

from helpers import ROOT

pytestmark = pytest.mark.gpu

REF_TESTS = os.path.join(ROOT, "baseline", "_ref", "_reference_tests")
# the four files SURVEY Appendix B names + the rest of the suite (the CLI tests render through the path as well)
FILES = ["test_raster.py", "test_grad.py", "test_shade.py", "test_optim.py", "test_cli.py", "test_scene.py",
         "test_camera.py", "test_blend.py", "test_testkit.py"]
# float64-tolerance assertions a float32 blend cannot meet (see the module docstring)
EXPECTED_FLOAT64_ONLY = {
    "TestDrawPixel::test_matches_render_forward_at_tau_zero",          # |draw_pixel - image| < 1e-12
    "TestRenderForward::test_matches_oracle_random_scenes",            # |image - oracle| < 1e-6 absolute
    "test_property_forward_equals_oracle",                             # the same, hypothesis-driven (SURVEY: "relaxed to 1e-5")
    "TestRenderBackward::test_gradcheck_small_scenes[pinhole-aa]",     # FD of the forward pass with float64 steps
    "TestRenderBackward::test_gradcheck_small_scenes[pinhole-6d]",
    "TestRenderBackward::test_gradcheck_small_scenes[orthographic-aa]",
}


def test_reference_test_files_pass_unchanged_on_the_gpu_path(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.isdir(REF_TESTS):
        pytest.skip("baseline/_ref/_reference_tests absent (the build hook copies it where /root/reference exists)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.path.join(ROOT, "tests") + os.pathsep + env.get("PYTHONPATH", "")
    env["HYPOTHESIS_STORAGE_DIRECTORY"] = str(tmp_path / "hyp")
    cmd = [sys.executable, "-m", "pytest", "-p", "refgpu_plugin", "-p", "no:cacheprovider", "-q", "--no-header",
           "-rf", "--tb=no", *FILES]
    r = subprocess.run(cmd, cwd=REF_TESTS, env=env, capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    # node ids are printed relative to pytest's rootdir: keep what follows the file name
    failed = set(re.findall(r"^FAILED \S*?(?:\.py)?::(\S+)", out, flags=re.M))
    m = re.search(r"(\d+) passed", out)
    passed = int(m.group(1)) if m else 0
    calls = re.search(r"render_forward calls on the GPU path: (\d+), render_backward: (\d+)", out)
    assert calls and int(calls.group(1)) > 500 and int(calls.group(2)) > 100, out[-2000:]  # the GPU path really ran
    assert "error" not in out.lower().split("short test summary")[0][-300:] or passed, out[-2000:]
    unexpected = failed - EXPECTED_FLOAT64_ONLY
    assert not unexpected, f"reference tests failing on the GPU path: {sorted(unexpected)}\n{out[-3000:]}"
    assert passed >= 159, out[-2000:]
