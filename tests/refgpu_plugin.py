"""pytest plugin (-p refgpu_plugin) for running the REFERENCE's own test files unchanged on the GPU path.

Loaded before the reference's test modules are imported: binds the reference package's `render_forward` /
`render_backward` names (in the modules that define or re-export them) to this repo's C-ABI path, so that
`from softsphere.raster import render_forward` in tests/test_raster.py etc. picks up the B200 implementation.
Everything else -- scene / camera types, `compute_bounds`, `draw_pixel`, `oracle_render`, `fd_gradient`, the fit
loop -- stays the reference's own code and is what the GPU results are compared against.
"""
import functools
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
for p in (ROOT, REF):
    if p not in sys.path:
        sys.path.insert(0, p)

import softsphere  # noqa: E402  (the unmodified reference, from baseline/_ref)
import softsphere.cli  # noqa: E402,F401
import softsphere.grad  # noqa: E402
import softsphere.optim  # noqa: E402
import softsphere.raster  # noqa: E402

import paper_2004_07484_b200 as pk  # noqa: E402

CALLS = {"forward": 0, "backward": 0}


@functools.wraps(softsphere.raster.render_forward)
def render_forward(*args, **kwargs):
    CALLS["forward"] += 1
    return pk.render_forward(*args, **kwargs)


@functools.wraps(softsphere.grad.render_backward)
def render_backward(*args, **kwargs):
    # the reference promises bit-identical gradients from run to run and for any worker count (grad.py:231-250,
    # tests/test_grad.py test_deterministic_across_workers): that is this path's deterministic mode
    CALLS["backward"] += 1
    kwargs.setdefault("deterministic", True)
    return pk.render_backward(*args, **kwargs)


for mod in (softsphere, softsphere.raster, softsphere.optim, softsphere.cli):
    if hasattr(mod, "render_forward"):
        mod.render_forward = render_forward
for mod in (softsphere, softsphere.grad, softsphere.optim, softsphere.cli):
    if hasattr(mod, "render_backward"):
        mod.render_backward = render_backward


def pytest_terminal_summary(terminalreporter):
    terminalreporter.write_line(f"refgpu: render_forward calls on the GPU path: {CALLS['forward']}, "
                                f"render_backward: {CALLS['backward']}")
