"""Shared helpers for the parity tests: golden fixtures, scene generators, tolerances."""
import glob
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")

# north_star tolerances: forward 1e-5 relative, gradients 1e-4 relative
FWD_RTOL, FWD_ATOL = 1e-5, 2e-6
GRAD_RTOL = 1e-4


def golden_names():
    """Render-path fixtures (fit_step.npz and extras.npz are the SURVEY 8(f) fixtures with their own tests)."""
    names = sorted(os.path.splitext(os.path.basename(p))[0] for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz")))
    return [n for n in names if not n.startswith(("fit_", "extras"))]


def load_golden(name):
    z = np.load(os.path.join(GOLDEN_DIR, name + ".npz"), allow_pickle=False)
    g = {k: z[k] for k in z.files}
    for k in ("width", "height", "top_k"):
        g[k] = int(g[k])
    for k in ("near", "far", "gamma", "eps", "tau"):
        g[k] = float(g[k])
    for k in ("normalize", "gate"):
        g[k] = bool(g[k])
    g["mode"] = str(g["mode"])
    return g


def make_random_scene(rng, m, d=3, depth=(25.0, 35.0), lateral=5.0, radius=(0.3, 2.0), opacity=(0.1, 1.0),
                      background=None):
    """Random scene in front of an identity camera; same distribution as the reference's
    tests/conftest.py:8-30, snapped to float32."""
    bg = rng.uniform(0, 1, d) if background is None else np.asarray(background)
    pos = np.column_stack([rng.uniform(-lateral, lateral, m), rng.uniform(-lateral, lateral, m),
                           rng.uniform(depth[0], depth[1], m)])
    f32 = np.float32
    return (pos.astype(f32), rng.uniform(radius[0], radius[1], m).astype(f32),
            rng.uniform(opacity[0], opacity[1], m).astype(f32), rng.uniform(0, 1, (m, d)).astype(f32),
            bg.astype(f32))


def assert_close(actual, expected, rtol, atol, what=""):
    a = np.asarray(actual, dtype=np.float64)
    e = np.asarray(expected, dtype=np.float64)
    assert a.shape == e.shape, f"{what}: shape {a.shape} vs {e.shape}"
    if a.size == 0:
        return
    err = np.abs(a - e)
    tol = atol + rtol * np.abs(e)
    bad = err > tol
    if bad.any():
        i = np.unravel_index(np.argmax(err - tol), err.shape)
        raise AssertionError(f"{what}: {int(bad.sum())}/{a.size} outside tolerance; worst at {i}: "
                             f"got {a[i]!r}, want {e[i]!r}, err {err[i]:.3e}")


def grad_close(actual, expected, what="", rtol=GRAD_RTOL, floor=1e-7):
    """1e-4 relative with an absolute floor tied to the array's magnitude (float32 atomics
    reorder sums; gradients of one sphere are sums of cancelling per-pixel terms)."""
    e = np.asarray(expected, dtype=np.float64)
    scale = float(np.abs(e).max()) if e.size else 0.0
    assert_close(actual, e, rtol, max(floor, rtol * scale * 0.05), what)
