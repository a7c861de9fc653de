"""ctypes front-end of the CPU parity oracle (oracle/ss_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  Nothing under
paper_2004_07484_b200/ imports this module.

The heavy per-pixel work is the float64 C restatement in ss_oracle.c (each
function there cites the reference file:line it follows).  This file restates
the small host-side pieces of the reference in NumPy:

* camera vector layouts and rotation maps  -- softsphere/camera.py:42-54,
  :79-97, :216-249;
* rotation-parameter VJPs                   -- softsphere/camera.py:57-76, :100-117;
* blend-parameter clamping / validation     -- softsphere/blend.py:38-45;
* scene validation                          -- softsphere/scene.py:91-114;
* the fit-loop step      -- softsphere/optim.py:87-154, :286-329.

Parity is pinned: oracle/pin_against_reference.py checks every entry point
against the imported reference and writes tests/golden/*.npz.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libss_oracle.so")
_lib = None

PINHOLE = "pinhole"
ORTHOGRAPHIC = "orthographic"
AXIS_ANGLE = "axis_angle"
SIX_D = "6d"


class OracleError(Exception):
    pass


class OracleValidationError(OracleError):
    pass


class OracleConfigurationError(OracleError):
    pass


def build(force: bool = False) -> str:
    """Compile libss_oracle.so with the committed Makefile (gcc, -fopenmp)."""
    src = os.path.join(_HERE, "ss_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-C", _HERE, "-B", "libss_oracle.so"], check=True,
                       stdout=subprocess.DEVNULL)
    return _LIB_PATH


class _Cam(C.Structure):
    _fields_ = [("t", C.c_double * 3), ("R", C.c_double * 9), ("focal", C.c_double),
                ("sensor_w", C.c_double), ("near", C.c_double), ("far", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("mode", C.c_int32),
                ("pad", C.c_int32)]


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_LIB_PATH)
        for name in ("or_compute_bounds", "or_sort_order", "or_bin_tiles", "or_render_forward",
                     "or_render_backward", "or_num_threads_available"):
            getattr(_lib, name).restype = C.c_int
    return _lib


def num_threads_available() -> int:
    return int(_load().or_num_threads_available())


# --------------------------------------------------------------------------- camera

def axis_angle_to_matrix(v):
    """Rodrigues; series below theta < 1e-8 (camera.py:42-54)."""
    v = np.asarray(v, dtype=np.float64).reshape(3)
    th2 = float(v @ v)
    th = np.sqrt(th2)
    k = np.array([[0.0, -v[2], v[1]], [v[2], 0.0, -v[0]], [-v[1], v[0], 0.0]])
    if th < 1e-8:
        a, b = 1.0 - th2 / 6.0, 0.5 - th2 / 24.0
    else:
        a, b = np.sin(th) / th, (1.0 - np.cos(th)) / th2
    return np.eye(3) + a * k + b * (k @ k)


def rotation_from_6d(a):
    """Gram-Schmidt, columns c1, c2, c1 x c2 (camera.py:79-97)."""
    a = np.asarray(a, dtype=np.float64).reshape(6)
    a1, a2 = a[:3], a[3:]
    n1 = np.linalg.norm(a1)
    if n1 < 1e-8:
        raise OracleConfigurationError("6d rotation: first column has near-zero norm")
    c1 = a1 / n1
    w = a2 - (c1 @ a2) * c1
    nw = np.linalg.norm(w)
    if nw < 1e-8:
        raise OracleConfigurationError("6d rotation: columns are near-parallel")
    c2 = w / nw
    return np.stack([c1, c2, np.cross(c1, c2)], axis=1)


def axis_angle_vjp(v, grad_matrix):
    """d loss / d v from d loss / d R (camera.py:57-76): closed-form Rodrigues derivative
    dR/dv_i = ((v_i [v]x + [v x (I-R) e_i]x) / |v|^2) R; generators at v = 0."""
    v = np.asarray(v, dtype=np.float64).reshape(3)
    g = np.asarray(grad_matrix, dtype=np.float64).reshape(3, 3)

    def skew(w):
        return np.array([[0.0, -w[2], w[1]], [w[2], 0.0, -w[0]], [-w[1], w[0], 0.0]])

    th2 = float(v @ v)
    out = np.zeros(3)
    if th2 < 1e-14:
        for i in range(3):
            out[i] = np.sum(g * skew(np.eye(3)[i]))
        return out
    r = axis_angle_to_matrix(v)
    imr = np.eye(3) - r
    for i in range(3):
        d_r = ((v[i] * skew(v) + skew(np.cross(v, imr[:, i]))) / th2) @ r
        out[i] = np.sum(g * d_r)
    return out


def rotation_6d_vjp(a, grad_matrix):
    """d loss / d a for R = rotation_from_6d(a) (camera.py:100-117): reverse-mode through
    normalise -> project -> normalise -> cross."""
    a = np.asarray(a, dtype=np.float64).reshape(6)
    g = np.asarray(grad_matrix, dtype=np.float64).reshape(3, 3)
    a1, a2 = a[:3], a[3:]
    n1 = np.linalg.norm(a1)
    c1 = a1 / n1
    w = a2 - (c1 @ a2) * c1
    nw = np.linalg.norm(w)
    c2 = w / nw
    g1, g2, g3 = g[:, 0], g[:, 1], g[:, 2]
    bar_c2 = g2 + np.cross(g3, c1)           # c3 = c1 x c2 contributes g3 x c1 to c2
    bar_w = (bar_c2 - (c2 @ bar_c2) * c2) / nw
    bar_a2 = bar_w - (c1 @ bar_w) * c1
    bar_c1 = g1 + np.cross(c2, g3) - (c1 @ bar_w) * a2 - (c1 @ a2) * bar_w
    bar_a1 = (bar_c1 - (c1 @ bar_c1) * c1) / n1
    return np.concatenate([bar_a1, bar_a2])


@dataclass
class OracleCamera:
    translation: np.ndarray
    rotation_param: np.ndarray
    rotation_type: str
    focal_length: float
    sensor_width: float
    width: int
    height: int
    near: float = 0.1
    far: float = 45.0
    mode: str = PINHOLE
    rotation: np.ndarray = field(default=None)

    def __post_init__(self):
        self.translation = np.asarray(self.translation, dtype=np.float64).reshape(3)
        self.rotation_param = np.asarray(self.rotation_param, dtype=np.float64).reshape(-1)
        if self.rotation_type == AXIS_ANGLE:
            self.rotation = axis_angle_to_matrix(self.rotation_param)
        elif self.rotation_type == SIX_D:
            self.rotation = rotation_from_6d(self.rotation_param)
        else:
            raise OracleConfigurationError(f"unknown rotation type {self.rotation_type!r}")
        if self.mode not in (PINHOLE, ORTHOGRAPHIC):
            raise OracleConfigurationError(f"unknown camera mode {self.mode!r}")
        if self.focal_length <= 0 or self.sensor_width <= 0:
            raise OracleConfigurationError("focal length and sensor width must be > 0")
        if self.width < 1 or self.height < 1:
            raise OracleConfigurationError("image size must be at least 1x1")
        if not (self.near < self.far) or self.near < 0 or self.far - self.near < 1e-12:
            raise OracleConfigurationError("need 0 <= near < far")

    def to_vector(self):
        return np.concatenate([self.translation, self.rotation_param,
                               [self.focal_length, self.sensor_width]])

    def _c(self) -> _Cam:
        s = _Cam()
        s.t[:] = list(self.translation)
        s.R[:] = list(self.rotation.reshape(-1))
        s.focal, s.sensor_w = float(self.focal_length), float(self.sensor_width)
        s.near, s.far = float(self.near), float(self.far)
        s.width, s.height = int(self.width), int(self.height)
        s.mode = 0 if self.mode == PINHOLE else 1
        return s


def camera_from_vector(vec, width, height, near=0.1, far=45.0, mode=PINHOLE) -> OracleCamera:
    """8 = t(3), axis-angle(3), f, s; 11 = t(3), 6d(6), f, s (camera.py:216-249)."""
    v = np.asarray(vec, dtype=np.float64).reshape(-1)
    if v.shape == (8,):
        rp, rt, f, s = v[3:6], AXIS_ANGLE, v[6], v[7]
    elif v.shape == (11,):
        rp, rt, f, s = v[3:9], SIX_D, v[9], v[10]
    else:
        raise OracleConfigurationError(f"camera vector must have 8 or 11 values, got {v.size}")
    return OracleCamera(v[:3], rp, rt, float(f), float(s), int(width), int(height),
                        float(near), float(far), mode)


# --------------------------------------------------------------------------- params / validation

def clamp_gamma(gamma: float) -> float:
    return float(np.clip(gamma, 1e-5, 1.0))  # blend.py:39


def check_blend(eps, tau, k):
    if eps <= 0:
        raise OracleValidationError("epsilon must be > 0")
    if not (0.0 <= tau < 1.0):
        raise OracleValidationError("tau must be in [0, 1)")
    if k < 1:
        raise OracleValidationError("top_k must be >= 1")


def validate_scene(pos, rad, opa, feat, bg):
    """scene.py:91-114."""
    m = pos.shape[0]
    if feat.shape[0] != m or feat.ndim != 2 or feat.shape[1] != bg.shape[0]:
        raise OracleValidationError("feature array shape does not match (M, d)")
    if not np.all(np.isfinite(bg)):
        raise OracleValidationError("background feature contains non-finite values")
    for name, arr in (("position", pos), ("radius", rad), ("opacity", opa), ("feature", feat)):
        if not np.all(np.isfinite(arr)):
            raise OracleValidationError(f"non-finite {name}")
    if np.any(rad <= 0):
        raise OracleValidationError("non-positive radius")


def _f64(a, shape=None):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if shape is not None:
        a = a.reshape(shape)
    return a


def _p(a, ty=C.c_double):
    return a.ctypes.data_as(C.POINTER(ty))


# --------------------------------------------------------------------------- entry points

def compute_bounds(pos, rad, cam: OracleCamera):
    lib = _load()
    pos, rad = _f64(pos, (-1, 3)), _f64(rad, (-1,))
    m = pos.shape[0]
    out = {
        "x_min": np.zeros(m, np.int64), "x_max": np.zeros(m, np.int64),
        "y_min": np.zeros(m, np.int64), "y_max": np.zeros(m, np.int64),
        "on_sensor": np.zeros(m, np.uint8), "proj_radius_px": np.zeros(m),
        "center_cam": np.zeros((m, 3)), "earliest": np.zeros(m),
    }
    c = cam._c()
    lib.or_compute_bounds(C.c_int64(m), _p(pos), _p(rad), C.byref(c),
                          _p(out["x_min"], C.c_int64), _p(out["x_max"], C.c_int64),
                          _p(out["y_min"], C.c_int64), _p(out["y_max"], C.c_int64),
                          _p(out["on_sensor"], C.c_uint8), _p(out["proj_radius_px"]),
                          _p(out["center_cam"]), _p(out["earliest"]))
    out["on_sensor"] = out["on_sensor"].astype(bool)
    return out


def sort_order(earliest):
    lib = _load()
    e = _f64(earliest, (-1,))
    order = np.zeros(e.shape[0], np.int64)
    lib.or_sort_order(C.c_int64(e.shape[0]), _p(e), _p(order, C.c_int64))
    return order


def tile_lists(pos, rad, cam: OracleCamera, tile: int = 16):
    """(sphere_ids grouped by tile in scan order, tile_starts).  Sphere ids are ORIGINAL
    scene indices: the reference's record_seq (raster.py:267-293) mapped through the
    depth-sort permutation (raster.py:239-244)."""
    lib = _load()
    b = compute_bounds(pos, rad, cam)
    order = sort_order(b["earliest"])
    n_active = int(b["on_sensor"].sum())
    ntx = (cam.width + tile - 1) // tile
    nty = (cam.height + tile - 1) // tile
    sx0, sx1 = np.ascontiguousarray(b["x_min"][order]), np.ascontiguousarray(b["x_max"][order])
    sy0, sy1 = np.ascontiguousarray(b["y_min"][order]), np.ascontiguousarray(b["y_max"][order])
    starts = np.zeros(ntx * nty + 1, np.int64)
    lib.or_bin_tiles(C.c_int64(n_active), _p(sx0, C.c_int64), _p(sx1, C.c_int64),
                     _p(sy0, C.c_int64), _p(sy1, C.c_int64), tile, ntx, nty, None,
                     _p(starts, C.c_int64))
    seq = np.zeros(max(int(starts[-1]), 1), np.int64)
    lib.or_bin_tiles(C.c_int64(n_active), _p(sx0, C.c_int64), _p(sx1, C.c_int64),
                     _p(sy0, C.c_int64), _p(sy1, C.c_int64), tile, ntx, nty,
                     _p(seq, C.c_int64), _p(starts, C.c_int64))
    seq = seq[: int(starts[-1])]
    return order[seq].astype(np.int64), starts


def render_forward(pos, rad, opa, feat, bg, cam: OracleCamera, gamma=0.1, eps=1e-2, tau=0.01,
                   top_k=5, tile=16, chunk=256, store_buffer=True, threads=1, validate=True):
    """raster.py:437-512.  Returns dict(image, bg_weight, ids, z, closeness, log_denom, stats)."""
    lib = _load()
    pos, rad, opa = _f64(pos, (-1, 3)), _f64(rad, (-1,)), _f64(opa, (-1,))
    bg = _f64(bg, (-1,))
    d = bg.shape[0]
    feat = _f64(feat, (-1, d))
    if validate:
        validate_scene(pos, rad, opa, feat, bg)
    gamma = clamp_gamma(gamma)
    check_blend(eps, tau, top_k)
    m, h, w, k = pos.shape[0], cam.height, cam.width, int(top_k)
    image = np.zeros((h, w, d))
    bgw = np.zeros((h, w))
    ids = np.full((h, w, k), -1, np.int32)
    z = np.zeros((h, w, k))
    clos = np.zeros((h, w, k))
    ld = np.zeros((h, w))
    stats = np.zeros(6, np.int64)
    c = cam._c()
    lib.or_render_forward(C.c_int64(m), d, _p(pos), _p(rad), _p(opa), _p(feat), _p(bg),
                          C.byref(c), C.c_double(gamma), C.c_double(eps), C.c_double(tau), k,
                          int(tile), int(chunk), int(bool(store_buffer)), int(threads),
                          _p(image), _p(bgw), _p(ids, C.c_int32), _p(z), _p(clos), _p(ld),
                          _p(stats, C.c_int64))
    return {
        "image": image, "bg_weight": bgw, "ids": ids, "z": z, "closeness": clos,
        "log_denom": ld,
        "stats": {"spheres_total": int(stats[0]), "spheres_on_sensor": int(stats[1]),
                  "candidates_tested": int(stats[2]), "hits_blended": int(stats[3]),
                  "pixels_early_stopped": int(stats[4]), "tiles": int(stats[5])},
        "gamma": gamma, "eps": float(eps), "top_k": k, "num_spheres": m,
    }


def render_backward(pos, rad, opa, feat, bg, cam: OracleCamera, buffer, upstream, gamma=None,
                    eps=None, normalize=True, gate=True, tile=16, threads=1):
    """grad.py:323-357.  `buffer` is the dict returned by render_forward (or any mapping
    with ids/z/closeness/log_denom + gamma/eps).  Returns dict with the SceneGradients and
    CameraGradients fields."""
    lib = _load()
    pos, rad, opa = _f64(pos, (-1, 3)), _f64(rad, (-1,)), _f64(opa, (-1,))
    bg = _f64(bg, (-1,))
    d = bg.shape[0]
    feat = _f64(feat, (-1, d))
    m = pos.shape[0]
    ids = np.ascontiguousarray(buffer["ids"], dtype=np.int32)
    h, w, k = ids.shape
    if "num_spheres" in buffer and buffer["num_spheres"] != m:
        raise OracleError("stale buffer")  # grad.py:340-343
    upstream = _f64(upstream)
    if upstream.shape != (h, w, d):
        raise OracleValidationError(f"upstream shape {upstream.shape} != {(h, w, d)}")
    gamma = clamp_gamma(buffer["gamma"] if gamma is None else gamma)
    eps = float(buffer["eps"] if eps is None else eps)
    z, clos, ld = _f64(buffer["z"]), _f64(buffer["closeness"]), _f64(buffer["log_denom"])
    d_pos, d_rad, d_opa = np.zeros((m, 3)), np.zeros(m), np.zeros(m)
    d_feat = np.zeros((m, d))
    cnt = np.zeros(m, np.int64)
    d_t, G = np.zeros(3), np.zeros(9)
    d_f, d_s = C.c_double(0.0), C.c_double(0.0)
    c = cam._c()
    lib.or_render_backward(C.c_int64(m), d, _p(pos), _p(rad), _p(opa), _p(feat), _p(bg),
                           C.byref(c), C.c_double(gamma), C.c_double(eps), k,
                           _p(ids, C.c_int32), _p(z), _p(clos), _p(ld), _p(upstream),
                           int(bool(normalize)), int(bool(gate)), int(tile), int(threads),
                           _p(d_pos), _p(d_rad), _p(d_opa), _p(d_feat), _p(cnt, C.c_int64),
                           _p(d_t), _p(G), C.byref(d_f), C.byref(d_s))
    G = G.reshape(3, 3)
    if cam.rotation_type == AXIS_ANGLE:
        d_rot = axis_angle_vjp(cam.rotation_param, G)
    else:
        d_rot = rotation_6d_vjp(cam.rotation_param, G)
    return {"d_position": d_pos, "d_radius": d_rad, "d_opacity": d_opa, "d_feature": d_feat,
            "pixel_count": cnt, "d_translation": d_t, "d_rotation": d_rot,
            "d_focal": float(d_f.value), "d_sensor_width": float(d_s.value),
            "grad_rot_matrix": G}


# --------------------------------------------------------------------------- synthetic inputs

def benchmark_scene(count, width, height, seed=0, d=3, profile="uniform", aspect_fill=False):
    """The reference benchmark's synthetic scene (cli.py:323-356) for the identity camera
    cam_vec = [0,0,0, 0,0,0, 5, 2], snapped to float32.  Returns (pos, rad, opa, feat, bg, cam_vec).
    With the identity pose camera_to_world is the identity map, so points are generated
    directly in world space.  d != 3 draws (count, d) features from the same stream."""
    rng = np.random.default_rng(seed)
    f, s = 5.0, 2.0
    px = s / width
    parts = []
    if profile == "occluded":
        side = int(np.ceil(np.sqrt(256)))
        depth_w = 5.0
        half = depth_w * (s / 2.0) / f
        gx, gy = np.meshgrid(np.linspace(-half, half, side), np.linspace(-half, half, side))
        wall = np.column_stack([gx.ravel(), gy.ravel(), np.full(side * side, depth_w)])
        r_wall = np.full(side * side, 2.2 * 2 * half / side)
        parts.append((wall, r_wall, np.ones(side * side), rng.uniform(0.2, 1.0, (side * side, d))))
        depth = rng.uniform(30.0, 43.0, count)
    elif profile == "uniform":
        depth = rng.uniform(6.0, 43.0, count)
    else:
        raise OracleConfigurationError(f"unknown profile {profile!r}")
    half_w = depth * (s / 2.0) / f
    x = rng.uniform(-1, 1, count) * half_w
    y = rng.uniform(-1, 1, count) * half_w * ((height / width) if aspect_fill else 1.0)
    pts = np.column_stack([x, y, depth])
    radius = 3.0 * depth * px / f
    parts.append((pts, radius, rng.uniform(0.5, 1.0, count), rng.uniform(0, 1, (count, d))))
    pos = np.concatenate([p[0] for p in parts]).astype(np.float32)
    rad = np.concatenate([p[1] for p in parts]).astype(np.float32)
    opa = np.concatenate([p[2] for p in parts]).astype(np.float32)
    feat = np.concatenate([p[3] for p in parts]).astype(np.float32)
    bg = np.zeros(d, np.float32)
    cam_vec = np.array([0, 0, 0, 0, 0, 0, f, s], dtype=np.float64)
    return pos, rad, opa, feat, bg, cam_vec


# --------------------------------------------------------------------------- fit-loop step
# NumPy restatements of softsphere/optim.py:87-97 (photometric_loss), :100-121
# (opacity_depth_regularizer) and :142-154 (adam_step); pinned by pin_against_reference.py.

def photometric_loss(rendered, target):
    """(mean |rendered - target|, sign(diff) / n)."""
    diff = np.asarray(rendered, dtype=np.float64) - np.asarray(target, dtype=np.float64)
    n = diff.size
    return float(np.abs(diff).sum() / n), np.sign(diff) / n


def opacity_depth_regularizer(pos, opa, cam: OracleCamera, lambda_od):
    """Energy sum(-lambda z_i o_i) and its gradients w.r.t. position and (unclamped) opacity."""
    pos = _f64(pos, (-1, 3))
    opa = _f64(opa, (-1,))
    m = pos.shape[0]
    if lambda_od == 0.0 or m == 0:
        return 0.0, np.zeros((m, 3)), np.zeros(m)
    zeta = ((pos - cam.translation) @ cam.rotation.T)[:, 2]
    span = cam.far - cam.near
    z = (cam.far - np.clip(zeta, cam.near, cam.far)) / span
    o = np.clip(opa, 0.0, 1.0)
    inside = (zeta > cam.near) & (zeta < cam.far)
    dzeta = np.where(inside, lambda_od * o / span, 0.0)
    return float(lambda_od * np.sum(-z * o)), dzeta[:, None] * cam.rotation[2][None, :], -lambda_od * z


def adam_step(params, grads, m, v, t, lr, beta1=0.9, beta2=0.999, adam_eps=1e-8):
    """One bias-corrected Adam update; returns (params', m', v', t + 1)."""
    params, grads = np.asarray(params, np.float64), np.asarray(grads, np.float64)
    t = t + 1
    m = beta1 * m + (1 - beta1) * grads
    v = beta2 * v + (1 - beta2) * grads * grads
    m_hat = m / (1 - beta1 ** t)
    v_hat = v / (1 - beta2 ** t)
    return params - lr * m_hat / (np.sqrt(v_hat) + adam_eps), m, v, t


def fit_step(scene, cam: OracleCamera, target, state, cfg, threads=1):
    """One iteration of the reference's fit loop body (optim.py:286-329) for one observation.
    scene = dict(pos, rad, opa, feat, bg) of float64 arrays (updated copies are returned);
    state = dict(group -> (m, v, t)) for groups pos/rad/opa/feat; cfg = dict with lr_* , beta1, beta2,
    adam_eps, gamma, epsilon, tau, top_k, lambda_od, radius_min, normalize_grads, gate.
    Returns (loss, scene', state', grads)."""
    f = render_forward(scene["pos"], scene["rad"], scene["opa"], scene["feat"], scene["bg"], cam,
                       gamma=cfg["gamma"], eps=cfg["epsilon"], tau=cfg["tau"], top_k=cfg["top_k"], threads=threads)
    loss, upstream = photometric_loss(f["image"], target)
    e, r_dpos, r_dopa = opacity_depth_regularizer(scene["pos"], scene["opa"], cam, cfg["lambda_od"])
    loss += e
    g = render_backward(scene["pos"], scene["rad"], scene["opa"], scene["feat"], scene["bg"], cam, f, upstream,
                        normalize=cfg["normalize_grads"], gate=cfg["gate"], threads=threads)
    g["d_position"] = g["d_position"] + r_dpos
    g["d_opacity"] = g["d_opacity"] + r_dopa
    new_scene, new_state = dict(scene), dict(state)
    for key, gname, lr in (("pos", "d_position", cfg["lr_position"]), ("rad", "d_radius", cfg["lr_radius"]),
                           ("opa", "d_opacity", cfg["lr_opacity"]), ("feat", "d_feature", cfg["lr_feature"])):
        if lr > 0:
            m, v, t = state[key]
            p, m, v, t = adam_step(scene[key], g[gname], m, v, t, lr, cfg["beta1"], cfg["beta2"], cfg["adam_eps"])
            if key == "rad":
                p = np.maximum(p, cfg["radius_min"])
            new_scene[key], new_state[key] = p, (m, v, t)
    return loss, new_scene, new_state, g
