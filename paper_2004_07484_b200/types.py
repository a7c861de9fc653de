"""Host-side mirror of the reference's data model for the render path.

Same names, fields, argument meaning and error behaviour as the reference package
`softsphere` (paths relative to pkg/src/softsphere/), so that code written against the
reference's `render_forward` / `render_backward` runs against the B200 path unchanged:

  errors                  errors.py:4-25
  BlendParams             blend.py:25-45      (gamma clamp, eps/tau/top_k validation)
  Camera, camera_from_vector, camera_to_vector
                          camera.py:130-177, :216-259
  rotation maps and VJPs  camera.py:42-117
  SphereScene, new_scene, add_sphere_arrays
                          scene.py:43-114, :117-176
  FeatureImage, BackwardBuffer, RenderStats
                          raster.py:79-123
  SceneGradients, CameraGradients
                          grad.py:45-69

Everything here is small float64 host math (a camera is 8 or 11 numbers); the per-sphere and
per-pixel work lives in the CUDA kernels.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

PINHOLE = "pinhole"
ORTHOGRAPHIC = "orthographic"
AXIS_ANGLE = "axis_angle"
SIX_D = "6d"

GAMMA_MIN = 1e-5
GAMMA_MAX = 1.0


# ----------------------------------------------------------------------------- errors
class SoftSphereError(Exception):
    """Base class for library errors."""


class ConfigurationError(SoftSphereError):
    """Invalid configuration value (dimensions, planes, parameter ranges)."""


class ValidationError(SoftSphereError):
    """Input data violates an invariant (NaN fields, bad radii, dim mismatch)."""


class FormatError(SoftSphereError):
    """A file does not conform to its declared on-disk format."""


class ContractViolation(SoftSphereError):
    """Mismatched pipeline artifacts, e.g. a stale backward buffer."""


class DivergenceError(SoftSphereError):
    """Optimization produced a non-finite loss."""


# ----------------------------------------------------------------------------- blend params
@dataclass
class BlendParams:
    gamma: float = 0.1
    epsilon: float = 1e-2
    tau: float = 0.01
    top_k: int = 5

    def __post_init__(self):
        self.gamma = float(min(max(float(self.gamma), GAMMA_MIN), GAMMA_MAX))
        if self.epsilon <= 0:
            raise ValidationError("epsilon must be > 0")
        if not (0.0 <= self.tau < 1.0):
            raise ValidationError("tau must be in [0, 1)")
        if self.top_k < 1:
            raise ValidationError("top_k must be >= 1")


# ----------------------------------------------------------------------------- rotations
def _hat(v):
    x, y, z = v
    return np.array([[0.0, -z, y], [z, 0.0, -x], [-y, x, 0.0]])


def axis_angle_to_matrix(v) -> np.ndarray:
    """R = I + a [v]x + b [v]x^2, a = sin(th)/th, b = (1 - cos th)/th^2; Taylor below 1e-8."""
    v = np.asarray(v, dtype=np.float64).reshape(3)
    t2 = float(np.dot(v, v))
    th = np.sqrt(t2)
    if th < 1e-8:
        a, b = 1.0 - t2 / 6.0, 0.5 - t2 / 24.0
    else:
        a, b = np.sin(th) / th, (1.0 - np.cos(th)) / t2
    k = _hat(v)
    return np.eye(3) + a * k + b * (k @ k)


def axis_angle_vjp(v, grad_matrix) -> np.ndarray:
    """Pull d loss / d R back to the axis-angle vector.

    Uses dR/dv_i = [ (v_i v + v x (I - R) e_i) / |v|^2 ]x R; at v = 0 the derivative is the
    generator [e_i]x."""
    v = np.asarray(v, dtype=np.float64).reshape(3)
    g = np.asarray(grad_matrix, dtype=np.float64).reshape(3, 3)
    t2 = float(np.dot(v, v))
    out = np.zeros(3)
    if t2 < 1e-14:
        for i in range(3):
            out[i] = float(np.sum(g * _hat(np.eye(3)[i])))
        return out
    r = axis_angle_to_matrix(v)
    imr = np.eye(3) - r
    for i in range(3):
        w = (v[i] * v + np.cross(v, imr[:, i])) / t2
        out[i] = float(np.sum(g * (_hat(w) @ r)))
    return out


def rotation_from_6d(a) -> np.ndarray:
    """Gram-Schmidt of two 3-vectors into columns (c1, c2, c1 x c2)."""
    a = np.asarray(a, dtype=np.float64).reshape(6)
    a1, a2 = a[:3], a[3:]
    n1 = float(np.linalg.norm(a1))
    if n1 < 1e-8:
        raise ConfigurationError("6d rotation: first column has near-zero norm")
    c1 = a1 / n1
    w = a2 - np.dot(c1, a2) * c1
    nw = float(np.linalg.norm(w))
    if nw < 1e-8:
        raise ConfigurationError("6d rotation: columns are near-parallel")
    c2 = w / nw
    return np.stack([c1, c2, np.cross(c1, c2)], axis=1)


def rotation_6d_vjp(a, grad_matrix) -> np.ndarray:
    """Reverse mode through normalise -> project -> normalise -> cross."""
    a = np.asarray(a, dtype=np.float64).reshape(6)
    g = np.asarray(grad_matrix, dtype=np.float64).reshape(3, 3)
    a1, a2 = a[:3], a[3:]
    n1 = float(np.linalg.norm(a1))
    c1 = a1 / n1
    s = float(np.dot(c1, a2))
    w = a2 - s * c1
    nw = float(np.linalg.norm(w))
    c2 = w / nw
    b1, b2, b3 = g[:, 0], g[:, 1], g[:, 2]
    bar_c2 = b2 + np.cross(b3, c1)
    bar_w = (bar_c2 - np.dot(c2, bar_c2) * c2) / nw
    bar_a2 = bar_w - np.dot(c1, bar_w) * c1
    bar_c1 = b1 + np.cross(c2, b3) - np.dot(c1, bar_w) * a2 - s * bar_w
    bar_a1 = (bar_c1 - np.dot(c1, bar_c1) * c1) / n1
    return np.concatenate([bar_a1, bar_a2])


# ----------------------------------------------------------------------------- camera
@dataclass(frozen=True)
class Camera:
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
    rotation: np.ndarray = field(init=False, repr=False)

    def __post_init__(self):
        object.__setattr__(self, "translation", np.asarray(self.translation, dtype=np.float64).reshape(3))
        object.__setattr__(self, "rotation_param",
                           np.asarray(self.rotation_param, dtype=np.float64).reshape(-1))
        if self.rotation_type == AXIS_ANGLE:
            if self.rotation_param.shape != (3,):
                raise ConfigurationError("axis-angle rotation needs 3 values")
            r = axis_angle_to_matrix(self.rotation_param)
        elif self.rotation_type == SIX_D:
            if self.rotation_param.shape != (6,):
                raise ConfigurationError("6d rotation needs 6 values")
            r = rotation_from_6d(self.rotation_param)
        else:
            raise ConfigurationError(f"unknown rotation type {self.rotation_type!r}")
        if np.abs(r.T @ r - np.eye(3)).max() >= 1e-6:
            raise ConfigurationError("rotation failed orthonormality check")
        object.__setattr__(self, "rotation", r)
        if self.mode not in (PINHOLE, ORTHOGRAPHIC):
            raise ConfigurationError(f"unknown camera mode {self.mode!r}")
        if self.focal_length <= 0 or self.sensor_width <= 0:
            raise ConfigurationError("focal length and sensor width must be > 0")
        if self.width < 1 or self.height < 1:
            raise ConfigurationError("image size must be at least 1x1")
        if not (self.near < self.far) or self.near < 0:
            raise ConfigurationError(f"need 0 <= near < far, got near={self.near} far={self.far}")
        if self.far - self.near < 1e-12:
            raise ConfigurationError("far - near underflows")

    @property
    def pixel_size(self) -> float:
        return self.sensor_width / self.width

    @property
    def sensor_height(self) -> float:
        return self.sensor_width * self.height / self.width

    def world_to_camera(self, points) -> np.ndarray:
        return (np.asarray(points, dtype=np.float64) - self.translation) @ self.rotation.T

    def camera_to_world(self, points) -> np.ndarray:
        return np.asarray(points, dtype=np.float64) @ self.rotation + self.translation


def camera_from_vector(vec, width: int, height: int, near: float = 0.1, far: float = 45.0,
                       mode: str = PINHOLE) -> Camera:
    """8 values: t(3), axis-angle(3), focal, sensor width; 11 values: t(3), 6d(6), focal, sensor."""
    v = np.asarray(vec, dtype=np.float64).reshape(-1)
    if v.shape == (8,):
        rp, rt, f, s = v[3:6], AXIS_ANGLE, v[6], v[7]
    elif v.shape == (11,):
        rp, rt, f, s = v[3:9], SIX_D, v[9], v[10]
    else:
        raise ConfigurationError(f"camera vector must have 8 or 11 values, got {v.size}")
    return Camera(translation=v[:3], rotation_param=rp, rotation_type=rt, focal_length=float(f),
                  sensor_width=float(s), width=int(width), height=int(height), near=float(near),
                  far=float(far), mode=mode)


def camera_to_vector(cam) -> np.ndarray:
    return np.concatenate([cam.translation, cam.rotation_param, [cam.focal_length, cam.sensor_width]])


# ----------------------------------------------------------------------------- scene
@dataclass
class SphereScene:
    feature_dim: int
    background: np.ndarray
    positions: np.ndarray = field(default=None)
    radii: np.ndarray = field(default=None)
    opacities: np.ndarray = field(default=None)
    features: np.ndarray = field(default=None)

    def __post_init__(self):
        d = self.feature_dim
        if self.positions is None:
            self.positions = np.zeros((0, 3))
        if self.radii is None:
            self.radii = np.zeros(0)
        if self.opacities is None:
            self.opacities = np.zeros(0)
        if self.features is None:
            self.features = np.zeros((0, d))
        self.background = np.asarray(self.background, dtype=np.float64).reshape(d)

    def __len__(self) -> int:
        return self.positions.shape[0]

    @property
    def num_spheres(self) -> int:
        return self.positions.shape[0]

    def copy(self) -> "SphereScene":
        return SphereScene(self.feature_dim, self.background.copy(), self.positions.copy(),
                           self.radii.copy(), self.opacities.copy(), self.features.copy())

    def validate(self) -> None:
        validate_arrays(self.positions, self.radii, self.opacities, self.features, self.background,
                        self.feature_dim)


def validate_arrays(positions, radii, opacities, features, background, feature_dim) -> None:
    """ValidationError on any NaN/Inf field or non-positive radius (host-side twin of the
    device-side scan in k_project)."""
    m = positions.shape[0]
    if tuple(features.shape) != (m, feature_dim):
        raise ValidationError(
            f"feature array shape {tuple(features.shape)} does not match (M={m}, d={feature_dim})")
    if not np.all(np.isfinite(background)):
        raise ValidationError("background feature contains non-finite values")
    for name, arr in (("position", positions), ("radius", radii), ("opacity", opacities),
                      ("feature", features)):
        bad = ~np.isfinite(arr)
        if bad.any():
            raise ValidationError(f"non-finite {name} at sphere index {int(np.argwhere(bad)[0][0])}")
    bad_r = radii <= 0
    if bad_r.any():
        raise ValidationError(f"non-positive radius at sphere index {int(np.argmax(bad_r))}")


def new_scene(feature_dim: int, background_feature) -> SphereScene:
    if int(feature_dim) < 1:
        raise ConfigurationError(f"feature_dim must be >= 1, got {feature_dim}")
    bg = np.atleast_1d(np.asarray(background_feature, dtype=np.float64))
    if bg.shape != (int(feature_dim),):
        raise ConfigurationError(f"background feature has length {bg.size}, expected {feature_dim}")
    return SphereScene(feature_dim=int(feature_dim), background=bg)


def add_sphere_arrays(scene: SphereScene, positions, radii, opacities, features) -> SphereScene:
    positions = np.asarray(positions, dtype=np.float64).reshape(-1, 3)
    radii = np.asarray(radii, dtype=np.float64).reshape(-1)
    opacities = np.asarray(opacities, dtype=np.float64).reshape(-1)
    features = np.atleast_2d(np.asarray(features, dtype=np.float64))
    n = positions.shape[0]
    if not (radii.shape[0] == opacities.shape[0] == features.shape[0] == n):
        raise ValidationError("sphere column arrays have mismatched lengths")
    if features.shape[1] != scene.feature_dim:
        raise ValidationError(f"feature dim {features.shape[1]} does not match scene d={scene.feature_dim}")
    validate_arrays(positions, radii, opacities, features, scene.background, scene.feature_dim)
    scene.positions = np.concatenate([scene.positions, positions])
    scene.radii = np.concatenate([scene.radii, radii])
    scene.opacities = np.concatenate([scene.opacities, opacities])
    scene.features = np.concatenate([scene.features, features])
    return scene


# ----------------------------------------------------------------------------- render artefacts
@dataclass
class FeatureImage:
    data: np.ndarray  # (H, W, d)
    background_weight: Optional[np.ndarray] = None  # (H, W)

    @property
    def height(self):
        return self.data.shape[0]

    @property
    def width(self):
        return self.data.shape[1]

    @property
    def feature_dim(self):
        return self.data.shape[2]


class BackwardBuffer:
    """Per-pixel top-K record feeding the backward pass (reference raster.py:97-110).

    The record stays on the GPU in the kernels' slot-major (K, H, W) layout; `ids`, `z`,
    `closeness` and `log_denom` materialise NumPy views in the reference's (H, W, K) layout
    on first access."""

    def __init__(self, dev, params: BlendParams, num_spheres: int, dtype=np.float32):
        self.dev = dev  # dict of CUDA tensors: ids/z/closeness (K,H,W), log_denom (H,W) (+ the forward token)
        self.params = params
        self.num_spheres = int(num_spheres)
        self.dtype = np.dtype(dtype)  # dtype of the float views (the reference's buffer has render_forward's dtype)
        self._np = {}

    def _get(self, name):
        if name not in self._np:
            t = self.dev[name]
            if t.dim() == 3:
                t = t.permute(1, 2, 0)
            a = t.contiguous().cpu().numpy()
            self._np[name] = a if name == "ids" else a.astype(self.dtype, copy=False)
        return self._np[name]

    @property
    def ids(self):
        return self._get("ids")

    @property
    def z(self):
        return self._get("z")

    @property
    def closeness(self):
        return self._get("closeness")

    @property
    def log_denom(self):
        return self._get("log_denom")


@dataclass
class RenderStats:
    spheres_total: int = 0
    spheres_on_sensor: int = 0
    candidates_tested: int = 0
    hits_blended: int = 0
    pixels_early_stopped: int = 0
    tiles: int = 0

    def early_stop_ratio(self, num_pixels: int) -> float:
        return self.pixels_early_stopped / num_pixels if num_pixels else 0.0


@dataclass
class SceneGradients:
    d_position: np.ndarray
    d_radius: np.ndarray
    d_opacity: np.ndarray
    d_feature: np.ndarray
    pixel_count: np.ndarray

    @staticmethod
    def zeros(m: int, d: int) -> "SceneGradients":
        return SceneGradients(np.zeros((m, 3)), np.zeros(m), np.zeros(m), np.zeros((m, d)),
                              np.zeros(m, dtype=np.int64))


@dataclass
class CameraGradients:
    d_translation: np.ndarray
    d_rotation: np.ndarray
    d_focal: float
    d_sensor_width: float
