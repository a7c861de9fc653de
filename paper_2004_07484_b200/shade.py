"""post-projection shading of the feature map on the device (reference
softsphere/shade.py).  Every shader is a per-pixel map with an explicit backward companion.

Reference signatures (NumPy / FeatureImage in, float64 NumPy out):
  shade_identity, shade_identity_backward            shade.py:66-77
  shade_diffuse, shade_diffuse_backward              shade.py:84-131
  view_direction_plane                               shade.py:138-142
  shade_linear, shade_linear_backward                shade.py:148-171
The `*_device` twins take and return float32 CUDA tensors (the image straight out of ss_forward) and do
not synchronise.  All arithmetic runs in csrc/ss_shade.cu through the C ABI; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .engine import CameraSpec, _ptr, _raise_for, default_engine
from .types import FeatureImage, ValidationError

MAX_LIGHTS = 8


@dataclass
class DirectionalLight:
    direction: np.ndarray  # unit vector, pointing from the light into the scene
    intensity: float = 1.0
    ambient: float = 0.0

    def __post_init__(self):
        d = np.asarray(self.direction, dtype=np.float64).reshape(3)
        n = np.linalg.norm(d)
        if n < 1e-12:
            raise ValidationError("light direction has zero norm")
        self.direction = d / n
        if self.intensity < 0 or not (0.0 <= self.ambient <= 1.0):
            raise ValidationError("intensity must be >= 0 and ambient in [0, 1]")


@dataclass
class LinearShader:
    """Per-pixel affine map from d feature channels (+3 view-direction channels) to RGB."""
    weight: np.ndarray  # (d_in, 3)
    bias: np.ndarray  # (3,)
    trainable: bool = True

    def __post_init__(self):
        self.weight = np.asarray(self.weight, dtype=np.float64)
        self.bias = np.asarray(self.bias, dtype=np.float64).reshape(3)
        if self.weight.ndim != 2 or self.weight.shape[1] != 3:
            raise ValidationError("shader weight must have shape (d_in, 3)")
        if not (np.isfinite(self.weight).all() and np.isfinite(self.bias).all()):
            raise ValidationError("shader parameters must be finite")


def _stream(dev):
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _check(rc):
    if rc != _lib.SS_OK:
        _raise_for(rc)


def _to_device(image, device="cuda") -> torch.Tensor:
    if isinstance(image, torch.Tensor):
        return image.to(dtype=torch.float32).contiguous()
    if isinstance(image, FeatureImage) or hasattr(image, "data") and not isinstance(image, np.ndarray):
        image = image.data
        if isinstance(image, torch.Tensor):
            return image.to(dtype=torch.float32).contiguous()
    dev = default_engine(device).device
    return torch.from_numpy(np.ascontiguousarray(np.asarray(image, dtype=np.float32))).to(dev)


def _host(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().astype(np.float64)


def _lights_c(lights):
    if len(lights) > MAX_LIGHTS:
        raise ValidationError(f"at most {MAX_LIGHTS} lights")
    arr = (_lib.SsLight * max(len(lights), 1))()
    for i, l in enumerate(lights):
        arr[i].direction[:] = [float(x) for x in np.asarray(l.direction).reshape(3)]
        arr[i].intensity, arr[i].ambient = float(l.intensity), float(l.ambient)
    return arr


# ------------------------------------------------------------------------------------------- identity
def shade_identity_device(f: torch.Tensor) -> torch.Tensor:
    if f.shape[-1] != 3:
        raise ValidationError(f"identity shading needs d=3, got d={f.shape[-1]}")
    out = torch.empty_like(f)
    _check(_lib.load().ss_shade_identity(_ptr(f), f.numel(), _ptr(out), _stream(f.device)))
    return out


def shade_identity_backward_device(f: torch.Tensor, upstream: torch.Tensor) -> torch.Tensor:
    out = torch.empty_like(f)
    _check(_lib.load().ss_shade_identity_backward(_ptr(f), _ptr(upstream.contiguous()), f.numel(), _ptr(out),
                                                  _stream(f.device)))
    return out


def shade_identity(image, device="cuda") -> np.ndarray:
    """Pass 3-channel features through, clamped to [0, 1]."""
    return _host(shade_identity_device(_to_device(image, device)))


def shade_identity_backward(image, upstream, device="cuda") -> np.ndarray:
    f = _to_device(image, device)
    return _host(shade_identity_backward_device(f, _to_device(upstream, device).to(f.device)))


# -------------------------------------------------------------------------------------------- diffuse
def _check_diffuse(f):
    if f.shape[-1] != 6:
        raise ValidationError(f"diffuse shading needs the [albedo:3, normal:3] layout, got d={f.shape[-1]}")


def shade_diffuse_device(f: torch.Tensor, lights) -> torch.Tensor:
    _check_diffuse(f)
    out = torch.empty(f.shape[:-1] + (3,), dtype=torch.float32, device=f.device)
    _check(_lib.load().ss_shade_diffuse(_ptr(f), f.numel() // 6, _lights_c(lights), len(lights), _ptr(out),
                                        _stream(f.device)))
    return out


def shade_diffuse_backward_device(f: torch.Tensor, lights, upstream: torch.Tensor) -> torch.Tensor:
    _check_diffuse(f)
    out = torch.empty_like(f)
    _check(_lib.load().ss_shade_diffuse_backward(_ptr(f), _ptr(upstream.contiguous()), f.numel() // 6,
                                                 _lights_c(lights), len(lights), _ptr(out), _stream(f.device)))
    return out


def shade_diffuse(image, lights, device="cuda") -> np.ndarray:
    """albedo * (ambient + sum_l intensity * max(0, n . -l)), clamped; zero normals get ambient only."""
    return _host(shade_diffuse_device(_to_device(image, device), lights))


def shade_diffuse_backward(image, lights, upstream, device="cuda") -> np.ndarray:
    f = _to_device(image, device)
    return _host(shade_diffuse_backward_device(f, lights, _to_device(upstream, device).to(f.device)))


# --------------------------------------------------------------------------------------------- linear
def view_direction_plane_device(camera, device="cuda") -> torch.Tensor:
    spec = camera if isinstance(camera, CameraSpec) else CameraSpec.from_camera(camera)
    dev = default_engine(device).device
    out = torch.empty((spec.height, spec.width, 3), dtype=torch.float32, device=dev)
    cam_c = spec.to_c()
    _check(_lib.load().ss_view_directions(C.byref(cam_c), _ptr(out), _stream(dev)))
    return out


def view_direction_plane(camera, device="cuda") -> np.ndarray:
    """(H, W, 3) unit view directions in the camera frame."""
    return _host(view_direction_plane_device(camera, device))


def _linear_args(f, shader, view_dirs):
    d = f.shape[-1]
    if view_dirs is not None and tuple(view_dirs.shape[:2]) != tuple(f.shape[:2]):
        raise ValidationError("view-direction plane does not match image size")
    d_in = d + (3 if view_dirs is not None else 0)
    if d_in != shader.weight.shape[0]:
        raise ValidationError(f"shader expects {shader.weight.shape[0]} inputs, image has {d_in}")
    w = torch.from_numpy(np.ascontiguousarray(shader.weight, dtype=np.float32)).to(f.device)
    b = torch.from_numpy(np.ascontiguousarray(shader.bias, dtype=np.float32)).to(f.device)
    return d, d_in, w, b


def shade_linear_device(f: torch.Tensor, shader: LinearShader, view_dirs: torch.Tensor = None) -> torch.Tensor:
    d, _, w, b = _linear_args(f, shader, view_dirs)
    out = torch.empty(f.shape[:-1] + (3,), dtype=torch.float32, device=f.device)
    _check(_lib.load().ss_shade_linear(_ptr(f), _ptr(view_dirs), f.numel() // d, d, _ptr(w), _ptr(b), _ptr(out),
                                       _stream(f.device)))
    return out


def shade_linear_backward_device(f, shader: LinearShader, upstream, view_dirs=None):
    """(d_features tensor, d_weight float64 tensor (d_in, 3) or None, d_bias float64 tensor (3) or None)."""
    d, d_in, w, b = _linear_args(f, shader, view_dirs)
    d_f = torch.empty_like(f)
    d_w = d_b = None
    if shader.trainable:
        d_w = torch.empty((d_in, 3), dtype=torch.float64, device=f.device)
        d_b = torch.empty(3, dtype=torch.float64, device=f.device)
    _check(_lib.load().ss_shade_linear_backward(_ptr(f), _ptr(view_dirs), f.numel() // d, d, _ptr(w), _ptr(b),
                                                _ptr(upstream.contiguous()), _ptr(d_f), _ptr(d_w), _ptr(d_b),
                                                _stream(f.device)))
    return d_f, d_w, d_b


def shade_linear(image, shader: LinearShader, view_dirs=None, device="cuda") -> np.ndarray:
    """Per-pixel affine map plus clamp; optionally view-direction conditioned."""
    f = _to_device(image, device)
    v = None if view_dirs is None else _to_device(view_dirs, device).to(f.device)
    return _host(shade_linear_device(f, shader, v))


def shade_linear_backward(image, shader: LinearShader, upstream, view_dirs=None, device="cuda"):
    """Returns (d_features, d_weight, d_bias); shader grads are None when the shader is frozen."""
    f = _to_device(image, device)
    v = None if view_dirs is None else _to_device(view_dirs, device).to(f.device)
    d_f, d_w, d_b = shade_linear_backward_device(f, shader, _to_device(upstream, device).to(f.device), v)
    if d_w is None:
        return _host(d_f), None, None
    return _host(d_f), d_w.cpu().numpy(), d_b.cpu().numpy()
