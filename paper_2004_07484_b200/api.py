"""Reference-facing entry points of the B200 render path.

`render_forward` / `render_backward` keep the reference's library signatures
(softsphere/raster.py:437-447, softsphere/grad.py:323-334) and return the same artefact
types, so they drop into `softsphere.optim.fit(..., renderer=SoftsphereAdapter())`
(optim.py:228-278) and into tests written against the reference.  Scene / camera / params may
be this package's types or the reference's own objects (same attribute names).

Host arrays are snapped to float32 on upload (the device path is float32 SoA + float64
geometry); outputs come back as float64 NumPy arrays like the reference's.
"""
from __future__ import annotations

import numpy as np
import torch

from .engine import CameraSpec, RenderEngine, default_engine
from .types import (AXIS_ANGLE, BackwardBuffer, BlendParams, CameraGradients, ConfigurationError,
                    ContractViolation, FeatureImage, RenderStats, SceneGradients, ValidationError,
                    axis_angle_vjp, rotation_6d_vjp)

DEFAULT_TILE_SIZE = 16
GATE_RADIUS_PX = 3.0


def _scene_arrays(scene):
    m = len(scene)
    d = int(scene.feature_dim)
    feats = np.asarray(scene.features)
    if tuple(feats.shape) != (m, d):
        raise ValidationError(f"feature array shape {tuple(feats.shape)} does not match (M={m}, d={d})")
    return (np.asarray(scene.positions), np.asarray(scene.radii), np.asarray(scene.opacities), feats,
            np.asarray(scene.background))


def _upload(scene, device):
    pos, rad, opa, feat, bg = _scene_arrays(scene)

    def up(a, shape):
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32).reshape(shape))
        return t.to(device, non_blocking=True)

    d = int(scene.feature_dim)
    return up(pos, (-1, 3)), up(rad, (-1,)), up(opa, (-1,)), up(feat, (-1, d)), up(bg, (-1,))


def render_forward(scene, camera, params, *, workers: int = 1, dtype=np.float64,
                   tile_size: int = DEFAULT_TILE_SIZE, store_buffer: bool = True, chunk_size: int = 256,
                   engine: RenderEngine = None):
    """Bounds, depth order, tile binning and tile draw on the GPU.

    Returns (FeatureImage, BackwardBuffer or None, RenderStats) like the reference.  `workers`
    and `dtype` are accepted for signature compatibility and ignored (the device path is
    deterministic and mixed float32/float64 by design)."""
    eng = engine or default_engine()
    if tile_size != DEFAULT_TILE_SIZE:
        raise ConfigurationError("the B200 path supports tile_size=16 only")
    if not (1 <= int(chunk_size) <= 256):
        raise ConfigurationError("chunk_size must be in 1..256")
    p = params if isinstance(params, BlendParams) else BlendParams(params.gamma, params.epsilon, params.tau,
                                                                   params.top_k)
    dev_in = _upload(scene, eng.device)
    # background is validated on the host (d numbers); per-sphere fields are scanned on the device
    if not np.all(np.isfinite(np.asarray(scene.background, dtype=np.float64))):
        raise ValidationError("background feature contains non-finite values")
    cam = CameraSpec.from_camera(camera)
    res = eng.forward(*dev_in, cam, gamma=p.gamma, eps=p.epsilon, tau=p.tau, top_k=p.top_k,
                      chunk=int(chunk_size), store_buffer=store_buffer, collect_stats=True, check=True)
    st = res["status"]
    image = FeatureImage(data=res["image"].cpu().numpy().astype(np.float64),
                         background_weight=res["bg_weight"].cpu().numpy().astype(np.float64))
    buffer = None
    if store_buffer:
        buffer = BackwardBuffer({k: res[k] for k in ("ids", "z", "closeness", "log_denom")}, p, len(scene))
        buffer._inputs = res["inputs"]
    ntx, nty = (cam.width + 15) // 16, (cam.height + 15) // 16
    stats = RenderStats(spheres_total=len(scene), spheres_on_sensor=st["spheres_on_sensor"],
                        candidates_tested=st["candidates_tested"], hits_blended=st["hits_blended"],
                        pixels_early_stopped=st["pixels_early_stopped"], tiles=ntx * nty)
    return image, buffer, stats


def render_backward(scene, camera, params, buffer: BackwardBuffer, upstream, *, workers: int = 1,
                    normalize: bool = True, gate: bool = True, tile_size: int = 16,
                    engine: RenderEngine = None):
    """Full backward pipeline; returns (SceneGradients, CameraGradients) as float64 NumPy."""
    eng = engine or default_engine()
    if buffer.num_spheres != len(scene):
        raise ContractViolation(f"buffer built for {buffer.num_spheres} spheres, scene has {len(scene)}")
    upstream = np.asarray(upstream, dtype=np.float64)
    k, h, w = buffer.dev["ids"].shape
    if upstream.shape != (h, w, scene.feature_dim):
        raise ValidationError(f"upstream shape {upstream.shape} != {(h, w, scene.feature_dim)}")
    bp = buffer.params
    cam = CameraSpec.from_camera(camera)
    dev_in = _upload(scene, eng.device)
    up = torch.from_numpy(np.ascontiguousarray(upstream, dtype=np.float32)).to(eng.device, non_blocking=True)
    out = eng.backward(*dev_in, cam, buffer.dev, up, gamma=bp.gamma, eps=bp.epsilon, normalize=normalize,
                       gate=gate, camera_grads=True)
    m, d = len(scene), int(scene.feature_dim)
    grads = SceneGradients(
        d_position=out["d_pos"].cpu().numpy().astype(np.float64).reshape(m, 3),
        d_radius=out["d_rad"].cpu().numpy().astype(np.float64),
        d_opacity=out["d_opa"].cpu().numpy().astype(np.float64),
        d_feature=out["d_feat"].cpu().numpy().astype(np.float64).reshape(m, d),
        pixel_count=out["pixel_count"].cpu().numpy().astype(np.int64),
    )
    cg = out["cam_grad"].cpu().numpy()
    g_rot = cg[3:12].reshape(3, 3)
    if camera.rotation_type == AXIS_ANGLE:
        d_rot = axis_angle_vjp(camera.rotation_param, g_rot)
    else:
        d_rot = rotation_6d_vjp(camera.rotation_param, g_rot)
    cam_grads = CameraGradients(d_translation=cg[0:3].copy(), d_rotation=d_rot, d_focal=float(cg[12]),
                                d_sensor_width=float(cg[13]))
    return grads, cam_grads


class SoftsphereAdapter:
    """`renderer=` plug-in for the reference's fit loop (optim.py:265-278): an object with
    forward(scene, camera, params) and backward(scene, camera, params, buffer, upstream)."""

    def __init__(self, normalize: bool = True, gate: bool = True, engine: RenderEngine = None):
        self.normalize = normalize
        self.gate = gate
        self.engine = engine

    def forward(self, scene, camera, params):
        return render_forward(scene, camera, params, engine=self.engine)

    def backward(self, scene, camera, params, buffer, upstream):
        return render_backward(scene, camera, params, buffer, upstream, normalize=self.normalize,
                               gate=self.gate, engine=self.engine)
