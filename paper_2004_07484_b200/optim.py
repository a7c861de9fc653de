"""the step either side of the render path in the reference's fit loop
(softsphere/optim.py), on the device.

  photometric_loss(rendered, target)        optim.py:87-97   (reference signature, NumPy in/out)
  adam_step(params, grads, state, lr, cfg)  optim.py:142-154 (reference signature, NumPy in/out)
  DeviceFit                                 the body of fit's loop (optim.py:280-329) for one observation:
                                            forward -> L1 loss + upstream -> backward -> regulariser +
                                            visibility + per-group Adam with radius floor, all device resident

Everything runs in the sm_100a kernels of csrc/ss_optim.cu (k_photometric, k_fit_step, k_adam_flat)
through the C ABI; there is no CPU fallback.  Pruning and subdivision are
DeviceFit.prune / DeviceFit.subdivide (surgery.py), checkpoints rank 3 (sceneio.py).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .engine import CameraSpec, RenderEngine, _ptr, _raise_for, default_engine
from .types import ConfigurationError, DivergenceError, ValidationError

RADIUS_MIN = 1e-6


@dataclass
class FitConfig:
    """The fields of the reference's FitConfig that the per-step update uses (optim.py:33-70)."""
    lr_position: float = 1e-3
    lr_radius: float = 1e-3
    lr_opacity: float = 1e-2
    lr_feature: float = 1e-2
    lr_camera: float = 0.0
    beta1: float = 0.9
    beta2: float = 0.999
    adam_eps: float = 1e-8
    gamma: float = 0.1
    epsilon: float = 1e-2
    tau: float = 0.01
    top_k: int = 5
    lambda_od: float = 0.0
    radius_min: float = RADIUS_MIN
    normalize_grads: bool = True
    gate: bool = True
    # blending schedule (optim.py:44-47, :72-79), pruning (:51-54) and subdivision (:55-57)
    steps: int = 500
    gamma_start: float = 0.1
    gamma_end: float = 1e-4
    prune_every: int = 0
    prune_opacity_min: float = 0.05
    prune_background_dist: float = 0.0
    subdivide_at: tuple = ()
    subdivide_scale: float = float(np.sqrt(2.0))
    seed: int = 0
    workers: int = 1  # accepted like the reference's field (optim.py:58); the device path has no worker pool

    def __post_init__(self):
        for name in ("lr_position", "lr_radius", "lr_opacity", "lr_feature", "lr_camera"):
            if getattr(self, name) < 0:
                raise ConfigurationError(f"{name} must be >= 0")
        for name in ("gamma_start", "gamma_end"):
            g = getattr(self, name)
            if not (1e-5 <= g <= 1.0):
                raise ConfigurationError(f"{name} must lie in [1e-5, 1]")

    def gamma_at(self, step: int) -> float:
        """Log-interpolated gamma schedule (optim.py:72-79)."""
        if self.steps <= 1:
            return self.gamma_start
        t = step / (self.steps - 1)
        return float(np.exp((1 - t) * np.log(self.gamma_start) + t * np.log(self.gamma_end)))


@dataclass
class AdamState:
    m: np.ndarray
    v: np.ndarray
    t: int = 0

    @staticmethod
    def like(x) -> "AdamState":
        return AdamState(m=np.zeros_like(x, dtype=np.float64), v=np.zeros_like(x, dtype=np.float64))


def _stream(dev):
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def photometric_loss_device(image: torch.Tensor, target: torch.Tensor):
    """Device tensors in, (loss tensor float64[1], upstream tensor) out; one kernel, no sync."""
    if image.shape != target.shape:
        raise ValidationError(f"rendered shape {tuple(image.shape)} != target {tuple(target.shape)}")
    lib = _lib.load()
    image, target = image.contiguous(), target.contiguous()
    upstream = torch.empty_like(image)
    loss = torch.empty(1, dtype=torch.float64, device=image.device)
    rc = lib.ss_photometric_loss(_ptr(image), _ptr(target), _ptr(upstream), image.numel(), _ptr(loss),
                                 _stream(image.device))
    if rc != _lib.SS_OK:
        _raise_for(rc)
    return loss, upstream


def photometric_loss(rendered, target, device="cuda"):
    """Mean absolute error and its subgradient image sign(diff)/n (reference signature)."""
    rendered = np.asarray(rendered, dtype=np.float64)
    target = np.asarray(target, dtype=np.float64)
    if rendered.shape != target.shape:
        raise ValidationError(f"rendered shape {rendered.shape} != target {target.shape}")
    dev = default_engine(device).device
    a = torch.from_numpy(rendered.astype(np.float32)).to(dev)
    b = torch.from_numpy(target.astype(np.float32)).to(dev)
    loss, up = photometric_loss_device(a, b)
    return float(loss.item()), up.cpu().numpy().astype(np.float64)


def adam_step(params, grads, state: AdamState, lr: float, config, device="cuda"):
    """Bias-corrected Adam on one array (reference signature); state is updated in place."""
    params = np.asarray(params, dtype=np.float64)
    grads = np.asarray(grads, dtype=np.float64)
    if params.shape != grads.shape or state.m.shape != params.shape:
        raise ValidationError("adam_step: parameter/gradient/state shape mismatch")
    lib = _lib.load()
    dev = default_engine(device).device
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(dev)
    p, g, m, v = t(params), t(grads), t(state.m), t(state.v)
    state.t += 1
    rc = lib.ss_adam_flat(_ptr(p), _ptr(g), _ptr(m), _ptr(v), p.numel(), float(lr), float(config.beta1),
                          float(config.beta2), float(config.adam_eps), int(state.t), 0, 0.0, _stream(dev))
    if rc != _lib.SS_OK:
        _raise_for(rc)
    state.m = m.cpu().numpy().astype(np.float64).reshape(params.shape)
    state.v = v.cpu().numpy().astype(np.float64).reshape(params.shape)
    return p.cpu().numpy().astype(np.float64).reshape(params.shape)


class DeviceFit:
    """Device-resident scene + Adam moments + visibility; `step` is one iteration of the reference's
    fit loop body for one observation (optim.py:286-329), without leaving the GPU."""

    def __init__(self, pos, rad, opa, feat, bg, config: FitConfig = None, engine: RenderEngine = None,
                 device="cuda"):
        self.cfg = config or FitConfig()
        self.engine = engine or RenderEngine(device)
        dev = self.engine.device
        f32 = lambda x, shape: torch.as_tensor(np.ascontiguousarray(x, dtype=np.float32)).reshape(shape).to(dev).clone()
        bg = np.asarray(bg, dtype=np.float32).reshape(-1)
        self.d = int(bg.shape[0])
        self.pos, self.rad = f32(pos, (-1, 3)), f32(rad, (-1,))
        self.opa, self.feat, self.bg = f32(opa, (-1,)), f32(feat, (-1, self.d)), f32(bg, (-1,))
        self.energy = torch.zeros(1, dtype=torch.float64, device=dev)
        self.last = None
        self._reset_state()

    @classmethod
    def from_device(cls, pos, rad, opa, feat, bg, config: FitConfig = None, engine: RenderEngine = None):
        """Adopt float32 device tensors (e.g. from sceneio.scene_from_bytes_device) without a host copy."""
        self = cls.__new__(cls)
        self.cfg = config or FitConfig()
        self.engine = engine or RenderEngine(pos.device)
        self.d = int(feat.shape[1])
        self.pos, self.rad, self.opa, self.feat, self.bg = pos, rad, opa, feat, bg
        self.energy = torch.zeros(1, dtype=torch.float64, device=pos.device)
        self.last = None
        self._reset_state()
        return self

    def _reset_state(self):
        """Fresh Adam moments, step counts and visibility for the current sphere set (optim.py:355-363)."""
        self.m = int(self.pos.shape[0])
        z = lambda t: torch.zeros_like(t)
        self.moments = {k: (z(t), z(t)) for k, t in (("pos", self.pos), ("rad", self.rad), ("opa", self.opa),
                                                     ("feat", self.feat))}
        self.steps = [0, 0, 0, 0]
        self.visibility = torch.zeros(self.m, dtype=torch.int32, device=self.pos.device)

    def prune(self):
        """prune + states[name].take(keep) + visibility reset (optim.py:345-353), all on the device.
        Returns the number of spheres kept."""
        from .surgery import prune_device
        cfg = self.cfg
        extra = [t for k in ("pos", "rad", "opa", "feat") for t in self.moments[k]]
        self.pos, self.rad, self.opa, self.feat, extra, _ = prune_device(
            self.pos, self.rad, self.opa, self.feat, self.bg, self.visibility, cfg.prune_opacity_min,
            cfg.prune_background_dist, extra)
        self.moments = {k: (extra[2 * i], extra[2 * i + 1]) for i, k in enumerate(("pos", "rad", "opa", "feat"))}
        self.m = int(self.pos.shape[0])
        self.visibility = torch.zeros(self.m, dtype=torch.int32, device=self.pos.device)
        return self.m

    def subdivide(self):
        """FCC x12 subdivision with fresh optimiser state (optim.py:355-363).  Returns the new count."""
        from .surgery import subdivide_device
        self.pos, self.rad, self.opa, self.feat = subdivide_device(self.pos, self.rad, self.opa, self.feat,
                                                                   self.cfg.subdivide_scale)
        self._reset_state()
        return self.m

    def apply_gradients(self, grads: dict, cam: CameraSpec):
        """k_fit_step on the outputs of RenderEngine.backward."""
        cfg, lib = self.cfg, _lib.load()
        a = _lib.SsFitStepArgs()
        a.num_spheres, a.feature_dim = self.m, self.d
        a.pos, a.rad, a.opa, a.feat = _ptr(self.pos), _ptr(self.rad), _ptr(self.opa), _ptr(self.feat)
        a.d_pos, a.d_rad = _ptr(grads["d_pos"]), _ptr(grads["d_rad"])
        a.d_opa, a.d_feat = _ptr(grads["d_opa"]), _ptr(grads["d_feat"])
        a.pixel_count, a.visibility = _ptr(grads["pixel_count"]), _ptr(self.visibility)
        (a.m_pos, a.v_pos), (a.m_rad, a.v_rad) = map(_ptr, self.moments["pos"]), map(_ptr, self.moments["rad"])
        (a.m_opa, a.v_opa), (a.m_feat, a.v_feat) = map(_ptr, self.moments["opa"]), map(_ptr, self.moments["feat"])
        lrs = (cfg.lr_position, cfg.lr_radius, cfg.lr_opacity, cfg.lr_feature)
        for g, lr in enumerate(lrs):
            if lr > 0:
                self.steps[g] += 1
            a.lr[g] = float(lr)
            a.step[g] = max(self.steps[g], 1)
        a.beta1, a.beta2, a.adam_eps = float(cfg.beta1), float(cfg.beta2), float(cfg.adam_eps)
        a.radius_min, a.lambda_od = float(cfg.radius_min), float(cfg.lambda_od)
        a.cam = cam.to_c()
        a.energy = _ptr(self.energy)
        rc = lib.ss_fit_step(C.byref(a), _stream(self.engine.device))
        if rc != _lib.SS_OK:
            _raise_for(rc)

    def step(self, target: torch.Tensor, cam: CameraSpec, gamma: float = None, check: bool = True):
        """forward -> loss/upstream -> backward -> fused update.  Returns the loss (float64 tensor [1]:
        photometric + regulariser energy of the scene BEFORE the update, like the reference's trace).
        check=True (default) reads the status block after the forward pass (one stream sync): invalid fields
        raise ValidationError like the reference's render_forward, a tile-pair overflow regrows the workspace
        and re-renders.  check=False never syncs; the caller then polls engine.read_status() itself -- an
        overflowed frame is background only and yields zero gradients."""
        cfg = self.cfg
        g = cfg.gamma if gamma is None else gamma
        f = self.engine.forward(self.pos, self.rad, self.opa, self.feat, self.bg, cam, gamma=g, eps=cfg.epsilon,
                                tau=cfg.tau, top_k=cfg.top_k, check=check)
        loss, upstream = photometric_loss_device(f["image"], target)
        grads = self.engine.backward(self.pos, self.rad, self.opa, self.feat, self.bg, cam, f, upstream, gamma=g,
                                     eps=cfg.epsilon, normalize=cfg.normalize_grads, gate=cfg.gate,
                                     camera_grads=cfg.lr_camera > 0)
        self.apply_gradients(grads, cam)
        self.engine.invalidate_records()  # k_fit_step moved the spheres behind torch's version counters
        self.last = {"image": f["image"], "grads": grads, "status": f["status"]}
        return loss + self.energy

    def check_finite(self, loss: torch.Tensor):
        if not bool(torch.isfinite(loss).all()):
            raise DivergenceError("non-finite loss")


# --------------------------------------------------------------------------------------------------
# The fit loop (optim.py:219-373): the caller of the render path.  Everything per sphere and per pixel stays on
# the device (DeviceFit.step / .prune / .subdivide); what remains on the host is the loop itself: the seeded
# epoch shuffling, the gamma schedule, the 8- or 11-value camera Adam step and the event / trace bookkeeping.
@dataclass
class Observation:
    """One posed training image (optim.py:25-30)."""
    image: np.ndarray  # (H, W, d)
    camera: object


@dataclass
class FitResult:
    scene: object
    cameras: list
    trace: np.ndarray  # per-step loss
    events: list = field(default_factory=list)  # (step, kind, detail)


def _adam_host(params, grads, state: AdamState, lr, cfg):
    """adam_step for the camera vector (8 or 11 float64 values): host arithmetic, optim.py:142-154."""
    state.t += 1
    state.m = cfg.beta1 * state.m + (1.0 - cfg.beta1) * grads
    state.v = cfg.beta2 * state.v + (1.0 - cfg.beta2) * grads * grads
    m_hat = state.m / (1.0 - cfg.beta1 ** state.t)
    v_hat = state.v / (1.0 - cfg.beta2 ** state.t)
    return params - lr * m_hat / (np.sqrt(v_hat) + cfg.adam_eps)


def fit(scene, observations, config: FitConfig, renderer=None, on_step=None, device="cuda") -> FitResult:
    """Reference signature (optim.py:228).  The device pipeline IS the renderer: `renderer` may be None or a
    SoftsphereAdapter (its engine and its normalize / gate flags are used, like the reference uses a plug-in's
    own settings, optim.py:273-278); any other plug-in object is refused -- hand that one to the reference's
    own fit loop.  on_step(step, loss, fit_state, cameras) receives the DeviceFit (device tensors) instead of
    a host scene; FitResult.scene is downloaded once at the end."""
    from .types import (AXIS_ANGLE, SphereScene, axis_angle_vjp, camera_from_vector, camera_to_vector,
                        rotation_6d_vjp)
    engine = None
    if renderer is not None:
        from .api import SoftsphereAdapter
        if not isinstance(renderer, SoftsphereAdapter):
            raise ConfigurationError("the device fit loop renders with its own kernels; pass renderer=None or a "
                                     "SoftsphereAdapter (other plug-ins belong to the reference's fit loop)")
        import dataclasses
        config = dataclasses.replace(config, normalize_grads=renderer.normalize, gate=renderer.gate)
        engine = renderer.engine
    if not observations:
        raise ValidationError("fit needs at least one observation")
    d = scene.feature_dim
    for i, ob in enumerate(observations):
        if tuple(np.shape(ob.image)) != (ob.camera.height, ob.camera.width, d):
            raise ValidationError(f"observation {i} image shape mismatch")
    dfit = DeviceFit(scene.positions, scene.radii, scene.opacities, scene.features, scene.background, config,
                     engine=engine, device=device)
    dev = dfit.engine.device
    targets = [torch.from_numpy(np.ascontiguousarray(ob.image, dtype=np.float32)).to(dev) for ob in observations]
    cameras = [ob.camera for ob in observations]
    cam_states = [AdamState.like(camera_to_vector(c)) for c in cameras]
    rng = np.random.default_rng(config.seed)
    trace = np.zeros(config.steps)
    events = []
    seen = np.zeros(len(observations), dtype=bool)
    order = []
    subdivide_at = set(config.subdivide_at)
    for step in range(config.steps):
        if not order:
            order = list(rng.permutation(len(observations)))
        idx = int(order.pop(0))
        seen[idx] = True
        cam = cameras[idx]
        loss_t = dfit.step(targets[idx], CameraSpec.from_camera(cam), gamma=config.gamma_at(step), check=True)
        loss = float(loss_t.item())
        if not np.isfinite(loss):
            raise DivergenceError(f"non-finite loss at step {step}")
        trace[step] = loss
        if config.lr_camera > 0:
            cg = dfit.last["grads"]["cam_grad"].cpu().numpy()
            g_rot = cg[3:12].reshape(3, 3)
            d_rot = (axis_angle_vjp(cam.rotation_param, g_rot) if cam.rotation_type == AXIS_ANGLE
                     else rotation_6d_vjp(cam.rotation_param, g_rot))
            gvec = np.concatenate([cg[0:3], d_rot, [cg[12], cg[13]]])
            new_vec = _adam_host(camera_to_vector(cam), gvec, cam_states[idx], config.lr_camera, config)
            cameras[idx] = camera_from_vector(new_vec, cam.width, cam.height, near=cam.near, far=cam.far,
                                              mode=cam.mode)
        if config.prune_every and (step + 1) % config.prune_every == 0 and seen.all():
            events.append((step, "prune", dfit.prune()))
            seen[:] = False
        if step in subdivide_at:
            events.append((step, "subdivide", dfit.subdivide()))
            seen[:] = False
        if on_step is not None:
            on_step(step, loss, dfit, cameras)
    f64 = lambda t: t.cpu().numpy().astype(np.float64)
    out = SphereScene(feature_dim=d, background=np.array(scene.background, dtype=np.float64),
                      positions=f64(dfit.pos), radii=f64(dfit.rad), opacities=f64(dfit.opa), features=f64(dfit.feat))
    return FitResult(scene=out, cameras=cameras, trace=trace, events=events)
