"""PyTorch front-end: `SphereRender` (torch.autograd.Function) and the paper-style `Renderer`
module (Listing 1: `Renderer(W, H, n)(pos, col, rad, cam, gamma=..., max_depth=...)`).

The Function only marshals pointers into the C-ABI library; all arithmetic happens in the
repo's sm_100a kernels.  The camera vector (8 = t, axis-angle, f, s; 11 = t, 6d, f, s) is host
data: it is turned into (t, R) on the host and its gradient is assembled on the host from the
kernel's 16-float camera block (d_t, dL/dR, d_f, d_s).
"""
from __future__ import annotations

import numpy as np
import torch

from .engine import CameraSpec, RenderEngine, default_engine
from .types import (AXIS_ANGLE, BlendParams, axis_angle_vjp, camera_from_vector, rotation_6d_vjp)


class SphereRender(torch.autograd.Function):
    @staticmethod
    def forward(ctx, pos, feat, rad, opa, cam_vec, bg, width, height, gamma, eps, tau, n_track, min_depth,
                max_depth, mode, normalize, gate, engine, check):
        eng: RenderEngine = engine or default_engine(pos.device)
        p = BlendParams(gamma, eps, tau, n_track)
        cam = camera_from_vector(cam_vec.detach().cpu().numpy(), width, height, near=min_depth, far=max_depth,
                                 mode=mode)
        spec = CameraSpec.from_camera(cam)
        res = eng.forward(pos.detach(), rad.detach(), opa.detach(), feat.detach(), bg.detach(), spec,
                          gamma=p.gamma, eps=p.epsilon, tau=p.tau, top_k=p.top_k, store_buffer=True,
                          check=check)
        ctx.eng, ctx.spec, ctx.cam, ctx.p = eng, spec, cam, p
        ctx.normalize, ctx.gate = normalize, gate
        ctx.buf = {k: res[k] for k in ("ids", "z", "closeness", "log_denom")}
        ctx.inputs = res["inputs"]
        ctx.cam_vec_meta = (cam_vec.device, cam_vec.dtype)
        ctx.mark_non_differentiable(res["bg_weight"])
        return res["image"], res["bg_weight"]

    @staticmethod
    def backward(ctx, grad_image, _grad_bgw):
        pos, rad, opa, feat, bg = ctx.inputs
        need_cam = ctx.needs_input_grad[4]
        out = ctx.eng.backward(pos, rad, opa, feat, bg, ctx.spec, ctx.buf, grad_image.contiguous(),
                               gamma=ctx.p.gamma, eps=ctx.p.epsilon, normalize=ctx.normalize, gate=ctx.gate,
                               camera_grads=need_cam)
        d_cam = None
        if need_cam:
            cg = out["cam_grad"].cpu().numpy()
            g_rot = cg[3:12].reshape(3, 3)
            cam = ctx.cam
            d_rot = (axis_angle_vjp if cam.rotation_type == AXIS_ANGLE else rotation_6d_vjp)(
                cam.rotation_param, g_rot)
            vec = np.concatenate([cg[0:3], d_rot, [cg[12], cg[13]]])
            dev, dt = ctx.cam_vec_meta
            d_cam = torch.from_numpy(vec).to(device=dev, dtype=dt)
        ctx.pixel_count = out["pixel_count"]
        return (out["d_pos"], out["d_feat"], out["d_rad"], out["d_opa"], d_cam, None, None, None, None, None,
                None, None, None, None, None, None, None, None, None)


class Renderer(torch.nn.Module):
    """Differentiable sphere renderer with a persistent workspace.

    forward(pos (M,3), feat (M,d), rad (M), cam_vec (8|11), opacity (M)=1, background (d)=0, gamma, ...)
    -> image (H, W, d).  Gradients flow to pos, feat, rad, opacity and cam_vec."""

    def __init__(self, width: int, height: int, n_track: int = 5, mode: str = "pinhole",
                 normalize: bool = True, gate: bool = True, device="cuda"):
        super().__init__()
        self.width, self.height, self.n_track, self.mode = int(width), int(height), int(n_track), mode
        self.normalize, self.gate = normalize, gate
        self.engine = RenderEngine(device)
        self.last_background_weight = None

    def forward(self, pos, feat, rad, cam_vec, opacity=None, background=None, gamma: float = 0.1,
                eps: float = 1e-2, tau: float = 0.01, min_depth: float = 0.1, max_depth: float = 45.0,
                check: bool = True):
        dev = self.engine.device
        if opacity is None:
            opacity = torch.ones(pos.shape[0], dtype=torch.float32, device=dev)
        if background is None:
            background = torch.zeros(feat.shape[1], dtype=torch.float32, device=dev)
        if not isinstance(cam_vec, torch.Tensor):
            cam_vec = torch.as_tensor(np.asarray(cam_vec, dtype=np.float64))
        image, bgw = SphereRender.apply(pos, feat, rad, opacity, cam_vec, background, self.width, self.height,
                                        gamma, eps, tau, self.n_track, min_depth, max_depth, self.mode,
                                        self.normalize, self.gate, self.engine, check)
        self.last_background_weight = bgw
        return image
