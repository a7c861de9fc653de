"""Host-buffer session: the reference-facing call for users whose scene lives in host memory
(as the reference's NumPy columns do).  Pinned staging buffers are allocated once; every
render_step copies the inputs host->device, runs ss_forward / ss_backward, and copies the image
and all gradients device->host.  This is the path bench.py times as `e2e`."""
from __future__ import annotations

import numpy as np
import torch

from .engine import CameraSpec, RenderEngine


class HostRenderSession:
    def __init__(self, num_spheres: int, feature_dim: int, width: int, height: int, top_k: int = 5,
                 engine: RenderEngine = None, device="cuda"):
        self.engine = engine or RenderEngine(device)
        dev = self.engine.device
        m, d, w, h = int(num_spheres), int(feature_dim), int(width), int(height)
        self.m, self.d, self.w, self.h, self.k = m, d, w, h, int(top_k)

        def pin(shape, dtype=torch.float32):
            return torch.empty(shape, dtype=dtype).pin_memory()

        def devt(shape, dtype=torch.float32):
            return torch.empty(shape, dtype=dtype, device=dev)

        # host (pinned) side
        self.h_pos, self.h_rad, self.h_opa, self.h_feat = pin((m, 3)), pin((m,)), pin((m,)), pin((m, d))
        self.h_bg, self.h_upstream = pin((d,)), pin((h, w, d))
        self.h_image = pin((h, w, d))
        self.h_d_pos, self.h_d_rad, self.h_d_opa, self.h_d_feat = pin((m, 3)), pin((m,)), pin((m,)), pin((m, d))
        self.h_count = pin((m,), torch.int32)
        self.h_cam_grad = pin((16,), torch.float64)
        # device side
        self.pos, self.rad, self.opa, self.feat = devt((m, 3)), devt((m,)), devt((m,)), devt((m, d))
        self.bg, self.upstream = devt((d,)), devt((h, w, d))
        self.out = {"d_pos": devt((m, 3)), "d_rad": devt((m,)), "d_opa": devt((m,)), "d_feat": devt((m, d)),
                    "pixel_count": devt((m,), torch.int32), "cam_grad": devt((16,), torch.float64)}
        self.h2d_bytes = 4 * (m * (5 + d) + d + h * w * d)
        self.d2h_bytes = 4 * (h * w * d + m * (5 + d) + m) + 16 * 8

    def set_scene(self, pos, rad, opa, feat, bg):
        for dst, src, shape in ((self.h_pos, pos, (self.m, 3)), (self.h_rad, rad, (self.m,)),
                                (self.h_opa, opa, (self.m,)), (self.h_feat, feat, (self.m, self.d)),
                                (self.h_bg, bg, (self.d,))):
            dst.copy_(torch.from_numpy(np.ascontiguousarray(src, dtype=np.float32).reshape(shape)))

    def render_step(self, cams, upstream_fn=None, gamma=0.1, eps=1e-2, tau=0.01, normalize=True, gate=True,
                    check=False, reduce_fn=None):
        """One host-to-host step over one or more views of the staged scene:
        H2D scene; per view: ss_forward, D2H image, [upstream_fn(view, host image) -> host upstream, else
        the staged h_upstream], H2D upstream, ss_backward (gradients summed over the views);
        optional reduce_fn(out) (the multi-GPU allreduce); D2H all gradients.  Returns after a
        stream sync with the last image and the gradient buffers (pinned host tensors)."""
        if not isinstance(cams, (list, tuple)):
            cams = [cams]
        nb = dict(non_blocking=True)
        self.pos.copy_(self.h_pos, **nb); self.rad.copy_(self.h_rad, **nb); self.opa.copy_(self.h_opa, **nb)
        self.feat.copy_(self.h_feat, **nb); self.bg.copy_(self.h_bg, **nb)
        for i, cam in enumerate(cams):
            f = self.engine.forward(self.pos, self.rad, self.opa, self.feat, self.bg, cam, gamma=gamma, eps=eps,
                                    tau=tau, top_k=self.k, check=check)
            self.h_image.copy_(f["image"], **nb)
            if upstream_fn is not None:
                torch.cuda.current_stream().synchronize()
                self.h_upstream.copy_(upstream_fn(i, self.h_image))
            self.upstream.copy_(self.h_upstream, **nb)
            self.engine.backward(self.pos, self.rad, self.opa, self.feat, self.bg, cam, f, self.upstream,
                                 gamma=gamma, eps=eps, normalize=normalize, gate=gate, camera_grads=True,
                                 out=self.out, accumulate=(i > 0))
        if reduce_fn is not None:
            reduce_fn(self.out)
        self.h_d_pos.copy_(self.out["d_pos"], **nb); self.h_d_rad.copy_(self.out["d_rad"], **nb)
        self.h_d_opa.copy_(self.out["d_opa"], **nb); self.h_d_feat.copy_(self.out["d_feat"], **nb)
        self.h_count.copy_(self.out["pixel_count"], **nb); self.h_cam_grad.copy_(self.out["cam_grad"], **nb)
        torch.cuda.current_stream().synchronize()
        return self.h_image, {"d_pos": self.h_d_pos, "d_rad": self.h_d_rad, "d_opa": self.h_d_opa,
                              "d_feat": self.h_d_feat, "pixel_count": self.h_count, "cam_grad": self.h_cam_grad}

    def bytes_per_step(self, views: int):
        m, d, w, h = self.m, self.d, self.w, self.h
        h2d = 4 * (m * (5 + d) + d) + views * 4 * h * w * d
        d2h = views * 4 * h * w * d + 4 * (m * (5 + d) + m) + 16 * 8
        return h2d, d2h
