"""Host-buffer session: the reference-facing call for users whose scene lives in host memory
(as the reference's NumPy columns do).  Pinned staging buffers are allocated once; every
render_step copies the inputs host->device, runs ss_forward / ss_backward, and copies the image
and all gradients device->host.  This is the path bench.py times as `e2e`.

Transfers are packed: the five scene columns travel as ONE pinned block / one H2D copy, all
gradients (+ pixel counts + the camera block) as ONE block / one D2H copy, and the image
download runs on a second stream so that it overlaps the upstream upload (the two PCIe
directions) and the start of the backward pass."""
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
        f32 = torch.float32

        # ---- inputs: one block of floats [pos 3m | rad m | opa m | feat m*d | bg d]
        n_in = m * (5 + d) + d
        self.h_in = torch.empty(n_in, dtype=f32).pin_memory()
        self.d_in = torch.empty(n_in, dtype=f32, device=dev)

        def carve_in(t):
            o = 0
            out = []
            for n, shape in ((3 * m, (m, 3)), (m, (m,)), (m, (m,)), (m * d, (m, d)), (d, (d,))):
                out.append(t[o:o + n].view(shape))
                o += n
            return out

        self.h_pos, self.h_rad, self.h_opa, self.h_feat, self.h_bg = carve_in(self.h_in)
        self.pos, self.rad, self.opa, self.feat, self.bg = carve_in(self.d_in)
        self.h_upstream = torch.empty((h, w, d), dtype=f32).pin_memory()
        self.upstream = torch.empty((h, w, d), dtype=f32, device=dev)
        self.h_image = torch.empty((h, w, d), dtype=f32).pin_memory()

        # ---- outputs: one block of 4-byte words [d_pos 3m | d_rad m | d_opa m | d_feat m*d | count m | cam 32]
        n_out = m * (6 + d) + 32
        n_out += n_out % 2  # keep the float64 camera block 8-byte aligned
        cam_off = n_out - 32
        self.h_out = torch.empty(n_out, dtype=f32).pin_memory()
        self.d_out = torch.empty(n_out, dtype=f32, device=dev)

        def carve_out(t):
            o = 0
            res = {}
            for name, n, shape in (("d_pos", 3 * m, (m, 3)), ("d_rad", m, (m,)), ("d_opa", m, (m,)),
                                   ("d_feat", m * d, (m, d))):
                res[name] = t[o:o + n].view(shape)
                o += n
            res["pixel_count"] = t[o:o + m].view(torch.int32)
            res["cam_grad"] = t[cam_off:cam_off + 32].view(torch.float64)
            return res

        self.out = carve_out(self.d_out)
        self.h_grads = carve_out(self.h_out)
        self.copy_stream = torch.cuda.Stream(device=dev)
        self.h2d_bytes = 4 * (n_in + h * w * d)
        self.d2h_bytes = 4 * (h * w * d + n_out)

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
        optional reduce_fn(out) (the multi-GPU allreduce); D2H all gradients.  Returns after the
        streams are synchronised, with the last image and the gradient views (pinned host tensors)."""
        if not isinstance(cams, (list, tuple)):
            cams = [cams]
        main = torch.cuda.current_stream(self.engine.device)
        self.d_in.copy_(self.h_in, non_blocking=True)
        for i, cam in enumerate(cams):
            if upstream_fn is None:  # upstream already staged on the host: upload it under the forward pass
                self.copy_stream.wait_stream(main)  # (orders it after the previous view's backward)
                with torch.cuda.stream(self.copy_stream):
                    self.upstream.copy_(self.h_upstream, non_blocking=True)
            f = self.engine.forward(self.pos, self.rad, self.opa, self.feat, self.bg, cam, gamma=gamma, eps=eps,
                                    tau=tau, top_k=self.k, check=check)
            image = f["image"]
            if upstream_fn is None:
                main.wait_stream(self.copy_stream)  # backward needs the uploaded upstream
            self.copy_stream.wait_stream(main)
            with torch.cuda.stream(self.copy_stream):  # image download overlaps the backward pass
                self.h_image.copy_(image, non_blocking=True)
                image.record_stream(self.copy_stream)
            if upstream_fn is not None:
                self.copy_stream.synchronize()
                self.h_upstream.copy_(upstream_fn(i, self.h_image))
                self.upstream.copy_(self.h_upstream, non_blocking=True)
            self.engine.backward(self.pos, self.rad, self.opa, self.feat, self.bg, cam, f, self.upstream,
                                 gamma=gamma, eps=eps, normalize=normalize, gate=gate, camera_grads=True,
                                 out=self.out, accumulate=(i > 0))
        if reduce_fn is not None:
            reduce_fn(self.out)
        self.h_out.copy_(self.d_out, non_blocking=True)
        main.synchronize()
        self.copy_stream.synchronize()
        return self.h_image, self.h_grads

    def bytes_per_step(self, views: int):
        m, d, w, h = self.m, self.d, self.w, self.h
        h2d = 4 * (m * (5 + d) + d) + views * 4 * h * w * d
        d2h = views * 4 * h * w * d + 4 * self.h_out.numel()
        return h2d, d2h
