"""View-sharded multi-GPU rendering: one process per GPU, views dealt round-robin to ranks, the
scene replicated, per-view gradients accumulated locally (normalisation and gating are per
view, before the sum -- the reference divides by the per-view pixel_count inside
render_backward, grad.py:273-286), then ONE sum-allreduce of the concatenated sphere-gradient
buffer (+ the int32 pixel counts) over NCCL/NVLink per step.  Camera gradients are per view
and are not reduced.

The reference has no multi-view call (optim.py:280-304 renders one view per step); the oracle
for this module is "sum over views of single-view render_backward".
"""
from __future__ import annotations

from typing import Callable, Dict, List, Optional, Sequence

import torch
import torch.distributed as dist


def shard_views(num_views: int, world_size: int, rank: int) -> List[int]:
    """View v is rendered by rank v mod world_size."""
    if not (0 <= rank < world_size):
        raise ValueError(f"rank {rank} outside world of size {world_size}")
    return list(range(rank, num_views, world_size))


class SphereGradBuffer:
    """Per-sphere gradients in ONE flat float32 tensor (so a single allreduce moves them) plus
    the int32 pixel counts.  Layout: d_pos (M,3) | d_rad (M) | d_opa (M) | d_feat (M,d)."""

    def __init__(self, num_spheres: int, feature_dim: int, device):
        m, d = int(num_spheres), int(feature_dim)
        self.m, self.d = m, d
        self.flat = torch.zeros(m * (5 + d), dtype=torch.float32, device=device)
        self.pixel_count = torch.zeros(m, dtype=torch.int32, device=device)
        self.d_pos = self.flat[: 3 * m].view(m, 3)
        self.d_rad = self.flat[3 * m: 4 * m]
        self.d_opa = self.flat[4 * m: 5 * m]
        self.d_feat = self.flat[5 * m:].view(m, d)

    def zero_(self):
        self.flat.zero_()
        self.pixel_count.zero_()

    def as_out(self) -> Dict[str, torch.Tensor]:
        return {"d_pos": self.d_pos, "d_rad": self.d_rad, "d_opa": self.d_opa, "d_feat": self.d_feat,
                "pixel_count": self.pixel_count}

    def allreduce_bytes(self) -> int:
        return self.flat.numel() * 4 + self.pixel_count.numel() * 4


class ViewShardedRenderer:
    """engine: object with forward(pos, rad, opa, feat, bg, cam, **blend) -> dict and
    backward(pos, rad, opa, feat, bg, cam, buf, upstream, gamma=, eps=, normalize=, gate=,
    camera_grads=, out=, accumulate=) -> dict  (RenderEngine, or a stand-in in CPU tests)."""

    def __init__(self, engine, group: Optional[dist.ProcessGroup] = None):
        self.engine = engine
        self.group = group
        self.distributed = dist.is_available() and dist.is_initialized()
        self.world_size = dist.get_world_size(group) if self.distributed else 1
        self.rank = dist.get_rank(group) if self.distributed else 0

    def local_views(self, num_views: int) -> List[int]:
        return shard_views(num_views, self.world_size, self.rank)

    def step(self, scene, cameras: Sequence, upstream_fn: Callable, grads: SphereGradBuffer, gamma=0.1,
             eps=1e-2, tau=0.01, top_k=5, normalize=True, gate=True, camera_grads=True, check=False):
        """One multi-view step.  scene = (pos, rad, opa, feat, bg) device tensors; cameras = the
        CameraSpec of EVERY view (all ranks hold the list); upstream_fn(view, image) -> dL/dimage.
        Fills `grads` with the sum over ALL views (after the allreduce) and returns
        {view: cam_grad tensor} for the local views."""
        pos, rad, opa, feat, bg = scene
        cam_out = {}
        out = grads.as_out()
        local = self.local_views(len(cameras))
        if not local:
            grads.zero_()
        for i, v in enumerate(local):
            cam = cameras[v]
            f = self.engine.forward(pos, rad, opa, feat, bg, cam, gamma=gamma, eps=eps, tau=tau, top_k=top_k,
                                    check=check)
            up = upstream_fn(v, f["image"])
            o = dict(out)
            res = self.engine.backward(pos, rad, opa, feat, bg, cam, f, up, gamma=gamma, eps=eps,
                                       normalize=normalize, gate=gate, camera_grads=camera_grads, out=o,
                                       accumulate=(i > 0))  # the first local view overwrites: no zero fill
            if camera_grads:
                cam_out[v] = res["cam_grad"]
        if self.world_size > 1:
            # one NCCL group: float sphere gradients + int pixel counts
            h1 = dist.all_reduce(grads.flat, op=dist.ReduceOp.SUM, group=self.group, async_op=True)
            h2 = dist.all_reduce(grads.pixel_count, op=dist.ReduceOp.SUM, group=self.group, async_op=True)
            h1.wait()
            h2.wait()
        return cam_out
