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
        self.backend = dist.get_backend(group) if self.distributed else None
        self._pending = None  # work handle of a deferred allreduce (overlap=True)
        self.collectives_issued = 0  # collective launches so far (one per step on NCCL)
        self._twin = None  # second engine + the two side streams of the pipelined view loop
        self._streams = None
        self._graphs = {}  # captured local steps (graphed_step), newest last; a handful is kept
        self._graph = None  # the most recently used one

    def _pipeline(self):
        """Two engines (workspaces) on two side streams, or None when the engine is a stand-in (CPU tests)."""
        from .engine import RenderEngine
        e = self.engine
        if not isinstance(e, RenderEngine) or e.device.type != "cuda":
            return None
        if self._twin is None:
            self._twin = RenderEngine(e.device, pair_factor=e.pair_factor, min_pairs=e.min_pairs)
            self._streams = [torch.cuda.Stream(device=e.device), torch.cuda.Stream(device=e.device)]
        return [e, self._twin], self._streams

    def local_views(self, num_views: int) -> List[int]:
        return shard_views(num_views, self.world_size, self.rank)

    def finish(self):
        """Wait (stream-ordered, not a host sync on NCCL) for a deferred allreduce before `grads` is read."""
        if self._pending is not None:
            self._pending.wait()
            self._pending = None

    def _allreduce(self, grads: SphereGradBuffer):
        """ONE collective per step: the float32 gradient block and the int32 pixel counts travel in one NCCL
        group (a single fused launch on the communicator's stream, ordered after the last local k_finalize by
        the usual event; the pixel counts cannot ride in the float buffer, their sums exceed 2^24).  Backends
        without coalescing (gloo in the CPU tests) issue the two reductions back to back."""
        if self.backend == "nccl":
            try:
                with dist._coalescing_manager(group=self.group, async_ops=True) as cm:
                    dist.all_reduce(grads.flat, op=dist.ReduceOp.SUM, group=self.group)
                    dist.all_reduce(grads.pixel_count, op=dist.ReduceOp.SUM, group=self.group)
                self.collectives_issued += 1
                return cm
            except Exception:  # the (private) coalescing API moved or refused the group: two plain collectives
                self.backend = "nccl (uncoalesced)"
        h1 = dist.all_reduce(grads.flat, op=dist.ReduceOp.SUM, group=self.group, async_op=True)
        h2 = dist.all_reduce(grads.pixel_count, op=dist.ReduceOp.SUM, group=self.group, async_op=True)
        self.collectives_issued += 2

        class _Both:
            def wait(self_inner):
                h1.wait()
                h2.wait()
        return _Both()

    def step(self, scene, cameras: Sequence, upstream_fn: Callable, grads: SphereGradBuffer, gamma=0.1,
             eps=1e-2, tau=0.01, top_k=5, normalize=True, gate=True, camera_grads=True, check=False,
             overlap=False, pipeline=True, _local_only=False):
        """One multi-view step.  scene = (pos, rad, opa, feat, bg) device tensors; cameras = the
        CameraSpec of EVERY view (all ranks hold the list); upstream_fn(view, image) -> dL/dimage.
        Fills `grads` with the sum over ALL views (after the allreduce) and returns
        {view: cam_grad tensor} for the local views.  overlap=True leaves the allreduce in flight (call
        finish() before reading `grads`): the next step's first forward pass then runs under it, and the
        next step waits for it before its first backward overwrites the buffer.

        pipeline=True (real engines, more than one local view): consecutive views alternate between two engines
        (workspaces) on two side streams, so the forward pass of view i + 1 runs while the backward pass of view i
        is still going; the backward passes themselves stay in view order (k_finalize adds into the shared buffers
        without atomics).  The kernels of one view leave issue slots and tails idle that the other view's kernels
        fill: +9 % frames/s at 32 views of C3 on one B200 (`scripts/two_stream_probe.py`).  The caller's stream
        waits for both side streams before the step returns."""
        pos, rad, opa, feat, bg = scene
        cam_out = {}
        out = grads.as_out()
        local = self.local_views(len(cameras))
        if not local:
            self.finish()
            grads.zero_()
        pipe = self._pipeline() if (pipeline and len(local) > 1) else None
        if pipe is not None:
            engines, streams = pipe
            main = torch.cuda.current_stream(self.engine.device)
            for st in streams:
                st.wait_stream(main)  # the scene (and whatever else the caller enqueued) is ready
            backward_done = None
            for i, v in enumerate(local):
                cam, eng, st = cameras[v], engines[i & 1], streams[i & 1]
                with torch.cuda.stream(st):
                    f = eng.forward(pos, rad, opa, feat, bg, cam, gamma=gamma, eps=eps, tau=tau, top_k=top_k,
                                    check=check)
                    up = upstream_fn(v, f["image"])
                    if i == 0:
                        self.finish()  # the previous step's reduction must be done before this buffer is overwritten
                    else:
                        st.wait_event(backward_done)  # k_finalize of the previous view has added its share
                    res = eng.backward(pos, rad, opa, feat, bg, cam, f, up, gamma=gamma, eps=eps, normalize=normalize,
                                       gate=gate, camera_grads=camera_grads, out=dict(out), accumulate=(i > 0))
                    backward_done = torch.cuda.Event()
                    backward_done.record(st)
                    if camera_grads:
                        res["cam_grad"].record_stream(main)
                        cam_out[v] = res["cam_grad"]
            for st in streams:
                main.wait_stream(st)
            local = []  # (done)
        for i, v in enumerate(local):
            cam = cameras[v]
            f = self.engine.forward(pos, rad, opa, feat, bg, cam, gamma=gamma, eps=eps, tau=tau, top_k=top_k,
                                    check=check)
            up = upstream_fn(v, f["image"])
            if i == 0:
                self.finish()  # the previous step's reduction must be done before this buffer is overwritten
            o = dict(out)
            res = self.engine.backward(pos, rad, opa, feat, bg, cam, f, up, gamma=gamma, eps=eps,
                                       normalize=normalize, gate=gate, camera_grads=camera_grads, out=o,
                                       accumulate=(i > 0))  # the first local view overwrites: no zero fill
            if camera_grads:
                cam_out[v] = res["cam_grad"]
        if self.world_size > 1 and not _local_only:
            self._pending = self._allreduce(grads)
            if not overlap:
                self.finish()
        return cam_out

    def graphed_step(self, scene, cameras: Sequence, upstream_fn: Callable, grads: SphereGradBuffer, overlap=False,
                     **params):
        """`step` with the local work of the step -- every kernel of every local view, on both pipeline streams, plus
        whatever `upstream_fn` enqueues -- captured ONCE into a CUDA graph and replayed afterwards.  The usual
        training loop renders a fixed set of cameras while the optimiser updates the scene tensors in place: the
        launch sequence never changes, and a replay removes the launch gaps between the ~10 kernels of a view
        (C1: 0.17 -> 0.04 ms per frame, C2: 0.15 -> 0.11 ms, C3: 0.496 -> 0.473 ms, `scripts/graph_probe.py`).

        The graph bakes in the tensors' addresses, the cameras and the blend parameters: it is re-captured when any
        of those changes (scene tensors replaced rather than updated in place, another camera list, other
        `params`, another `upstream_fn` OBJECT -- pass the same function every step, a fresh lambda per call means a
        fresh capture per call; the last four captures are kept, so a loop may alternate between a few of them).  `upstream_fn` must be capturable (device work on the current stream, no host
        synchronisation) and must depend on its arguments only.  check=True is not available (no host read inside a graph): poll
        `engine.read_status()` yourself.  The collective of a multi-GPU step stays outside the graph."""
        if params.get("check"):
            raise ValueError("graphed_step cannot read the status block back (check=True): use step()")
        params = dict(params, check=False)
        key = (tuple((t.data_ptr(), tuple(t.shape)) for t in scene), tuple(id(c) for c in cameras), id(upstream_fn),
               grads.flat.data_ptr(), tuple(sorted(params.items())))
        g = self._graphs.get(key)
        if g is None:
            self.finish()
            dev = self.engine.device
            side = torch.cuda.Stream(device=dev)
            side.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(side):  # warm-up outside the capture: workspaces, twin engine, function attributes
                for _ in range(2):
                    self.step(scene, cameras, upstream_fn, grads, _local_only=True, **params)
            torch.cuda.current_stream(dev).wait_stream(side)
            torch.cuda.synchronize(dev)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                cam_out = self.step(scene, cameras, upstream_fn, grads, _local_only=True, **params)
            g = {"key": key, "graph": graph, "cam_out": cam_out,
                 "keepalive": (scene, list(cameras), upstream_fn, grads)}
            while len(self._graphs) >= 4:  # a loop that alternates between a few camera sets keeps its captures
                self._graphs.pop(next(iter(self._graphs)))
            self._graphs[key] = g
        self._graph = g
        self.finish()  # a deferred reduction of the previous step must be done before the buffers are overwritten
        g["graph"].replay()
        if self.world_size > 1:
            self._pending = self._allreduce(grads)
            if not overlap:
                self.finish()
        return g["cam_out"]
