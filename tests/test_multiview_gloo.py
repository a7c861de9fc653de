"""CPU, world_size 2, gloo: the view-sharding + allreduce host logic.  The per-view renderer is
a stand-in backed by the CPU oracle (tests may use the oracle; the product engine needs a GPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import make_random_scene
from oracle import oracle as orc
from paper_2004_07484_b200.multiview import SphereGradBuffer, ViewShardedRenderer, shard_views


class OracleEngine:
    """Same dict interface as RenderEngine, float64 oracle inside (test stand-in only)."""

    def forward(self, pos, rad, opa, feat, bg, cam, gamma, eps, tau, top_k, check=False):
        f = orc.render_forward(pos.numpy(), rad.numpy(), opa.numpy(), feat.numpy(), bg.numpy(), cam,
                               gamma=gamma, eps=eps, tau=tau, top_k=top_k)
        f["image"] = torch.from_numpy(f["image"])
        return f

    def backward(self, pos, rad, opa, feat, bg, cam, buf, upstream, gamma, eps, normalize, gate, camera_grads,
                 out, accumulate):
        g = orc.render_backward(pos.numpy(), rad.numpy(), opa.numpy(), feat.numpy(), bg.numpy(), cam, buf,
                                upstream.numpy().astype(np.float64), normalize=normalize, gate=gate)
        if not accumulate:
            for k in ("d_pos", "d_rad", "d_opa", "d_feat", "pixel_count"):
                out[k].zero_()
        out["d_pos"] += torch.from_numpy(g["d_position"]).float()
        out["d_rad"] += torch.from_numpy(g["d_radius"]).float()
        out["d_opa"] += torch.from_numpy(g["d_opacity"]).float()
        out["d_feat"] += torch.from_numpy(g["d_feature"]).float()
        out["pixel_count"] += torch.from_numpy(g["pixel_count"]).int()
        out["cam_grad"] = torch.from_numpy(np.concatenate([g["d_translation"], g["grad_rot_matrix"].ravel(),
                                                           [g["d_focal"], g["d_sensor_width"], 0, 0]]))
        return out


def _scene_and_cameras(num_views=5):
    rng = np.random.default_rng(5)
    pos, rad, opa, feat, bg = make_random_scene(rng, 60)
    cams = []
    for v in range(num_views):
        th = 2 * np.pi * v / num_views
        vec = [0.3 * np.cos(th), 0.3 * np.sin(th), 0, 0, 0.02 * np.sin(th), 0, 5.0, 2.0]
        cams.append(orc.camera_from_vector(vec, 32, 32))
    scene = tuple(torch.from_numpy(x) for x in (pos, rad, opa, feat, bg))
    return scene, cams


def _upstream(v, image):
    return torch.sign(image - 0.5) * (1.0 + 0.1 * v)


def _worker(rank, world, port, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        scene, cams = _scene_and_cameras()
        r = ViewShardedRenderer(OracleEngine())
        assert r.world_size == world and r.rank == rank
        grads = SphereGradBuffer(scene[0].shape[0], 3, "cpu")
        cam_out = r.step(scene, cams, _upstream, grads, gamma=0.1, tau=0.0)
        ret[rank] = (grads.flat.clone(), grads.pixel_count.clone(), sorted(cam_out.keys()))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_views_partition():
    for world in (1, 2, 3, 8):
        seen = sorted(v for r in range(world) for v in shard_views(64, world, r))
        assert seen == list(range(64))
    assert shard_views(5, 2, 0) == [0, 2, 4] and shard_views(5, 2, 1) == [1, 3]
    with pytest.raises(ValueError):
        shard_views(4, 2, 2)


def test_grad_buffer_views_alias_one_flat_tensor():
    g = SphereGradBuffer(7, 3, "cpu")
    g.d_pos[2, 1] = 5.0
    g.d_feat[6, 2] = 3.0
    assert g.flat[2 * 3 + 1] == 5.0 and g.flat[-1] == 3.0
    assert g.flat.numel() == 7 * 8 and g.allreduce_bytes() == 7 * 8 * 4 + 7 * 4


def test_two_rank_step_equals_sum_over_views():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(world, port, ret), nprocs=world, join=True)
    # single-process reference: sum over all views
    scene, cams = _scene_and_cameras()
    grads = SphereGradBuffer(scene[0].shape[0], 3, "cpu")
    ViewShardedRenderer(OracleEngine()).step(scene, cams, _upstream, grads, gamma=0.1, tau=0.0)
    for rank in range(world):
        flat, cnt, views = ret[rank]
        assert torch.allclose(flat, grads.flat, rtol=1e-5, atol=1e-7)
        assert torch.equal(cnt, grads.pixel_count)
        assert views == shard_views(len(cams), world, rank)
    assert grads.pixel_count.sum() > 0 and grads.flat.abs().sum() > 0


def _worker_overlap(rank, world, port, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        scene, cams = _scene_and_cameras()
        r = ViewShardedRenderer(OracleEngine())
        grads = SphereGradBuffer(scene[0].shape[0], 3, "cpu")
        # two steps with the reduction left in flight: the second step must wait for the first one's
        # allreduce before its first backward overwrites the buffer, finish() before the buffer is read
        r.step(scene, cams, _upstream, grads, gamma=0.1, tau=0.0, overlap=True)
        assert r._pending is not None
        r.step(scene, cams, _upstream, grads, gamma=0.1, tau=0.0, overlap=True)
        r.finish()
        assert r._pending is None
        ret[rank] = (grads.flat.clone(), grads.pixel_count.clone(), r.collectives_issued)
    finally:
        dist.destroy_process_group()


def test_deferred_allreduce_gives_the_same_sums():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker_overlap, args=(world, port, ret), nprocs=world, join=True)
    scene, cams = _scene_and_cameras()
    grads = SphereGradBuffer(scene[0].shape[0], 3, "cpu")
    ViewShardedRenderer(OracleEngine()).step(scene, cams, _upstream, grads, gamma=0.1, tau=0.0)
    for rank in range(world):
        flat, cnt, n_coll = ret[rank]
        assert torch.allclose(flat, grads.flat, rtol=1e-5, atol=1e-7) and torch.equal(cnt, grads.pixel_count)
        assert n_coll == 4  # gloo: two reductions per step (NCCL: one coalesced group per step)
