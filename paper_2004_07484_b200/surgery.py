"""scene surgery on the device (reference softsphere/optim.py:161-213).

  prune(scene, visibility, config) -> (scene', keep_mask)     optim.py:161-183 (reference signature)
  subdivide(scene, config) -> scene'                          optim.py:186-213 (reference signature)
  prune_device / subdivide_device                             the same on device tensors, no host round trip;
                                                              DeviceFit.prune / DeviceFit.subdivide use them
                                                              (optim.py:345-367: moments are compacted with the
                                                              scene on prune and reset on subdivide)

The mask, the stream compaction and the x12 expansion run in csrc/ss_scene.cu through the C ABI; there
is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .engine import _ptr, _raise_for, default_engine
from .types import SphereScene, ValidationError


def _stream(dev):
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _check(rc):
    if rc != _lib.SS_OK:
        _raise_for(rc)


def prune_mask_device(opa, feat, bg, visibility, opacity_min: float, background_dist: float) -> torch.Tensor:
    """uint8 keep mask (M) on the device."""
    lib = _lib.load()
    m, d = int(opa.shape[0]), int(feat.shape[1])
    keep = torch.empty(m, dtype=torch.uint8, device=opa.device)
    _check(lib.ss_prune_mask(_ptr(opa), _ptr(feat), _ptr(bg), _ptr(visibility), m, d, float(opacity_min),
                             float(background_dist), _ptr(keep), _stream(opa.device)))
    return keep


def compact_device(keep: torch.Tensor, columns):
    """Stable compaction of per-sphere device tensors (any trailing shape, 4-byte dtypes) by `keep`.
    Returns (list of compacted tensors, count).  One host sync to read the count."""
    lib = _lib.load()
    m = int(keep.shape[0])
    dev = keep.device
    columns = [c.contiguous() for c in columns]
    if len(columns) > 16:
        raise ValidationError("at most 16 columns per compaction")
    outs = [torch.empty_like(c) for c in columns]
    arr = (_lib.SsColumn * max(len(columns), 1))()
    for i, (c, o) in enumerate(zip(columns, outs)):
        if c.shape[0] != m or c.element_size() != 4:
            raise ValidationError("compaction columns need M rows of 4-byte elements")
        arr[i].src, arr[i].dst = c.data_ptr(), o.data_ptr()
        arr[i].row_bytes = (c.numel() // max(m, 1)) * 4 if m else 4
    nb = C.c_size_t()
    _check(lib.ss_compact_workspace_bytes(m, C.byref(nb)))
    ws = torch.empty(max(nb.value, 256), dtype=torch.uint8, device=dev)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    _check(lib.ss_compact_rows(_ptr(keep), m, arr, len(columns), _ptr(ws), ws.numel(), _ptr(count), _stream(dev)))
    n = int(count.item())
    return [o[:n] for o in outs], n


def prune_device(pos, rad, opa, feat, bg, visibility, opacity_min, background_dist, extra=()):
    """(pos', rad', opa', feat', extra', keep): `extra` are further per-sphere tensors (Adam moments)."""
    keep = prune_mask_device(opa, feat, bg, visibility, opacity_min, background_dist)
    cols, n = compact_device(keep, [pos, rad, opa, feat, *extra])
    return cols[0], cols[1], cols[2], cols[3], cols[4:], keep


def subdivide_device(pos, rad, opa, feat, scale: float):
    lib = _lib.load()
    m, d = int(pos.shape[0]), int(feat.shape[1])
    dev = pos.device
    po = torch.empty((12 * m, 3), dtype=torch.float32, device=dev)
    ro = torch.empty(12 * m, dtype=torch.float32, device=dev)
    oo = torch.empty(12 * m, dtype=torch.float32, device=dev)
    fo = torch.empty((12 * m, d), dtype=torch.float32, device=dev)
    _check(lib.ss_subdivide(_ptr(pos.contiguous()), _ptr(rad.contiguous()), _ptr(opa.contiguous()),
                            _ptr(feat.contiguous()), m, d, float(scale), _ptr(po), _ptr(ro), _ptr(oo), _ptr(fo),
                            _stream(dev)))
    return po, ro, oo, fo


def _upload(scene: SphereScene, dev):
    f32 = lambda a, shape: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).reshape(shape).to(dev)
    d = scene.feature_dim
    return (f32(scene.positions, (-1, 3)), f32(scene.radii, (-1,)), f32(scene.opacities, (-1,)),
            f32(scene.features, (-1, d)), f32(scene.background, (d,)))


def _download(d, bg, pos, rad, opa, feat) -> SphereScene:
    f64 = lambda t: t.cpu().numpy().astype(np.float64)
    return SphereScene(feature_dim=d, background=np.array(bg, dtype=np.float64), positions=f64(pos),
                       radii=f64(rad), opacities=f64(opa), features=f64(feat))


def prune(scene: SphereScene, visibility, config, device="cuda"):
    """Reference signature (optim.py:161): returns (scene', keep_mask)."""
    dev = default_engine(device).device
    vis_np = np.asarray(visibility).reshape(len(scene))
    pos, rad, opa, feat, bg = _upload(scene, dev)
    vis = torch.from_numpy(np.clip(vis_np, 0, np.iinfo(np.int32).max).astype(np.int32)).to(dev)
    pos, rad, opa, feat, _, keep = prune_device(pos, rad, opa, feat, bg, vis, config.prune_opacity_min,
                                                config.prune_background_dist)
    return _download(scene.feature_dim, scene.background, pos, rad, opa, feat), keep.cpu().numpy().astype(bool)


def subdivide(scene: SphereScene, config, device="cuda") -> SphereScene:
    """Reference signature (optim.py:197)."""
    dev = default_engine(device).device
    pos, rad, opa, feat, _ = _upload(scene, dev)
    out = subdivide_device(pos, rad, opa, feat, config.subdivide_scale)
    return _download(scene.feature_dim, scene.background, *out)
