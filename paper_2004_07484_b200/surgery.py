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


def _f64(a, shape, dev):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).reshape(shape).to(dev)


def prune(scene: SphereScene, visibility, config, device="cuda"):
    """Reference signature (optim.py:161): returns (scene', keep_mask).  The mask is decided on the device from
    the scene's own float64 values (k_prune_flags<double>); the survivors are exact float64 copies like the
    reference's `scene.positions[keep]` (optim.py:176-181)."""
    lib = _lib.load()
    dev = default_engine(device).device
    m, d = len(scene), int(scene.feature_dim)
    vis_np = np.asarray(visibility).reshape(m)
    keep_t = torch.empty(max(m, 1), dtype=torch.uint8, device=dev)
    if m:
        with torch.cuda.device(dev):
            opa, feat, bg = _f64(scene.opacities, (-1,), dev), _f64(scene.features, (-1, d), dev), _f64(scene.background, (d,), dev)
            vis = torch.from_numpy(np.clip(vis_np, 0, np.iinfo(np.int32).max).astype(np.int32)).to(dev)
            _check(lib.ss_prune_mask_f64(_ptr(opa), _ptr(feat), _ptr(bg), _ptr(vis), m, d,
                                         float(config.prune_opacity_min), float(config.prune_background_dist),
                                         _ptr(keep_t), _stream(dev)))
    keep = keep_t[:m].cpu().numpy().astype(bool)
    out = SphereScene(feature_dim=d, background=np.array(scene.background, dtype=np.float64),
                      positions=np.asarray(scene.positions)[keep], radii=np.asarray(scene.radii)[keep],
                      opacities=np.asarray(scene.opacities)[keep], features=np.asarray(scene.features)[keep])
    return out, keep


def subdivide(scene: SphereScene, config, device="cuda") -> SphereScene:
    """Reference signature (optim.py:197); float64 columns in and out (k_subdivide<double>)."""
    lib = _lib.load()
    dev = default_engine(device).device
    m, d = len(scene), int(scene.feature_dim)
    with torch.cuda.device(dev):
        pos, rad = _f64(scene.positions, (-1, 3), dev), _f64(scene.radii, (-1,), dev)
        opa, feat = _f64(scene.opacities, (-1,), dev), _f64(scene.features, (-1, d), dev)
        f64 = dict(dtype=torch.float64, device=dev)
        po, ro, oo = torch.empty((12 * m, 3), **f64), torch.empty(12 * m, **f64), torch.empty(12 * m, **f64)
        fo = torch.empty((12 * m, d), **f64)
        _check(lib.ss_subdivide_f64(_ptr(pos), _ptr(rad), _ptr(opa), _ptr(feat), m, d, float(config.subdivide_scale),
                                    _ptr(po), _ptr(ro), _ptr(oo), _ptr(fo), _stream(dev)))
    return SphereScene(feature_dim=d, background=np.array(scene.background, dtype=np.float64),
                       positions=po.cpu().numpy(), radii=ro.cpu().numpy(), opacities=oo.cpu().numpy(),
                       features=fo.cpu().numpy())
