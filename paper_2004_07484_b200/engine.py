"""Device-side driver of the C-ABI hot path: owns the workspace, fills the POD argument structs
and enqueues ss_forward / ss_backward on the current CUDA stream.

PyTorch is used for device memory and streams only; every kernel that runs is one of this
repo's sm_100a kernels inside libss_b200.so (no eager/PyTorch fallback exists).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from .types import (ORTHOGRAPHIC, PINHOLE, ConfigurationError, ContractViolation, SoftSphereError,
                    ValidationError)


@dataclass
class CameraSpec:
    """Plain-number camera handed to the ABI (SsCamera)."""
    t: np.ndarray          # (3,)
    R: np.ndarray          # (3,3) row-major, p_cam = R (p - t)
    focal: float
    sensor_w: float
    width: int
    height: int
    near: float = 0.1
    far: float = 45.0
    mode: str = PINHOLE

    @staticmethod
    def from_camera(cam) -> "CameraSpec":
        """Accepts this package's Camera or the reference's (same attribute names)."""
        return CameraSpec(np.asarray(cam.translation, np.float64), np.asarray(cam.rotation, np.float64),
                          float(cam.focal_length), float(cam.sensor_width), int(cam.width),
                          int(cam.height), float(cam.near), float(cam.far), cam.mode)

    def to_c(self) -> _lib.SsCamera:
        c = _lib.SsCamera()
        c.t[:] = [float(x) for x in np.asarray(self.t).reshape(3)]
        c.R[:] = [float(x) for x in np.asarray(self.R).reshape(9)]
        c.focal, c.sensor_w = float(self.focal), float(self.sensor_w)
        c.near_, c.far_ = float(self.near), float(self.far)
        c.width, c.height = int(self.width), int(self.height)
        if self.mode == PINHOLE:
            c.mode = _lib.MODE_PINHOLE
        elif self.mode == ORTHOGRAPHIC:
            c.mode = _lib.MODE_ORTHOGRAPHIC
        else:
            raise ConfigurationError(f"unknown camera mode {self.mode!r}")
        return c


def _raise_for(code: int):
    msg = _lib.status_string(code)
    if code in (_lib.SS_ERR_DIMS, _lib.SS_ERR_CAMERA, _lib.SS_ERR_UNSUPPORTED):
        raise ConfigurationError(msg)
    if code == _lib.SS_ERR_PARAMS:
        raise ValidationError(msg)
    raise SoftSphereError(msg)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _dev_f32(x, device, shape=None) -> torch.Tensor:
    if not isinstance(x, torch.Tensor):
        x = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float32)))
    x = x.to(device=device, dtype=torch.float32, non_blocking=True).contiguous()
    if shape is not None:
        x = x.reshape(shape)
    return x


class RenderEngine:
    """One workspace + launch helper per device.  Not thread-safe per instance (like one
    reference call at a time); use one engine per stream."""

    def __init__(self, device="cuda", pair_factor: float = 4.0, min_pairs: int = 1 << 16):
        if not torch.cuda.is_available():
            raise _lib.NativeLibraryError("CUDA device required: the render path has no CPU fallback")
        self.lib = _lib.load()
        self.device = torch.device(device)
        if self.device.type != "cuda":
            raise _lib.NativeLibraryError("RenderEngine needs a CUDA device")
        self.pair_factor = float(pair_factor)
        self.min_pairs = int(min_pairs)
        self._ws: Optional[torch.Tensor] = None
        self._ws_dims = None
        self._pair_capacity = 0
        # Record reuse (SS_OPT_REUSE_RECORDS): the workspace holds the draw records of exactly one forward call.
        # Every forward gets a token; backward skips re-projection only for the buffer that carries the token of
        # the workspace's LAST forward, and only while that call's input tensors (kept alive here, so their
        # addresses cannot be recycled) are the ones handed to backward, unmodified (torch version counters).
        self._fwd_seq = 0
        self._last_fwd = None
        self._det_ws: Optional[torch.Tensor] = None  # scratch of the deterministic backward

    # -- workspace -------------------------------------------------------------------
    def _dims(self, m, d, w, h, k, max_pairs) -> _lib.SsDims:
        return _lib.SsDims(int(m), int(max_pairs), int(d), int(w), int(h), int(k))

    def _ensure_workspace(self, m, d, w, h, k, need_pairs=None):
        n_tiles = ((w + 15) // 16) * ((h + 15) // 16)
        # baseline: 4 pairs per sphere, and room for a few dozen image-filling spheres (64 pairs per tile)
        cap = max(self._pair_capacity, self.min_pairs, int(self.pair_factor * m), 64 * n_tiles)
        if need_pairs is not None:
            cap = max(cap, int(need_pairs * 1.25) + 1024)
        key = (m, d, w, h, k, cap)
        if self._ws is not None and self._ws_dims == key:
            return self._dims(*key[:5], cap)
        dims = self._dims(m, d, w, h, k, cap)
        nbytes = C.c_size_t()
        rc = self.lib.ss_workspace_bytes(C.byref(dims), C.byref(nbytes))
        if rc != _lib.SS_OK:
            _raise_for(rc)
        if self._ws is None or self._ws.numel() < nbytes.value:
            self._ws = torch.empty(nbytes.value, dtype=torch.uint8, device=self.device)
        # a (re)laid-out workspace must not carry a stale "accumulators are clean" tag (ss_workspace_init)
        with torch.cuda.device(self.device):
            rc = self.lib.ss_workspace_init(C.byref(dims), _ptr(self._ws), self._ws.numel(), self._stream())
        if rc != _lib.SS_OK:
            _raise_for(rc)
        self._ws_dims = key
        self._pair_capacity = cap
        self._last_fwd = None
        return dims

    def invalidate_records(self):
        """Forget the last forward's draw records (call after editing scene tensors behind torch's back,
        e.g. from a raw kernel): the next backward re-projects like the reference (grad.py:213, :351)."""
        self._last_fwd = None

    @staticmethod
    def _cam_key(cam: CameraSpec):
        return (tuple(np.asarray(cam.t, np.float64).reshape(-1).tolist()),
                tuple(np.asarray(cam.R, np.float64).reshape(-1).tolist()), float(cam.focal), float(cam.sensor_w),
                int(cam.width), int(cam.height), float(cam.near), float(cam.far), cam.mode)

    def _records_current(self, buf: dict, tensors, cam: CameraSpec) -> bool:
        last = self._last_fwd
        if last is None or self._ws is None or buf.get("fwd_token") != last["token"]:
            return False
        if last["cam"] != self._cam_key(cam):
            return False
        for t, (ref, ver) in zip(tensors, last["inputs"]):
            if t is not ref and (t.data_ptr() != ref.data_ptr() or t.shape != ref.shape):
                return False
            if ref._version != ver or t._version != ver:
                return False
        return True

    def _stream(self):
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def read_status(self) -> dict:
        st = _lib.SsStatus()
        with torch.cuda.device(self.device):
            rc = self.lib.ss_read_status(_ptr(self._ws), C.byref(st), self._stream())
        if rc != _lib.SS_OK:
            _raise_for(rc)
        return {f: int(getattr(st, f)) for f, _ in _lib.SsStatus._fields_ if f != "reserved"}

    # -- forward ---------------------------------------------------------------------
    def forward(self, pos, rad, opa, feat, bg, cam: CameraSpec, gamma=0.1, eps=1e-2, tau=0.01, top_k=5,
                chunk=256, tile=16, store_buffer=True, collect_stats=False, validate=True,
                check=True, debug=False, image=None, bg_weight=None, band_events=None, after_launch=None):
        """Enqueue the forward pipeline.  Inputs: float32 CUDA tensors (or array-likes, which are
        copied to the device).  Returns a dict of CUDA tensors; with check=True the status block
        is read back (one stream sync), validation / overflow are handled and `status` is set.

        band_events: a list of torch.cuda.Event -- the image is then drawn in that many bands of tile rows
        (ss_forward_banded) and event b is recorded when the rows `band_rows(height, n, b)` are final, so that a
        copy stream can download the upper bands while the lower ones are still being drawn.  after_launch: called
        right after the kernels have been enqueued, i.e. before a check=True status read synchronises the stream
        (the place to enqueue such downloads; called again if an overflow makes the engine render a second time)."""
        dev = self.device
        bg = _dev_f32(bg, dev, (-1,))
        d = bg.shape[0]
        pos = _dev_f32(pos, dev, (-1, 3))
        m = pos.shape[0]
        rad, opa = _dev_f32(rad, dev, (-1,)), _dev_f32(opa, dev, (-1,))
        feat = _dev_f32(feat, dev, (-1, d)) if m else torch.zeros((0, d), device=dev)
        if rad.shape[0] != m or opa.shape[0] != m or feat.shape[0] != m:
            raise ValidationError("sphere column arrays have mismatched lengths")
        w, h, k = int(cam.width), int(cam.height), int(top_k)
        if store_buffer:
            ids = torch.empty((k, h, w), dtype=torch.int32, device=dev)
            z = torch.empty((k, h, w), dtype=torch.float32, device=dev)
            clos = torch.empty((k, h, w), dtype=torch.float32, device=dev)
            log_denom = torch.empty((h, w), dtype=torch.float32, device=dev)
        else:
            ids = z = clos = log_denom = None
        if image is None:
            image = torch.empty((h, w, d), dtype=torch.float32, device=dev)
        if bg_weight is None:
            bg_weight = torch.empty((h, w), dtype=torch.float32, device=dev)
        bgw = bg_weight
        for t, shape in ((image, (h, w, d)), (bgw, (h, w))):
            if tuple(t.shape) != shape or t.dtype != torch.float32 or not t.is_contiguous() or not t.is_cuda:
                raise ValidationError("caller-provided image / bg_weight must be contiguous float32 CUDA tensors "
                                      f"of shape {shape}")
        dbg = {}
        if debug:
            dbg = {"rect": torch.empty((m, 4), dtype=torch.int32, device=dev),
                   "on_sensor": torch.empty((m,), dtype=torch.uint8, device=dev),
                   "earliest": torch.empty((m,), dtype=torch.float64, device=dev),
                   "proj_radius_px": torch.empty((m,), dtype=torch.float64, device=dev)}
        flags = 0
        if store_buffer:
            flags |= _lib.OPT_STORE_BUFFER
        if collect_stats:
            flags |= _lib.OPT_COLLECT_STATS
        if not validate:
            flags |= _lib.OPT_SKIP_VALIDATE
        ccam = cam.to_c()
        need_pairs = None
        status = None
        for _attempt in range(3):
            dims = self._ensure_workspace(m, d, w, h, k, need_pairs)
            a = _lib.SsForwardArgs()
            a.dims, a.cam = dims, ccam
            a.blend = _lib.SsBlend(float(gamma), float(eps), float(tau), int(tile), int(chunk), flags, 0)
            a.pos, a.rad, a.opa, a.feat, a.bg = _ptr(pos), _ptr(rad), _ptr(opa), _ptr(feat), _ptr(bg)
            a.workspace, a.workspace_bytes = _ptr(self._ws), self._ws.numel()
            a.image, a.bg_weight = _ptr(image), _ptr(bgw)
            a.ids, a.z, a.closeness, a.log_denom = _ptr(ids), _ptr(z), _ptr(clos), _ptr(log_denom)
            a.rect, a.on_sensor = _ptr(dbg.get("rect")), _ptr(dbg.get("on_sensor"))
            a.earliest, a.proj_radius_px = _ptr(dbg.get("earliest")), _ptr(dbg.get("proj_radius_px"))
            with torch.cuda.device(dev):  # kernels launch on the current device: make it the engine's
                if band_events:
                    stream = torch.cuda.current_stream(dev)
                    for e in band_events:  # a torch event only gets its CUDA handle on first record
                        if not e.cuda_event:
                            e.record(stream)
                    evs = (C.c_void_p * len(band_events))(*[C.c_void_p(e.cuda_event) for e in band_events])
                    rc = self.lib.ss_forward_banded(C.byref(a), len(band_events), evs, self._stream())
                else:
                    rc = self.lib.ss_forward(C.byref(a), self._stream())
            if rc != _lib.SS_OK:
                _raise_for(rc)
            if after_launch is not None:
                after_launch()
            if not check:
                break
            status = self.read_status()
            if status["flags"] & _lib.FLAG_INVALID_INPUT:
                raise ValidationError(
                    f"non-finite field or non-positive radius at sphere index {status['first_invalid']}")
            if status["flags"] & _lib.FLAG_PAIR_OVERFLOW:
                need_pairs = status["num_pairs"]
                continue
            break
        else:
            raise SoftSphereError("tile-sphere pair workspace overflow persisted after regrowth")
        self._fwd_seq += 1
        token = (id(self), self._fwd_seq)
        self._last_fwd = {"token": token, "cam": self._cam_key(cam),
                          "inputs": tuple((t, t._version) for t in (pos, rad, opa))}
        out = {"image": image, "bg_weight": bgw, "ids": ids, "z": z, "closeness": clos,
               "log_denom": log_denom, "status": status, "num_spheres": m,
               "inputs": (pos, rad, opa, feat, bg), "fwd_token": token}
        out.update(dbg)
        return out

    def band_rows(self, height: int, n_bands: int, band: int):
        """(row_begin, row_end) of band `band` when an image of `height` rows is drawn in `n_bands` bands."""
        r0, r1 = C.c_int(), C.c_int()
        rc = self.lib.ss_band_rows(int(height), int(n_bands), int(band), C.byref(r0), C.byref(r1))
        if rc != _lib.SS_OK:
            _raise_for(rc)
        return r0.value, r1.value

    def tile_lists(self, m, d, w, h, k):
        """(tile_starts, sphere ids grouped by tile in scan order) of the last forward (parity)."""
        dims = self._dims(*self._ws_dims)
        ntx, nty = (w + 15) // 16, (h + 15) // 16
        starts = torch.empty(ntx * nty + 1, dtype=torch.int32, device=self.device)
        ids = torch.empty(max(int(dims.max_pairs), 1), dtype=torch.int32, device=self.device)
        rc = self.lib.ss_debug_tile_lists(C.byref(dims), _ptr(self._ws), _ptr(starts), _ptr(ids), self._stream())
        if rc != _lib.SS_OK:
            _raise_for(rc)
        starts = starts.cpu().numpy().astype(np.int64)
        return starts, ids[: int(starts[-1])].cpu().numpy()

    # -- backward --------------------------------------------------------------------
    def backward(self, pos, rad, opa, feat, bg, cam: CameraSpec, buf: dict, upstream, gamma, eps,
                 normalize=True, gate=True, camera_grads=True, out: Optional[dict] = None,
                 accumulate=False, tile=16, deterministic=False):
        """Enqueue the backward pipeline.  `buf` holds ids/z/closeness (K,H,W) + log_denom (H,W)
        CUDA tensors.  Returns dict of CUDA tensors d_pos, d_rad, d_opa, d_feat, pixel_count and
        cam_grad (16 float64: d_t[3], dL/dR[9], d_focal, d_sensor).  deterministic=True selects the
        bit-reproducible accumulation (SS_OPT_DETERMINISTIC: about twice the backward time), the counterpart
        of the reference's fixed-order merge (grad.py:231-250)."""
        dev = self.device
        bg = _dev_f32(bg, dev, (-1,))
        d = bg.shape[0]
        pos = _dev_f32(pos, dev, (-1, 3))
        m = pos.shape[0]
        rad, opa = _dev_f32(rad, dev, (-1,)), _dev_f32(opa, dev, (-1,))
        feat = _dev_f32(feat, dev, (-1, d)) if m else torch.zeros((0, d), device=dev)
        ids = buf["ids"]
        k, h, w = ids.shape
        if (h, w) != (int(cam.height), int(cam.width)):
            raise ContractViolation("buffer resolution does not match the camera")
        upstream = _dev_f32(upstream, dev)
        if tuple(upstream.shape) != (h, w, d):
            raise ValidationError(f"upstream shape {tuple(upstream.shape)} != {(h, w, d)}")
        if out is None:
            out = {"d_pos": torch.empty((m, 3), dtype=torch.float32, device=dev),
                   "d_rad": torch.empty((m,), dtype=torch.float32, device=dev),
                   "d_opa": torch.empty((m,), dtype=torch.float32, device=dev),
                   "d_feat": torch.empty((m, d), dtype=torch.float32, device=dev),
                   "pixel_count": torch.empty((m,), dtype=torch.int32, device=dev)}
            accumulate = False
        if camera_grads and "cam_grad" not in out:
            out["cam_grad"] = torch.empty(16, dtype=torch.float64, device=dev)  # fully written by the kernels
        dims = self._ensure_workspace(m, d, w, h, k)  # (a re-laid-out workspace forgets the last forward)
        reuse = self._records_current(buf, (pos, rad, opa), cam)
        flags = 0
        if normalize:
            flags |= _lib.OPT_NORMALIZE
        if gate:
            flags |= _lib.OPT_GATE
        if camera_grads:
            flags |= _lib.OPT_CAMERA_GRADS
        if accumulate:
            flags |= _lib.OPT_ACCUMULATE
        if reuse:
            flags |= _lib.OPT_REUSE_RECORDS
        det_ws = None
        if deterministic and m > 0:
            flags |= _lib.OPT_DETERMINISTIC
            nb = C.c_size_t()
            rc = self.lib.ss_deterministic_workspace_bytes(C.byref(dims), C.byref(nb))
            if rc != _lib.SS_OK:
                _raise_for(rc)
            if self._det_ws is None or self._det_ws.numel() < nb.value:
                self._det_ws = torch.empty(nb.value, dtype=torch.uint8, device=dev)
            det_ws = self._det_ws
        a = _lib.SsBackwardArgs()
        a.dims, a.cam = dims, cam.to_c()
        a.blend = _lib.SsBlend(float(gamma), float(eps), 0.0, int(tile), 256, flags, 0)
        a.pos, a.rad, a.opa, a.feat, a.bg = _ptr(pos), _ptr(rad), _ptr(opa), _ptr(feat), _ptr(bg)
        a.workspace, a.workspace_bytes = _ptr(self._ws), self._ws.numel()
        a.ids, a.z, a.closeness = _ptr(ids), _ptr(buf["z"]), _ptr(buf["closeness"])
        a.log_denom, a.upstream = _ptr(buf["log_denom"]), _ptr(upstream)
        a.d_pos, a.d_rad, a.d_opa = _ptr(out["d_pos"]), _ptr(out["d_rad"]), _ptr(out["d_opa"])
        a.d_feat, a.pixel_count = _ptr(out["d_feat"]), _ptr(out["pixel_count"])
        a.cam_grad = _ptr(out.get("cam_grad"))
        a.det_workspace, a.det_workspace_bytes = _ptr(det_ws), (det_ws.numel() if det_ws is not None else 0)
        with torch.cuda.device(dev):
            rc = self.lib.ss_backward(C.byref(a), self._stream())
        if rc != _lib.SS_OK:
            _raise_for(rc)
        out["_keepalive"] = (pos, rad, opa, feat, bg, upstream)
        return out


_engines = {}


def default_engine(device="cuda") -> RenderEngine:
    if not torch.cuda.is_available():
        raise _lib.NativeLibraryError("CUDA device required: the render path has no CPU fallback")
    dev = torch.device(device)
    if dev.type == "cuda" and dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    if dev not in _engines:
        _engines[dev] = RenderEngine(dev)
    return _engines[dev]
