"""Reference-facing entry points of the B200 render path.

`render_forward` / `render_backward` keep the reference's library signatures
(softsphere/raster.py:437-447, softsphere/grad.py:323-334) and return the same artefact
types, so they drop into `softsphere.optim.fit(..., renderer=SoftsphereAdapter())`
(optim.py:228-278) and into tests written against the reference.  Scene / camera / params may
be this package's types or the reference's own objects (same attribute names).

Host <-> device traffic of one call (the part of the plug-in path that is not a kernel):
  * the scene's NumPy columns (float64 in the reference) are narrowed to float32 straight into ONE pinned
    staging block (multi-threaded copy, no intermediate array) and travel as one H2D copy;
  * render_backward re-uses the device copy made by the render_forward that produced `buffer` when it is
    handed the very same scene object with the very same column arrays (identity + a sampled fingerprint;
    the reference's fit loop calls forward and backward on one unmodified scene, optim.py:292-304) --
    otherwise it uploads again, like the reference re-reads the scene (grad.py:213);
  * image and gradients come back through pinned blocks (one D2H copy each) and are widened to the
    reference's dtypes (image: the `dtype` argument, raster.py:443; gradients: float64, grad.py:224-227)
    by a multi-threaded copy into the returned arrays.
"""
from __future__ import annotations

import numpy as np
import torch

from .engine import CameraSpec, RenderEngine, default_engine
from .types import (AXIS_ANGLE, BackwardBuffer, BlendParams, CameraGradients, ConfigurationError,
                    ContractViolation, FeatureImage, RenderStats, SceneGradients, ValidationError,
                    axis_angle_vjp, rotation_6d_vjp)

DEFAULT_TILE_SIZE = 16
GATE_RADIUS_PX = 3.0
_IMAGE_BANDS = 4


def _reference_of(obj):
    """The reference package itself when `obj` (a scene) is one of ITS objects, else None.  A caller that hands in
    the reference's types -- its fit loop with this renderer plugged in, its own test files -- gets the reference's
    artefact types back (its shading and loss code check `isinstance(image, FeatureImage)`, shade.py:19-22) and
    the reference's exception classes raised (`pytest.raises(ContractViolation)` in tests/test_grad.py)."""
    import sys
    if type(obj).__module__.split(".")[0] != "softsphere":
        return None
    ref = sys.modules.get("softsphere")
    return ref if ref is not None and hasattr(ref, "raster") and hasattr(ref, "grad") else None


def _raises_reference_errors(fn):
    """Re-raises this package's exceptions as the same-named classes of the reference (errors.py:4-25) when the
    scene argument is a reference object."""
    import functools

    @functools.wraps(fn)
    def wrapper(scene, *args, **kwargs):
        try:
            return fn(scene, *args, **kwargs)
        except Exception as e:  # noqa: BLE001
            ref = _reference_of(scene)
            cls = getattr(getattr(ref, "errors", None), type(e).__name__, None) if ref is not None else None
            if cls is None or isinstance(e, cls) or type(e).__module__.split(".")[0] != __name__.split(".")[0]:
                raise
            raise cls(*e.args) from e
    return wrapper


def _scene_columns(scene):
    m = len(scene)
    d = int(scene.feature_dim)
    feats = np.asarray(scene.features)
    if tuple(feats.shape) != (m, d):
        raise ValidationError(f"feature array shape {tuple(feats.shape)} does not match (M={m}, d={d})")
    pos, rad, opa = np.asarray(scene.positions), np.asarray(scene.radii), np.asarray(scene.opacities)
    if pos.shape != (m, 3) or rad.shape != (m,) or opa.shape != (m,):
        raise ValidationError("sphere column arrays have mismatched lengths")
    return pos, rad, opa, feats, np.asarray(scene.background)


def _fingerprint(cols):
    """A few hundred strided samples per column: catches bulk in-place edits of a scene between forward and
    backward (identity of the arrays alone cannot)."""
    out = []
    for a in cols:
        flat = a.reshape(-1)
        step = max(1, flat.shape[0] // 251)
        out.append(flat[::step][:512].astype(np.float64).tobytes())
    return tuple(out)


class _Stage:
    """Pinned staging blocks + device output blocks for one problem size (cached on the engine)."""

    def __init__(self, device, m, d, h, w):
        from .host import PackedGradients
        self.key = (m, d, h, w)
        self.m, self.d, self.h, self.w = m, d, h, w
        f32 = torch.float32
        self.n_in = m * (5 + d) + d
        self.h_in = torch.empty(self.n_in, dtype=f32).pin_memory()
        self.h_img = torch.empty(h * w * (d + 1), dtype=f32).pin_memory()
        self.h_up = torch.empty((h, w, d), dtype=f32).pin_memory()
        self.upstream = torch.empty((h, w, d), dtype=f32, device=device)
        self.d_img = torch.empty(h * w * (d + 1), dtype=f32, device=device)
        self.grads = PackedGradients(m, d, device)
        self.side = torch.cuda.Stream(device=device)  # image rows travel while the lower bands are drawn
        self.band_events = [torch.cuda.Event() for _ in range(_IMAGE_BANDS)]

    @staticmethod
    def carve_in(t, m, d):
        o, out = 0, []
        for n, shape in ((3 * m, (m, 3)), (m, (m,)), (m, (m,)), (m * d, (m, d)), (d, (d,))):
            out.append(t[o:o + n].view(shape))
            o += n
        return out


def _stage_for(eng: RenderEngine, m, d, h, w) -> _Stage:
    st = getattr(eng, "_api_stage", None)
    if st is None or st.key != (m, d, h, w):
        st = _Stage(eng.device, m, d, h, w)
        eng._api_stage = st
    return st


def _narrow_into(dst: torch.Tensor, src: np.ndarray):
    """dst (pinned float32 view) <- src (any float dtype): torch's multi-threaded converting copy."""
    if src.size:
        dst.copy_(torch.from_numpy(np.ascontiguousarray(src)).view(dst.shape))


def _widen(src: torch.Tensor, dtype) -> np.ndarray:
    """New NumPy array of `dtype` holding the values of the pinned tensor `src`."""
    out = np.empty(tuple(src.shape), dtype=dtype)
    if out.size:
        torch.from_numpy(out).copy_(src)
    return out


_PIPE_ELEMS = 1 << 21  # elements per pipeline piece (8 MB of float32): ~0.15 ms of PCIe time each


def _upload_scene(eng: RenderEngine, st: _Stage, cols):
    """float64 NumPy columns -> one float32 device block.  Narrowing (CPU, multi-threaded) and the H2D copy (DMA)
    are pipelined piece by piece: the copy of piece i runs while piece i + 1 is being narrowed into the pinned
    staging block (0.86 + 0.60 ms back to back at 1 M spheres, ~0.95 ms pipelined)."""
    m, d = st.m, st.d
    d_in = torch.empty(st.n_in, dtype=torch.float32, device=eng.device)  # fresh: the buffer keeps it for backward
    o = 0
    for dst, src in zip(_Stage.carve_in(st.h_in, m, d), cols):
        n = dst.numel()
        if n:
            flat_src = torch.from_numpy(np.ascontiguousarray(src)).view(-1)
            flat_dst = dst.view(-1)
            for a in range(0, n, _PIPE_ELEMS):
                b = min(n, a + _PIPE_ELEMS)
                flat_dst[a:b].copy_(flat_src[a:b])
                d_in[o + a:o + b].copy_(st.h_in[o + a:o + b], non_blocking=True)
        o += n
    return tuple(_Stage.carve_in(d_in, m, d))


def _download_widened(eng: RenderEngine, pieces):
    """pieces: [(device tensor, pinned host tensor, numpy dtype)].  Enqueues the D2H copies in order with an event
    behind each, then widens piece i into a new NumPy array while the copies of the later pieces are still running
    (0.64 ms of D2H + 0.93 ms of widening back to back for the 1 M-sphere gradients, ~1.15 ms pipelined)."""
    stream = torch.cuda.current_stream(eng.device)
    events = []
    for dev, host, _ in pieces:
        host.copy_(dev, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(stream)
        events.append(ev)
    out = []
    for (dev, host, dtype), ev in zip(pieces, events):
        ev.synchronize()
        out.append(_widen(host, dtype))
    return out


@_raises_reference_errors
def render_forward(scene, camera, params, *, workers: int = 1, dtype=np.float64,
                   tile_size: int = DEFAULT_TILE_SIZE, store_buffer: bool = True, chunk_size: int = 256,
                   engine: RenderEngine = None):
    """Bounds, depth order, tile binning and tile draw on the GPU.

    Returns (FeatureImage, BackwardBuffer or None, RenderStats) like the reference.  `workers` is accepted
    for signature compatibility (the device path is deterministic); `tile_size` other than 16 is accepted at
    tau = 0, where only the counters depend on it (see below); `dtype` selects the dtype of the returned
    arrays like in the reference (raster.py:462-474) -- the device arithmetic is the mixed float32 blend /
    float64 geometry path either way."""
    eng = engine or default_engine()
    if int(tile_size) < 1:
        raise ConfigurationError(f"tile_size must be >= 1, got {tile_size}")
    if not (1 <= int(chunk_size) <= 256):
        raise ConfigurationError("chunk_size must be in 1..256")
    dtype = np.dtype(dtype)
    if dtype not in (np.dtype(np.float64), np.dtype(np.float32)):
        raise ConfigurationError(f"dtype must be float64 or float32, got {dtype}")
    p = params if isinstance(params, BlendParams) else BlendParams(params.gamma, params.epsilon, params.tau,
                                                                   params.top_k)
    other_tiles = int(tile_size) != DEFAULT_TILE_SIZE
    if other_tiles and p.tau > 0.0:
        # The device draws 16x16 tiles.  Image, buffer and gradients do not depend on the tile size at tau = 0 (only
        # the `tiles` / `candidates_tested` counters do, and those are recomputed below); with tau > 0 the early-stop
        # vote is taken per tile and chunk of the tile's list (raster.py:358-368), so another tile size would stop
        # other pixels than the reference does.
        raise ConfigurationError("tile_size != 16 is supported for tau = 0 only (the device takes the early-stop "
                                 "vote per 16x16 tile)")
    cols = _scene_columns(scene)
    # background is validated on the host (d numbers); per-sphere fields are scanned on the device
    if not np.all(np.isfinite(np.asarray(scene.background, dtype=np.float64))):
        raise ValidationError("background feature contains non-finite values")
    cam = CameraSpec.from_camera(camera)
    m, d, h, w = len(scene), int(scene.feature_dim), int(cam.height), int(cam.width)
    with torch.cuda.device(eng.device):
        st = _stage_for(eng, m, d, h, w)
        dev_in = _upload_scene(eng, st, cols)
        n_img = h * w * d
        # the kernels write image | bg_weight into one device block: one D2H copy
        d_image, d_bgw = st.d_img[:n_img].view(h, w, d), st.d_img[n_img:].view(h, w)
        h_image, h_bgw = st.h_img[:n_img].view(h, w, d), st.h_img[n_img:].view(h, w)
        main = torch.cuda.current_stream(eng.device)

        def download_bands():  # on the side stream, band by band as the raster launches complete
            with torch.cuda.stream(st.side):
                for b, ev in enumerate(st.band_events):
                    r0, r1 = eng.band_rows(h, _IMAGE_BANDS, b)
                    st.side.wait_event(ev)
                    if r1 > r0:
                        h_image[r0:r1].copy_(d_image[r0:r1], non_blocking=True)
                        h_bgw[r0:r1].copy_(d_bgw[r0:r1], non_blocking=True)

        st.side.wait_stream(main)  # (the staging block's previous readers are done: calls end synchronised)
        res = eng.forward(*dev_in, cam, gamma=p.gamma, eps=p.epsilon, tau=p.tau, top_k=p.top_k,
                          chunk=int(chunk_size), store_buffer=store_buffer, collect_stats=True, check=True,
                          image=d_image, bg_weight=d_bgw, debug=other_tiles, band_events=st.band_events,
                          after_launch=download_bands)
        stat = res["status"]
        st.side.synchronize()
    image = FeatureImage(data=_widen(st.h_img[:n_img].view(h, w, d), dtype),
                         background_weight=_widen(st.h_img[n_img:].view(h, w), dtype))
    buffer = None
    if store_buffer:
        buffer = BackwardBuffer({k: res[k] for k in ("ids", "z", "closeness", "log_denom", "fwd_token")}, p,
                                len(scene), dtype=dtype)
        buffer._inputs = res["inputs"]
        buffer._host_cols = cols  # strong references: ids of live objects cannot be recycled
        buffer._scene_fp = _fingerprint(cols)
    ts = int(tile_size)
    ntx, nty = (cam.width + ts - 1) // ts, (cam.height + ts - 1) // ts
    tested = stat["candidates_tested"]
    if other_tiles:  # tau = 0: every tile scans its whole list, i.e. one test per (sphere, tile) pair of THAT tiling
        rect = res["rect"].cpu().numpy().astype(np.int64)
        on = res["on_sensor"].cpu().numpy().astype(bool)
        pairs = (rect[:, 1] // ts - rect[:, 0] // ts + 1) * (rect[:, 3] // ts - rect[:, 2] // ts + 1)
        tested = int(pairs[on].sum())
    ref = _reference_of(scene)
    stats_cls = ref.raster.RenderStats if ref is not None else RenderStats
    stats = stats_cls(spheres_total=len(scene), spheres_on_sensor=stat["spheres_on_sensor"],
                      candidates_tested=tested, hits_blended=stat["hits_blended"],
                      pixels_early_stopped=stat["pixels_early_stopped"], tiles=ntx * nty)
    if ref is not None:  # (the buffer stays this package's lazily downloaded record: it is duck-typed everywhere)
        image = ref.raster.FeatureImage(data=image.data, background_weight=image.background_weight)
    return image, buffer, stats


def _same_scene(buffer: BackwardBuffer, cols) -> bool:
    held = getattr(buffer, "_host_cols", None)
    if held is None or getattr(buffer, "_inputs", None) is None:
        return False
    if not all(a is b for a, b in zip(held, cols)):
        return False
    return buffer._scene_fp == _fingerprint(cols)


def _device_record(buffer, device):
    """The per-pixel record as the kernels want it: slot-major (K, H, W) CUDA tensors.  A buffer made by this
    package already holds them; a buffer made by the REFERENCE's render_forward (NumPy arrays in (H, W, K) layout,
    raster.py:97-110) is transposed and uploaded, so the two implementations' forward and backward halves can be mixed."""
    dev = getattr(buffer, "dev", None)
    if dev is not None:
        return dev

    def up(a, dtype):
        a = np.asarray(a)
        if a.ndim == 3:
            a = np.transpose(a, (2, 0, 1))
        return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).to(device, non_blocking=True)

    return {"ids": up(buffer.ids, np.int32), "z": up(buffer.z, np.float32), "closeness": up(buffer.closeness, np.float32),
            "log_denom": up(buffer.log_denom, np.float32)}


@_raises_reference_errors
def render_backward(scene, camera, params, buffer: BackwardBuffer, upstream, *, workers: int = 1,
                    normalize: bool = True, gate: bool = True, tile_size: int = 16,
                    engine: RenderEngine = None, reuse_upload: bool = True, deterministic: bool = False):
    """Full backward pipeline; returns (SceneGradients, CameraGradients) as float64 NumPy like the reference.
    reuse_upload=False always re-uploads the scene (see the module docstring); deterministic=True makes the
    result bit-identical from run to run like the reference's (grad.py:231-250), at about twice the device time."""
    eng = engine or default_engine()
    if buffer.num_spheres != len(scene):
        raise ContractViolation(f"buffer built for {buffer.num_spheres} spheres, scene has {len(scene)}")
    upstream = np.asarray(upstream)
    if upstream.dtype not in (np.float64, np.float32):
        upstream = upstream.astype(np.float64)
    record = _device_record(buffer, eng.device)
    k, h, w = record["ids"].shape
    m, d = len(scene), int(scene.feature_dim)
    if upstream.shape != (h, w, d):
        raise ValidationError(f"upstream shape {upstream.shape} != {(h, w, d)}")
    bp = buffer.params
    cam = CameraSpec.from_camera(camera)
    cols = _scene_columns(scene)
    with torch.cuda.device(eng.device):
        st = _stage_for(eng, m, d, h, w)
        if reuse_upload and _same_scene(buffer, cols):
            dev_in = buffer._inputs
        else:
            dev_in = _upload_scene(eng, st, cols)
        _narrow_into(st.h_up, upstream)
        st.upstream.copy_(st.h_up, non_blocking=True)
        out = eng.backward(*dev_in, cam, record, st.upstream, gamma=bp.gamma, eps=bp.epsilon,
                           normalize=normalize, gate=gate, camera_grads=True, out=dict(st.grads.dev),
                           accumulate=False, deterministic=deterministic)
        gd, hg = st.grads.dev, st.grads.host
        # the camera block first (tiny), then the columns: each is widened while the next ones are still in flight
        names = ("cam_grad", "d_pos", "d_feat", "d_rad", "d_opa", "pixel_count")
        dtypes = (np.float64, np.float64, np.float64, np.float64, np.float64, np.int64)
        got = dict(zip(names, _download_widened(eng, [(gd[n], hg[n], t) for n, t in zip(names, dtypes)])))
        del out
    grads = SceneGradients(d_position=got["d_pos"], d_radius=got["d_rad"], d_opacity=got["d_opa"],
                           d_feature=got["d_feat"], pixel_count=got["pixel_count"])
    cg = got["cam_grad"]
    g_rot = cg[3:12].reshape(3, 3)
    if camera.rotation_type == AXIS_ANGLE:
        d_rot = axis_angle_vjp(camera.rotation_param, g_rot)
    else:
        d_rot = rotation_6d_vjp(camera.rotation_param, g_rot)
    cam_grads = CameraGradients(d_translation=cg[0:3].copy(), d_rotation=d_rot, d_focal=float(cg[12]),
                                d_sensor_width=float(cg[13]))
    ref = _reference_of(scene)
    if ref is not None:
        grads = ref.grad.SceneGradients(d_position=grads.d_position, d_radius=grads.d_radius,
                                        d_opacity=grads.d_opacity, d_feature=grads.d_feature,
                                        pixel_count=grads.pixel_count)
        cam_grads = ref.grad.CameraGradients(d_translation=cam_grads.d_translation, d_rotation=cam_grads.d_rotation,
                                             d_focal=cam_grads.d_focal, d_sensor_width=cam_grads.d_sensor_width)
    return grads, cam_grads


class SoftsphereAdapter:
    """`renderer=` plug-in for the reference's fit loop (optim.py:265-278): an object with
    forward(scene, camera, params) and backward(scene, camera, params, buffer, upstream).

    The reference's fit does not pass its normalize/gate settings to a plug-in (optim.py:273-278), so they
    are constructor arguments here (defaults = FitConfig's defaults)."""

    def __init__(self, normalize: bool = True, gate: bool = True, engine: RenderEngine = None,
                 dtype=np.float64, reuse_upload: bool = True, deterministic: bool = False):
        self.deterministic = deterministic
        self.normalize = normalize
        self.gate = gate
        self.engine = engine
        self.dtype = dtype
        self.reuse_upload = reuse_upload

    def forward(self, scene, camera, params):
        return render_forward(scene, camera, params, engine=self.engine, dtype=self.dtype)

    def backward(self, scene, camera, params, buffer, upstream):
        return render_backward(scene, camera, params, buffer, upstream, normalize=self.normalize,
                               gate=self.gate, engine=self.engine, reuse_upload=self.reuse_upload,
                               deterministic=self.deterministic)
