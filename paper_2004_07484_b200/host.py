"""Host-buffer session: the reference-facing call for users whose scene lives in host memory
(as the reference's NumPy columns do).  Pinned staging buffers are allocated once; a render_step
copies what changed host->device, runs ss_forward / ss_backward, and copies the image and the
gradients device->host.  This is the path bench.py times as `e2e`.

Transfers are packed and minimal:
  * the five scene columns travel as ONE pinned block / one H2D copy, and only when `set_scene` has
    been called since the last step (a static scene stays resident on the device);
  * gradients come back either dense (ONE block: all M rows + pixel counts + the camera block) or
    `compact=True`: only the U rows of spheres that received gradient (pixel_count > 0), preceded by
    their sphere indices -- ss_mask_nonzero_i32 + ss_compact_rows on the device interleave them into one
    array of records (C3: 36 MB -> 12.7 MB), written by the compaction kernel straight into the mapped pinned
    host array together with the row count (CompactGradients(zero_copy=True); a device array + one copy otherwise);
  * the image download runs on a second stream so that it overlaps the upstream upload (the two
    PCIe directions); the forward pass draws the image in `bands` bands of tile rows (ss_forward_banded) and
    every band is downloaded as soon as it is final -- the upper bands under the raster kernel of the lower
    ones, the last one under the backward pass (2 bands by default: each band is a raster launch of its own and
    pays its own partial waves; measured 1 / 2 / 3 / 4 / 8 bands, scripts/e2e_bands.py)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

from . import _lib
from .engine import CameraSpec, RenderEngine, _ptr, _raise_for


class PackedGradients:
    """All per-sphere gradients of one backward call in ONE device block of 4-byte words
    [d_pos 3m | d_rad m | d_opa m | d_feat m*d | pixel_count m | camera block 16 float64] and its pinned
    host twin, carved into views (`dev`, `host`): one D2H copy moves everything."""

    def __init__(self, num_spheres: int, feature_dim: int, device):
        m, d = int(num_spheres), int(feature_dim)
        self.m, self.d = m, d
        n_out = m * (6 + d) + 32
        n_out += n_out % 2  # keep the float64 camera block 8-byte aligned
        self.cam_off = n_out - 32
        self.d_out = torch.empty(n_out, dtype=torch.float32, device=device)
        self.h_out = torch.empty(n_out, dtype=torch.float32).pin_memory()
        self.dev = self._carve(self.d_out)
        self.host = self._carve(self.h_out)

    def _carve(self, t):
        m, d = self.m, self.d
        o, res = 0, {}
        for name, n, shape in (("d_pos", 3 * m, (m, 3)), ("d_rad", m, (m,)), ("d_opa", m, (m,)),
                               ("d_feat", m * d, (m, d))):
            res[name] = t[o:o + n].view(shape)
            o += n
        res["pixel_count"] = t[o:o + m].view(torch.int32)
        res["cam_grad"] = t[self.cam_off:self.cam_off + 32].view(torch.float64)
        return res

    def download(self, stream=None):
        """Enqueue the single D2H copy; the caller synchronises.  Returns the pinned host views."""
        self.h_out.copy_(self.d_out, non_blocking=True)
        return self.host

    def nbytes(self) -> int:
        return 4 * self.h_out.numel()


class CompactGradients:
    """Rows of the spheres that received gradient, gathered on the device into ONE array of records
    [index i32 | pixel_count i32 | d_pos 3 | d_rad | d_opa | d_feat d] (7 + d words each) and downloaded with a
    single copy; the host views are columns of that record array."""

    def __init__(self, num_spheres: int, feature_dim: int, device, zero_copy=None):
        m, d = int(num_spheres), int(feature_dim)
        self.m, self.d, self.device = m, d, device
        self.lib = _lib.load()
        self.words = 7 + d
        # zero_copy: the compaction kernel writes the records (and the count) straight into the pinned host array
        # -- whole 128-byte lines over PCIe while it runs -- instead of into a device array that a copy then
        # downloads: no staging pass, no speculative size, never a second round trip.  SS_COMPACT_ZERO_COPY=0/1.
        if zero_copy is None:
            zero_copy = os.environ.get("SS_COMPACT_ZERO_COPY", "1") != "0"
        self.zero_copy = bool(zero_copy)
        self.index = torch.arange(m, dtype=torch.int32, device=device)  # one-time iota (source of the index column)
        self.keep = torch.empty(max(m, 1), dtype=torch.uint8, device=device)
        self.count = torch.zeros(1, dtype=torch.int64, device=device)
        self.h_count = torch.zeros(1, dtype=torch.int64).pin_memory()
        self.d_rec = torch.empty(max(m, 1) * self.words, dtype=torch.float32, device=device)
        self.h_rec = torch.empty(max(m, 1) * self.words, dtype=torch.float32).pin_memory()
        nb = C.c_size_t()
        rc = self.lib.ss_compact_workspace_bytes(m, C.byref(nb))
        if rc != _lib.SS_OK:
            _raise_for(rc)
        self.ws = torch.empty(max(nb.value, 256), dtype=torch.uint8, device=device)
        self._last_count = None
        self.last_bytes = 0

    def estimate(self) -> int:
        """Rows downloaded speculatively together with the count: what the previous call needed + 5 %, rounded up to
        whole blocks of 4096 rows (a captured step bakes this size in: it should not change from step to step)."""
        if self.zero_copy:
            return self.m  # (nothing is downloaded speculatively: the kernel writes exactly `count` records)
        if self._last_count is None:
            return 0
        est = int(self._last_count * 1.05) + 1024
        return min(self.m, (est + 4095) // 4096 * 4096)

    def enqueue(self, grads: dict, stream, est: int) -> None:
        """Device side of `gather` (no host synchronisation: capturable): mask, compaction into records, download of
        the count and of the first `est` records."""
        m, d, words = self.m, self.d, self.words
        sp = C.c_void_p(stream.cuda_stream)
        rc = self.lib.ss_mask_nonzero_i32(_ptr(grads["pixel_count"]), m, _ptr(self.keep), sp)
        if rc != _lib.SS_OK:
            _raise_for(rc)
        cols = ((self.index, 1), (grads["pixel_count"], 1), (grads["d_pos"], 3), (grads["d_rad"], 1),
                (grads["d_opa"], 1), (grads["d_feat"], d))
        arr = (_lib.SsColumn * len(cols))()
        off = 0
        rec_ptr = self.h_rec.data_ptr() if self.zero_copy else self.d_rec.data_ptr()
        count = self.h_count if self.zero_copy else self.count
        for i, (src, w) in enumerate(cols):  # interleave the columns into records: dst offset inside the first record
            arr[i].src, arr[i].dst = src.data_ptr(), rec_ptr + 4 * off
            arr[i].row_bytes, arr[i].dst_stride_bytes = 4 * w, 4 * words
            off += w
        rc = self.lib.ss_compact_rows(_ptr(self.keep), m, arr, len(cols), _ptr(self.ws), self.ws.numel(),
                                      _ptr(count), sp)
        if rc != _lib.SS_OK:
            _raise_for(rc)
        if self.zero_copy:
            return
        # One round trip instead of two: the count travels together with a SPECULATIVE download of as many rows as
        # the previous call needed (+5 %); only when this call touched more spheres is the remainder fetched.
        self.h_count.copy_(self.count, non_blocking=True)
        if est:
            self.h_rec[: est * words].copy_(self.d_rec[: est * words], non_blocking=True)

    def finish(self, stream, est: int) -> dict:
        """Host side of `gather`: waits for `stream`, fetches the rows beyond the speculative download if there are
        any, returns the pinned host views."""
        words = self.words
        stream.synchronize()
        n = int(self.h_count[0])
        if n > est:
            self.h_rec[est * words: n * words].copy_(self.d_rec[est * words: n * words], non_blocking=True)
            stream.synchronize()
        self._last_count = n
        rec = self.h_rec[: n * words].view(n, words)
        irec = rec.view(torch.int32)
        self.last_bytes = 8 + 4 * (n if self.zero_copy else max(n, est)) * words
        return {"count": n, "index": irec[:, 0], "pixel_count": irec[:, 1], "d_pos": rec[:, 2:5], "d_rad": rec[:, 5],
                "d_opa": rec[:, 6], "d_feat": rec[:, 7:], "records": rec}

    def gather(self, grads: dict, stream) -> dict:
        """grads: dense device gradients (d_pos, d_rad, d_opa, d_feat, pixel_count).  Returns pinned host views
        of `count` rows after synchronising `stream`."""
        est = self.estimate()
        self.enqueue(grads, stream, est)
        return self.finish(stream, est)


class HostRenderSession:
    def __init__(self, num_spheres: int, feature_dim: int, width: int, height: int, top_k: int = 5,
                 engine: RenderEngine = None, device="cuda", bands: int = 2):
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

        # forward outputs and the argument blocks of the two C calls are allocated / filled once: the per-step
        # Python work before the first kernel launch is GPU idle time on this path (it was 0.1 ms of a 1 ms step)
        k = self.k
        # two image buffers, alternating by view: the download of view i must not hold back the forward of view i + 1
        # (a ring of image buffers: the pipelined multi-view step uses all four, so that the forward pass of view
        # i + 2 does not wait for the download of image i; the other paths alternate between the first two)
        self._images = [torch.empty((h, w, d), dtype=f32, device=dev) for _ in range(4)]
        self._image_copied = [torch.cuda.Event() for _ in range(4)]
        # "lane" j = an engine (workspace) + its forward outputs + its upstream buffer + its argument blocks.  Lane 0
        # serves single views; multi-view steps alternate views between lane 0 and lane 1 (allocated on first use)
        # on two compute streams, so the forward of view i + 1 runs under the backward of view i.
        self._lanes = [self._new_lane(self.engine, self.upstream)]
        self._compute_streams = None

        self.packed = PackedGradients(m, d, dev)
        self.out, self.h_grads = self.packed.dev, self.packed.host
        self.d_out, self.h_out = self.packed.d_out, self.packed.h_out
        self._compact = None
        self.copy_stream = torch.cuda.Stream(device=dev)
        self._upload_stream = None  # H2D stream of the pipelined multi-view step
        self.bands = max(1, int(bands))
        self._band_events = [torch.cuda.Event() for _ in range(self.bands)]
        self._band_rows = [self.engine.band_rows(h, self.bands, b) for b in range(self.bands)]
        self._scene_dirty = True
        self.last_h2d_bytes = 0
        self.last_d2h_bytes = 0
        self._step_graphs = {}  # captured single-view steps (render_step(..., graph=True)), newest last

    def _new_lane(self, engine, upstream):
        dev, f32 = engine.device, torch.float32
        h, w, k = self.h, self.w, self.k
        return {"engine": engine, "upstream": upstream, "key": None, "fa": None, "ba": None, "events_c": None,
                "bg_weight": torch.empty((h, w), dtype=f32, device=dev),
                "ids": torch.empty((k, h, w), dtype=torch.int32, device=dev),
                "z": torch.empty((k, h, w), dtype=f32, device=dev),
                "closeness": torch.empty((k, h, w), dtype=f32, device=dev),
                "log_denom": torch.empty((h, w), dtype=f32, device=dev)}

    def _lane(self, j):
        while len(self._lanes) <= j:
            e = self.engine
            twin = RenderEngine(e.device, pair_factor=e.pair_factor, min_pairs=e.min_pairs)
            self._lanes.append(self._new_lane(twin, torch.empty_like(self.upstream)))
        return self._lanes[j]

    def _prepared(self, lane):
        """Argument blocks of ss_forward / ss_backward with every pointer filled in; rebuilt only when the lane's
        workspace moved or was re-laid out (the first lane's engine may be shared with other callers)."""
        eng = lane["engine"]
        dims = eng._ensure_workspace(self.m, self.d, self.w, self.h, self.k)
        key = (eng._ws.data_ptr(), eng._ws.numel(), int(dims.max_pairs))
        if key != lane["key"]:
            fa, ba = _lib.SsForwardArgs(), _lib.SsBackwardArgs()
            for a in (fa, ba):
                a.dims = dims
                a.pos, a.rad, a.opa, a.feat, a.bg = (_ptr(self.pos), _ptr(self.rad), _ptr(self.opa), _ptr(self.feat),
                                                     _ptr(self.bg))
                a.workspace, a.workspace_bytes = _ptr(eng._ws), eng._ws.numel()
                a.ids, a.z, a.closeness, a.log_denom = (_ptr(lane["ids"]), _ptr(lane["z"]), _ptr(lane["closeness"]),
                                                        _ptr(lane["log_denom"]))
            fa.bg_weight = _ptr(lane["bg_weight"])
            ba.upstream = _ptr(lane["upstream"])
            o = self.out
            ba.d_pos, ba.d_rad, ba.d_opa, ba.d_feat = _ptr(o["d_pos"]), _ptr(o["d_rad"]), _ptr(o["d_opa"]), _ptr(o["d_feat"])
            ba.pixel_count, ba.cam_grad = _ptr(o["pixel_count"]), _ptr(o["cam_grad"])
            lane["fa"], lane["ba"], lane["key"], lane["events_c"] = fa, ba, key, None
        return lane["fa"], lane["ba"]

    def _forward_fast(self, cam, gamma, eps, tau, events, stream, image, lane=None):
        """ss_forward[_banded] on the session's own buffers without the engine's per-call checks and allocations
        (no status read: the caller polls engine.read_status(), like engine.forward(check=False))."""
        lane = lane or self._lanes[0]
        fa, _ = self._prepared(lane)
        fa.cam, fa.image = cam.to_c(), _ptr(image)
        fa.blend = _lib.SsBlend(float(gamma), float(eps), float(tau), 16, 256, _lib.OPT_STORE_BUFFER, 0)
        lib, sp = lane["engine"].lib, C.c_void_p(stream.cuda_stream)
        if events:
            if lane["events_c"] is None or len(lane["events_c"]) != len(events):
                for e in events:  # a torch event only gets its CUDA handle on first record
                    if not e.cuda_event:
                        e.record(stream)
                lane["events_c"] = (C.c_void_p * len(events))(*[C.c_void_p(e.cuda_event) for e in events])
            rc = lib.ss_forward_banded(C.byref(fa), len(events), lane["events_c"], sp)
        else:
            rc = lib.ss_forward(C.byref(fa), sp)
        if rc != _lib.SS_OK:
            _raise_for(rc)
        lane["engine"]._last_fwd = None  # (the engine's own record-reuse bookkeeping does not cover this call)

    def _backward_fast(self, cam, gamma, eps, normalize, gate, accumulate, stream, lane=None):
        lane = lane or self._lanes[0]
        _, ba = self._prepared(lane)
        ba.cam = cam.to_c()
        # the draw records in the workspace are those of the forward call just made on the same, untouched inputs
        flags = _lib.OPT_CAMERA_GRADS | _lib.OPT_REUSE_RECORDS
        flags |= (_lib.OPT_NORMALIZE if normalize else 0) | (_lib.OPT_GATE if gate else 0)
        flags |= _lib.OPT_ACCUMULATE if accumulate else 0
        ba.blend = _lib.SsBlend(float(gamma), float(eps), 0.0, 16, 256, flags, 0)
        rc = lane["engine"].lib.ss_backward(C.byref(ba), C.c_void_p(stream.cuda_stream))
        if rc != _lib.SS_OK:
            _raise_for(rc)

    def _views_pipelined(self, cams, gamma, eps, tau, normalize, gate, main):
        """Multi-view body of render_step for an upstream that is already staged on the host: views alternate between
        two lanes on two compute streams (forward of view i + 1 under the backward of view i; the backward passes stay
        in view order: k_finalize adds into the shared gradient buffers without atomics), uploads and downloads ride
        on the copy stream.  Returns the H2D byte count."""
        dev = self.engine.device
        if self._compute_streams is None:
            self._compute_streams = [torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)]
        copy = self.copy_stream
        if self._upload_stream is None:
            self._upload_stream = torch.cuda.Stream(device=dev)
        upload = self._upload_stream
        for st in self._compute_streams:
            st.wait_stream(main)  # scene upload / earlier work of the caller
        copy.wait_stream(main)
        upload.wait_stream(main)
        bwd_done, last_bwd, h2d = [None, None], None, 0
        with torch.cuda.device(dev):
            for i, cam in enumerate(cams):
                j = i & 1
                lane, st = self._lane(j), self._compute_streams[j]
                last = i == len(cams) - 1
                events = self._band_events[:self.bands] if (last and self.bands > 1) else None
                with torch.cuda.stream(upload):  # upstream of view i -> lane j, once backward(i - 2) has consumed it
                    if bwd_done[j] is not None:
                        upload.wait_event(bwd_done[j])
                    lane["upstream"].copy_(self.h_upstream, non_blocking=True)
                    up_ready = torch.cuda.Event()
                    up_ready.record(upload)
                h2d += 4 * self.h_upstream.numel()
                r = i & 3
                image = self._images[r]
                if i > 3:  # this image buffer was last used four views ago: its download must have read it
                    st.wait_event(self._image_copied[r])
                with torch.cuda.stream(st):  # (a lane's first use initialises its workspace on the current stream)
                    self._forward_fast(cam, gamma, eps, tau, events, st, image, lane)
                fwd_done = torch.cuda.Event()
                fwd_done.record(st)
                with torch.cuda.stream(copy):
                    if events:
                        for b, ev in enumerate(events):
                            r0, r1 = self._band_rows[b]
                            copy.wait_event(ev)
                            if r1 > r0:
                                self.h_image[r0:r1].copy_(image[r0:r1], non_blocking=True)
                    else:
                        copy.wait_event(fwd_done)
                        self.h_image.copy_(image, non_blocking=True)
                    self._image_copied[r].record(copy)
                st.wait_event(up_ready)
                if last_bwd is not None:
                    st.wait_event(last_bwd)
                with torch.cuda.stream(st):
                    self._backward_fast(cam, gamma, eps, normalize, gate, i > 0, st, lane)
                last_bwd = torch.cuda.Event()
                last_bwd.record(st)
                bwd_done[j] = last_bwd
        for st in self._compute_streams:
            main.wait_stream(st)
        return h2d

    def _enqueue_single_view(self, cam, gamma, eps, tau, normalize, gate, est):
        """Every device operation of a one-view step with a staged upstream and compact gradient rows, without a
        host synchronisation (so that it can be captured): upstream H2D on the copy stream under the banded forward
        pass, image rows D2H band by band, backward pass, compaction, count + speculative rows + camera block D2H."""
        dev = self.engine.device
        main = torch.cuda.current_stream(dev)
        cs = self.copy_stream
        cs.wait_stream(main)
        with torch.cuda.stream(cs):
            self.upstream.copy_(self.h_upstream, non_blocking=True)
        events = self._band_events[:self.bands] if self.bands > 1 else None
        image = self._images[0]
        with torch.cuda.device(dev):
            self._forward_fast(cam, gamma, eps, tau, events, main, image)
        main.wait_stream(cs)  # backward needs the uploaded upstream
        with torch.cuda.stream(cs):
            if events:
                for b, ev in enumerate(events):
                    r0, r1 = self._band_rows[b]
                    cs.wait_event(ev)
                    if r1 > r0:
                        self.h_image[r0:r1].copy_(image[r0:r1], non_blocking=True)
            else:
                cs.wait_stream(main)
                self.h_image.copy_(image, non_blocking=True)
            self._image_copied[0].record(cs)
        with torch.cuda.device(dev):
            self._backward_fast(cam, gamma, eps, normalize, gate, False, main)
        self._compact.enqueue(self.out, main, est)
        self.h_out[self.packed.cam_off:].copy_(self.d_out[self.packed.cam_off:], non_blocking=True)
        main.wait_stream(cs)  # the copy stream rejoins: the step ends on one stream

    def _render_step_graphed(self, cam, gamma, eps, tau, normalize, gate):
        """render_step for ONE view with a staged upstream and compact rows, replayed from a CUDA graph: the ~15 launches
        and copies of the step cost the host 0.15 ms of enqueueing, during which the GPU waits between the short
        kernels of the forward pass; a replay is one launch.  The capture bakes in the camera, the parameters and
        the size of the speculative row download; the last four are kept."""
        dev = self.engine.device
        if self._compact is None:
            self._compact = CompactGradients(self.m, self.d, dev)
        est = self._compact.estimate()
        key = (bytes(cam.to_c()), float(gamma), float(eps), float(tau), bool(normalize), bool(gate), est,
               self._lanes[0]["key"])
        g = self._step_graphs.get(key)
        if g is None:
            # warm-up outside the capture (workspace, argument blocks, event handles, function attributes)
            self._enqueue_single_view(cam, gamma, eps, tau, normalize, gate, est)
            torch.cuda.synchronize(dev)
            key = key[:-1] + (self._lanes[0]["key"],)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._enqueue_single_view(cam, gamma, eps, tau, normalize, gate, est)
            while len(self._step_graphs) >= 4:
                self._step_graphs.pop(next(iter(self._step_graphs)))
            self._step_graphs[key] = g
        g.replay()
        main = torch.cuda.current_stream(dev)
        grads = self._compact.finish(main, est)
        grads["cam_grad"] = self.h_grads["cam_grad"]
        self.last_h2d_bytes = 4 * self.h_upstream.numel()
        self.last_d2h_bytes = 4 * self.h_image.numel() + self._compact.last_bytes + 4 * 32
        return self.h_image, grads

    def set_scene(self, pos, rad, opa, feat, bg):
        """Stage a (new) scene: uploaded by the next render_step, resident afterwards."""
        for dst, src, shape in ((self.h_pos, pos, (self.m, 3)), (self.h_rad, rad, (self.m,)),
                                (self.h_opa, opa, (self.m,)), (self.h_feat, feat, (self.m, self.d)),
                                (self.h_bg, bg, (self.d,))):
            dst.copy_(torch.from_numpy(np.ascontiguousarray(src)).view(shape))
        self._scene_dirty = True

    def render_step(self, cams, upstream_fn=None, gamma=0.1, eps=1e-2, tau=0.01, normalize=True, gate=True,
                    check=False, reduce_fn=None, compact=False, always_upload=False, pipeline=True, graph=False):
        """One host-to-host step over one or more views of the staged scene:
        [H2D scene if set_scene was called since the last step]; per view: ss_forward, D2H image,
        [upstream_fn(view, host image) -> host upstream, else the staged h_upstream], H2D upstream, ss_backward
        (gradients summed over the views); optional reduce_fn(out) (the multi-GPU allreduce); D2H gradients
        (dense block, or compact rows of the touched spheres).  Returns after the streams are synchronised,
        with the last image and the gradient views (pinned host tensors).
        graph=True: a one-view step with the staged upstream (no upstream_fn), compact rows and a resident scene is
        replayed from a CUDA graph captured on its first use (same results; any other combination is enqueued call
        by call as without the flag)."""
        if not isinstance(cams, (list, tuple)):
            cams = [cams]
        dev = self.engine.device
        main = torch.cuda.current_stream(dev)
        h2d = 0
        # graph=True: a one-view step with a staged upstream and compact rows is replayed from a CUDA graph (any other
        # combination takes the stream-launched path below)
        if (graph and len(cams) == 1 and upstream_fn is None and not check and reduce_fn is None and compact
                and not always_upload and not self._scene_dirty):
            return self._render_step_graphed(cams[0], gamma, eps, tau, normalize, gate)
        if self._scene_dirty or always_upload:
            self.d_in.copy_(self.h_in, non_blocking=True)
            self._scene_dirty = False
            h2d += 4 * self.h_in.numel()
        if upstream_fn is None and not check and len(cams) > 1 and pipeline:
            h2d += self._views_pipelined(cams, gamma, eps, tau, normalize, gate, main)
            cams_serial = []
        else:
            cams_serial = cams
        for i, cam in enumerate(cams_serial):
            if upstream_fn is None:  # upstream already staged on the host: upload it under the forward pass
                self.copy_stream.wait_stream(main)  # (orders it after the previous view's backward)
                with torch.cuda.stream(self.copy_stream):
                    self.upstream.copy_(self.h_upstream, non_blocking=True)
            # the image is drawn in bands of tile rows; the copy stream downloads band b as soon as its event has
            # completed, i.e. while the raster kernel of band b + 1 is running (and the last band under the backward)
            # Only the LAST view of a step is banded: an earlier view's download hides under the next view's
            # forward pass anyway, and a band boundary costs a few microseconds of raster time.
            nb = self.bands if (not check and i == len(cams_serial) - 1) else 1  # (check=True may re-render after a regrowth)
            events = self._band_events[:nb] if nb > 1 else None
            if i > 1:  # this image buffer was last used two views ago: its download must have read it
                main.wait_event(self._image_copied[i & 1])
            if check:
                f = self.engine.forward(self.pos, self.rad, self.opa, self.feat, self.bg, cam, gamma=gamma, eps=eps,
                                        tau=tau, top_k=self.k, check=True, band_events=events)
                image = f["image"]
            else:
                image = self._images[i & 1]
                with torch.cuda.device(dev):
                    self._forward_fast(cam, gamma, eps, tau, events, main, image)
                f = None
            if upstream_fn is None:
                main.wait_stream(self.copy_stream)  # backward needs the uploaded upstream
            with torch.cuda.stream(self.copy_stream):
                if events:
                    for b, ev in enumerate(events):
                        r0, r1 = self._band_rows[b]
                        self.copy_stream.wait_event(ev)
                        if r1 > r0:
                            self.h_image[r0:r1].copy_(image[r0:r1], non_blocking=True)
                else:
                    self.copy_stream.wait_stream(main)
                    self.h_image.copy_(image, non_blocking=True)
                image.record_stream(self.copy_stream)
                self._image_copied[i & 1].record(self.copy_stream)
            if upstream_fn is not None:
                self.copy_stream.synchronize()
                self.h_upstream.copy_(upstream_fn(i, self.h_image))
                self.upstream.copy_(self.h_upstream, non_blocking=True)
            h2d += 4 * self.h_upstream.numel()
            if f is not None:
                self.engine.backward(self.pos, self.rad, self.opa, self.feat, self.bg, cam, f, self.upstream,
                                     gamma=gamma, eps=eps, normalize=normalize, gate=gate, camera_grads=True,
                                     out=self.out, accumulate=(i > 0))
            else:
                with torch.cuda.device(dev):
                    self._backward_fast(cam, gamma, eps, normalize, gate, i > 0, main)
        if reduce_fn is not None:
            reduce_fn(self.out)
        d2h = len(cams) * 4 * self.h_image.numel()
        if compact:
            if self._compact is None:
                self._compact = CompactGradients(self.m, self.d, dev)
            grads = self._compact.gather(self.out, main)
            self.h_out[self.packed.cam_off:].copy_(self.d_out[self.packed.cam_off:], non_blocking=True)
            grads["cam_grad"] = self.h_grads["cam_grad"]
            d2h += self._compact.last_bytes + 4 * 32
        else:
            self.packed.download()
            grads = self.h_grads
            d2h += self.packed.nbytes()
        main.synchronize()
        self.copy_stream.synchronize()
        self.last_h2d_bytes, self.last_d2h_bytes = h2d, d2h
        return self.h_image, grads

    def bytes_per_step(self, views: int):
        """(h2d, d2h) bytes of the LAST render_step (counted from the tensors that were copied)."""
        return self.last_h2d_bytes, self.last_d2h_bytes
