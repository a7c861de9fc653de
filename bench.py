#!/usr/bin/env python
"""Headline benchmark: fwd+bwd of the differentiable sphere renderer, BASELINE.json config 3
(1M spheres @ 1024x1024, n_track = 5, all gradients incl. camera), frames/s.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One process per GPU (under torchrun for N > 1; RANK/LOCAL_RANK/WORLD_SIZE from the env).
A step = every rank renders `views_per_rank` views of the shared scene (forward + backward each,
gradients accumulated) and, for N > 1, one sum-allreduce of the sphere-gradient buffer.  N = 1
runs config 3 itself (1 view, identity camera); N > 1 runs config 4's orbit, 8 views per rank
(64 views at N = 8), weak scaling.

Timing: CUDA events on the launching stream around each step, L2 flushed (256 MB write) between
steps outside the timed region, max over ranks.  The step is `ViewShardedRenderer.graphed_step`: its
local work is captured once into a CUDA graph and replayed (what a training loop over a fixed set of
cameras runs); `stream_launches` in the line is the same step enqueued kernel by kernel.
`--impl reference` times the unmodified reference's own CPU path (baseline/_ref, one core; its float64
C port on all host threads is reported beside it) on the same config.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

COUNT, SIZE, TOP_K, D = 1_000_000, 1024, 5, 3
GAMMA, EPS, TAU = 0.1, 1e-2, 0.01
NCU_KERNELS_JSON = "profiles/ncu_kernels.json"  # per-kernel ncu --set full figures, written by scripts/ncu_extract.py
METRIC = "fwd+bwd frames/s, 1M spheres @1024^2 n_track=5 (ms/frame = ms_per_step / views_per_rank)"
WORKLOAD = ("C3: 1M uniform 3px spheres (cli.py:_benchmark_scene, seed 0), 1024x1024, d=3, n_track=5, "
            "gamma=0.1 eps=0.01 tau=0.01, full fwd+bwd incl. camera gradients, upstream=sign(image-0.5)")


class ClockSampler(threading.Thread):
    """Samples SM clock and throttle reasons through NVML while the timed region runs."""

    def __init__(self, index: int, period: float = 0.01):
        super().__init__(daemon=True)
        self.index, self.period = index, period
        self.samples, self.reasons, self.sm_max = [], set(), None
        self._halt = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.sm_max = int(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.ok = True
        except Exception:
            self.ok = False

    def _sample(self):
        nv = self.nv
        self.samples.append(int(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
        try:
            r = int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
        except Exception:
            r = int(nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h))
        names = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
                 0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting",
                 0x100: "display_clock_setting", 0x10: "sync_boost"}
        for bit, name in names.items():
            if r & bit:
                self.reasons.add(name)

    def run(self):
        if not self.ok:
            return
        while not self._halt.is_set():
            try:
                self._sample()
            except Exception:
                pass
            self._halt.wait(self.period)

    def stop(self):
        self._halt.set()
        if self.ok and not self.samples:
            try:
                self._sample()
            except Exception:
                pass
        return {"sm_mhz": (float(np.median(self.samples)) if self.samples else None), "sm_max_mhz": self.sm_max,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def algorithmic_bytes(T, S, U, M=COUNT, P=SIZE * SIZE, d=D, K=TOP_K):
    """SURVEY.md 8(d) byte model (float32 device layout).  T pairs, S filled slots, U touched spheres."""
    fwd = M * (20 + 4 * d) + 8 * T + T * (24 + 4 * d) + P * (4 * d + 4) + P * (12 * K + 4)
    bwd = P * (12 * K + 4) + P * 4 * d + U * (20 + 4 * d) + 2 * M * (32 + 4 * d) + M * (24 + 4 * d)
    raster = T * (4 + 24 + 4 * d) + P * (4 * d + 4) + P * (12 * K + 4)
    # k_project: inputs read once, 96 B of records / keys / rectangles / filter per sphere + 4 B per tile bucket entry
    project = M * (20 + 4 * d) + M * 96 + 4 * T
    # k_backward: buffer + upstream read, one gather and one accumulator row per touched sphere
    backward = P * (12 * K + 4) + P * 4 * d + U * (20 + 4 * d) + U * (32 + 4 * d)
    return fwd, bwd, {"k_raster": raster, "k_project": project, "k_backward": backward}


def host_threads():
    """Host cores this process may use (torchrun exports OMP_NUM_THREADS=1, so do not ask OpenMP)."""
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return max(1, os.cpu_count() or 1)


def cpu_frame_seconds(threads, repeats=1):
    """One full C3 frame (fwd + bwd) on the CPU oracle port of the reference; returns seconds/frame."""
    from oracle import oracle as orc
    from paper_2004_07484_b200.synthetic import benchmark_scene
    pos, rad, opa, feat, bg, vec = benchmark_scene(COUNT, SIZE, SIZE, seed=0)
    cam = orc.camera_from_vector(vec, SIZE, SIZE)
    best = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        f = orc.render_forward(pos, rad, opa, feat, bg, cam, gamma=GAMMA, eps=EPS, tau=TAU, top_k=TOP_K,
                               threads=threads, validate=True)
        up = np.sign(f["image"] - 0.5)
        orc.render_backward(pos, rad, opa, feat, bg, cam, f, up, threads=threads)
        best.append(time.perf_counter() - t0)
    return best


def reference_package():
    """The unmodified reference (pure Python / NumPy), installed by __graft_entry__.build() into the
    git-ignored baseline/_ref, or None.  /root/reference itself is never read at run time."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "softsphere")):
        return None
    if ref_dir not in sys.path:
        sys.path.append(ref_dir)
    try:
        import softsphere
        return softsphere
    except Exception:
        return None


def reference_frame_seconds(ss, frames=1, budget_s=150.0):
    """Full C3 frames through the reference's own render_forward / render_backward (cli.py:377-389 protocol:
    float64, workers=1 -- its thread pool does not scale under the GIL), as many of `frames` as fit the budget."""
    from paper_2004_07484_b200.synthetic import benchmark_scene
    pos, rad, opa, feat, bg, vec = benchmark_scene(COUNT, SIZE, SIZE, seed=0)
    scene = ss.new_scene(D, bg.astype(np.float64))
    scene.positions, scene.radii = pos.astype(np.float64), rad.astype(np.float64)
    scene.opacities, scene.features = opa.astype(np.float64), feat.astype(np.float64)
    cam = ss.camera_from_vector(vec, SIZE, SIZE)
    params = ss.BlendParams(gamma=GAMMA, epsilon=EPS, tau=TAU, top_k=TOP_K)
    times, t_start = [], time.perf_counter()
    for _ in range(frames):
        t0 = time.perf_counter()
        image, buf, _ = ss.render_forward(scene, cam, params, workers=1)
        ss.render_backward(scene, cam, params, buf, np.sign(image.data - 0.5), workers=1)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start + times[-1] > budget_s:
            break
    return times


def cpu_baseline_block(threads, frames=1, budget_s=150.0):
    """cpu_baseline for the JSON line: the real reference when it is installed (kind "reference", 1 core),
    else the float64 C port of it (kind "port", OpenMP over tiles)."""
    ss = reference_package()
    port = cpu_frame_seconds(threads, repeats=1)[0]
    if ss is not None:
        times = reference_frame_seconds(ss, frames, budget_s)
        total = float(np.sum(times))
        return times, {"value": len(times) / total, "unit": "frames/s", "cores": 1, "kind": "reference",
                       "sample": f"{len(times)} full C3 frame(s) (fwd+bwd, tau=0.01) through the unmodified reference's "
                                 "render_forward/render_backward from baseline/_ref, float64, workers=1 (its thread "
                                 "pool does not scale under the GIL)",
                       "port": {"value": 1.0 / port, "unit": "frames/s", "cores": threads,
                                "note": "oracle/ss_oracle.c, the float64 C restatement, OpenMP over tiles"}}
    return [port], {"value": 1.0 / port, "unit": "frames/s", "cores": threads, "kind": "port",
                    "sample": "1 full C3 frame (fwd+bwd, tau=0.01) on the float64 oracle port, OpenMP over tiles "
                              "(baseline/_ref not installed on this box)"}


def run_reference(args, rank):
    """CPU arm: the reference's own CPU implementation of the path on this box's host cores (rank 0 only;
    under torchrun the other ranks exit without work -- the CPU arm does not scale with --gpus)."""
    if rank != 0:
        return
    from oracle import oracle as orc
    orc.build()
    threads = host_threads()
    times, block = cpu_baseline_block(threads, frames=max(1, min(args.steps, 3)))
    total = float(np.sum(times))
    value = len(times) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": len(times), "warmup": 0, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "views_per_rank": 1,
                   "note": "CPU arm: runs on rank 0 only and does not scale with --gpus; frames are whole C3 frames, "
                           "bounded to ~150 s of CPU time (no warm-up frame: a frame takes about a minute)"},
        "cpu_baseline": block,
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--views-per-rank", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    args.warmup = max(args.warmup, 3)

    import torch
    import torch.distributed as dist
    from paper_2004_07484_b200 import CameraSpec, RenderEngine, _lib, camera_from_vector
    from paper_2004_07484_b200.host import HostRenderSession
    from paper_2004_07484_b200.multiview import SphereGradBuffer, ViewShardedRenderer
    from paper_2004_07484_b200.synthetic import benchmark_scene, orbit_camera_vectors

    assert torch.cuda.is_available(), "bench.py needs a CUDA device (no CPU fallback)"
    # One GPU per rank.  SS_DIST_BACKEND=gloo lets several ranks share a GPU to smoke-test the N > 1 code
    # path on a single-GPU box (NCCL refuses duplicate devices); the real run uses NCCL over NVLink.
    backend = os.environ.get("SS_DIST_BACKEND", "nccl")
    dev_index = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(dev_index)
    device = torch.device("cuda", dev_index)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group(backend)
    vpr = args.views_per_rank or (1 if world == 1 else 8)
    n_views = vpr * world

    pos, rad, opa, feat, bg, vec = benchmark_scene(COUNT, SIZE, SIZE, seed=0)
    scene = tuple(torch.from_numpy(x).to(device) for x in (pos, rad, opa, feat, bg))
    cam_vecs = [vec] if n_views == 1 else orbit_camera_vectors(64)[:n_views] if n_views <= 64 else \
        orbit_camera_vectors(n_views)
    cams = [CameraSpec.from_camera(camera_from_vector(v, SIZE, SIZE)) for v in cam_vecs]

    eng = RenderEngine(device)
    mv = ViewShardedRenderer(eng)
    # upstream per local view = sign(image - 0.5) (cli.py:384), computed once outside the timed region
    upstreams, status = {}, None
    for v in mv.local_views(n_views):
        f = eng.forward(*scene, cams[v], gamma=GAMMA, eps=EPS, tau=TAU, top_k=TOP_K, collect_stats=True)
        upstreams[v] = torch.sign(f["image"] - 0.5)
        status = f["status"]
        filled = int((f["ids"] >= 0).sum().item())

    # (allocated after the engine's workspace: k_project streams through ten per-sphere arrays at once and its time
    # moves between 56 and 90 us with where the allocator places them relative to each other -- scripts/bench_probe.py;
    # workspace first, gradient buffers second is the 56 us order)
    grads = SphereGradBuffer(COUNT, D, device)

    def upstream_fn(v, image):
        return upstreams[v]

    def step():
        return mv.step(scene, cams, upstream_fn, grads, gamma=GAMMA, eps=EPS, tau=TAU, top_k=TOP_K,
                       normalize=True, gate=True, camera_grads=True, check=False)

    def upstream_fn_timed(v, image):  # a second function OBJECT: a second capture of the same step (see below)
        return upstreams[v]

    def graphed(timed=True):
        return mv.graphed_step(scene, cams, upstream_fn_timed if timed else upstream_fn, grads, gamma=GAMMA, eps=EPS,
                               tau=TAU, top_k=TOP_K, normalize=True, gate=True, camera_grads=True)

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)
    # ---- headline: the step as the training loop of a fixed camera set runs it -- the local work of the step (all
    # kernels of all local views, both pipeline streams, the upstream callback) captured once into a CUDA graph and
    # replayed (ViewShardedRenderer.graphed_step); the collective of an N > 1 step stays outside the graph.  The
    # dominant kernel's in-step launch duration feeds `roofline`: the step is captured twice, once with one EXTERNAL
    # event-record pair around k_raster inside the graph and once without, and every `sample_every`-th timed step
    # replays the capture with the pair (read back after that step: a device synchronisation outside the event
    # brackets).  A pair costs ~12 us inside a graph -- 2.5 % of the step -- so it is not paid on every step.
    sample_every = max(1, min(10, args.steps // 4))  # >= 4 timed launches whenever there are >= 4 steps
    _lib.profile_captured_reset()
    use_graph = True
    try:
        _lib.profile_enable_only(["k_raster"])
        for _ in range(args.warmup):
            flush.zero_()
            graphed(timed=True)
        torch.cuda.synchronize()
        if sample_every > 1:
            _lib.profile_enable(False)
            for _ in range(args.warmup):
                flush.zero_()
                graphed(timed=False)
            torch.cuda.synchronize()
            _lib.profile_enable_only(["k_raster"])
    except Exception as exc:  # capture refused (driver / torch mismatch): time the stream-launched step instead
        print(f"bench: CUDA-graph capture failed ({exc!r}); the headline falls back to stream launches", file=sys.stderr)
        use_graph = False
        _lib.profile_enable_only(["k_raster"])
        torch.cuda.synchronize()
        for _ in range(args.warmup):
            flush.zero_()
            step()
    torch.cuda.synchronize()
    _lib.profile_collect()  # (drop the stream-launched warm-up pairs of the capture)
    l0 = _lib.launch_count()
    step()  # kernels per step, counted on one stream-launched step (a replay does not pass through the counter)
    launches_per_step = _lib.launch_count() - l0
    _lib.profile_collect()
    touched = int((grads.pixel_count > 0).sum().item())
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(dev_index)
    sampler.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    raster_ms, raster_n = 0.0, 0
    torch.cuda.synchronize()
    for i, (a, b) in enumerate(ev):
        sampled = not use_graph or i % sample_every == 0
        flush.zero_()
        a.record()
        if use_graph:
            graphed(timed=sampled)
        else:
            step()
        b.record()
        if sampled:
            got = (_lib.profile_collect_captured() if use_graph else _lib.profile_collect()).get("k_raster", (0.0, 0))
            raster_ms, raster_n = raster_ms + got[0], raster_n + got[1]  # (the collect synchronises)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    prof = {"k_raster": (raster_ms, raster_n)}
    launches = launches_per_step * args.steps
    total_ms = float(sum(a.elapsed_time(b) for a, b in ev))
    # ---- the same step with plain stream launches (mv.step), same flush / event protocol, one event pair around
    # k_raster: what a caller pays who changes cameras or parameters every step
    s_steps = max(3, min(args.steps, 50))
    for _ in range(3):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    _lib.profile_collect()
    sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(s_steps)]
    for a, b in sev:
        flush.zero_()
        a.record()
        step()
        b.record()
    torch.cuda.synchronize()
    stream_prof = _lib.profile_collect()
    stream_ms = float(sum(a.elapsed_time(b) for a, b in sev))
    # per-kernel breakdown: a short extra pass with every kernel bracketed by events (stream launches)
    _lib.profile_enable(True)
    for _ in range(min(args.steps, 20)):
        flush.zero_()
        step()
    breakdown = _lib.profile_collect()
    _lib.profile_enable(False)
    if world > 1:
        t = torch.tensor([total_ms, stream_ms], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, stream_ms = float(t[0].item()), float(t[1].item())
    value = n_views * args.steps / (total_ms / 1e3)

    # ---- end to end with HOST buffers (copies inside the timed region, wall clock around synchronised steps)
    local = mv.local_views(n_views)
    local_cams = [cams[v] for v in local]
    e2e_steps = max(3, min(args.steps, 20))

    def reduce_fn(out):  # multi-GPU: sphere gradients are reduced on the device before the download
        if world > 1:
            for k in ("d_pos", "d_rad", "d_opa", "d_feat", "pixel_count"):
                dist.all_reduce(out[k])

    def timed(fn, steps):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            fn()
        torch.cuda.synchronize()
        secs = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([secs], dtype=torch.float64, device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            secs = float(t.item())
        return n_views * steps / secs

    # (1) `e2e`: the C-ABI session call.  Pinned host buffers; the scene is uploaded when it changes (set_scene)
    #     and stays resident; every step uploads the upstream image and downloads the image and the gradient
    #     rows of the spheres that received gradient (device-side compaction).
    sess = HostRenderSession(COUNT, D, SIZE, SIZE, TOP_K, engine=eng)
    sess.set_scene(pos, rad, opa, feat, bg)
    sess.h_upstream.copy_(upstreams[local[0]].cpu())
    compact = world == 1  # the allreduced buffer of a multi-GPU step is dense
    e2e_stream = timed(lambda: sess.render_step(local_cams, gamma=GAMMA, eps=EPS, tau=TAU, reduce_fn=reduce_fn,
                                                compact=compact), e2e_steps)
    h2d_b, d2h_b = sess.bytes_per_step(len(local_cams))
    # one view per step on one GPU: the same call with graph=True -- launches and copies of the step captured once and
    # replayed (the host needs 0.15 ms to enqueue them one by one, during which the GPU waits between the short
    # kernels of the forward pass); every other combination has no captured form and keeps the stream-launched figure
    e2e_graphed = world == 1 and len(local_cams) == 1
    e2e_graph_error = None
    if e2e_graphed:
        try:
            e2e_value = timed(lambda: sess.render_step(local_cams, gamma=GAMMA, eps=EPS, tau=TAU, compact=True,
                                                       graph=True), e2e_steps)
            h2d_b, d2h_b = sess.bytes_per_step(len(local_cams))
        except Exception as exc:  # reported in the line (e2e.graph_error); e2e then is the stream-launched figure
            e2e_graph_error = repr(exc)
            e2e_graphed = False
            torch.cuda.synchronize()
            e2e_value = e2e_stream
    else:
        e2e_value = e2e_stream
    # (2) the same session re-uploading the whole scene and downloading all M gradient rows every step
    #     (what round 1 reported as e2e: a scene that changes on the host between steps)
    e2e_dense = timed(lambda: sess.render_step(local_cams, gamma=GAMMA, eps=EPS, tau=TAU, reduce_fn=reduce_fn,
                                               compact=False, always_upload=True), e2e_steps)
    dense_h2d, dense_d2h = sess.bytes_per_step(len(local_cams))
    # (3) `e2e_plugin`: the reference-facing plug-in call itself -- SoftsphereAdapter.forward / .backward on a
    #     SphereScene of float64 NumPy columns, NumPy image / SceneGradients out (optim.py:265-304), N = 1 only
    plugin = None
    if world == 1:
        import paper_2004_07484_b200 as pk
        scene_np = pk.new_scene(D, bg.astype(np.float64))
        scene_np.positions, scene_np.radii = pos.astype(np.float64), rad.astype(np.float64)
        scene_np.opacities, scene_np.features = opa.astype(np.float64), feat.astype(np.float64)
        cam_np = camera_from_vector(cam_vecs[0], SIZE, SIZE)
        params_np = pk.BlendParams(gamma=GAMMA, epsilon=EPS, tau=TAU, top_k=TOP_K)
        adapter = pk.SoftsphereAdapter(engine=eng)

        # protocol of the reference's own benchmark (cli.py:378-389): forward and backward are timed, the host
        # upstream sign(image - 0.5) between them is the caller's NumPy work and is not
        plug_steps = max(3, min(args.steps, 20))
        t_f = t_b = 0.0
        for it in range(plug_steps + 3):
            t0 = time.perf_counter()
            image, buf, _ = adapter.forward(scene_np, cam_np, params_np)
            t1 = time.perf_counter()
            up_np = np.sign(image.data - 0.5)
            t2 = time.perf_counter()
            adapter.backward(scene_np, cam_np, params_np, buf, up_np)
            t3 = time.perf_counter()
            if it >= 3:  # 3 warm-up frames
                t_f += t1 - t0
                t_b += t3 - t2
        plugin = {"value": plug_steps / (t_f + t_b), "unit": "frames/s", "steps": plug_steps,
                  "forward_ms": 1e3 * t_f / plug_steps, "backward_ms": 1e3 * t_b / plug_steps,
                  "h2d_bytes_per_step": 4 * (COUNT * (5 + D) + D) + 4 * SIZE * SIZE * D,
                  "d2h_bytes_per_step": 4 * SIZE * SIZE * (D + 1) + 4 * (COUNT * (6 + D) + 32),
                  "path": "SoftsphereAdapter.forward / .backward(SphereScene float64 NumPy, Camera, BlendParams), each "
                          "call returning synchronised NumPy results: float64 columns narrowed into pinned staging + "
                          "1 H2D, ss_forward, image + bg_weight -> float64 NumPy | upstream float64 -> pinned + H2D, "
                          "ss_backward (scene upload shared with the forward call), all gradients -> float64 NumPy; "
                          "the host-side upstream sign(image - 0.5) between the calls is not timed (cli.py:378-389)"}

    if rank == 0:
        peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
        if os.path.exists(peaks_path):
            peak, peak_src = float(json.load(open(peaks_path))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        else:
            peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
        T = status["num_pairs"]
        fwd_b, bwd_b, kbytes = algorithmic_bytes(T, filled, touched)
        try:
            ncu = json.load(open(os.path.join(ROOT, NCU_KERNELS_JSON)))
        except Exception:
            ncu = {}
        sm_mhz = clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 1965.0
        per_kernel = {}
        for kname, nbytes in kbytes.items():
            ms_k, n_k = prof.get(kname, (0.0, 0))
            timed_in = "timed region"
            if not n_k:  # not bracketed inside the timed region: the separate all-kernels pass
                ms_k, n_k = breakdown.get(kname, (0.0, 0))
                timed_in = "separate pass (every kernel bracketed by events)"
            if not n_k:
                continue
            us = 1e3 * ms_k / n_k
            gbs = nbytes / (us * 1e-6) / 1e9
            entry = {"avg_launch_us": us, "launches_timed": n_k, "timed_in": timed_in,
                     "algorithmic_bytes_per_launch": nbytes,
                     "achieved_GBps": gbs, "frac": gbs / peak}
            nk = ncu.get(kname)
            if nk:
                entry["traffic"] = nk.get("dram_bytes")
                if nk.get("inst_executed"):
                    # time the launch would take if one of the 4 x 148 warp schedulers issued an instruction every cycle
                    issue_us = nk["inst_executed"] / (592.0 * sm_mhz)
                    entry["issue_frac"] = issue_us / us
                    entry["warp_instructions"] = nk["inst_executed"]
            per_kernel[kname] = entry
        rk = per_kernel.get("k_raster", {})
        raster_ms = rk.get("avg_launch_us", 0.0) / 1e3
        achieved = rk.get("achieved_GBps", 0.0)
        step_ms = total_ms / args.steps / vpr
        kernels = {k: {"us": round(1e3 * ms / n, 2), "launches": n} for k, (ms, n) in breakdown.items() if n}
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 blend + f64 geometry", "data": "synthetic",
            "config": {"workload": WORKLOAD, "views_per_rank": vpr, "views_total": n_views,
                       "cache": "L2 flushed between timed steps (256 MB write, outside the timed region)",
                       "pairs_T": T, "filled_slots_S": filled, "touched_spheres_U": touched,
                       "step_path": ("ViewShardedRenderer.graphed_step: the step's kernels replayed from one CUDA graph "
                                     "(captured once; fixed cameras, scene tensors updated in place)" if use_graph else
                                     "ViewShardedRenderer.step, stream launches (CUDA-graph capture failed on this box)"),
                       "timed_region_note": f"every {sample_every}-th timed step replays a second capture of the same "
                                            "step that carries 1 external CUDA-event pair around k_raster (read back "
                                            "after that step; the pair costs ~12 us of a step, the other steps replay "
                                            "the capture without it): roofline.kernels.k_raster.launches_timed of the "
                                            "timed region's launches; k_project / k_backward durations come from the "
                                            "separate stream-launched all-kernels pass",
                       "collective": ("none" if world == 1 else
                                      f"1 {backend} sum-allreduce group of {grads.allreduce_bytes()} B per step")},
            "clocks": clocks,
            "e2e": {"value": e2e_value, "unit": "frames/s", "h2d_bytes_per_step": h2d_b, "d2h_bytes_per_step": d2h_b,
                    "steps": e2e_steps,
                    "stream_launched_value": e2e_stream,
                    "graph_replay": bool(e2e_graphed), "graph_error": e2e_graph_error,
                    "path": ("[the step's launches and copies replayed from one CUDA graph, render_step(graph=True); "
                             "stream_launched_value is the same step enqueued call by call] " if e2e_graphed else "") +
                            "HostRenderSession.render_step (C ABI, pinned host buffers): scene resident on the device "
                            "(uploaded by set_scene when it changes), argument blocks prepared once; per step and view upstream "
                            "H2D, ss_forward (last view: ss_forward_banded, 2 bands of tile rows, each band's image rows "
                            "downloaded as soon as its event completes), image D2H, ss_backward; then " +
                            ("the gradient rows of the touched spheres (index + count + grads) compacted on the device, "
                             "the compaction kernel writing the records straight into the mapped pinned host array "
                             "(counted in d2h_bytes_per_step), + camera block D2H" if compact else
                             "the allreduce of the sphere gradients and one D2H block with all M gradient rows")},
            "e2e_dense_reupload": {"value": e2e_dense, "unit": "frames/s", "h2d_bytes_per_step": dense_h2d,
                                   "d2h_bytes_per_step": dense_d2h,
                                   "path": "same call, whole scene uploaded and all M gradient rows downloaded every step "
                                           "(round 1's e2e)"},
            "stream_launches": {"value": n_views * s_steps / (stream_ms / 1e3), "unit": "frames/s",
                                "ms_per_step": stream_ms / s_steps, "steps": s_steps,
                                "k_raster_us": (1e3 * stream_prof["k_raster"][0] / max(1, stream_prof["k_raster"][1])
                                                if "k_raster" in stream_prof else None),
                                "path": "ViewShardedRenderer.step: the same step enqueued kernel by kernel on the "
                                        "stream (no graph), same flush and event protocol, one event pair around "
                                        "k_raster"},
            "gpu_launches": int(launches),
            "roofline": {"kernel": "k_raster", "bound": "hbm", "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": rk.get("traffic"),
                         "issue_frac": rk.get("issue_frac"),
                         "traffic_source": f"dram__bytes_read.sum + dram__bytes_write.sum of one launch, ncu --set full, "
                                           f"{ncu.get('_source', 'unavailable')} via {NCU_KERNELS_JSON}",
                         "issue_bound_note": "k_raster is instruction-issue bound, not HBM bound (SURVEY 8d): issue_frac = "
                                             "warp instructions (ncu) / (592 schedulers x SM clock) / measured launch time",
                         "peak_source": peak_src, "algorithmic_bytes_per_launch": kbytes["k_raster"],
                         "avg_launch_ms": raster_ms,
                         "kernels": per_kernel,
                         "step": {"algorithmic_bytes_fwd": fwd_b, "algorithmic_bytes_bwd": bwd_b,
                                  "ms_per_frame": step_ms,
                                  "achieved_GBps": (fwd_b + bwd_b) / (step_ms * 1e-3) / 1e9,
                                  "frac": (fwd_b + bwd_b) / (step_ms * 1e-3) / 1e9 / peak},
                         "kernels_separate_pass": kernels},
        }
        if plugin is not None:
            line["e2e_plugin"] = plugin
        if world == 1 and not args.no_cpu_baseline:
            from oracle import oracle as orc
            orc.build()
            _, line["cpu_baseline"] = cpu_baseline_block(host_threads(), frames=1)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
