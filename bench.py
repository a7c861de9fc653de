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
steps outside the timed region, max over ranks.  `--impl reference` times the CPU implementation
(the float64 oracle port of the reference, all host threads) on the same config.
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
NCU_RASTER_DRAM_BYTES = 180_676_352  # one k_raster launch at this config: 117.48 MB read + 63.19 MB written (ncu, r01n)
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
    return fwd, bwd, raster


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


def run_reference(args, rank):
    """CPU arm: the oracle port of the reference (float64, OpenMP over tiles), all host threads."""
    if rank != 0:
        return
    from oracle import oracle as orc
    orc.build()
    threads = host_threads()
    warm = cpu_frame_seconds(threads) if args.warmup > 0 else []
    # bounded sample: full frames, as many of the K requested as fit in ~2 minutes of CPU time
    first = cpu_frame_seconds(threads, repeats=1)
    budget_frames = max(1, int(120.0 / max(first[0], 1e-3)))
    times = first + (cpu_frame_seconds(threads, repeats=min(args.steps, budget_frames) - 1)
                     if min(args.steps, budget_frames) > 1 else [])
    total = float(np.sum(times))
    value = len(times) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": len(times), "warmup": len(warm), "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "views_per_rank": 1},
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": threads, "kind": "port",
                         "sample": f"{len(times)} full C3 frame(s) of the {args.steps} requested (capped at ~120 s), "
                                   "fwd+bwd, tau=0.01, float64 oracle port, OpenMP over tiles"},
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
    grads = SphereGradBuffer(COUNT, D, device)
    # upstream per local view = sign(image - 0.5) (cli.py:384), computed once outside the timed region
    upstreams, status = {}, None
    for v in mv.local_views(n_views):
        f = eng.forward(*scene, cams[v], gamma=GAMMA, eps=EPS, tau=TAU, top_k=TOP_K, collect_stats=True)
        upstreams[v] = torch.sign(f["image"] - 0.5)
        status = f["status"]
        filled = int((f["ids"] >= 0).sum().item())

    def upstream_fn(v, image):
        return upstreams[v]

    def step():
        return mv.step(scene, cams, upstream_fn, grads, gamma=GAMMA, eps=EPS, tau=TAU, top_k=TOP_K,
                       normalize=True, gate=True, camera_grads=True, check=False)

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)
    for _ in range(args.warmup):
        flush.zero_()
        step()
    touched = int((grads.pixel_count > 0).sum().item())
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(dev_index)
    sampler.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = _lib.launch_count()
    _lib.profile_enable_only(["k_raster"])  # dominant kernel: one event pair per step inside the timed region
    torch.cuda.synchronize()
    for a, b in ev:
        flush.zero_()
        a.record()
        step()
        b.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    prof = _lib.profile_collect()
    launches = _lib.launch_count() - launches0
    # per-kernel breakdown: a short extra pass with every kernel bracketed by events (not the headline)
    _lib.profile_enable(True)
    for _ in range(min(args.steps, 20)):
        flush.zero_()
        step()
    breakdown = _lib.profile_collect()
    _lib.profile_enable(False)
    total_ms = float(sum(a.elapsed_time(b) for a, b in ev))
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = n_views * args.steps / (total_ms / 1e3)

    # ---- end to end through the host-buffer API (pinned host buffers, H2D + D2H inside the timed region)
    sess = HostRenderSession(COUNT, D, SIZE, SIZE, TOP_K, engine=eng)
    sess.set_scene(pos, rad, opa, feat, bg)
    local = mv.local_views(n_views)
    sess.h_upstream.copy_(upstreams[local[0]].cpu())
    e2e_steps = max(3, min(args.steps, 20))
    local_cams = [cams[v] for v in local]

    def reduce_fn(out):  # multi-GPU: sphere gradients are reduced on the device before the download
        if world > 1:
            for k in ("d_pos", "d_rad", "d_opa", "d_feat", "pixel_count"):
                dist.all_reduce(out[k])

    for _ in range(3):
        sess.render_step(local_cams, gamma=GAMMA, eps=EPS, tau=TAU, reduce_fn=reduce_fn)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        sess.render_step(local_cams, gamma=GAMMA, eps=EPS, tau=TAU, reduce_fn=reduce_fn)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    h2d_b, d2h_b = sess.bytes_per_step(len(local_cams))
    e2e_value = n_views * e2e_steps / e2e_s

    if rank == 0:
        peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
        if os.path.exists(peaks_path):
            peak, peak_src = float(json.load(open(peaks_path))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        else:
            peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
        T = status["num_pairs"]
        fwd_b, bwd_b, raster_b = algorithmic_bytes(T, filled, touched)
        ms_r, n_r = prof["k_raster"]
        raster_ms = ms_r / max(n_r, 1)
        achieved = raster_b / (raster_ms * 1e-3) / 1e9
        step_ms = total_ms / args.steps / vpr
        kernels = {k: {"us": round(1e3 * ms / n, 2), "launches": n} for k, (ms, n) in breakdown.items() if n}
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 blend + f64 geometry", "data": "synthetic",
            "config": {"workload": WORKLOAD, "views_per_rank": vpr, "views_total": n_views,
                       "cache": "L2 flushed between timed steps (256 MB write, outside the timed region)",
                       "pairs_T": T, "filled_slots_S": filled, "touched_spheres_U": touched,
                       "collective": ("none" if world == 1 else
                                      f"1 {backend} sum-allreduce of {grads.allreduce_bytes()} B per step")},
            "clocks": clocks,
            "e2e": {"value": e2e_value, "unit": "frames/s", "h2d_bytes_per_step": h2d_b, "d2h_bytes_per_step": d2h_b,
                    "steps": e2e_steps,
                    "path": "HostRenderSession.render_step: pinned host scene+upstream -> device, "
                            "ss_forward, image -> host, ss_backward, all gradients -> host"},
            "gpu_launches": int(launches),
            "roofline": {"kernel": "k_raster", "bound": "hbm", "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": NCU_RASTER_DRAM_BYTES,
                         "traffic_source": "dram__bytes_read.sum + dram__bytes_write.sum of one k_raster launch, "
                                           "ncu --set full, profiles/r01_summary.md (r01n)",
                         "issue_bound_note": "k_raster is instruction-issue bound, not HBM bound (SURVEY 8d): ncu "
                                             "smsp__issue_active 72%, 213 M warp instructions, l1tex (shared-memory wavefronts) 68%, DRAM 8% of peak",
                         "peak_source": peak_src, "algorithmic_bytes_per_launch": raster_b,
                         "avg_launch_ms": raster_ms,
                         "step": {"algorithmic_bytes_fwd": fwd_b, "algorithmic_bytes_bwd": bwd_b,
                                  "ms_per_frame": step_ms,
                                  "achieved_GBps": (fwd_b + bwd_b) / (step_ms * 1e-3) / 1e9,
                                  "frac": (fwd_b + bwd_b) / (step_ms * 1e-3) / 1e9 / peak},
                         "kernels_separate_pass": kernels},
        }
        if world == 1 and not args.no_cpu_baseline:
            from oracle import oracle as orc
            orc.build()
            threads = host_threads()
            secs = cpu_frame_seconds(threads, repeats=1)[0]
            line["cpu_baseline"] = {"value": 1.0 / secs, "unit": "frames/s", "cores": threads, "kind": "port",
                                    "sample": "1 full C3 frame (fwd+bwd, tau=0.01) on the float64 oracle port, "
                                              "OpenMP over tiles"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
