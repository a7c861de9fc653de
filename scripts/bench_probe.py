"""Why does bench.py's frame take 0.51 ms when quick_time.py's takes 0.484 ms?  (development probe)"""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2004_07484_b200 import CameraSpec, RenderEngine, _lib, camera_from_vector
from paper_2004_07484_b200.multiview import SphereGradBuffer, ViewShardedRenderer
from paper_2004_07484_b200.synthetic import benchmark_scene

pos, rad, opa, feat, bg, vec = benchmark_scene(1_000_000, 1024, 1024, seed=0)
scene = tuple(torch.from_numpy(x).cuda() for x in (pos, rad, opa, feat, bg))
cam = CameraSpec.from_camera(camera_from_vector(vec, 1024, 1024))
eng = RenderEngine("cuda")
mv = ViewShardedRenderer(eng)
if os.environ.get("PROBE_GRADS_FIRST", "1") == "1":
    grads = SphereGradBuffer(1_000_000, 3, "cuda")
f = eng.forward(*scene, cam, gamma=0.1, tau=0.01, collect_stats=True)
if os.environ.get("PROBE_GRADS_FIRST", "1") != "1":
    grads = SphereGradBuffer(1_000_000, 3, "cuda")
up = torch.sign(f["image"] - 0.5)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
N = 100


def direct():
    f = eng.forward(*scene, cam, gamma=0.1, eps=1e-2, tau=0.01, top_k=5, check=False)
    eng.backward(*scene, cam, f, up, gamma=0.1, eps=1e-2)


def direct_out():
    f = eng.forward(*scene, cam, gamma=0.1, eps=1e-2, tau=0.01, top_k=5, check=False)
    eng.backward(*scene, cam, f, up, gamma=0.1, eps=1e-2, out=dict(grads.as_out()), camera_grads=True)


def mvstep():
    mv.step(scene, [cam], lambda v, im: up, grads, gamma=0.1, eps=1e-2, tau=0.01, top_k=5, check=False)


def run(fn, prof):
    for _ in range(10):
        flush.zero_(); fn()
    torch.cuda.synchronize()
    if prof == "three":
        _lib.profile_enable_only(["k_raster", "k_backward", "k_project"])
    elif prof == "all":
        _lib.profile_enable(True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(N)]
    for a, b in ev:
        flush.zero_(); a.record(); fn(); b.record()
    torch.cuda.synchronize()
    p = _lib.profile_collect() if prof else {}
    _lib.profile_enable(False)
    ms = np.array([a.elapsed_time(b) for a, b in ev])
    kp = {k: round(1e3 * v[0] / v[1], 1) for k, v in p.items() if v[1] and k in ("k_project", "k_raster", "k_backward")}
    return f"{np.mean(ms):.4f} ms (median {np.median(ms):.4f}) {kp}"


for name, fn in (("direct", direct),):
    for prof in (None, "all"):
        print(f"{name:11s} prof={prof}: {run(fn, prof)}", flush=True)
