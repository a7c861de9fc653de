"""External event pairs inside a captured step: do they read the right duration, what do they cost?  (probe)"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2004_07484_b200 import CameraSpec, RenderEngine, _lib, camera_from_vector
from paper_2004_07484_b200.multiview import SphereGradBuffer, ViewShardedRenderer
from paper_2004_07484_b200.synthetic import benchmark_scene

pos, rad, opa, feat, bg, vec = benchmark_scene(1_000_000, 1024, 1024, seed=0)
scene = tuple(torch.from_numpy(x).cuda() for x in (pos, rad, opa, feat, bg))
cams = [CameraSpec.from_camera(camera_from_vector(vec, 1024, 1024))]
eng = RenderEngine("cuda")
f = eng.forward(*scene, cams[0], gamma=0.1, tau=0.01)
up = torch.sign(f["image"] - 0.5)
grads = SphereGradBuffer(1_000_000, 3, "cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
kw = dict(gamma=0.1, eps=1e-2, tau=0.01, top_k=5)


def upstream_fn(v, im):
    return up


for names in ([], ["k_raster"], ["k_raster", "k_project", "k_backward"]):
    mv = ViewShardedRenderer(eng)
    _lib.profile_captured_reset()
    _lib.profile_enable_only(names)
    for _ in range(5):
        flush.zero_(); mv.graphed_step(scene, cams, upstream_fn, grads, **kw)
    torch.cuda.synchronize()
    ts, ks = [], []
    for _ in range(50):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush.zero_(); a.record(); mv.graphed_step(scene, cams, upstream_fn, grads, **kw); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
        if names:
            ks.append({k: v[0] for k, v in _lib.profile_collect_captured().items() if v[1]})
    _lib.profile_enable(False)
    kavg = {k: round(1e3 * np.mean([x[k] for x in ks]), 1) for k in (ks[0] if ks else {})}
    print(f"captured pairs {names}: {np.mean(ts):.4f} ms per step (per-step sync), kernels (us): {kavg}", flush=True)
