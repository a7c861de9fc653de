"""Repeat timing of HostRenderSession.render_step (development aid)."""
import os, sys, time
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2004_07484_b200 import CameraSpec, RenderEngine, camera_from_vector
from paper_2004_07484_b200.host import HostRenderSession
from paper_2004_07484_b200.synthetic import benchmark_scene
pos, rad, opa, feat, bg, vec = benchmark_scene(1_000_000, 1024, 1024, seed=0)
cam = CameraSpec.from_camera(camera_from_vector(vec, 1024, 1024))
eng = RenderEngine("cuda")
for bands in (1, 2, 2, 1, 4, 2):
    s = HostRenderSession(1_000_000, 3, 1024, 1024, 5, engine=eng, bands=bands)
    s.set_scene(pos, rad, opa, feat, bg)
    s.h_upstream.copy_(torch.sign(torch.rand(1024, 1024, 3) - 0.5))
    for _ in range(5):
        s.render_step([cam], gamma=0.1, eps=1e-2, tau=0.01, compact=True)
    res = []
    for rep in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(20):
            s.render_step([cam], gamma=0.1, eps=1e-2, tau=0.01, compact=True)
        torch.cuda.synchronize()
        res.append(20 / (time.perf_counter() - t0))
    print(f"bands={bands}: " + " ".join(f"{r:.0f}" for r in res), flush=True)
    del s
