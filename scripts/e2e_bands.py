"""Band count of the banded forward pass inside the graph-replayed host-to-host step (development aid):
python scripts/e2e_bands.py  ->  e2e frames/s at C3 for 1 / 2 / 4 / 8 / 16 bands, two repeats each."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_07484_b200 as pk
from paper_2004_07484_b200.host import HostRenderSession
from paper_2004_07484_b200.synthetic import benchmark_scene

M, S = 1_000_000, 1024
pos, rad, opa, feat, bg, vec = benchmark_scene(M, S, S, seed=0)
cam = pk.CameraSpec.from_camera(pk.camera_from_vector(vec, S, S))
eng = pk.RenderEngine("cuda")
scene = tuple(torch.from_numpy(x).cuda() for x in (pos, rad, opa, feat, bg))
f = eng.forward(*scene, cam, gamma=0.1, eps=1e-2, tau=0.01, top_k=5)
up = torch.sign(f["image"] - 0.5).cpu()
for rep in range(2):
    for bands in [int(x) for x in os.environ.get("BANDS", "1,2,4,8,16").split(",")]:
        sess = HostRenderSession(M, 3, S, S, 5, engine=eng, bands=bands)
        sess.set_scene(pos, rad, opa, feat, bg)
        sess.h_upstream.copy_(up)
        for graph in (False, True):
            fn = lambda: sess.render_step([cam], gamma=0.1, eps=1e-2, tau=0.01, compact=True, graph=graph)
            for _ in range(5):
                fn()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(40):
                fn()
            torch.cuda.synchronize()
            print("bands %2d graph %d: %.1f frames/s" % (bands, graph, 40 / (time.perf_counter() - t0)), flush=True)
        del sess
