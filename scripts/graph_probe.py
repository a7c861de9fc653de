"""Can a whole frame (ss_forward + ss_backward through the engine) be captured in a CUDA graph and replayed?
What does it buy on the launch-bound small configurations?  (development probe)"""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2004_07484_b200 import CameraSpec, RenderEngine, camera_from_vector
from paper_2004_07484_b200.synthetic import benchmark_scene

for count, size in ((1000, 64), (100_000, 512), (1_000_000, 1024)):
    pos, rad, opa, feat, bg, vec = benchmark_scene(count, size, size, seed=0)
    scene = tuple(torch.from_numpy(x).cuda() for x in (pos, rad, opa, feat, bg))
    cam = CameraSpec.from_camera(camera_from_vector(vec, size, size))
    eng = RenderEngine("cuda")
    f = eng.forward(*scene, cam, gamma=0.1, tau=0.01)
    up = torch.sign(f["image"] - 0.5)
    ref = eng.backward(*scene, cam, f, up, gamma=0.1, eps=1e-2)
    ref = {k: ref[k].clone() for k in ("d_pos", "d_feat", "pixel_count")}
    ref_img = f["image"].clone()

    def frame():
        f = eng.forward(*scene, cam, gamma=0.1, tau=0.01, check=False)
        o = eng.backward(*scene, cam, f, up, gamma=0.1, eps=1e-2)
        return f, o

    def timeit(fn, n=200):
        for _ in range(20):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        torch.cuda.synchronize()
        return 1e3 * (time.perf_counter() - t0) / n

    t_stream = timeit(frame)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        for _ in range(3):
            frame()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        gf, go = frame()
    g.replay()
    torch.cuda.synchronize()
    ok = (torch.equal(gf["image"], ref_img) and torch.equal(go["pixel_count"], ref["pixel_count"])
          and torch.allclose(go["d_feat"], ref["d_feat"], rtol=1e-4, atol=1e-6))
    t_graph = timeit(g.replay)
    print(f"M={count} {size}x{size}: stream launches {t_stream:.3f} ms/frame, graph replay {t_graph:.3f} ms/frame, "
          f"results equal: {ok}", flush=True)
