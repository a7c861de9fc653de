"""Does running two views concurrently on two streams (two engines / workspaces) raise multi-view throughput?
Development probe: python scripts/two_stream_probe.py"""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2004_07484_b200 import CameraSpec, RenderEngine, camera_from_vector
from paper_2004_07484_b200.synthetic import benchmark_scene, orbit_camera_vectors

pos, rad, opa, feat, bg, vec = benchmark_scene(1_000_000, 1024, 1024, seed=0)
scene = tuple(torch.from_numpy(x).cuda() for x in (pos, rad, opa, feat, bg))
cams = [CameraSpec.from_camera(camera_from_vector(v, 1024, 1024)) for v in orbit_camera_vectors(64)[:32]]
engs = [RenderEngine("cuda"), RenderEngine("cuda")]
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
up = torch.sign(engs[0].forward(*scene, cams[0], gamma=0.1, tau=0.01)["image"] - 0.5)
outs = [None, None]


def run(n_streams):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i, cam in enumerate(cams):
        j = i % n_streams
        with torch.cuda.stream(streams[j]):
            f = engs[j].forward(*scene, cam, gamma=0.1, tau=0.01, check=False)
            outs[j] = engs[j].backward(*scene, cam, f, up, gamma=0.1, eps=1e-2, out=outs[j])
    torch.cuda.synchronize()
    return len(cams) / (time.perf_counter() - t0)


for n in (1, 2, 1, 2):
    run(n)
    print(f"{n} stream(s): {run(n):.0f} frames/s")
