"""cProfile of the 64-view host-to-host step (development aid): where the host time of _views_pipelined goes."""
import cProfile, os, pstats, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_07484_b200 as pk
from paper_2004_07484_b200.host import HostRenderSession
from paper_2004_07484_b200.synthetic import benchmark_scene, orbit_camera_vectors

M, S = 1_000_000, 1024
pos, rad, opa, feat, bg, vec = benchmark_scene(M, S, S, seed=0)
cams = [pk.CameraSpec.from_camera(pk.camera_from_vector(v, S, S)) for v in orbit_camera_vectors(64)]
eng = pk.RenderEngine("cuda")
sess = HostRenderSession(M, 3, S, S, 5, engine=eng)
sess.set_scene(pos, rad, opa, feat, bg)
sess.h_upstream.copy_(torch.sign(torch.rand(S, S, 3) - 0.5))
fn = lambda: sess.render_step(cams, gamma=0.1, eps=1e-2, tau=0.01, compact=True)
for _ in range(3):
    fn()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    fn()
torch.cuda.synchronize()
print("64-view step: %.2f ms (%.1f frames/s)" % (1e3 * (time.perf_counter() - t0) / 5, 64 * 5 / (time.perf_counter() - t0)))
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    fn()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
