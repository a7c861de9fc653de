"""Where the host time of the plug-in call goes (development aid): python scripts/plugin_profile.py"""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_07484_b200 as pk
from paper_2004_07484_b200 import api
from paper_2004_07484_b200.synthetic import benchmark_scene

M, S = 1_000_000, 1024
pos, rad, opa, feat, bg, vec = benchmark_scene(M, S, S, seed=0)
scene = pk.new_scene(3, bg.astype(np.float64))
scene.positions, scene.radii = pos.astype(np.float64), rad.astype(np.float64)
scene.opacities, scene.features = opa.astype(np.float64), feat.astype(np.float64)
cam = pk.camera_from_vector(vec, S, S)
params = pk.BlendParams(gamma=0.1, epsilon=1e-2, tau=0.01, top_k=5)
eng = pk.RenderEngine("cuda")
print("torch threads", torch.get_num_threads(), "cpus", len(os.sched_getaffinity(0)))

def t(fn, n=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t0) / n

image, buf, _ = pk.render_forward(scene, cam, params, engine=eng)
up = np.sign(image.data - 0.5)
print("render_forward  %.2f ms" % t(lambda: pk.render_forward(scene, cam, params, engine=eng)))
print("render_forward f32 out %.2f ms" % t(lambda: pk.render_forward(scene, cam, params, engine=eng, dtype=np.float32)))
print("render_backward %.2f ms" % t(lambda: pk.render_backward(scene, cam, params, buf, up, engine=eng)))
print("np.sign(image-0.5) %.2f ms" % t(lambda: np.sign(image.data - 0.5)))
st = api._stage_for(eng, M, 3, S, S)
cols = api._scene_columns(scene)
print("  narrow scene into pinned %.2f ms" % t(lambda: [api._narrow_into(d, s) for d, s in zip(api._Stage.carve_in(st.h_in, M, 3), cols)]))
print("  fingerprint %.3f ms" % t(lambda: api._fingerprint(cols)))
d_in = torch.empty(st.n_in, dtype=torch.float32, device="cuda")
print("  H2D scene %.2f ms" % t(lambda: d_in.copy_(st.h_in, non_blocking=True)))
print("  alloc device scene %.3f ms" % t(lambda: torch.empty(st.n_in, dtype=torch.float32, device="cuda")))
dev_in = api._upload_scene(eng, st, cols)
spec = pk.CameraSpec.from_camera(cam)
print("  engine.forward check=True %.2f ms" % t(lambda: eng.forward(*dev_in, spec, gamma=0.1, tau=0.01, top_k=5, collect_stats=True, check=True)))
print("  engine.forward check=False %.2f ms" % t(lambda: eng.forward(*dev_in, spec, gamma=0.1, tau=0.01, top_k=5, check=False)))
print("  D2H image block %.2f ms" % t(lambda: st.h_img.copy_(st.d_img, non_blocking=True)))
print("  widen image f64 %.2f ms" % t(lambda: api._widen(st.h_img[:S * S * 3].view(S, S, 3), np.float64)))
print("  widen image f32 %.2f ms" % t(lambda: api._widen(st.h_img[:S * S * 3].view(S, S, 3), np.float32)))
print("  narrow upstream %.2f ms" % t(lambda: api._narrow_into(st.h_up, up)))
print("  D2H grads block %.2f ms" % t(lambda: st.grads.download()))
hg = st.grads.host
print("  widen grads f64 %.2f ms" % t(lambda: [api._widen(hg[k], np.float64) for k in ("d_pos", "d_rad", "d_opa", "d_feat")] + [api._widen(hg["pixel_count"], np.int64)]))
print("  np.empty 3M f64 + fill %.2f ms" % t(lambda: np.empty((M, 3)).fill(0)))
