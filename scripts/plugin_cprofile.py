"""cProfile of the plug-in calls at C3 (development aid): python scripts/plugin_cprofile.py"""
import cProfile, os, pstats, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_07484_b200 as pk
from paper_2004_07484_b200.synthetic import benchmark_scene

M, S = 1_000_000, 1024
pos, rad, opa, feat, bg, vec = benchmark_scene(M, S, S, seed=0)
scene = pk.new_scene(3, bg.astype(np.float64))
scene.positions, scene.radii = pos.astype(np.float64), rad.astype(np.float64)
scene.opacities, scene.features = opa.astype(np.float64), feat.astype(np.float64)
cam = pk.camera_from_vector(vec, S, S)
params = pk.BlendParams(gamma=0.1, epsilon=1e-2, tau=0.01, top_k=5)
eng = pk.RenderEngine("cuda")
for _ in range(3):
    image, buf, _ = pk.render_forward(scene, cam, params, engine=eng)
    up = np.sign(image.data - 0.5)
    pk.render_backward(scene, cam, params, buf, up, engine=eng)
for name, fn in (("forward", lambda: pk.render_forward(scene, cam, params, engine=eng)),
                 ("backward", lambda: pk.render_backward(scene, cam, params, buf, up, engine=eng))):
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(20):
        fn()
    pr.disable()
    print("=====", name, "(20 calls)")
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)
