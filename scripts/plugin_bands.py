"""Band count of the plug-in's render_forward (development aid): python scripts/plugin_bands.py"""
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
for rep in range(3):
    for bands in (1, 2, 4, 8):
        api._IMAGE_BANDS = bands
        eng._api_stage = None
        for _ in range(5):
            pk.render_forward(scene, cam, params, engine=eng)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(30):
            pk.render_forward(scene, cam, params, engine=eng)
        torch.cuda.synchronize()
        print("bands %d: render_forward %.3f ms" % (bands, 1e3 * (time.perf_counter() - t0) / 30), flush=True)
