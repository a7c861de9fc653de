"""Run one BASELINE.json-style configuration on the GPU, optionally compare with the CPU oracle, and
print per-kernel timings.  Development / evidence script (not the bench contract).

  python scripts/run_config.py --count 10000000 --width 1920 --height 1080 --d 16 --k 32 --oracle
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2004_07484_b200 import CameraSpec, RenderEngine, _lib, camera_from_vector
from paper_2004_07484_b200.synthetic import benchmark_scene


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--count", type=int, default=1_000_000)
    ap.add_argument("--width", type=int, default=1024)
    ap.add_argument("--height", type=int, default=1024)
    ap.add_argument("--d", type=int, default=3)
    ap.add_argument("--k", type=int, default=5)
    ap.add_argument("--tau", type=float, default=0.0)
    ap.add_argument("--profile", default="uniform")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--oracle", action="store_true")
    a = ap.parse_args()
    pos, rad, opa, feat, bg, vec = benchmark_scene(a.count, a.width, a.height, seed=0, d=a.d, profile=a.profile,
                                                   aspect_fill=(a.width != a.height))
    spec = CameraSpec.from_camera(camera_from_vector(vec, a.width, a.height))
    eng = RenderEngine("cuda")
    dev = [torch.from_numpy(x).cuda() for x in (pos, rad, opa, feat, bg)]
    f = eng.forward(*dev, spec, gamma=0.1, tau=a.tau, top_k=a.k, collect_stats=True)
    status = f["status"]
    print("status", status, "workspace MB", eng._ws.numel() / 1e6)
    up = torch.sign(f["image"] - 0.5)
    out = eng.backward(*dev, spec, f, up, gamma=0.1, eps=1e-2)
    torch.cuda.synchronize()
    _lib.profile_enable(True)
    t = []
    for _ in range(a.steps):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        f = eng.forward(*dev, spec, gamma=0.1, tau=a.tau, top_k=a.k, check=False)
        e1.record()
        out = eng.backward(*dev, spec, f, up, gamma=0.1, eps=1e-2)
        e2.record()
        torch.cuda.synchronize()
        t.append((e0.elapsed_time(e1), e1.elapsed_time(e2)))
    t = np.array(t)
    print(f"fwd {np.median(t[:, 0]):.3f} ms  bwd {np.median(t[:, 1]):.3f} ms  total {np.median(t.sum(1)):.3f} ms")
    for k, (ms, n) in _lib.profile_collect().items():
        if n:
            print(f"  {k:20s} {ms / n * 1000:10.1f} us x {n}")
    _lib.profile_enable(False)
    if a.oracle:
        from oracle import oracle as orc
        ocam = orc.camera_from_vector(vec, a.width, a.height)
        thr = orc.num_threads_available()
        t0 = time.perf_counter()
        ref = orc.render_forward(pos, rad, opa, feat, bg, ocam, gamma=0.1, tau=a.tau, top_k=a.k, threads=thr)
        t1 = time.perf_counter()
        gr = orc.render_backward(pos, rad, opa, feat, bg, ocam, ref, up.cpu().numpy().astype(np.float64), threads=thr)
        t2 = time.perf_counter()
        print(f"oracle ({thr} threads): fwd {t1 - t0:.1f} s  bwd {t2 - t1:.1f} s", ref["stats"])
        ids = f["ids"].permute(1, 2, 0).cpu().numpy()
        print("id mismatches:", int((ids != ref["ids"]).sum()), "of", ids.size)
        img = f["image"].cpu().numpy().astype(np.float64)
        err = np.abs(img - ref["image"])
        print("image max abs err %.3e, max rel err %.3e" % (err.max(), (err / np.maximum(np.abs(ref["image"]), 1e-2)).max()))
        print("stats equal:", status["hits_blended"] == ref["stats"]["hits_blended"],
              status["candidates_tested"] == ref["stats"]["candidates_tested"])
        print("pixel_count equal:", bool(np.array_equal(out["pixel_count"].cpu().numpy(), gr["pixel_count"])))
        for name, key in (("d_pos", "d_position"), ("d_rad", "d_radius"), ("d_opa", "d_opacity"), ("d_feat", "d_feature")):
            g = out[name].cpu().numpy().astype(np.float64)
            e = np.abs(g - gr[key])
            print(f"  {name}: max abs err {e.max():.3e} (max |ref| {np.abs(gr[key]).max():.3e})")
        cg = out["cam_grad"].cpu().numpy()
        print("  cam d_t", cg[:3], "ref", gr["d_translation"])


if __name__ == "__main__":
    main()
