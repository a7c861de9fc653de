"""Times the SURVEY 8(f) rank-1 kernels (photometric loss, fused fit step) and a full device-resident
fit iteration at C3 size; prints achieved GB/s against the measured HBM peak."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2004_07484_b200 as pk
from paper_2004_07484_b200.synthetic import benchmark_scene


def timed(fn, n=20, flush=None):
    ts = []
    for _ in range(n):
        if flush is not None:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    m, size, d = 1_000_000, 1024, 3
    pos, rad, opa, feat, bg, vec = benchmark_scene(m, size, size, seed=0)
    spec = pk.CameraSpec.from_camera(pk.camera_from_vector(vec, size, size))
    cfg = pk.FitConfig(lambda_od=0.05, tau=0.01)
    fit = pk.DeviceFit(pos, rad, opa, feat, bg, cfg)
    target = torch.rand((size, size, d), device="cuda")
    peak = 6550.1
    pp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pp):
        peak = float(json.load(open(pp))["hbm_gbs"])
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        fit.step(target, spec)
    img = fit.last["image"]
    grads = fit.last["grads"]
    t_loss = timed(lambda: pk.photometric_loss_device(img, target), flush=flush)
    b_loss = 3 * img.numel() * 4
    t_upd = timed(lambda: fit.apply_gradients(grads, spec), flush=flush)
    # per sphere: 5 + d parameters read + written, 5 + d gradients read, pixel_count read, visibility
    # read + written, two moments per parameter read + written
    b_upd = m * ((5 + d) * 4 * 2 + (5 + d) * 4 + 4 + 4 * 2 + (5 + d) * 4 * 4)
    t_step = timed(lambda: fit.step(target, spec), flush=flush)
    print(f"k_photometric: {t_loss * 1e3:.1f} us, {b_loss / t_loss / 1e6:.0f} GB/s = {b_loss / t_loss / 1e6 / peak:.2f} of measured HBM peak")
    print(f"k_fit_step:    {t_upd * 1e3:.1f} us, {b_upd / t_upd / 1e6:.0f} GB/s = {b_upd / t_upd / 1e6 / peak:.2f} of measured HBM peak")
    print(f"full fit iteration (forward + loss + backward + fused update), C3: {t_step:.3f} ms")


if __name__ == "__main__":
    main()
