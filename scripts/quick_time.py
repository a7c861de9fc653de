"""Quick per-kernel timing of the hot path on one GPU (development aid, not the bench contract)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as orc  # scene generator only
from paper_2004_07484_b200 import CameraSpec, RenderEngine, _lib, camera_from_vector


def main():
    count = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    size = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    tau = float(sys.argv[3]) if len(sys.argv) > 3 else 0.01
    det = len(sys.argv) > 4 and sys.argv[4] == "det"  # time the SS_OPT_DETERMINISTIC backward
    steps = int(os.environ.get("QT_STEPS", "10"))
    pos, rad, opa, feat, bg, vec = orc.benchmark_scene(count, size, size, seed=0)
    cam = camera_from_vector(vec, size, size)
    spec = CameraSpec.from_camera(cam)
    eng = RenderEngine("cuda")
    dev = [torch.from_numpy(x).cuda() for x in (pos, rad, opa, feat, bg)]
    f = eng.forward(*dev, spec, gamma=0.1, tau=tau, top_k=5, collect_stats=True)
    print("status", f["status"])
    up = torch.sign(f["image"] - 0.5)
    out = eng.backward(*dev, spec, f, up, gamma=0.1, eps=1e-2)
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    # QT_FLUSH=drain: read a second buffer after the write so that the dirty lines are written back before the frame
    drain = torch.zeros(32 << 20, dtype=torch.int64, device="cuda") if os.environ.get("QT_FLUSH") == "drain" else None
    for collect in (False, True):
        _lib.profile_enable(collect)
        e0 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        e1 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        e2 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        for i in range(steps):
            if os.environ.get("QT_FLUSH") != "none":
                flush.zero_()
            if drain is not None:
                drain.sum()
            e0[i].record()
            f = eng.forward(*dev, spec, gamma=0.1, tau=tau, top_k=5, check=False)
            e1[i].record()
            out = eng.backward(*dev, spec, f, up, gamma=0.1, eps=1e-2, deterministic=det)
            e2[i].record()
        torch.cuda.synchronize()
        fw = np.array([a.elapsed_time(b) for a, b in zip(e0, e1)])
        bw = np.array([a.elapsed_time(b) for a, b in zip(e1, e2)])
        print(f"profile={collect}: fwd {np.median(fw):.3f} ms  bwd {np.median(bw):.3f} ms  "
              f"total {np.median(fw + bw):.3f} ms (min {np.min(fw + bw):.3f})")
        if collect:
            prof = _lib.profile_collect()
            for k, (ms, n) in prof.items():
                if n:
                    print(f"  {k:20s} {ms / n * 1000:9.1f} us x {n}")
    _lib.profile_enable(False)


if __name__ == "__main__":
    main()
