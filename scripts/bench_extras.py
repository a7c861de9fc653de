"""Times the SURVEY 8(f) rank 2-4 kernels at benchmark sizes (L2 flushed between runs, CUDA events) and
prints achieved GB/s of their algorithmic bytes against the measured HBM peak.  Evidence script."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2004_07484_b200 import shade, surgery, sceneio, _lib  # noqa: E402
from paper_2004_07484_b200.engine import _ptr  # noqa: E402
import ctypes as C  # noqa: E402

PEAK = 6557.1
try:
    PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    pass
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=10):
    ts = []
    for _ in range(reps + 2):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts[2:]))


def report(name, us, nbytes):
    gbs = nbytes / us / 1e3
    print(f"{name:34s} {us:8.1f} us  {nbytes / 1e6:8.1f} MB  {gbs:7.0f} GB/s  {gbs / PEAK:5.2f} of peak")


def main():
    rng = np.random.default_rng(0)
    m, d = 1_000_000, 3
    t = lambda a: torch.from_numpy(a).cuda()
    pos, rad = t(rng.normal(size=(m, 3)).astype(np.float32)), t(rng.uniform(0.1, 1, m).astype(np.float32))
    opa, feat = t(rng.uniform(-0.1, 1.1, m).astype(np.float32)), t(rng.uniform(0, 1, (m, d)).astype(np.float32))
    bg = t(np.full(d, 0.5, np.float32))
    vis = t(rng.integers(0, 3, m).astype(np.int32))
    lib = _lib.load()
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    keep = torch.empty(m, dtype=torch.uint8, device="cuda")
    report("k_prune_flags (1M, d=3)", timed(lambda: lib.ss_prune_mask(_ptr(opa), _ptr(feat), _ptr(bg), _ptr(vis), m, d, 0.2, 0.3, _ptr(keep), st)),
           m * (4 + 4 * d + 4 + 1))
    kept = int(keep.sum().item())
    cols = [pos, rad, opa, feat]
    outs = [torch.empty_like(c) for c in cols]
    arr = (_lib.SsColumn * 4)()
    for i, (c, o) in enumerate(zip(cols, outs)):
        arr[i].src, arr[i].dst, arr[i].row_bytes = c.data_ptr(), o.data_ptr(), c.numel() // m * 4
    nb = C.c_size_t(); lib.ss_compact_workspace_bytes(m, C.byref(nb))
    ws = torch.empty(nb.value, dtype=torch.uint8, device="cuda"); cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    report(f"compaction, 4 columns ({kept} kept)", timed(lambda: lib.ss_compact_rows(_ptr(keep), m, arr, 4, _ptr(ws), ws.numel(), _ptr(cnt), st)),
           2 * m + 2 * kept * (20 + 4 * d))
    po = torch.empty((12 * m, 3), device="cuda"); ro = torch.empty(12 * m, device="cuda")
    oo = torch.empty(12 * m, device="cuda"); fo = torch.empty((12 * m, d), device="cuda")
    report("k_subdivide (1M -> 12M)", timed(lambda: lib.ss_subdivide(_ptr(pos), _ptr(rad), _ptr(opa), _ptr(feat), m, d, 0.8, _ptr(po), _ptr(ro), _ptr(oo), _ptr(fo), st)),
           13 * m * (20 + 4 * d))
    rec = torch.empty(m * (5 + d), device="cuda")
    report("k_psc1 pack (1M, d=3)", timed(lambda: lib.ss_psc1_pack(_ptr(pos), _ptr(rad), _ptr(opa), _ptr(feat), m, d, _ptr(rec), st)), 2 * m * (20 + 4 * d))
    report("k_psc1 unpack (1M, d=3)", timed(lambda: lib.ss_psc1_unpack(_ptr(rec), m, d, _ptr(pos), _ptr(rad), _ptr(opa), _ptr(feat), st)), 2 * m * (20 + 4 * d))
    h = w = 1024
    dd = 16
    f = t((rng.normal(size=(h, w, dd)) * 0.4).astype(np.float32)); up = t(rng.normal(size=(h, w, 3)).astype(np.float32))
    sh = shade.LinearShader(rng.normal(size=(dd, 3)) * 0.3, np.array([0.4, 0.5, 0.3]))
    wt, b = t(sh.weight.astype(np.float32)), t(sh.bias.astype(np.float32))
    out = torch.empty((h, w, 3), device="cuda"); d_f = torch.empty_like(f)
    d_w = torch.empty((dd, 3), dtype=torch.float64, device="cuda"); d_b = torch.empty(3, dtype=torch.float64, device="cuda")
    n = h * w
    report("k_shade_linear (1024^2, d=16)", timed(lambda: lib.ss_shade_linear(_ptr(f), None, n, dd, _ptr(wt), _ptr(b), _ptr(out), st)), n * (4 * dd + 12))
    report("k_shade_linear_bwd (+ d_w, d_b)", timed(lambda: lib.ss_shade_linear_backward(_ptr(f), None, n, dd, _ptr(wt), _ptr(b), _ptr(up), _ptr(d_f), _ptr(d_w), _ptr(d_b), st)),
           n * (8 * dd + 12))
    f6 = t(rng.normal(size=(h, w, 6)).astype(np.float32))
    lights = shade._lights_c([shade.DirectionalLight([0.1, 0.2, 1.0], 0.8, 0.1)])
    d6 = torch.empty_like(f6)
    report("k_shade_diffuse (1024^2)", timed(lambda: lib.ss_shade_diffuse(_ptr(f6), n, lights, 1, _ptr(out), st)), n * 36)
    report("k_shade_diffuse_bwd", timed(lambda: lib.ss_shade_diffuse_backward(_ptr(f6), _ptr(up), n, lights, 1, _ptr(d6), st)), n * 60)


if __name__ == "__main__":
    main()
