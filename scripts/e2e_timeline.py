"""Where one HostRenderSession.render_step goes (development aid): CUDA events recorded on both streams
at the phase boundaries of a hand-inlined copy of render_step(compact=True)."""
import os, sys, time
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2004_07484_b200 import CameraSpec, RenderEngine, camera_from_vector
from paper_2004_07484_b200.host import HostRenderSession, CompactGradients
from paper_2004_07484_b200.synthetic import benchmark_scene

bands = int(sys.argv[1]) if len(sys.argv) > 1 else 2
pos, rad, opa, feat, bg, vec = benchmark_scene(1_000_000, 1024, 1024, seed=0)
cam = CameraSpec.from_camera(camera_from_vector(vec, 1024, 1024))
eng = RenderEngine("cuda")
s = HostRenderSession(1_000_000, 3, 1024, 1024, 5, engine=eng, bands=bands)
s.set_scene(pos, rad, opa, feat, bg)
s.h_upstream.copy_(torch.sign(torch.rand(1024, 1024, 3) - 0.5))
for _ in range(5):
    s.render_step([cam], gamma=0.1, eps=1e-2, tau=0.01, compact=True)
torch.cuda.synchronize()
main = torch.cuda.current_stream()
cs = s.copy_stream
names = ["start", "h2d_up_done", "fwd_done", "band0_copied", "img_copied", "bwd_done", "compact_done", "rows_copied"]
acc = {n: 0.0 for n in names}
host_acc = {}
N = 20
for it in range(N):
    ev = {n: torch.cuda.Event(enable_timing=True) for n in names}
    th = [time.perf_counter()]
    ev["start"].record(main)
    cs.wait_stream(main)
    with torch.cuda.stream(cs):
        s.upstream.copy_(s.h_upstream, non_blocking=True)
        ev["h2d_up_done"].record(cs)
    events = s._band_events[:bands] if bands > 1 else None
    f = eng.forward(s.pos, s.rad, s.opa, s.feat, s.bg, cam, gamma=0.1, eps=1e-2, tau=0.01, top_k=5, check=False,
                    band_events=events)
    ev["fwd_done"].record(main)
    th.append(time.perf_counter())
    main.wait_stream(cs)
    with torch.cuda.stream(cs):
        if events:
            for b, e in enumerate(events):
                r0, r1 = s._band_rows[b]
                cs.wait_event(e)
                s.h_image[r0:r1].copy_(f["image"][r0:r1], non_blocking=True)
                if b == 0:
                    ev["band0_copied"].record(cs)
        else:
            cs.wait_stream(main)
            s.h_image.copy_(f["image"], non_blocking=True)
            ev["band0_copied"].record(cs)
        ev["img_copied"].record(cs)
    eng.backward(s.pos, s.rad, s.opa, s.feat, s.bg, cam, f, s.upstream, gamma=0.1, eps=1e-2, normalize=True, gate=True,
                 camera_grads=True, out=s.out, accumulate=False)
    ev["bwd_done"].record(main)
    th.append(time.perf_counter())
    if s._compact is None:
        s._compact = CompactGradients(s.m, s.d, eng.device)
    c = s._compact
    # inline of gather() up to the sync
    import ctypes as C
    from paper_2004_07484_b200 import _lib
    from paper_2004_07484_b200.engine import _ptr
    sp = C.c_void_p(main.cuda_stream)
    c.lib.ss_mask_nonzero_i32(_ptr(s.out["pixel_count"]), s.m, _ptr(c.keep), sp)
    cols = ((c.index, 1), (s.out["pixel_count"], 1), (s.out["d_pos"], 3), (s.out["d_rad"], 1), (s.out["d_opa"], 1), (s.out["d_feat"], 3))
    arr = (_lib.SsColumn * len(cols))()
    off = 0
    for i, (src, w) in enumerate(cols):
        arr[i].src, arr[i].dst = src.data_ptr(), c.d_rec.data_ptr() + 4 * off
        arr[i].row_bytes, arr[i].dst_stride_bytes = 4 * w, 4 * c.words
        off += w
    c.lib.ss_compact_rows(_ptr(c.keep), s.m, arr, len(cols), _ptr(c.ws), c.ws.numel(), _ptr(c.count), sp)
    ev["compact_done"].record(main)
    est = 335000
    c.h_count.copy_(c.count, non_blocking=True)
    c.h_rec[: est * c.words].copy_(c.d_rec[: est * c.words], non_blocking=True)
    ev["rows_copied"].record(main)
    th.append(time.perf_counter())
    main.synchronize(); cs.synchronize()
    th.append(time.perf_counter())
    if it >= 2:
        for n in names:
            acc[n] += ev["start"].elapsed_time(ev[n])
        for i, n in enumerate(["fwd_enqueued", "bwd_enqueued", "all_enqueued", "synced"]):
            host_acc[n] = host_acc.get(n, 0.0) + (th[i + 1] - th[0]) * 1e3
print(f"bands={bands}; GPU event times since step start (ms):")
for n in names:
    print(f"  {n:14s} {acc[n] / (N - 2):.3f}")
print("host clock since step start (ms):", {k: round(v / (N - 2), 3) for k, v in host_acc.items()})
