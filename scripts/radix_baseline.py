"""Head-to-head for DESIGN section 4 (tile binning): what the classic design -- ONE device-wide radix sort of the
T (tile, depth) keys, as north_star sketches it -- would cost on this GPU, measured with the library radix sort
(torch.sort -> CUB DeviceRadixSort).  Library code is used here as a yardstick only; the product path does not sort
globally (per-tile buckets + per-tile sort, csrc/ss_project.cu)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2004_07484_b200 import CameraSpec, RenderEngine, _lib, camera_from_vector
from paper_2004_07484_b200.synthetic import benchmark_scene

for count, w, h, d, k in ((1_000_000, 1024, 1024, 3, 5), (10_000_000, 1920, 1080, 16, 32)):
    pos, rad, opa, feat, bg, vec = benchmark_scene(count, w, h, seed=0, d=d, aspect_fill=(w != h))
    cam = CameraSpec.from_camera(camera_from_vector(vec, w, h))
    eng = RenderEngine("cuda")
    dev = [torch.from_numpy(x).cuda() for x in (pos, rad, opa, feat, bg)]
    f = eng.forward(*dev, cam, gamma=0.1, tau=0.01, top_k=k, collect_stats=True, debug=True)
    T = f["status"]["num_pairs"]
    starts, ids = eng.tile_lists(count, d, w, h, k)
    starts = torch.as_tensor(np.asarray(starts)).cuda().long()
    ids = torch.as_tensor(np.asarray(ids)).cuda()[:T].long()
    tiles = torch.repeat_interleave(torch.arange(starts.numel() - 1, device="cuda"), starts[1:] - starts[:-1])
    depth_bits = f["earliest"][ids].view(torch.int64) & ((1 << 52) - 1)  # positive doubles: bits are order-preserving
    keys = (tiles << 52) | (depth_bits >> 12)  # 12-bit tile id (C3) / 13-bit (C5) + depth
    perm = torch.randperm(T, device="cuda")
    keys = keys[perm].contiguous()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(12):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); torch.sort(keys); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    _lib.profile_enable(True)
    for _ in range(5):
        flush.zero_()
        eng.forward(*dev, cam, gamma=0.1, tau=0.01, top_k=k, check=False)
    p = _lib.profile_collect()
    _lib.profile_enable(False)
    ours = {n: round(1e3 * ms / c, 1) for n, (ms, c) in p.items() if c and n in ("k_scan", "k_emit", "k_tile_sort_small", "k_tile_sort_big")}
    print(f"M={count} T={T}: library radix sort of T 64-bit (tile, depth) keys + payload: median {np.median(ts[2:]):.1f} us; "
          f"this path's binning kernels after k_project (us per launch, k_tile_sort_big = mid + big): {ours}")
    del eng, f, dev
    torch.cuda.empty_cache()
