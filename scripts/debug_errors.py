"""Development aid: error statistics of the GPU forward against the oracle on a benchmark config."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as orc
from paper_2004_07484_b200 import CameraSpec, RenderEngine, camera_from_vector

count = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
size = int(sys.argv[2]) if len(sys.argv) > 2 else 512
gamma = float(sys.argv[3]) if len(sys.argv) > 3 else 0.1
pos, rad, opa, feat, bg, vec = orc.benchmark_scene(count, size, size, seed=0)
cam = camera_from_vector(vec, size, size)
ocam = orc.camera_from_vector(vec, size, size)
spec = CameraSpec.from_camera(cam)
eng = RenderEngine("cuda")
ref = orc.render_forward(pos, rad, opa, feat, bg, ocam, gamma=gamma, tau=0.0, top_k=5, threads=orc.num_threads_available())
f = eng.forward(pos, rad, opa, feat, bg, spec, gamma=gamma, tau=0.0, top_k=5, collect_stats=True)
hwk = lambda t: t.permute(1, 2, 0).cpu().numpy()
ids = hwk(f["ids"])
print("id mismatches", int((ids != ref["ids"]).sum()), "hits", f["status"]["hits_blended"], ref["stats"]["hits_blended"])
for name, a, e in (("image", f["image"].cpu().numpy(), ref["image"]), ("z", hwk(f["z"]), ref["z"]),
                   ("closeness", hwk(f["closeness"]), ref["closeness"]),
                   ("log_denom", f["log_denom"].cpu().numpy(), ref["log_denom"])):
    err = np.abs(a.astype(np.float64) - e)
    rel = err / np.maximum(np.abs(e), 1e-30)
    tol = 2e-6 + 1e-5 * np.abs(e)
    print(f"{name:10s} max abs {err.max():.3e}  p99.9 abs {np.quantile(err, 0.999):.3e}  mean abs {err.mean():.3e}  "
          f"max err/tol {np.max(err / tol):.3f}  n>tol {int((err > tol).sum())}")
# all hits, not only the top 5: K = 32 buffers
K = 32
ref2 = orc.render_forward(pos, rad, opa, feat, bg, ocam, gamma=gamma, tau=0.0, top_k=K, threads=orc.num_threads_available())
f2 = eng.forward(pos, rad, opa, feat, bg, spec, gamma=gamma, tau=0.0, top_k=K, collect_stats=True)
ids2 = hwk(f2["ids"])
print("K=32 id mismatches", int((ids2 != ref2["ids"]).sum()))
for name in ("z", "closeness"):
    a, e = hwk(f2[name]), ref2[name]
    err = np.abs(a.astype(np.float64) - e)
    i = np.unravel_index(np.argmax(err), err.shape)
    print(f"K=32 {name}: max abs {err.max():.3e} at {i}: got {a[i]!r} want {e[i]!r} id {ids2[i]}")
err = np.abs(f["log_denom"].cpu().numpy().astype(np.float64) - ref["log_denom"])
i = np.unravel_index(np.argmax(err), err.shape)
print("worst log_denom pixel", i, "gpu", f["log_denom"].cpu().numpy()[i], "ref", ref["log_denom"][i])
print(" ids", ids2[i][:12]); print(" z gpu", hwk(f2["z"])[i][:12]); print(" z ref", ref2["z"][i][:12])
print(" c gpu", hwk(f2["closeness"])[i][:12]); print(" c ref", ref2["closeness"][i][:12])
print(" opa", opa[ids2[i][:12]])
