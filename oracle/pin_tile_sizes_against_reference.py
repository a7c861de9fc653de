"""Pins the oracle's `tile` parameter against the reference's `tile_size` (raster.py:437-447, :420-434) and writes
the REFERENCE's outputs for tile sizes 8 / 24 / 32 to tests/golden/extras_tile_sizes.npz.

Run in the build container, where the reference is importable:
    python oracle/pin_tile_sizes_against_reference.py [--no-write]
TEST INFRASTRUCTURE ONLY: nothing in the product imports this.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, "/root/reference/pkg/src")

import softsphere as ss  # noqa: E402
from helpers import make_random_scene  # noqa: E402
from oracle import oracle as orc  # noqa: E402


def main():
    rng = np.random.default_rng(5)
    pos, rad, opa, feat, bg = make_random_scene(rng, 150)
    vec = np.array([0.1, -0.05, 0.2, 0.01, 0.02, -0.01, 5.0, 2.0])
    w, h = 70, 50
    scene = ss.new_scene(3, bg.astype(np.float64))
    scene.positions, scene.radii = pos.astype(np.float64), rad.astype(np.float64)
    scene.opacities, scene.features = opa.astype(np.float64), feat.astype(np.float64)
    cam, ocam = ss.camera_from_vector(vec, w, h), orc.camera_from_vector(vec, w, h)
    out = {"pos": pos, "rad": rad, "opa": opa, "feat": feat, "bg": bg, "cam_vec": vec, "width": w, "height": h,
           "tile_sizes": np.array([8, 24, 32])}
    for tile in (8, 16, 24, 32):
        for tau in (0.0, 0.01):
            img, buf, st = ss.render_forward(scene, cam, ss.BlendParams(gamma=0.1, tau=tau, top_k=5), tile_size=tile)
            o = orc.render_forward(pos, rad, opa, feat, bg, ocam, gamma=0.1, tau=tau, top_k=5, tile=tile)
            assert np.array_equal(buf.ids, o["ids"]), (tile, tau)
            assert np.abs(img.data - o["image"]).max() < 1e-9, (tile, tau)
            got = [o["stats"][k] for k in ("candidates_tested", "hits_blended", "pixels_early_stopped", "tiles")]
            assert got == [st.candidates_tested, st.hits_blended, st.pixels_early_stopped, st.tiles], (tile, tau)
            if tau == 0.0 and tile != 16:
                out[f"image_{tile}"] = img.data
                out[f"ids_{tile}"] = buf.ids
                out[f"stats_{tile}"] = np.array([st.spheres_total, st.spheres_on_sensor, st.candidates_tested,
                                                 st.hits_blended, st.pixels_early_stopped, st.tiles])
            print(f"tile {tile:2d} tau {tau}: ok (candidates {st.candidates_tested}, tiles {st.tiles})")
    if "--no-write" not in sys.argv:
        np.savez_compressed(os.path.join(ROOT, "tests", "golden", "extras_tile_sizes.npz"), **out)
        print("wrote tests/golden/extras_tile_sizes.npz")


if __name__ == "__main__":
    main()
