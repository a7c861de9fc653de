#!/usr/bin/env python
"""Pin oracle/extras.py against the imported reference and (re)generate
tests/golden/extras.npz and tests/golden/cloud.ply.

Runs ONLY in the build container (reference mounted read-only at /root/reference).  For prune,
subdivide, PSC1 / PSK1 bytes, PLY import and every shader it runs the REFERENCE on float32-snapped
inputs, asserts that the restatement agrees (masks, bytes and integer outputs exactly, floats to 1e-12)
and stores inputs + the REFERENCE's outputs.

Usage:  python oracle/pin_extras_against_reference.py [--no-write]
"""
from __future__ import annotations

import argparse
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import softsphere as ss  # noqa: E402  (the reference)
from softsphere import optim as ss_optim, scene as ss_scene, shade as ss_shade  # noqa: E402
from softsphere.camera import camera_from_vector, camera_to_vector  # noqa: E402

from oracle import extras as ex  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")


def snap(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def close(a, b, what, tol=1e-12):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    assert a.shape == b.shape, f"{what}: shape {a.shape} vs {b.shape}"
    err = np.abs(a - b).max() if a.size else 0.0
    assert err <= tol * max(1.0, np.abs(b).max() if b.size else 1.0), f"{what}: max error {err}"


def make_scene(rng, m, d):
    sc = ss_scene.new_scene(d, snap(rng.uniform(0, 1, d)))
    pos = snap(np.column_stack([rng.uniform(-5, 5, m), rng.uniform(-5, 5, m), rng.uniform(20, 40, m)]))
    ss_scene.add_sphere_arrays(sc, pos, snap(rng.uniform(0.2, 2.0, m)), snap(rng.uniform(-0.2, 1.2, m)),
                               snap(rng.uniform(0, 1, (m, d))))
    return sc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--no-write", action="store_true")
    args = ap.parse_args()
    rng = np.random.default_rng(20240607)
    g = {}

    # ---- rank 2: prune / subdivide
    for tag, m, d, bgdist in (("a", 700, 3, 0.0), ("b", 1500, 5, 0.55)):
        sc = make_scene(rng, m, d)
        sc.features[: m // 7] = sc.background + snap(rng.uniform(-0.2, 0.2, (m // 7, d)))  # near the background
        sc.features = snap(sc.features)
        vis = rng.integers(0, 4, m) * rng.integers(0, 2, m)
        cfg = ss_optim.FitConfig(prune_opacity_min=0.3, prune_background_dist=bgdist)
        out, keep = ss_optim.prune(sc, vis, cfg)
        o = ex.prune(sc.positions, sc.radii, sc.opacities, sc.features, sc.background, vis, 0.3, bgdist)
        assert np.array_equal(o[4], keep)
        for a, b, n in zip(o[:4], (out.positions, out.radii, out.opacities, out.features), "prof"):
            close(a, b, f"prune {tag} {n}", 0.0)
        g.update({f"prune_{tag}_pos": sc.positions, f"prune_{tag}_rad": sc.radii, f"prune_{tag}_opa": sc.opacities,
                  f"prune_{tag}_feat": sc.features, f"prune_{tag}_bg": sc.background, f"prune_{tag}_vis": vis,
                  f"prune_{tag}_cfg": np.array([0.3, bgdist]), f"prune_{tag}_keep": keep,
                  f"prune_{tag}_out_pos": out.positions, f"prune_{tag}_out_feat": out.features})
    sc = make_scene(rng, 333, 4)
    cfg = ss_optim.FitConfig(subdivide_scale=0.8)
    sub = ss_optim.subdivide(sc, cfg)
    o = ex.subdivide(sc.positions, sc.radii, sc.opacities, sc.features, 0.8)
    for a, b, n in zip(o, (sub.positions, sub.radii, sub.opacities, sub.features), "prof"):
        close(a, b, f"subdivide {n}")
    g.update({"sub_pos": sc.positions, "sub_rad": sc.radii, "sub_opa": sc.opacities, "sub_feat": sc.features,
              "sub_scale": np.array(0.8), "sub_out_pos": sub.positions, "sub_out_rad": sub.radii,
              "sub_out_opa": sub.opacities, "sub_out_feat": sub.features})

    # ---- rank 3: PSC1, PSK1, PLY
    for tag, m, d in (("d3", 257, 3), ("d15", 40, 15), ("empty", 0, 2)):
        sc = make_scene(rng, m, d)
        sc.opacities = np.clip(sc.opacities, 0.0, 1.0)
        blob = ss_scene.scene_to_bytes(sc)
        assert blob == ex.psc1_encode(sc.positions, sc.radii, sc.opacities, sc.features, sc.background)
        back = ss_scene.scene_from_bytes(blob)
        dec = ex.psc1_decode(blob)
        for a, b, n in zip(dec, (back.positions, back.radii, back.opacities, back.features, back.background), "profb"):
            close(a, b, f"psc1 {tag} {n}", 0.0)
        g.update({f"psc1_{tag}_blob": np.frombuffer(blob, np.uint8), f"psc1_{tag}_pos": back.positions,
                  f"psc1_{tag}_rad": back.radii, f"psc1_{tag}_opa": back.opacities, f"psc1_{tag}_feat": back.features,
                  f"psc1_{tag}_bg": back.background})
    sc = make_scene(rng, 64, 3)
    sc.opacities = np.clip(sc.opacities, 0.0, 1.0)
    cams = [camera_from_vector([0.1, -0.2, 0.3, 0.01, 0.02, -0.03, 5.0, 2.0], 48, 32),
            camera_from_vector([0, 0, 0, 1, 0, 0, 0, 1, 0, 4.0, 6.0], 40, 40, near=0.5, far=60.0, mode="orthographic")]
    states = {}
    for name, arr in (("position", sc.positions), ("radius", sc.radii), ("opacity", sc.opacities),
                      ("feature", sc.features)):
        st = ss_optim.AdamState.like(arr)
        st.m = snap(rng.normal(size=arr.shape) * 1e-2)
        st.v = snap(rng.uniform(0, 1e-3, size=arr.shape))
        st.t = 7
        states[name] = st
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "c.psk")
        ss_optim.save_checkpoint(path, sc, cams, states, meta={"step": 7, "note": "golden"})
        ck = open(path, "rb").read()
    mine = ex.psk1_encode(ss_scene.scene_to_bytes(sc), [camera_to_vector(c) for c in cams],
                          [{"width": c.width, "height": c.height, "near": c.near, "far": c.far, "mode": c.mode}
                           for c in cams], {k: (s.m, s.v, s.t) for k, s in states.items()},
                          meta={"step": 7, "note": "golden"})
    assert mine == ck, "PSK1 bytes differ"
    g.update({"psk1_blob": np.frombuffer(ck, np.uint8), "psk1_pos": sc.positions, "psk1_rad": sc.radii,
              "psk1_opa": sc.opacities, "psk1_feat": sc.features, "psk1_bg": sc.background,
              "psk1_cam0": camera_to_vector(cams[0]), "psk1_cam1": camera_to_vector(cams[1])})
    for name, st in states.items():
        g[f"psk1_m_{name}"], g[f"psk1_v_{name}"] = st.m, st.v
    ply = ["ply", "format ascii 1.0", "comment golden cloud", "element vertex 5", "property float x",
           "property float y", "property float z", "property uchar red", "property uchar green",
           "property uchar blue", "element face 0", "property list uchar int vertex_indices", "end_header"]
    for i in range(5):
        ply.append(f"{0.5 * i - 1:.3f} {0.25 * i:.3f} {20 + i} {50 * i} {255 - 40 * i} {7 * i}")
    ply_text = "\n".join(ply) + "\n"
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "c.ply")
        open(path, "w").write(ply_text)
        pc = ss_scene.import_point_cloud(path, 0.05, 0.8)
    g.update({"ply_pos": pc.positions, "ply_rad": pc.radii, "ply_opa": pc.opacities, "ply_feat": pc.features})

    # ---- rank 4: shading
    f3 = snap(rng.uniform(-0.3, 1.3, (9, 11, 3)))
    up3 = snap(rng.normal(size=(9, 11, 3)))
    close(ex.shade_identity(f3), ss_shade.shade_identity(f3), "identity")
    close(ex.shade_identity_backward(f3, up3), ss_shade.shade_identity_backward(f3, up3), "identity bwd")
    g.update({"id_f": f3, "id_up": up3, "id_out": ss_shade.shade_identity(f3),
              "id_bwd": ss_shade.shade_identity_backward(f3, up3)})
    f6 = snap(np.concatenate([rng.uniform(0, 1.2, (13, 7, 3)), rng.normal(size=(13, 7, 3))], axis=-1))
    f6[0, 0, 3:] = 0.0  # zero normal: ambient only
    lights = [ss_shade.DirectionalLight([0.2, -0.5, 1.0], 0.9, 0.15), ss_shade.DirectionalLight([-1.0, 0.1, 0.3], 0.4, 0.05)]
    lt = [(l.direction, l.intensity, l.ambient) for l in lights]
    close(ex.shade_diffuse(f6, lt), ss_shade.shade_diffuse(f6, lights), "diffuse")
    close(ex.shade_diffuse_backward(f6, lt, up3[:1].repeat(13, 0)[:, :7]),
          ss_shade.shade_diffuse_backward(f6, lights, up3[:1].repeat(13, 0)[:, :7]), "diffuse bwd")
    upd = snap(rng.normal(size=(13, 7, 3)))
    g.update({"df_f": f6, "df_up": upd, "df_lights": np.array([[*l.direction, l.intensity, l.ambient] for l in lights]),
              "df_out": ss_shade.shade_diffuse(f6, lights), "df_bwd": ss_shade.shade_diffuse_backward(f6, lights, upd)})
    cam = camera_from_vector([0, 0, 0, 0, 0, 0, 3.0, 2.5], 21, 14)
    vd = ss_shade.view_direction_plane(cam)
    close(ex.view_direction_plane(21, 14, 3.0, 2.5), vd, "view dirs")
    g.update({"vd_cam": np.array([21, 14, 3.0, 2.5]), "vd_out": vd})
    for tag, d, use_view in (("plain", 16, False), ("view", 5, True)):
        f = snap(rng.normal(size=(14, 21, d)) * 0.5)
        d_in = d + (3 if use_view else 0)
        sh = ss_shade.LinearShader(snap(rng.normal(size=(d_in, 3)) * 0.4), snap(rng.uniform(0.2, 0.6, 3)))
        up = snap(rng.normal(size=(14, 21, 3)))
        v = snap(vd) if use_view else None
        out = ss_shade.shade_linear(f, sh, v)
        d_f, d_w, d_b = ss_shade.shade_linear_backward(f, sh, up, v)
        close(ex.shade_linear(f, sh.weight, sh.bias, v), out, f"linear {tag}")
        o = ex.shade_linear_backward(f, sh.weight, sh.bias, up, v)
        close(o[0], d_f, f"linear {tag} d_f"); close(o[1], d_w, f"linear {tag} d_w"); close(o[2], d_b, f"linear {tag} d_b")
        g.update({f"lin_{tag}_f": f, f"lin_{tag}_w": sh.weight, f"lin_{tag}_b": sh.bias, f"lin_{tag}_up": up,
                  f"lin_{tag}_out": out, f"lin_{tag}_df": d_f, f"lin_{tag}_dw": d_w, f"lin_{tag}_db": d_b})
        if use_view:
            g[f"lin_{tag}_v"] = v
    # ---- the fit loop around the path (optim.py:228-373): reference trace / events for a small problem
    truth = make_scene(rng, 40, 3)
    truth.opacities = np.clip(truth.opacities, 0.3, 1.0)
    truth.positions[:, 2] = snap(rng.uniform(8, 14, 40))
    truth.positions[:, :2] = snap(rng.uniform(-1.6, 1.6, (40, 2)))
    truth.radii = snap(rng.uniform(0.25, 0.6, 40))
    cam_vecs = [[0.05, -0.02, 0.0, 0.0, 0.01, 0.0, 5.0, 2.0], [-0.3, 0.1, 0.2, 0.01, 0.04, -0.02, 5.0, 2.0]]
    fit_cams = [camera_from_vector(v, 32, 24) for v in cam_vecs]
    params = ss.BlendParams(gamma=0.1, epsilon=1e-2, tau=0.0, top_k=5)
    obs = [ss_optim.Observation(image=snap(ss.render_forward(truth, c, params)[0].data), camera=c) for c in fit_cams]
    start = truth.copy()
    start.positions = snap(start.positions + rng.normal(size=start.positions.shape) * 0.03)
    start.features = snap(np.clip(start.features + rng.normal(size=start.features.shape) * 0.2, 0, 1))
    fcfg = dict(lr_position=2e-3, lr_radius=1e-3, lr_opacity=5e-3, lr_feature=2e-2, lr_camera=1e-4, steps=14,
                gamma_start=0.2, gamma_end=0.05, epsilon=1e-2, tau=0.0, top_k=5, lambda_od=0.01, prune_every=6,
                prune_opacity_min=0.05, subdivide_at=(8,), subdivide_scale=0.6, seed=3)
    res = ss_optim.fit(start, obs, ss_optim.FitConfig(**fcfg))
    g.update({"fit_pos": start.positions, "fit_rad": start.radii, "fit_opa": start.opacities, "fit_feat": start.features,
              "fit_bg": start.background, "fit_cam_vecs": np.array(cam_vecs), "fit_img0": obs[0].image,
              "fit_img1": obs[1].image, "fit_trace": res.trace,
              "fit_events": np.array([[e[0], 0 if e[1] == "prune" else 1, e[2]] for e in res.events]),
              "fit_out_count": np.array(len(res.scene)),
              "fit_out_cam0": camera_to_vector(res.cameras[0]), "fit_out_cam1": camera_to_vector(res.cameras[1])})
    print("reference fit: events", res.events, "trace", np.round(res.trace, 5))
    print("oracle/extras.py pinned against the reference:", len(g), "arrays")
    if not args.no_write:
        np.savez_compressed(os.path.join(GOLDEN, "extras.npz"), **g)
        open(os.path.join(GOLDEN, "cloud.ply"), "w").write(ply_text)
        print("wrote tests/golden/extras.npz, tests/golden/cloud.ply")


if __name__ == "__main__":
    main()
