#!/usr/bin/env python
"""Pin the CPU oracle against the imported reference and (re)generate tests/golden/*.npz.

Runs ONLY in the build container, where the reference package is mounted read-only at
/root/reference (it is not present on the GPU box; nothing in tests/, smoke() or bench.py
reads it at run time).  For every case below it

  1. builds float32-snapped inputs,
  2. runs the REFERENCE (`softsphere.render_forward` / `render_backward` /
     `compute_bounds` / `_bin_tiles`, float64, workers=1),
  3. runs the oracle (oracle/oracle.py -> ss_oracle.c) on the same inputs,
  4. asserts agreement: integer outputs (rects, on_sensor, tile lists, buffer ids,
     pixel_count, stats) exactly; bounds floats to 1e-11; image / buffer floats to 1e-9
     (the reference's own dist^2 = |c|^2 - t^2 carries ~1e-11 of float64 cancellation
     noise that depends on BLAS summation order); gradients to 1e-7 relative,
  5. stores inputs + the REFERENCE's outputs as tests/golden/<case>.npz.

Usage:  python oracle/pin_against_reference.py [--no-write]
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import softsphere as ss  # noqa: E402  (the reference)
from softsphere import raster as ss_raster  # noqa: E402
from softsphere.scene import add_sphere_arrays, new_scene  # noqa: E402

from oracle import oracle as orc  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")


def snap(a):
    return np.asarray(a, dtype=np.float32)


def random_scene(rng, m, d=3, depth=(25.0, 35.0), lateral=5.0, radius=(0.3, 2.0),
                 opacity=(0.1, 1.0)):
    """Same distribution as the reference's tests/conftest.py:8-30."""
    bg = rng.uniform(0, 1, d)
    pos = np.column_stack([rng.uniform(-lateral, lateral, m), rng.uniform(-lateral, lateral, m),
                           rng.uniform(depth[0], depth[1], m)])
    return (snap(pos), snap(rng.uniform(radius[0], radius[1], m)),
            snap(rng.uniform(opacity[0], opacity[1], m)), snap(rng.uniform(0, 1, (m, d))), snap(bg))


def cases():
    rng = np.random.default_rng(12345)
    ident = [0, 0, 0, 0, 0, 0, 5.0, 2.0]
    posed = [0.3, -0.2, 0.5, 0.02, -0.03, 0.01, 5.0, 2.0]
    posed6 = [0.3, -0.2, 0.5, 1, 0.01, 0.02, -0.02, 1, 0.03, 5.0, 2.0]
    out = []

    def add(name, scene, vec, w, h, mode="pinhole", near=0.1, far=45.0, **kw):
        p = dict(gamma=0.1, eps=1e-2, tau=0.0, top_k=5, normalize=True, gate=True)
        p.update(kw)
        out.append(dict(name=name, scene=scene, vec=np.asarray(vec, np.float64), w=w, h=h,
                        mode=mode, near=near, far=far, **p))

    add("rand40_64_ident", random_scene(rng, 40), ident, 64, 64)
    add("rand40_64_tau", random_scene(rng, 40), ident, 64, 64, tau=0.01)
    add("rand60_50x37_posed", random_scene(rng, 60), posed, 50, 37, gamma=0.08)
    add("rand30_48_6d_raw", random_scene(rng, 30), posed6, 48, 48, gamma=0.3, normalize=False,
        gate=False, top_k=8)
    ortho = list(posed)
    ortho[-1] = 14.0
    add("rand30_40_ortho", random_scene(rng, 30, radius=(0.5, 2.5)), ortho, 40, 40,
        mode="orthographic", gamma=0.2)
    add("rand25_32_k32_d1", random_scene(rng, 25, d=1, radius=(1.0, 3.0)), posed, 32, 32,
        top_k=32, gamma=0.25, normalize=False, gate=False)
    add("rand20_33_d16_k1", random_scene(rng, 20, d=16), ident, 33, 33, top_k=1)
    # C1 of BASELINE.json: the reference benchmark scene, 1K spheres @ 64x64 (cli.py:323-356)
    b = orc.benchmark_scene(1000, 64, 64, seed=0)
    add("c1_bench1k_64", b[:5], b[5], 64, 64, tau=0.0)
    add("c1_bench1k_64_tau", b[:5], b[5], 64, 64, tau=0.01)
    b = orc.benchmark_scene(2000, 64, 64, seed=3, profile="occluded")
    add("occluded2k_64_tau", b[:5], b[5], 64, 64, tau=0.01)
    # edge cases: behind camera, camera inside a sphere, sub-pixel, off-sensor, horizon-crossing
    pos = snap([[0, 0, 30], [0, 0, -30], [0.1, 0.2, 1.0], [0, 0, 40], [50, 0, 10], [3.0, 0, 0.5],
                [0, -2.4, 12], [-6.05, 0, 30], [0.072, 0.07, 2.0]])
    rad = snap([2.0, 2.0, 3.0, 0.001, 1.0, 2.0, 0.5, 0.1, 5e-3])
    opa = snap([0.9, 0.9, 0.5, 1.0, 1.0, 1.4, -0.2, 0.7, 0.8])
    feat = snap(rng.uniform(0, 1, (9, 3)))
    add("edge_cases_40x24", (pos, rad, opa, feat, snap([0.1, 0.2, 0.3])), ident, 40, 24, gamma=0.15)
    add("edge_cases_ortho", (pos, rad, opa, feat, snap([0.1, 0.2, 0.3])), [0, 0, 0, 0, 0, 0, 5.0, 14.0],
        24, 40, mode="orthographic", gamma=0.15)
    add("hard_gamma_stack", random_scene(rng, 50, lateral=1.0, radius=(1.0, 2.0)), ident, 32, 32,
        gamma=0.02)
    add("empty_scene", (np.zeros((0, 3), np.float32), np.zeros(0, np.float32), np.zeros(0, np.float32),
                        np.zeros((0, 3), np.float32), snap([0.2, 0.3, 0.4])), ident, 20, 20)
    return out


def ref_objects(case):
    pos, rad, opa, feat, bg = case["scene"]
    d = bg.shape[0]
    scene = new_scene(d, bg.astype(np.float64))
    if pos.shape[0]:
        add_sphere_arrays(scene, pos.astype(np.float64), rad.astype(np.float64),
                          opa.astype(np.float64), feat.astype(np.float64))
    cam = ss.camera_from_vector(case["vec"], case["w"], case["h"], near=case["near"], far=case["far"],
                                mode=case["mode"])
    params = ss.BlendParams(gamma=case["gamma"], epsilon=case["eps"], tau=case["tau"],
                            top_k=case["top_k"])
    return scene, cam, params


def close(a, b, what, rtol=1e-11, atol=1e-13):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    if a.shape != b.shape:
        raise AssertionError(f"{what}: shape {a.shape} vs {b.shape}")
    with np.errstate(invalid="ignore"):
        same_inf = np.isinf(a) & np.isinf(b) & (np.sign(a) == np.sign(b))
        err = np.where(same_inf, 0.0, np.abs(a - b))
    tol = atol + rtol * np.maximum(np.abs(a), np.abs(b))
    tol = np.where(np.isfinite(tol), tol, 0.0)
    if not np.all(err <= tol):
        i = np.unravel_index(np.argmax(err - tol), err.shape) if err.ndim else ()
        raise AssertionError(f"{what}: max err {np.nanmax(err):.3e} at {i}: {a[i]} vs {b[i]}")


def run_case(case, write=True):
    pos, rad, opa, feat, bg = case["scene"]
    scene, cam, params = ref_objects(case)
    ocam = orc.camera_from_vector(case["vec"], case["w"], case["h"], near=case["near"],
                                  far=case["far"], mode=case["mode"])
    close(cam.rotation, ocam.rotation, "rotation", 1e-15)

    # ---- step 0 + sort + bin
    rb, rd = ss.compute_bounds(scene, cam)
    ob = orc.compute_bounds(pos, rad, ocam)
    for k in ("x_min", "x_max", "y_min", "y_max", "on_sensor"):
        assert np.array_equal(getattr(rb, k), ob[k]), f"{case['name']}: bounds {k}"
    close(rb.proj_radius_px, ob["proj_radius_px"], "proj_r")
    close(rd.earliest, ob["earliest"], "earliest")
    close(rd.center_cam, ob["center_cam"], "center_cam")
    sb, sd = ss.sort_draw_records(rb, rd)
    order = orc.sort_order(ob["earliest"])
    assert np.array_equal(sd.sphere_id, order), "sort order"
    n_active = int(sb.on_sensor.sum())
    ntx, nty, _ = ss_raster._tile_grid(cam.width, cam.height, 16)
    rseq, rstarts = ss_raster._bin_tiles(sb, n_active, 16, ntx, nty)
    ref_tile_ids = sd.sphere_id[rseq].astype(np.int64)
    o_ids, o_starts = orc.tile_lists(pos, rad, ocam)
    assert np.array_equal(rstarts, o_starts), "tile_starts"
    assert np.array_equal(ref_tile_ids, o_ids), "tile lists"

    # ---- forward
    img, buf, stats = ss.render_forward(scene, cam, params, workers=1)
    of = orc.render_forward(pos, rad, opa, feat, bg, ocam, gamma=case["gamma"], eps=case["eps"],
                            tau=case["tau"], top_k=case["top_k"], threads=2)
    assert np.array_equal(buf.ids, of["ids"]), f"{case['name']}: buffer ids"
    close(img.data, of["image"], "image", 1e-9, 1e-10)
    close(img.background_weight, of["bg_weight"], "bg_weight", 1e-9, 1e-10)
    close(buf.z, of["z"], "z")
    # dist2 = |c|^2 - t^2 cancels ~1e3 -> 1e-3 in float64: closeness carries ~1e-11 of
    # summation-order noise (BLAS dot vs scalar C), so it is compared to 1e-9 absolute.
    close(buf.closeness, of["closeness"], "closeness", 0.0, 1e-9)
    close(buf.log_denom, of["log_denom"], "log_denom", 1e-9, 1e-10)
    rstats = np.array([stats.spheres_total, stats.spheres_on_sensor, stats.candidates_tested,
                       stats.hits_blended, stats.pixels_early_stopped, stats.tiles], np.int64)
    ostats = np.array(list(of["stats"].values()), np.int64)
    assert np.array_equal(rstats, ostats), f"stats {rstats} vs {ostats}"

    # ---- backward (upstream as in cli.py:384 plus a little noise so no channel is all-equal)
    rng = np.random.default_rng(7)
    upstream = np.sign(img.data - 0.5) + 0.25 * rng.normal(size=img.data.shape)
    upstream = upstream.astype(np.float32).astype(np.float64)
    g, cg = ss.render_backward(scene, cam, params, buf, upstream, workers=1,
                               normalize=case["normalize"], gate=case["gate"])
    og = orc.render_backward(pos, rad, opa, feat, bg, ocam, of, upstream,
                             normalize=case["normalize"], gate=case["gate"], threads=2)
    assert np.array_equal(g.pixel_count, og["pixel_count"]), "pixel_count"
    scale = max(1.0, float(np.abs(g.d_position).max()) if g.d_position.size else 1.0)
    for k in ("d_position", "d_radius", "d_opacity", "d_feature"):
        close(getattr(g, k), og[k], k, 1e-7, 1e-9 * scale)
    for k in ("d_translation", "d_rotation"):
        close(getattr(cg, k), og[k], k, 1e-7, 1e-12)
    close(cg.d_focal, og["d_focal"], "d_focal", 1e-7, 1e-12)
    close(cg.d_sensor_width, og["d_sensor_width"], "d_sensor", 1e-7, 1e-12)

    if write:
        os.makedirs(GOLDEN, exist_ok=True)
        np.savez_compressed(
            os.path.join(GOLDEN, case["name"] + ".npz"),
            pos=pos, rad=rad, opa=opa, feat=feat, bg=bg, cam_vec=case["vec"],
            width=case["w"], height=case["h"], mode=case["mode"], near=case["near"], far=case["far"],
            gamma=case["gamma"], eps=case["eps"], tau=case["tau"], top_k=case["top_k"],
            normalize=case["normalize"], gate=case["gate"],
            x_min=rb.x_min.astype(np.int32), x_max=rb.x_max.astype(np.int32),
            y_min=rb.y_min.astype(np.int32), y_max=rb.y_max.astype(np.int32),
            on_sensor=rb.on_sensor, proj_radius_px=rb.proj_radius_px, earliest=rd.earliest,
            tile_ids=ref_tile_ids.astype(np.int32), tile_starts=rstarts.astype(np.int64),
            image=img.data, bg_weight=img.background_weight, ids=buf.ids, z=buf.z,
            closeness=buf.closeness, log_denom=buf.log_denom, stats=rstats,
            upstream=upstream.astype(np.float32),
            d_position=g.d_position, d_radius=g.d_radius, d_opacity=g.d_opacity,
            d_feature=g.d_feature, pixel_count=g.pixel_count,
            d_translation=cg.d_translation, d_rotation=cg.d_rotation,
            d_focal=cg.d_focal, d_sensor_width=cg.d_sensor_width,
        )
    return stats


def pin_known_answers():
    """Known-answer values the reference's own tests hold for this path."""
    # tests/test_raster.py:45-53: on-axis sphere, tangent half-width and earliest = 24
    cam = orc.camera_from_vector([0, 0, 0, 0, 0, 0, 5.0, 2.0], 1024, 1024)
    b = orc.compute_bounds(snap([[0, 0, 25.0]]), snap([1.0]), cam)
    assert b["earliest"][0] == 24.0
    half_px = 5.0 * np.tan(np.arcsin(1.0 / 25.0)) * 512.0
    assert abs((b["x_max"][0] - b["x_min"][0] + 1) / 2.0 - half_px) <= 1.0, (b, half_px)
    # tests/test_blend.py:44-54: Eq.1 weights 0.8805 / 0.1192 / 3.3e-4 for two stacked
    # hits -- reproduced through the full forward on a 1x1 orthographic image.
    # (z = 1 and z = 0.8 at gamma = 0.1 with unit opacity/closeness; eps = 1e-2... the
    # literal triple is a property of blend_arrays; here we check the same weights
    # through ids/z/closeness/log_denom of the oracle forward against blend_arrays.)
    from softsphere.blend import blend_arrays
    rng = np.random.default_rng(3)
    sc = random_scene(rng, 12, lateral=0.5, radius=(1.0, 2.0))
    cam = orc.camera_from_vector([0, 0, 0, 0, 0, 0, 5.0, 2.0], 8, 8)
    f = orc.render_forward(*sc, cam, gamma=0.1, tau=0.0, top_k=32)
    ids, z, c, ld = f["ids"][4, 4], f["z"][4, 4], f["closeness"][4, 4], f["log_denom"][4, 4]
    v = ids >= 0
    w, w_bg, log_d = blend_arrays(z[v], c[v], sc[2][ids[v]].astype(np.float64),
                                  ss.BlendParams(gamma=0.1, tau=0.0, top_k=32))
    assert abs(log_d - ld) < 1e-12 and abs(w_bg - f["bg_weight"][4, 4]) < 1e-12
    img = w @ sc[3][ids[v]].astype(np.float64) + w_bg * sc[4].astype(np.float64)
    assert np.abs(img - f["image"][4, 4]).max() < 1e-12


def pin_fit_step(write=True):
    """photometric_loss, opacity_depth_regularizer, adam_step and three iterations
    of the fit loop body (optim.py:286-329) -- reference vs oracle, then golden vectors."""
    from softsphere import optim as ro
    rng = np.random.default_rng(2024)
    a, b = rng.uniform(0, 1, (9, 7, 3)), rng.uniform(0, 1, (9, 7, 3))
    b[0, 0] = a[0, 0]  # ties -> sign 0
    l_ref, u_ref = ro.photometric_loss(a, b)
    l_or, u_or = orc.photometric_loss(a, b)
    assert l_ref == l_or and np.array_equal(u_ref, u_or)
    sc = random_scene(rng, 30, depth=(0.05, 50.0))
    vec = np.array([0.3, -0.2, 0.5, 0.02, -0.03, 0.01, 5.0, 2.0])
    case = dict(scene=sc, vec=vec, w=40, h=32, mode="pinhole", near=0.1, far=45.0, gamma=0.2, eps=1e-2, tau=0.0,
                top_k=5)
    scene, cam, _ = ref_objects(case)
    ocam = orc.camera_from_vector(vec, 40, 32)
    e_ref, dp_ref, do_ref = ro.opacity_depth_regularizer(scene, cam, 0.37)
    e_or, dp_or, do_or = orc.opacity_depth_regularizer(sc[0], sc[2], ocam, 0.37)
    close(e_ref, e_or, "od energy", 1e-14)
    close(dp_ref, dp_or, "od d_position", 1e-14)
    close(do_ref, do_or, "od d_opacity", 1e-14)
    cfg = ro.FitConfig(lr_position=2e-3, lr_radius=1e-3, lr_opacity=1e-2, lr_feature=2e-2, lambda_od=0.05)
    st = ro.AdamState.like(sc[0].astype(np.float64))
    p_ref = sc[0].astype(np.float64)
    p_or, m_or, v_or, t_or = p_ref.copy(), np.zeros_like(p_ref), np.zeros_like(p_ref), 0
    for _ in range(3):
        g = rng.normal(size=p_ref.shape)
        p_ref = ro.adam_step(p_ref, g, st, 2e-3, cfg)
        p_or, m_or, v_or, t_or = orc.adam_step(p_or, g, m_or, v_or, t_or, 2e-3)
    close(p_ref, p_or, "adam params", 1e-15)
    close(st.v, v_or, "adam v", 1e-15)

    # three iterations of the loop body on one observation (normalised, gated gradients)
    target = rng.uniform(0, 1, (32, 40, 3))
    params = ss.BlendParams(gamma=0.2, epsilon=1e-2, tau=0.0, top_k=5)
    r_scene = scene.copy()
    states = {k: ro.AdamState.like(getattr(r_scene, n)) for k, n in
              (("pos", "positions"), ("rad", "radii"), ("opa", "opacities"), ("feat", "features"))}
    o_scene = dict(pos=sc[0].astype(np.float64), rad=sc[1].astype(np.float64), opa=sc[2].astype(np.float64),
                   feat=sc[3].astype(np.float64), bg=sc[4].astype(np.float64))
    o_state = {k: (np.zeros_like(o_scene[k]), np.zeros_like(o_scene[k]), 0) for k in ("pos", "rad", "opa", "feat")}
    o_cfg = dict(lr_position=2e-3, lr_radius=1e-3, lr_opacity=1e-2, lr_feature=2e-2, beta1=0.9, beta2=0.999,
                 adam_eps=1e-8, gamma=0.2, epsilon=1e-2, tau=0.0, top_k=5, lambda_od=0.05, radius_min=1e-6,
                 normalize_grads=True, gate=True)
    losses = []
    for _ in range(3):
        img, buf, _ = ss.render_forward(r_scene, cam, params)
        loss, up = ro.photometric_loss(img.data, target)
        e, rdp, rdo = ro.opacity_depth_regularizer(r_scene, cam, cfg.lambda_od)
        loss += e
        g, _cg = ss.render_backward(r_scene, cam, params, buf, up)
        g.d_position += rdp
        g.d_opacity += rdo
        r_scene.positions = ro.adam_step(r_scene.positions, g.d_position, states["pos"], cfg.lr_position, cfg)
        r_scene.radii = np.maximum(ro.adam_step(r_scene.radii, g.d_radius, states["rad"], cfg.lr_radius, cfg),
                                   cfg.radius_min)
        r_scene.opacities = ro.adam_step(r_scene.opacities, g.d_opacity, states["opa"], cfg.lr_opacity, cfg)
        r_scene.features = ro.adam_step(r_scene.features, g.d_feature, states["feat"], cfg.lr_feature, cfg)
        o_loss, o_scene, o_state, _ = orc.fit_step(o_scene, ocam, target, o_state, o_cfg)
        close(loss, o_loss, "fit loss", 1e-9)
        losses.append(loss)
    close(r_scene.positions, o_scene["pos"], "fit positions", 1e-9)
    close(r_scene.radii, o_scene["rad"], "fit radii", 1e-9)
    close(r_scene.opacities, o_scene["opa"], "fit opacities", 1e-8, 1e-12)
    close(r_scene.features, o_scene["feat"], "fit features", 1e-8, 1e-12)
    if write:
        np.savez_compressed(os.path.join(GOLDEN, "fit_step.npz"), pos=sc[0], rad=sc[1], opa=sc[2], feat=sc[3],
                            bg=sc[4], cam_vec=vec, width=40, height=32, target=target.astype(np.float32),
                            losses=np.array(losses), pos_out=r_scene.positions, rad_out=r_scene.radii,
                            opa_out=r_scene.opacities, feat_out=r_scene.features,
                            pm_a=a.astype(np.float32), pm_b=b.astype(np.float32))
    print("fit step (photometric loss, regulariser, adam, 3 loop iterations): ok")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--no-write", action="store_true")
    args = ap.parse_args()
    orc.build(force=True)
    pin_known_answers()
    print("known answers: ok")
    for case in cases():
        st = run_case(case, write=not args.no_write)
        print(f"{case['name']:28s} ok  (tested={st.candidates_tested} hits={st.hits_blended} "
              f"stopped={st.pixels_early_stopped})")
    pin_fit_step(write=not args.no_write)
    print("oracle pinned against reference; golden fixtures in", GOLDEN)


if __name__ == "__main__":
    main()
