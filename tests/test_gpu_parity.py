"""GPU parity: CUDA path (through the C ABI) vs the committed golden fixtures (outputs of the
reference itself) and vs the CPU oracle on seeded inputs.

Bars (north_star): sphere ids, rectangles, tile lists, pixel counts bit-exact; forward floats
1e-5 relative; gradients 1e-4 relative.
"""
import numpy as np
import pytest

from helpers import (FWD_ATOL, FWD_RTOL, assert_close, golden_names, grad_close, load_golden,
                     make_random_scene)

pytestmark = pytest.mark.gpu


def _spec(g):
    from paper_2004_07484_b200 import CameraSpec, camera_from_vector
    cam = camera_from_vector(g["cam_vec"], g["width"], g["height"], near=g["near"], far=g["far"], mode=g["mode"])
    return cam, CameraSpec.from_camera(cam)


def _hwk(t):
    return t.permute(1, 2, 0).cpu().numpy()


@pytest.mark.parametrize("name", golden_names())
def test_golden_forward(engine, name):
    g = load_golden(name)
    cam, spec = _spec(g)
    f = engine.forward(g["pos"], g["rad"], g["opa"], g["feat"], g["bg"], spec, gamma=g["gamma"], eps=g["eps"],
                       tau=g["tau"], top_k=g["top_k"], collect_stats=True, debug=True)
    m = g["pos"].shape[0]
    # step 0: integer rectangles and visibility are exact
    rect = f["rect"].cpu().numpy()
    assert np.array_equal(rect[:, 0], g["x_min"]) and np.array_equal(rect[:, 1], g["x_max"])
    assert np.array_equal(rect[:, 2], g["y_min"]) and np.array_equal(rect[:, 3], g["y_max"])
    assert np.array_equal(f["on_sensor"].cpu().numpy().astype(bool), g["on_sensor"])
    e_gpu, e_ref = f["earliest"].cpu().numpy(), g["earliest"]
    assert np.array_equal(np.isinf(e_gpu), np.isinf(e_ref))
    fin = np.isfinite(e_ref)
    assert_close(e_gpu[fin], e_ref[fin], 1e-12, 1e-12, "earliest")
    assert_close(f["proj_radius_px"].cpu().numpy(), g["proj_radius_px"], 1e-12, 1e-12, "proj_radius_px")
    # tile lists: exact sequence (depth order, ties by index)
    starts, ids = engine.tile_lists(m, g["feat"].shape[1] if m else 3, g["width"], g["height"], g["top_k"])
    assert np.array_equal(starts, g["tile_starts"])
    assert np.array_equal(ids, g["tile_ids"])
    # per-pixel record: ids exact, floats 1e-5
    assert np.array_equal(_hwk(f["ids"]), g["ids"])
    assert_close(f["image"].cpu().numpy(), g["image"], FWD_RTOL, FWD_ATOL, "image")
    assert_close(f["bg_weight"].cpu().numpy(), g["bg_weight"], FWD_RTOL, FWD_ATOL, "bg_weight")
    assert_close(_hwk(f["z"]), g["z"], FWD_RTOL, FWD_ATOL, "z")
    assert_close(_hwk(f["closeness"]), g["closeness"], FWD_RTOL, FWD_ATOL, "closeness")
    assert_close(f["log_denom"].cpu().numpy(), g["log_denom"], FWD_RTOL, FWD_ATOL, "log_denom")
    st = f["status"]
    got = [m, st["spheres_on_sensor"], st["candidates_tested"], st["hits_blended"], st["pixels_early_stopped"]]
    assert got == [int(x) for x in g["stats"][:5]]


@pytest.mark.parametrize("name", golden_names())
def test_golden_backward(engine, name):
    g = load_golden(name)
    cam, spec = _spec(g)
    f = engine.forward(g["pos"], g["rad"], g["opa"], g["feat"], g["bg"], spec, gamma=g["gamma"], eps=g["eps"],
                       tau=g["tau"], top_k=g["top_k"])
    assert np.array_equal(_hwk(f["ids"]), g["ids"])
    out = engine.backward(g["pos"], g["rad"], g["opa"], g["feat"], g["bg"], spec, f, g["upstream"],
                          gamma=g["gamma"], eps=g["eps"], normalize=g["normalize"], gate=g["gate"])
    assert np.array_equal(out["pixel_count"].cpu().numpy(), g["pixel_count"])
    grad_close(out["d_pos"].cpu().numpy(), g["d_position"], "d_position")
    grad_close(out["d_rad"].cpu().numpy(), g["d_radius"], "d_radius")
    grad_close(out["d_opa"].cpu().numpy(), g["d_opacity"], "d_opacity")
    grad_close(out["d_feat"].cpu().numpy(), g["d_feature"], "d_feature")
    from paper_2004_07484_b200 import AXIS_ANGLE, axis_angle_vjp, rotation_6d_vjp
    cg = out["cam_grad"].cpu().numpy()
    vjp = axis_angle_vjp if cam.rotation_type == AXIS_ANGLE else rotation_6d_vjp
    d_rot = vjp(cam.rotation_param, cg[3:12].reshape(3, 3))
    cam_vec_grad = np.concatenate([cg[0:3], d_rot, [cg[12], cg[13]]])
    want = np.concatenate([g["d_translation"], g["d_rotation"], [g["d_focal"], g["d_sensor_width"]]])
    grad_close(cam_vec_grad, want, "camera gradient")


@pytest.mark.parametrize("m,size,mode,k,d", [(300, 96, "pinhole", 5, 3), (200, 80, "orthographic", 5, 3),
                                             (150, 64, "pinhole", 3, 4), (120, 64, "pinhole", 8, 2),
                                             (100, 48, "pinhole", 12, 7), (80, 40, "pinhole", 40, 20)])
def test_random_scene_vs_oracle(engine, m, size, mode, k, d):
    from oracle import oracle as orc
    from paper_2004_07484_b200 import CameraSpec, camera_from_vector
    rng = np.random.default_rng(1000 + m)
    pos, rad, opa, feat, bg = make_random_scene(rng, m, d=d)
    vec = [0.3, -0.2, 0.5, 0.02, -0.03, 0.01, 5.0, 14.0 if mode == "orthographic" else 2.0]
    cam = camera_from_vector(vec, size, size - 7, mode=mode)
    ocam = orc.camera_from_vector(vec, size, size - 7, mode=mode)
    spec = CameraSpec.from_camera(cam)
    ref = orc.render_forward(pos, rad, opa, feat, bg, ocam, gamma=0.12, tau=0.0, top_k=k)
    f = engine.forward(pos, rad, opa, feat, bg, spec, gamma=0.12, tau=0.0, top_k=k, collect_stats=True)
    assert np.array_equal(_hwk(f["ids"]), ref["ids"])
    assert_close(f["image"].cpu().numpy(), ref["image"], FWD_RTOL, FWD_ATOL, "image")
    assert_close(f["log_denom"].cpu().numpy(), ref["log_denom"], FWD_RTOL, FWD_ATOL, "log_denom")
    assert f["status"]["hits_blended"] == ref["stats"]["hits_blended"]
    assert f["status"]["candidates_tested"] == ref["stats"]["candidates_tested"]
    up = rng.normal(size=ref["image"].shape).astype(np.float32)
    out = engine.backward(pos, rad, opa, feat, bg, spec, f, up, gamma=0.12, eps=1e-2)
    gr = orc.render_backward(pos, rad, opa, feat, bg, ocam, ref, up.astype(np.float64))
    assert np.array_equal(out["pixel_count"].cpu().numpy(), gr["pixel_count"])
    grad_close(out["d_pos"].cpu().numpy(), gr["d_position"], "d_position")
    grad_close(out["d_rad"].cpu().numpy(), gr["d_radius"], "d_radius")
    grad_close(out["d_opa"].cpu().numpy(), gr["d_opacity"], "d_opacity")
    grad_close(out["d_feat"].cpu().numpy(), gr["d_feature"], "d_feature")
    cg = out["cam_grad"].cpu().numpy()
    grad_close(cg[0:3], gr["d_translation"], "d_translation")
    grad_close(cg[3:12].reshape(3, 3), gr["grad_rot_matrix"], "dL/dR")
    grad_close(cg[12:14], [gr["d_focal"], gr["d_sensor_width"]], "d_focal/d_sensor")


@pytest.mark.parametrize("count,size", [(100_000, 512), (1_000_000, 1024)])
def test_benchmark_configs_vs_oracle(engine, count, size):
    """C2 and C3 of BASELINE.json at full size against the oracle (OpenMP, a few seconds)."""
    from oracle import oracle as orc
    from paper_2004_07484_b200 import CameraSpec, camera_from_vector
    pos, rad, opa, feat, bg, vec = orc.benchmark_scene(count, size, size, seed=0)
    cam = camera_from_vector(vec, size, size)
    ocam = orc.camera_from_vector(vec, size, size)
    spec = CameraSpec.from_camera(cam)
    thr = orc.num_threads_available()
    ref = orc.render_forward(pos, rad, opa, feat, bg, ocam, gamma=0.1, tau=0.0, top_k=5, threads=thr)
    f = engine.forward(pos, rad, opa, feat, bg, spec, gamma=0.1, tau=0.0, top_k=5, collect_stats=True)
    ids = _hwk(f["ids"])
    assert np.array_equal(ids, ref["ids"]), f"{int((ids != ref['ids']).sum())} id mismatches"
    assert_close(f["image"].cpu().numpy(), ref["image"], FWD_RTOL, FWD_ATOL, "image")
    assert_close(_hwk(f["z"]), ref["z"], FWD_RTOL, FWD_ATOL, "z")
    assert_close(_hwk(f["closeness"]), ref["closeness"], FWD_RTOL, FWD_ATOL, "closeness")
    assert f["status"]["candidates_tested"] == ref["stats"]["candidates_tested"]
    assert f["status"]["hits_blended"] == ref["stats"]["hits_blended"]
    up = np.sign(ref["image"] - 0.5).astype(np.float32)
    out = engine.backward(pos, rad, opa, feat, bg, spec, f, up, gamma=0.1, eps=1e-2)
    gr = orc.render_backward(pos, rad, opa, feat, bg, ocam, ref, up.astype(np.float64), threads=thr)
    assert np.array_equal(out["pixel_count"].cpu().numpy(), gr["pixel_count"])
    grad_close(out["d_pos"].cpu().numpy(), gr["d_position"], "d_position")
    grad_close(out["d_rad"].cpu().numpy(), gr["d_radius"], "d_radius")
    grad_close(out["d_opa"].cpu().numpy(), gr["d_opacity"], "d_opacity")
    grad_close(out["d_feat"].cpu().numpy(), gr["d_feature"], "d_feature")
    cg = out["cam_grad"].cpu().numpy()
    grad_close(cg[0:3], gr["d_translation"], "d_translation")
    grad_close(cg[3:12].reshape(3, 3), gr["grad_rot_matrix"], "dL/dR")
    grad_close(cg[12:14], [gr["d_focal"], gr["d_sensor_width"]], "d_focal/d_sensor")
