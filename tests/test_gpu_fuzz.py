"""GPU: randomised geometry against the oracle -- wide and narrow fields of view, rotated cameras,
spheres in front of / around / behind / containing the camera, sub-pixel to screen-filling radii,
ragged image sizes.  Exercises the conservative float32 filter, the per-warp culling masks and the
trig fall-back of the extents; ids, tile lists and counters must stay exact."""
import numpy as np
import pytest

from helpers import FWD_ATOL, FWD_RTOL, assert_close, grad_close

pytestmark = pytest.mark.gpu


def _random_case(seed):
    rng = np.random.default_rng(seed)
    mode = "orthographic" if seed % 4 == 3 else "pinhole"
    w, h = int(rng.integers(17, 90)), int(rng.integers(17, 90))
    focal = float(rng.uniform(0.8, 6.0))
    sensor = float(rng.uniform(1.0, 4.0)) if mode == "pinhole" else float(rng.uniform(6.0, 20.0))
    m = int(rng.integers(5, 120))
    d = int(rng.choice([1, 2, 3, 4, 6]))
    k = int(rng.choice([1, 3, 5, 8, 11]))
    if seed % 3 == 0:   # cloud in front of the camera
        pos = np.column_stack([rng.uniform(-4, 4, m), rng.uniform(-4, 4, m), rng.uniform(2, 40, m)])
        rad = rng.uniform(0.01, 2.5, m)
    elif seed % 3 == 1:  # cloud all around the camera, some spheres contain it
        pos = rng.uniform(-6, 6, (m, 3))
        rad = rng.uniform(0.05, 4.0, m)
    else:                # mixture of tiny far spheres and huge near ones
        pos = np.column_stack([rng.uniform(-8, 8, m), rng.uniform(-8, 8, m), rng.uniform(-2, 44, m)])
        rad = np.where(rng.uniform(size=m) < 0.2, rng.uniform(3, 12, m), rng.uniform(1e-3, 0.3, m))
    opa = rng.uniform(-0.2, 1.3, m)
    feat = rng.uniform(0, 1, (m, d))
    bg = rng.uniform(0, 1, d)
    t = rng.uniform(-0.5, 0.5, 3)
    if seed % 2 == 0:
        vec = np.concatenate([t, rng.uniform(-0.4, 0.4, 3), [focal, sensor]])
    else:
        a6 = np.array([1, 0, 0, 0, 1, 0], float) + rng.uniform(-0.3, 0.3, 6)
        vec = np.concatenate([t, a6, [focal, sensor]])
    f32 = np.float32
    return dict(pos=pos.astype(f32), rad=rad.astype(f32), opa=opa.astype(f32), feat=feat.astype(f32),
                bg=bg.astype(f32), vec=vec, w=w, h=h, mode=mode, k=k, gamma=float(rng.uniform(0.03, 0.6)),
                tau=0.0 if seed % 5 else 0.02, near=0.1, far=float(rng.uniform(20, 60)), rng=rng)


@pytest.mark.parametrize("seed", range(40))
def test_random_geometry_vs_oracle(engine, seed):
    from oracle import oracle as orc
    from paper_2004_07484_b200 import CameraSpec, camera_from_vector
    c = _random_case(seed)
    cam = camera_from_vector(c["vec"], c["w"], c["h"], near=c["near"], far=c["far"], mode=c["mode"])
    ocam = orc.camera_from_vector(c["vec"], c["w"], c["h"], near=c["near"], far=c["far"], mode=c["mode"])
    spec = CameraSpec.from_camera(cam)
    args = (c["pos"], c["rad"], c["opa"], c["feat"], c["bg"])
    ref = orc.render_forward(*args, ocam, gamma=c["gamma"], tau=c["tau"], top_k=c["k"])
    f = engine.forward(*args, spec, gamma=c["gamma"], tau=c["tau"], top_k=c["k"], collect_stats=True, debug=True)
    b = orc.compute_bounds(c["pos"], c["rad"], ocam)
    rect = f["rect"].cpu().numpy()
    on = f["on_sensor"].cpu().numpy().astype(bool)
    assert np.array_equal(on, b["on_sensor"])
    for j, name in enumerate(("x_min", "x_max", "y_min", "y_max")):
        assert np.array_equal(rect[:, j], b[name]), name
    starts, ids = engine.tile_lists(len(c["rad"]), c["feat"].shape[1], c["w"], c["h"], c["k"])
    o_ids, o_starts = orc.tile_lists(c["pos"], c["rad"], ocam)
    assert np.array_equal(starts, o_starts) and np.array_equal(ids, o_ids)
    st = f["status"]
    assert st["hits_blended"] == ref["stats"]["hits_blended"]
    if c["tau"] == 0.0:
        assert st["candidates_tested"] == ref["stats"]["candidates_tested"]
        assert np.array_equal(f["ids"].permute(1, 2, 0).cpu().numpy(), ref["ids"])
    assert_close(f["image"].cpu().numpy(), ref["image"], 2 * FWD_RTOL, 2 * FWD_ATOL, "image")
    if c["tau"] == 0.0:
        up = c["rng"].normal(size=ref["image"].shape).astype(np.float32)
        out = engine.backward(*args, spec, f, up, gamma=c["gamma"], eps=1e-2, normalize=bool(seed % 2),
                              gate=bool(seed % 2))
        gr = orc.render_backward(*args, ocam, ref, up.astype(np.float64), normalize=bool(seed % 2),
                                 gate=bool(seed % 2))
        assert np.array_equal(out["pixel_count"].cpu().numpy(), gr["pixel_count"])
        grad_close(out["d_pos"].cpu().numpy(), gr["d_position"], "d_position")
        grad_close(out["d_rad"].cpu().numpy(), gr["d_radius"], "d_radius")
        grad_close(out["d_opa"].cpu().numpy(), gr["d_opacity"], "d_opacity")
        grad_close(out["d_feat"].cpu().numpy(), gr["d_feature"], "d_feature")
        cg = out["cam_grad"].cpu().numpy()
        grad_close(cg[0:3], gr["d_translation"], "d_translation")
        grad_close(cg[3:12].reshape(3, 3), gr["grad_rot_matrix"], "dL/dR")
        grad_close(cg[12:14], [gr["d_focal"], gr["d_sensor_width"]], "intrinsics")


@pytest.mark.parametrize("case", ["equal_depth_ortho", "duplicates", "outlier_range", "near_ties"])
def test_tile_sort_tie_paths_vs_oracle(engine, case):
    """The per-tile sort packs (key, position) into 32 bits when a segment has <= 512 pairs; these scenes force its
    three regimes -- runs of tied 23-bit parts ranked exactly, too many ties (64-bit network instead) and a range
    stretched by one outlier -- and the order must stay the reference's (earliest, then index)."""
    from oracle import oracle as orc
    from paper_2004_07484_b200 import CameraSpec, camera_from_vector
    rng = np.random.default_rng(11)
    m, w, h = 900, 48, 32
    mode = "pinhole"
    pos = np.column_stack([rng.uniform(-1.5, 1.5, m), rng.uniform(-1.0, 1.0, m), rng.uniform(8, 30, m)])
    rad = rng.uniform(0.05, 0.4, m)
    vec = [0, 0, 0, 0, 0, 0, 5.0, 2.0]
    if case == "equal_depth_ortho":   # every earliest = c_z - r identical: all ties, order by index
        mode = "orthographic"
        vec = [0, 0, 0, 0, 0, 0, 5.0, 6.0]
        rad = np.full(m, 0.25)
        pos[:, 2] = 12.0
        pos[:, :2] = rng.uniform(-2.5, 2.5, (m, 2))
    elif case == "duplicates":        # 10 % exact duplicates: runs of two equal keys inside otherwise distinct keys
        dup = rng.choice(m, m // 10, replace=False)
        src = rng.choice(m, m // 10, replace=False)
        pos[dup], rad[dup] = pos[src], rad[src]
    elif case == "outlier_range":     # one huge far sphere in every tile: the 23-bit parts of the rest collapse
        pos[:, 2] = rng.uniform(8.0, 8.0004, m)
        pos[0], rad[0] = (0.0, 0.0, 4000.0), 3000.0
    elif case == "near_ties":         # 30 distinct depths on the axis: long runs of EQUAL keys (the float32 cast below
        # removes the 2^-50 perturbation; keys that differ in their last float64 bits need a float64 camera
        # translation and are covered by tests/test_gpu_round2.py::test_last_bit_float64_key_ties)
        base = rng.uniform(8, 30, 30)
        pos[:, 2] = base[rng.integers(0, 30, m)] * (1.0 + rng.integers(0, 4, m) * 2.0 ** -50)
        pos[:, :2] = 0.0
        rad[:] = 0.2
    f32 = np.float32
    pos, rad = pos.astype(f32), rad.astype(f32)
    opa, feat, bg = rng.uniform(0.2, 1, m).astype(f32), rng.uniform(0, 1, (m, 3)).astype(f32), np.zeros(3, f32)
    cam = camera_from_vector(vec, w, h, mode=mode)
    ocam = orc.camera_from_vector(vec, w, h, mode=mode)
    f = engine.forward(pos, rad, opa, feat, bg, CameraSpec.from_camera(cam), gamma=0.1, tau=0.0, top_k=5)
    starts, ids = engine.tile_lists(m, 3, w, h, 5)
    o_ids, o_starts = orc.tile_lists(pos, rad, ocam)
    assert np.array_equal(starts, o_starts)
    assert np.array_equal(ids, o_ids)
    seg = np.diff(o_starts)
    assert seg.max() <= 2048 and (seg > 64).any()  # exercises the multi-block packed path
    ref = orc.render_forward(pos, rad, opa, feat, bg, ocam, gamma=0.1, tau=0.0, top_k=5)
    assert np.array_equal(f["ids"].permute(1, 2, 0).cpu().numpy(), ref["ids"])


@pytest.mark.parametrize("dense", [0, 2500, 5000])
def test_bucket_and_fallback_list_paths_vs_oracle(engine, dense):
    """Tile lists come from per-tile buckets filled by the projection kernel (spheres touching > 4 tiles fill a
    bucket from its far end): <= 512 per tile sort as packed words in registers, <= 4096 as packed words in shared
    memory (persistent CTAs); one tile with more than 4096 spheres switches the whole frame to the
    count/scan/emit path (SS_FLAG_LIST_FALLBACK).  All must give the reference's lists."""
    from oracle import oracle as orc
    from paper_2004_07484_b200 import CameraSpec, camera_from_vector
    rng = np.random.default_rng(21)
    w, h = 80, 48
    vec = [0.1, -0.05, 0, 0.01, 0.02, 0, 5.0, 2.0]
    m = 1500
    pos = np.column_stack([rng.uniform(-3, 3, m), rng.uniform(-2, 2, m), rng.uniform(8, 30, m)])
    rad = np.where(rng.uniform(size=m) < 0.1, rng.uniform(1.0, 4.0, m), rng.uniform(0.02, 0.3, m))  # some span many tiles
    if dense:  # tiny spheres behind one pixel block
        extra = np.column_stack([rng.uniform(-0.02, 0.02, dense), rng.uniform(-0.02, 0.02, dense), rng.uniform(9, 35, dense)])
        pos, rad = np.vstack([pos, extra]), np.concatenate([rad, rng.uniform(0.005, 0.02, dense)])
        m += dense
    f32 = np.float32
    pos, rad = pos.astype(f32), rad.astype(f32)
    opa, feat, bg = rng.uniform(0.2, 1, m).astype(f32), rng.uniform(0, 1, (m, 3)).astype(f32), np.zeros(3, f32)
    cam, ocam = camera_from_vector(vec, w, h), orc.camera_from_vector(vec, w, h)
    f = engine.forward(pos, rad, opa, feat, bg, CameraSpec.from_camera(cam), gamma=0.1, tau=0.0, top_k=5,
                       collect_stats=True)
    assert bool(f["status"]["flags"] & 4) == (dense > 4096)
    starts, ids = engine.tile_lists(m, 3, w, h, 5)
    o_ids, o_starts = orc.tile_lists(pos, rad, ocam)
    assert (np.diff(o_starts).max() > 4096) == (dense > 4096) and (np.diff(o_starts).max() > 2048) == (dense > 0)
    assert np.array_equal(starts, o_starts) and np.array_equal(ids, o_ids)
    ref = orc.render_forward(pos, rad, opa, feat, bg, ocam, gamma=0.1, tau=0.0, top_k=5)
    assert np.array_equal(f["ids"].permute(1, 2, 0).cpu().numpy(), ref["ids"])
    assert f["status"]["hits_blended"] == ref["stats"]["hits_blended"]


@pytest.mark.parametrize("d,k", [(16, 32), (32, 64), (32, 5), (7, 64)])
def test_feature_maps_and_long_records_vs_oracle(engine, d, k):
    """The template corners of the raster / backward kernels: d up to 32 channels, n_track up to 64."""
    from oracle import oracle as orc
    from paper_2004_07484_b200 import CameraSpec, camera_from_vector
    rng = np.random.default_rng(100 + d + k)
    m, w, h = 400, 40, 24
    pos, rad, opa, feat, bg = make_random_scene_d(rng, m, d)
    vec = [0.1, 0.0, 0.0, 0.0, 0.02, 0.0, 5.0, 2.0]
    cam, ocam = camera_from_vector(vec, w, h), orc.camera_from_vector(vec, w, h)
    spec = CameraSpec.from_camera(cam)
    ref = orc.render_forward(pos, rad, opa, feat, bg, ocam, gamma=0.15, tau=0.0, top_k=k)
    f = engine.forward(pos, rad, opa, feat, bg, spec, gamma=0.15, tau=0.0, top_k=k, collect_stats=True)
    assert np.array_equal(f["ids"].permute(1, 2, 0).cpu().numpy(), ref["ids"])
    assert f["status"]["hits_blended"] == ref["stats"]["hits_blended"]
    assert_close(f["image"].cpu().numpy(), ref["image"], FWD_RTOL, FWD_ATOL, "image")
    up = rng.normal(size=ref["image"].shape).astype(np.float32)
    out = engine.backward(pos, rad, opa, feat, bg, spec, f, up, gamma=0.15, eps=1e-2)
    gr = orc.render_backward(pos, rad, opa, feat, bg, ocam, ref, up.astype(np.float64))
    assert np.array_equal(out["pixel_count"].cpu().numpy(), gr["pixel_count"])
    grad_close(out["d_pos"].cpu().numpy(), gr["d_position"], "d_position")
    grad_close(out["d_rad"].cpu().numpy(), gr["d_radius"], "d_radius")
    grad_close(out["d_opa"].cpu().numpy(), gr["d_opacity"], "d_opacity")
    grad_close(out["d_feat"].cpu().numpy(), gr["d_feature"], "d_feature")
    cg = out["cam_grad"].cpu().numpy()
    grad_close(cg[0:3], gr["d_translation"], "d_translation")
    grad_close(cg[12:14], [gr["d_focal"], gr["d_sensor_width"]], "intrinsics")


def make_random_scene_d(rng, m, d):
    pos = np.column_stack([rng.uniform(-2.5, 2.5, m), rng.uniform(-1.5, 1.5, m), rng.uniform(10, 30, m)])
    f32 = np.float32
    return (pos.astype(f32), rng.uniform(0.1, 0.8, m).astype(f32), rng.uniform(0.1, 1.0, m).astype(f32),
            rng.uniform(0, 1, (m, d)).astype(f32), rng.uniform(0, 1, d).astype(f32))


@pytest.mark.parametrize("case", ["equal_depth", "duplicates", "near_ties"])
def test_long_segment_sort_tie_paths_vs_oracle(engine, case):
    """The same tie regimes for one tile of 3000 spheres: packed words with 12 position bits in the persistent
    sort kernel (exact ranking of tied runs, 64-bit network when too many tie)."""
    from oracle import oracle as orc
    from paper_2004_07484_b200 import CameraSpec, camera_from_vector
    rng = np.random.default_rng(31)
    m, w, h = 3000, 16, 16
    pos = np.column_stack([rng.uniform(-0.05, 0.05, m), rng.uniform(-0.05, 0.05, m), rng.uniform(10, 40, m)])
    rad = rng.uniform(0.01, 0.05, m)
    if case == "equal_depth":
        pos[:, 2], rad[:] = 20.0, 0.03
        pos[:, :2] = 0.0  # identical earliest for every sphere: order by index
    elif case == "duplicates":
        dup, src = rng.choice(m, 300, replace=False), rng.choice(m, 300, replace=False)
        pos[dup], rad[dup] = pos[src], rad[src]
    else:
        base = rng.uniform(10, 40, 40)
        pos[:, 2] = base[rng.integers(0, 40, m)] * (1.0 + rng.integers(0, 4, m) * 2.0 ** -50)
        pos[:, :2], rad[:] = 0.0, 0.03
    f32 = np.float32
    pos, rad = pos.astype(f32), rad.astype(f32)
    opa, feat, bg = rng.uniform(0.2, 1, m).astype(f32), rng.uniform(0, 1, (m, 3)).astype(f32), np.zeros(3, f32)
    vec = [0, 0, 0, 0, 0, 0, 5.0, 2.0]
    cam, ocam = camera_from_vector(vec, w, h), orc.camera_from_vector(vec, w, h)
    f = engine.forward(pos, rad, opa, feat, bg, CameraSpec.from_camera(cam), gamma=0.1, tau=0.0, top_k=5,
                       collect_stats=True)
    assert not f["status"]["flags"] & 4  # bucket path
    starts, ids = engine.tile_lists(m, 3, w, h, 5)
    o_ids, o_starts = orc.tile_lists(pos, rad, ocam)
    assert int(np.diff(o_starts).max()) > 2048
    assert np.array_equal(starts, o_starts) and np.array_equal(ids, o_ids)
