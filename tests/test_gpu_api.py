"""GPU: reference-facing API (render_forward / render_backward / adapter / autograd Function),
error behaviour, early stop, determinism and full-size properties."""
import numpy as np
import pytest

from helpers import FWD_ATOL, FWD_RTOL, assert_close, grad_close, load_golden, make_random_scene

pytestmark = pytest.mark.gpu


def _scene_obj(pk, pos, rad, opa, feat, bg):
    s = pk.new_scene(bg.shape[0], bg.astype(np.float64))
    if pos.shape[0]:
        pk.add_sphere_arrays(s, pos.astype(np.float64), rad.astype(np.float64), opa.astype(np.float64),
                             feat.astype(np.float64))
    return s


def test_reference_signature_roundtrip(engine):
    """render_forward / render_backward with the reference's signatures and artefact types,
    checked against the golden C1 vectors (reference outputs)."""
    import paper_2004_07484_b200 as pk
    g = load_golden("c1_bench1k_64")
    scene = _scene_obj(pk, g["pos"], g["rad"], g["opa"], g["feat"], g["bg"])
    cam = pk.camera_from_vector(g["cam_vec"], g["width"], g["height"])
    params = pk.BlendParams(gamma=g["gamma"], epsilon=g["eps"], tau=g["tau"], top_k=g["top_k"])
    image, buffer, stats = pk.render_forward(scene, cam, params, workers=4)
    assert isinstance(image, pk.FeatureImage) and image.data.shape == (64, 64, 3) and image.data.dtype == np.float64
    assert buffer.ids.shape == (64, 64, 5) and buffer.num_spheres == 1000
    assert np.array_equal(buffer.ids, g["ids"])
    assert_close(image.data, g["image"], FWD_RTOL, FWD_ATOL, "image")
    assert [stats.spheres_total, stats.spheres_on_sensor, stats.candidates_tested, stats.hits_blended,
            stats.pixels_early_stopped, stats.tiles] == [int(x) for x in g["stats"]]
    grads, cg = pk.render_backward(scene, cam, params, buffer, g["upstream"].astype(np.float64))
    assert np.array_equal(grads.pixel_count, g["pixel_count"]) and grads.pixel_count.dtype == np.int64
    grad_close(grads.d_position, g["d_position"], "d_position")
    grad_close(grads.d_feature, g["d_feature"], "d_feature")
    grad_close(cg.d_translation, g["d_translation"], "d_translation")
    grad_close(cg.d_rotation, g["d_rotation"], "d_rotation")
    grad_close([cg.d_focal, cg.d_sensor_width], [g["d_focal"], g["d_sensor_width"]], "intrinsics")
    # store_buffer=False returns no buffer (raster.py:445)
    _, none_buf, _ = pk.render_forward(scene, cam, params, store_buffer=False)
    assert none_buf is None


def test_error_behaviour_matches_reference(engine):
    import paper_2004_07484_b200 as pk
    rng = np.random.default_rng(3)
    pos, rad, opa, feat, bg = make_random_scene(rng, 20)
    cam = pk.camera_from_vector([0, 0, 0, 0, 0, 0, 5.0, 2.0], 32, 32)
    params = pk.BlendParams(tau=0.0)
    scene = _scene_obj(pk, pos, rad, opa, feat, bg)
    bad = scene.copy()
    bad.radii[7] = -1.0  # ValidationError from the device-side scan (scene.py:110-113)
    with pytest.raises(pk.ValidationError, match="index 7"):
        pk.render_forward(bad, cam, params)
    bad = scene.copy()
    bad.features[3, 1] = np.nan
    with pytest.raises(pk.ValidationError, match="index 3"):
        pk.render_forward(bad, cam, params)
    bad = scene.copy()
    bad.background = np.array([0.0, np.inf, 0.0])
    with pytest.raises(pk.ValidationError):
        pk.render_forward(bad, cam, params)
    image, buffer, _ = pk.render_forward(scene, cam, params)
    small = _scene_obj(pk, pos[:5], rad[:5], opa[:5], feat[:5], bg)
    with pytest.raises(pk.ContractViolation):  # stale buffer, grad.py:340-343
        pk.render_backward(small, cam, params, buffer, np.zeros((32, 32, 3)))
    with pytest.raises(pk.ValidationError):  # upstream shape, grad.py:346-349
        pk.render_backward(scene, cam, params, buffer, np.zeros((32, 31, 3)))
    with pytest.raises(pk.ConfigurationError):  # other tile sizes only at tau = 0 (test_other_tile_sizes_at_tau_zero)
        pk.render_forward(scene, cam, pk.BlendParams(tau=0.01), tile_size=8)


def test_zero_upstream_and_offscreen_sphere(engine):
    """tests/test_grad.py:59-67 and :115-129 of the reference."""
    import paper_2004_07484_b200 as pk
    scene = pk.new_scene(3, [0, 0, 0])
    pk.add_sphere_arrays(scene, [[0, 0, 30.0], [0, 0, -30.0]], [2.0, 2.0], [0.9, 0.9], [[1, 0, 0], [0, 1, 0]])
    cam = pk.camera_from_vector([0, 0, 0, 0, 0, 0, 5.0, 2.0], 24, 24)
    params = pk.BlendParams(gamma=0.1, tau=0.0)
    image, buffer, stats = pk.render_forward(scene, cam, params)
    assert stats.spheres_on_sensor == 1
    g, cg = pk.render_backward(scene, cam, params, buffer, np.zeros_like(image.data))
    assert np.all(g.d_position == 0) and np.all(g.d_feature == 0) and np.all(cg.d_translation == 0)
    g, _ = pk.render_backward(scene, cam, params, buffer, np.ones_like(image.data), gate=False)
    assert g.pixel_count[1] == 0 and np.all(g.d_position[1] == 0) and np.all(g.d_feature[1] == 0)
    assert g.pixel_count[0] > 0


def test_empty_scene_and_background(engine):
    import paper_2004_07484_b200 as pk
    scene = pk.new_scene(3, [0.2, 0.4, 0.6])
    cam = pk.camera_from_vector([0, 0, 0, 0, 0, 0, 5.0, 2.0], 20, 17)
    image, buffer, stats = pk.render_forward(scene, cam, pk.BlendParams())
    assert np.allclose(image.data, [0.2, 0.4, 0.6], atol=1e-7) and np.all(image.background_weight == 1.0)
    assert np.all(buffer.ids == -1) and stats.candidates_tested == 0
    g, cg = pk.render_backward(scene, cam, pk.BlendParams(), buffer, np.ones((17, 20, 3)))
    assert g.d_position.shape == (0, 3) and np.all(cg.d_translation == 0) and cg.d_focal == 0.0


def test_gating_and_normalisation_rules(engine):
    """grad.py:262-320: pixel-mean normalisation, 1e-3/area camera scale, gate at proj radius <= 3 px."""
    import paper_2004_07484_b200 as pk
    from oracle import oracle as orc
    rng = np.random.default_rng(11)
    pos, rad, opa, feat, bg = make_random_scene(rng, 30, radius=(0.05, 1.5))
    vec = [0, 0, 0, 0, 0, 0, 5.0, 2.0]
    cam = pk.camera_from_vector(vec, 64, 64)
    spec = pk.CameraSpec.from_camera(cam)
    f = engine.forward(pos, rad, opa, feat, bg, spec, gamma=0.1, tau=0.0, top_k=5, debug=True)
    up = rng.normal(size=(64, 64, 3)).astype(np.float32)
    raw = engine.backward(pos, rad, opa, feat, bg, spec, f, up, gamma=0.1, eps=1e-2, normalize=False, gate=False)
    nrm = engine.backward(pos, rad, opa, feat, bg, spec, f, up, gamma=0.1, eps=1e-2, normalize=True, gate=True)
    cnt = raw["pixel_count"].cpu().numpy()
    pr = f["proj_radius_px"].cpu().numpy()
    gated = pr <= 3.0
    assert gated.any() and (~gated & (cnt > 0)).any()
    div = np.maximum(cnt, 1)[:, None]
    # two launches sum their float32 atomics in different orders: compare to atomics tolerance
    grad_close(nrm["d_feat"].cpu().numpy(), raw["d_feat"].cpu().numpy() / div, "d_feature / count", rtol=2e-5)
    dp = nrm["d_pos"].cpu().numpy()
    assert np.all(dp[gated] == 0) and np.all(nrm["d_rad"].cpu().numpy()[gated] == 0)
    grad_close(dp[~gated], (raw["d_pos"].cpu().numpy() / div)[~gated], "d_position / count", rtol=2e-5)
    ocam = orc.camera_from_vector(vec, 64, 64)
    ref = orc.render_forward(pos, rad, opa, feat, bg, ocam, gamma=0.1, tau=0.0)
    gr = orc.render_backward(pos, rad, opa, feat, bg, ocam, ref, up.astype(np.float64))
    grad_close(nrm["cam_grad"].cpu().numpy()[0:3], gr["d_translation"], "normalised d_translation")


@pytest.mark.parametrize("chunk", [256, 64, 7])
def test_early_stop_bound_and_chunk_sizes(engine, chunk):
    """tau > 0: image within tau/(1-tau) of the tau = 0 image, counters shrink (tests/test_raster.py:285-306);
    stats and image equal the oracle's for the same chunk size."""
    from oracle import oracle as orc
    from paper_2004_07484_b200 import CameraSpec, camera_from_vector
    from paper_2004_07484_b200.synthetic import benchmark_scene
    pos, rad, opa, feat, bg, vec = benchmark_scene(20000, 96, 96, seed=2, profile="occluded")
    spec = CameraSpec.from_camera(camera_from_vector(vec, 96, 96))
    ocam = orc.camera_from_vector(vec, 96, 96)
    f0 = engine.forward(pos, rad, opa, feat, bg, spec, gamma=0.1, tau=0.0, top_k=5, chunk=chunk, collect_stats=True)
    f1 = engine.forward(pos, rad, opa, feat, bg, spec, gamma=0.1, tau=0.01, top_k=5, chunk=chunk, collect_stats=True)
    i0, i1 = f0["image"].cpu().numpy(), f1["image"].cpu().numpy()
    assert np.abs(i0 - i1).max() <= 0.01 / 0.99 * max(1.0, np.abs(i0).max())
    assert f1["status"]["pixels_early_stopped"] > 0
    assert f1["status"]["candidates_tested"] < f0["status"]["candidates_tested"]
    ref = orc.render_forward(pos, rad, opa, feat, bg, ocam, gamma=0.1, tau=0.01, top_k=5, chunk=chunk)
    assert f1["status"]["candidates_tested"] == ref["stats"]["candidates_tested"]
    assert f1["status"]["pixels_early_stopped"] == ref["stats"]["pixels_early_stopped"]
    assert_close(i1, ref["image"], FWD_RTOL, FWD_ATOL, "image (tau=0.01)")


def test_pair_overflow_regrows_workspace():
    """A full-cover sphere lands in every tile (tests/test_raster.py:308-313): more pairs than
    the initial capacity -> overflow flag -> workspace regrown -> same result as the oracle."""
    import paper_2004_07484_b200 as pk
    from oracle import oracle as orc
    eng = pk.RenderEngine("cuda", pair_factor=1.0, min_pairs=8)
    pos = np.array([[0, 0, 3.0], [0.5, 0.2, 20.0], [0, 0, 10.0]], np.float32)
    rad = np.array([2.9, 1.0, 30.0], np.float32)  # third: camera inside the sphere -> full image
    opa = np.array([0.6, 0.9, 0.3], np.float32)
    feat = np.eye(3, dtype=np.float32)
    bg = np.zeros(3, np.float32)
    vec = [0, 0, 0, 0, 0, 0, 5.0, 2.0]
    spec = pk.CameraSpec.from_camera(pk.camera_from_vector(vec, 64, 64))
    f = eng.forward(pos, rad, opa, feat, bg, spec, gamma=0.2, tau=0.0, collect_stats=True)
    ref = orc.render_forward(pos, rad, opa, feat, bg, orc.camera_from_vector(vec, 64, 64), gamma=0.2, tau=0.0)
    assert f["status"]["num_pairs"] == ref["stats"]["candidates_tested"] > 8
    assert f["status"]["hits_blended"] == ref["stats"]["hits_blended"]
    assert np.array_equal(f["ids"].permute(1, 2, 0).cpu().numpy(), ref["ids"])
    assert_close(f["image"].cpu().numpy(), ref["image"], FWD_RTOL, FWD_ATOL, "image")


def test_long_tile_lists_use_the_big_sort_paths(engine):
    """> 2048 and > 8192 candidates in one tile: dynamic-smem and global-memory bitonic paths."""
    from oracle import oracle as orc
    from paper_2004_07484_b200 import CameraSpec, camera_from_vector
    rng = np.random.default_rng(9)
    vec = [0, 0, 0, 0, 0, 0, 5.0, 2.0]
    for m in (3000, 9000):
        pos = np.column_stack([rng.uniform(-0.05, 0.05, m), rng.uniform(-0.05, 0.05, m),
                               rng.uniform(10, 40, m)]).astype(np.float32)
        rad = rng.uniform(0.01, 0.05, m).astype(np.float32)
        opa = rng.uniform(0.2, 1.0, m).astype(np.float32)
        feat = rng.uniform(0, 1, (m, 3)).astype(np.float32)
        bg = np.zeros(3, np.float32)
        spec = CameraSpec.from_camera(camera_from_vector(vec, 16, 16))
        f = engine.forward(pos, rad, opa, feat, bg, spec, gamma=0.1, tau=0.0, collect_stats=True)
        starts, ids = engine.tile_lists(m, 3, 16, 16, 5)
        o_ids, o_starts = orc.tile_lists(pos, rad, orc.camera_from_vector(vec, 16, 16))
        assert int(np.diff(o_starts).max()) > (2048 if m == 3000 else 8192)
        assert np.array_equal(starts, o_starts) and np.array_equal(ids, o_ids)
        ref = orc.render_forward(pos, rad, opa, feat, bg, orc.camera_from_vector(vec, 16, 16), gamma=0.1, tau=0.0)
        assert np.array_equal(f["ids"].permute(1, 2, 0).cpu().numpy(), ref["ids"])


def test_many_long_tiles_beside_short_ones_sort_exactly_every_time(engine):
    """The small-segment sort runs beside the two long-segment kernels (side stream), and the second long-segment kernel
    skips the list entries the first one has marked: 64 tiles of ~1 500 candidates (k_tile_sort_mid), one tile beyond
    4 096 (k_tile_sort_big) and short tiles in one frame, five frames in a row, lists equal to the oracle's each time."""
    from oracle import oracle as orc
    from paper_2004_07484_b200 import CameraSpec, camera_from_vector
    rng = np.random.default_rng(21)
    vec = [0, 0, 0, 0, 0, 0, 5.0, 2.0]
    w = h = 256
    ocam = orc.camera_from_vector(vec, w, h)
    # a dense 128 x 128 px patch (64 tiles), a pile on one tile, a sparse rest
    def patch(n, lo, hi, z=(10, 40)):
        zz = rng.uniform(*z, n)
        sx = rng.uniform(lo, hi, n) * zz / 5.0
        sy = rng.uniform(lo, hi, n) * zz / 5.0
        return np.column_stack([sx, sy, zz])
    half = 1.0  # sensor half-width: sensor_w = 2 (vec[7])
    pos = np.concatenate([patch(90_000, -0.98 * half, 0.0), patch(6_000, 0.30 * half, 0.34 * half),
                          patch(3_000, -half, half)]).astype(np.float32)
    m = len(pos)
    rad = rng.uniform(0.002, 0.01, m).astype(np.float32)
    opa = rng.uniform(0.2, 1.0, m).astype(np.float32)
    feat = rng.uniform(0, 1, (m, 3)).astype(np.float32)
    bg = np.zeros(3, np.float32)
    spec = CameraSpec.from_camera(camera_from_vector(vec, w, h))
    o_ids, o_starts = orc.tile_lists(pos, rad, ocam)
    lens = np.diff(o_starts)
    assert (lens > 512).sum() >= 32 and lens.max() > 4096 and (lens[lens > 0] <= 512).any(), np.sort(lens)[-5:]
    for _ in range(5):
        engine.forward(pos, rad, opa, feat, bg, spec, gamma=0.1, tau=0.0, collect_stats=True)
        starts, ids = engine.tile_lists(m, 3, w, h, 5)
        assert np.array_equal(starts, o_starts) and np.array_equal(ids, o_ids)


def test_forward_is_deterministic_and_order_invariant(engine):
    """Bit-identical across runs (tests/test_raster.py:259-269); permuting the input spheres
    permutes the ids and leaves the image unchanged to rounding (:271-283)."""
    from paper_2004_07484_b200 import CameraSpec, camera_from_vector
    from paper_2004_07484_b200.synthetic import benchmark_scene
    pos, rad, opa, feat, bg, vec = benchmark_scene(200_000, 512, 512, seed=4)
    spec = CameraSpec.from_camera(camera_from_vector(vec, 512, 512))
    a = engine.forward(pos, rad, opa, feat, bg, spec, gamma=0.1, tau=0.0)
    a_img, a_ids, a_z = a["image"].clone(), a["ids"].clone(), a["z"].clone()
    b = engine.forward(pos, rad, opa, feat, bg, spec, gamma=0.1, tau=0.0)
    assert (a_img == b["image"]).all() and (a_ids == b["ids"]).all() and (a_z == b["z"]).all()
    perm = np.random.default_rng(0).permutation(pos.shape[0])
    c = engine.forward(pos[perm], rad[perm], opa[perm], feat[perm], bg, spec, gamma=0.1, tau=0.0)
    ids_c = c["ids"].cpu().numpy()
    mapped = np.where(ids_c >= 0, perm[np.maximum(ids_c, 0)], -1)
    ids_a = a_ids.cpu().numpy()
    # identical sets per pixel; order can differ only between exactly tied depths
    assert (np.sort(mapped, axis=0) == np.sort(ids_a, axis=0)).all()
    assert np.abs(c["image"].cpu().numpy() - a_img.cpu().numpy()).max() < 2e-6


def test_weights_partition_unity_at_full_size(engine):
    """Size-independent property at C3 scale: with unit features and zero background the image
    equals 1 - background_weight in every pixel; buffer depths are sorted nearest-first."""
    from paper_2004_07484_b200 import CameraSpec, camera_from_vector
    from paper_2004_07484_b200.synthetic import benchmark_scene
    pos, rad, opa, feat, bg, vec = benchmark_scene(1_000_000, 1024, 1024, seed=1)
    feat[:] = 1.0
    spec = CameraSpec.from_camera(camera_from_vector(vec, 1024, 1024))
    f = engine.forward(pos, rad, opa, feat, bg, spec, gamma=0.1, tau=0.0, top_k=5)
    img, bgw = f["image"], f["bg_weight"]
    assert float((img.sum(dim=2) / 3.0 + bgw - 1.0).abs().max()) < 5e-6
    z, ids = f["z"], f["ids"]
    assert bool((z[:-1] >= z[1:]).all())
    assert bool(((ids[:-1] >= 0) | (ids[1:] < 0)).all())  # empty slots only at the tail
    # linearity of the backward pass in the upstream gradient
    up1 = (img * 0 + 1.0)
    g1 = engine.backward(pos, rad, opa, feat, bg, spec, f, up1, gamma=0.1, eps=1e-2, normalize=False, gate=False)
    d1 = g1["d_opa"].clone()
    g2 = engine.backward(pos, rad, opa, feat, bg, spec, f, 2.0 * up1, gamma=0.1, eps=1e-2, normalize=False, gate=False)
    scale = float(d1.abs().max())
    assert float((g2["d_opa"] - 2.0 * d1).abs().max()) <= 1e-4 * scale


def test_autograd_function_matches_oracle(engine):
    import torch
    import paper_2004_07484_b200 as pk
    from oracle import oracle as orc
    rng = np.random.default_rng(21)
    pos, rad, opa, feat, bg = make_random_scene(rng, 50, radius=(0.8, 2.5))
    vec = np.array([0.3, -0.2, 0.5, 0.02, -0.03, 0.01, 5.0, 2.0])
    target = rng.uniform(0, 1, (48, 48, 3)).astype(np.float32)
    r = pk.Renderer(48, 48, n_track=8, normalize=False, gate=False)
    t = {k: torch.tensor(v, device="cuda", requires_grad=True) for k, v in
         dict(pos=pos, feat=feat, rad=rad, opa=opa).items()}
    cam_vec = torch.tensor(vec, dtype=torch.float64, requires_grad=True)
    img = r(t["pos"], t["feat"], t["rad"], cam_vec, opacity=t["opa"], background=torch.tensor(bg, device="cuda"),
            gamma=0.2, tau=0.0)
    loss = 0.5 * ((img - torch.tensor(target, device="cuda")) ** 2).sum()
    loss.backward()
    ocam = orc.camera_from_vector(vec, 48, 48)
    ref = orc.render_forward(pos, rad, opa, feat, bg, ocam, gamma=0.2, tau=0.0, top_k=8)
    gr = orc.render_backward(pos, rad, opa, feat, bg, ocam, ref, ref["image"] - target.astype(np.float64),
                             normalize=False, gate=False)
    assert_close(img.detach().cpu().numpy(), ref["image"], FWD_RTOL, FWD_ATOL, "image")
    grad_close(t["pos"].grad.cpu().numpy(), gr["d_position"], "d_position")
    grad_close(t["rad"].grad.cpu().numpy(), gr["d_radius"], "d_radius")
    grad_close(t["opa"].grad.cpu().numpy(), gr["d_opacity"], "d_opacity")
    grad_close(t["feat"].grad.cpu().numpy(), gr["d_feature"], "d_feature")
    want = np.concatenate([gr["d_translation"], gr["d_rotation"], [gr["d_focal"], gr["d_sensor_width"]]])
    grad_close(cam_vec.grad.numpy(), want, "cam_vec gradient")


def test_host_session_matches_device_path(engine):
    import torch
    import paper_2004_07484_b200 as pk
    from paper_2004_07484_b200.host import HostRenderSession
    from paper_2004_07484_b200.synthetic import benchmark_scene
    pos, rad, opa, feat, bg, vec = benchmark_scene(5000, 128, 128, seed=6)
    spec = pk.CameraSpec.from_camera(pk.camera_from_vector(vec, 128, 128))
    f = engine.forward(pos, rad, opa, feat, bg, spec, gamma=0.1, tau=0.0)
    up = torch.sign(f["image"] - 0.5)
    ref = engine.backward(pos, rad, opa, feat, bg, spec, f, up, gamma=0.1, eps=1e-2)
    ref_feat = ref["d_feat"].cpu().numpy().copy()
    sess = HostRenderSession(5000, 3, 128, 128, 5, engine=engine)
    sess.set_scene(pos, rad, opa, feat, bg)
    image, grads = sess.render_step(spec, upstream_fn=lambda i, im: torch.sign(im - 0.5), gamma=0.1, tau=0.0)
    assert np.array_equal(image.numpy(), f["image"].cpu().numpy())
    assert np.array_equal(grads["pixel_count"].numpy(), ref["pixel_count"].cpu().numpy())
    grad_close(grads["d_feat"].numpy(), ref_feat, "host-session d_feature", rtol=1e-5)
    # resident scene (no re-upload) + compact download: only the rows of the spheres that received gradient
    dense = {k: grads[k].numpy().copy() for k in ("d_pos", "d_rad", "d_opa", "d_feat", "pixel_count")}
    for rep in range(3):  # the second and third call use the speculative one-round-trip download
        image, cg = sess.render_step(spec, upstream_fn=lambda i, im: torch.sign(im - 0.5), gamma=0.1, tau=0.0,
                                     compact=True)
        assert sess.last_h2d_bytes == 4 * 128 * 128 * 3  # upstream only: the scene stayed on the device
        idx = cg["index"].numpy()
        touched = np.flatnonzero(dense["pixel_count"] > 0)
        assert cg["count"] == touched.size and np.array_equal(idx, touched)
        assert np.array_equal(cg["pixel_count"].numpy(), dense["pixel_count"][touched])
        for k in ("d_pos", "d_rad", "d_opa", "d_feat"):
            grad_close(cg[k].numpy(), dense[k][touched], f"compact {k}", rtol=2e-5)
        grad_close(cg["cam_grad"].numpy()[:14], ref["cam_grad"].cpu().numpy()[:14], "compact cam_grad", rtol=2e-5)
    # a smaller scene afterwards touches MORE spheres than the speculative estimate of a fresh session would cover
    sess2 = HostRenderSession(5000, 3, 128, 128, 5, engine=engine)
    sess2.set_scene(pos, rad * 0.3, opa, feat, bg)
    _, few = sess2.render_step(spec, upstream_fn=lambda i, im: torch.sign(im - 0.5), gamma=0.1, tau=0.0, compact=True)
    sess2.set_scene(pos, rad, opa, feat, bg)
    _, more = sess2.render_step(spec, upstream_fn=lambda i, im: torch.sign(im - 0.5), gamma=0.1, tau=0.0, compact=True)
    assert more["count"] == touched.size and np.array_equal(more["index"].numpy(), touched)
    assert np.array_equal(more["pixel_count"].numpy(), dense["pixel_count"][touched])


@pytest.mark.parametrize("m,d", [(1, 3), (255, 1), (4099, 3), (100000, 16), (20000, 32)])
def test_compact_gradient_records_device_array_and_mapped_host_array(engine, m, d):
    """CompactGradients: records [index | pixel_count | d_pos | d_rad | d_opa | d_feat] of the rows with pixel_count > 0,
    bit-identical to the dense columns, for the device record array + copy (zero_copy=False) and for the compaction
    kernel writing into the mapped pinned host array (zero_copy=True); ragged block ends, empty and full masks."""
    import torch
    from paper_2004_07484_b200.host import CompactGradients
    dev = engine.device
    g = torch.Generator().manual_seed(m + d)
    for density in (0.0, 0.3, 1.0):
        pc = ((torch.rand(m, generator=g) < density).to(torch.int32) * torch.randint(1, 900, (m,), generator=g,
                                                                                     dtype=torch.int32))
        dense = {"pixel_count": pc, "d_pos": torch.randn(m, 3, generator=g), "d_rad": torch.randn(m, generator=g),
                 "d_opa": torch.randn(m, generator=g), "d_feat": torch.randn(m, d, generator=g)}
        on_dev = {k: v.to(dev) for k, v in dense.items()}
        touched = np.flatnonzero(pc.numpy() > 0)
        for zero_copy in (False, True):
            cg = CompactGradients(m, d, dev, zero_copy=zero_copy)
            for rep in range(2):  # (the second call of the copying form downloads speculatively)
                got = cg.gather(on_dev, torch.cuda.current_stream(dev))
                assert got["count"] == touched.size
                assert np.array_equal(got["index"].numpy(), touched)
                for k in ("pixel_count", "d_pos", "d_rad", "d_opa", "d_feat"):
                    assert np.array_equal(got[k].numpy(), dense[k].numpy()[touched]), (k, zero_copy, density)
                assert cg.last_bytes >= 8 + 4 * touched.size * (7 + d)


def test_host_session_graph_replayed_step_equals_the_stream_launched_one(engine):
    """render_step(..., graph=True): the one-view step with a staged upstream and compact rows captured once and
    replayed; same image bits, same touched rows, same gradients as the stream-launched step, also after the scene
    was replaced (set_scene: one stream-launched step uploads it, the replays see the new values) and for a second
    camera (its own capture)."""
    import torch
    import paper_2004_07484_b200 as pk
    from paper_2004_07484_b200.host import HostRenderSession
    from paper_2004_07484_b200.synthetic import benchmark_scene
    pos, rad, opa, feat, bg, vec = benchmark_scene(20000, 160, 128, seed=16)
    spec = pk.CameraSpec.from_camera(pk.camera_from_vector(vec, 160, 128))
    vec2 = list(vec)
    vec2[3] += 0.05
    spec2 = pk.CameraSpec.from_camera(pk.camera_from_vector(vec2, 160, 128))
    sess = HostRenderSession(20000, 3, 160, 128, 5, engine=engine)
    sess.h_upstream.copy_(torch.sign(torch.rand(128, 160, 3, generator=torch.Generator().manual_seed(3)) - 0.5))

    def snapshot(image, g):
        return (image.numpy().copy(), int(g["count"]), g["index"].numpy().copy(), g["pixel_count"].numpy().copy(),
                {k: g[k].numpy().copy() for k in ("d_pos", "d_rad", "d_opa", "d_feat", "cam_grad")})

    for scene_radius in (1.0, 0.6):
        sess.set_scene(pos, rad * scene_radius, opa, feat, bg)
        for cam in (spec, spec2):
            ref = snapshot(*sess.render_step(cam, gamma=0.1, tau=0.01, compact=True))
            ref = snapshot(*sess.render_step(cam, gamma=0.1, tau=0.01, compact=True))  # (speculative download primed)
            for rep in range(3):
                got = snapshot(*sess.render_step(cam, gamma=0.1, tau=0.01, compact=True, graph=True))
                assert np.array_equal(got[0], ref[0])
                assert got[1] == ref[1] and np.array_equal(got[2], ref[2]) and np.array_equal(got[3], ref[3])
                for k in ref[4]:
                    a, e = got[4][k], ref[4][k]
                    if k == "cam_grad":
                        a, e = a[:14], e[:14]
                    grad_close(a, e, f"graph-replayed {k}", rtol=2e-5)
    assert 1 <= len(sess._step_graphs) <= 4


def test_accumulator_reuse_protocol(engine):
    """ss_backward re-zeroes only the accumulator rows it touched and trusts a tag on the next call.
    Repeated calls, a layout change in between, and a fresh engine must all give the same gradients."""
    import torch
    import paper_2004_07484_b200 as pk
    from paper_2004_07484_b200.synthetic import benchmark_scene

    def grads_of(eng, scene, spec):
        f = eng.forward(*scene, spec, gamma=0.1, tau=0.0)
        up = torch.sign(f["image"] - 0.5)
        o = eng.backward(*scene, spec, f, up, gamma=0.1, eps=1e-2)
        return {k: o[k].clone() for k in ("d_pos", "d_rad", "d_opa", "d_feat", "pixel_count", "cam_grad")}

    a = benchmark_scene(20000, 128, 128, seed=11)
    b = benchmark_scene(7000, 96, 96, seed=12)
    spec_a = pk.CameraSpec.from_camera(pk.camera_from_vector(a[5], 128, 128))
    spec_b = pk.CameraSpec.from_camera(pk.camera_from_vector(b[5], 96, 96))
    ref = grads_of(pk.RenderEngine("cuda"), a[:5], spec_a)
    runs = [grads_of(engine, a[:5], spec_a), grads_of(engine, a[:5], spec_a)]
    grads_of(engine, b[:5], spec_b)  # different layout on the same workspace memory
    runs.append(grads_of(engine, a[:5], spec_a))
    for r in runs:
        assert torch.equal(r["pixel_count"], ref["pixel_count"])
        for k in ("d_pos", "d_rad", "d_opa", "d_feat"):
            grad_close(r[k].cpu().numpy(), ref[k].cpu().numpy(), k, rtol=2e-5)
        grad_close(r["cam_grad"].cpu().numpy(), ref["cam_grad"].cpu().numpy(), "cam_grad", rtol=2e-5)


def test_other_tile_sizes_at_tau_zero(engine):
    """The reference accepts any tile_size (raster.py:437-447).  At tau = 0 image, buffer and gradients do not
    depend on it, only the `tiles` / `candidates_tested` counters do: checked against the REFERENCE's outputs for
    tile sizes 8 / 24 / 32 (tests/golden/extras_tile_sizes.npz).  With tau > 0 the vote is per tile: refused."""
    import os
    import paper_2004_07484_b200 as pk
    from helpers import GOLDEN_DIR
    g = np.load(os.path.join(GOLDEN_DIR, "extras_tile_sizes.npz"))
    scene = _scene_obj(pk, g["pos"], g["rad"], g["opa"], g["feat"], g["bg"])
    cam = pk.camera_from_vector(g["cam_vec"], int(g["width"]), int(g["height"]))
    p0 = pk.BlendParams(gamma=0.1, tau=0.0, top_k=5)
    base, buf16, _ = pk.render_forward(scene, cam, p0, engine=engine)
    up = np.random.default_rng(0).normal(size=base.data.shape)
    g16, _ = pk.render_backward(scene, cam, p0, buf16, up, engine=engine)
    for tile in g["tile_sizes"]:
        image, buf, st = pk.render_forward(scene, cam, p0, tile_size=int(tile), engine=engine)
        assert np.array_equal(buf.ids, g[f"ids_{tile}"])
        assert_close(image.data, g[f"image_{tile}"], FWD_RTOL, FWD_ATOL, f"image, tile_size {tile}")
        assert [st.spheres_total, st.spheres_on_sensor, st.candidates_tested, st.hits_blended,
                st.pixels_early_stopped, st.tiles] == [int(x) for x in g[f"stats_{tile}"]]
        gt, _ = pk.render_backward(scene, cam, p0, buf, up, tile_size=int(tile), engine=engine)
        assert np.array_equal(gt.pixel_count, g16.pixel_count)
        grad_close(gt.d_position, g16.d_position, f"d_position, tile_size {tile}", rtol=2e-5)
    with pytest.raises(pk.ConfigurationError, match="tau = 0"):
        pk.render_forward(scene, cam, pk.BlendParams(gamma=0.1, tau=0.01), tile_size=8, engine=engine)
    with pytest.raises(pk.ConfigurationError):
        pk.render_forward(scene, cam, p0, tile_size=0, engine=engine)


@pytest.mark.parametrize("n_bands", [1, 2, 3, 7, 16])
def test_banded_forward_is_identical_and_bands_complete_in_order(engine, n_bands):
    """ss_forward_banded draws the image in bands of tile rows (one raster launch each) and records an event per
    band so that a host caller can download the upper rows early.  Tiles are independent: every output and every
    counter must equal the single-launch forward bit for bit, for band counts that do not divide the tile rows
    (H = 100: 7 tile rows) and for more bands than tile rows (empty bands)."""
    import torch
    import paper_2004_07484_b200 as pk
    from paper_2004_07484_b200.synthetic import benchmark_scene
    w, h = 136, 100
    pos, rad, opa, feat, bg, vec = benchmark_scene(20000, w, h, seed=3)
    spec = pk.CameraSpec.from_camera(pk.camera_from_vector(vec, w, h))
    ref = engine.forward(pos, rad, opa, feat, bg, spec, gamma=0.1, tau=0.01, collect_stats=True)
    events = [torch.cuda.Event() for _ in range(n_bands)]
    out = engine.forward(pos, rad, opa, feat, bg, spec, gamma=0.1, tau=0.01, collect_stats=True, band_events=events)
    for k in ("image", "bg_weight", "ids", "z", "closeness", "log_denom"):
        assert torch.equal(out[k], ref[k]), k
    for k in ("num_pairs", "candidates_tested", "hits_blended", "pixels_early_stopped", "spheres_on_sensor"):
        assert out["status"][k] == ref["status"][k], k
    rows = [engine.band_rows(h, n_bands, b) for b in range(n_bands)]
    assert rows[0][0] == 0 and rows[-1][1] == h
    for (a0, a1), (b0, b1) in zip(rows, rows[1:]):
        assert a1 == b0 and a0 <= a1  # contiguous, top to bottom
    assert all(r0 % 16 == 0 for r0, _ in rows)
    torch.cuda.synchronize()
    assert all(e.query() for e in events)
    # rows of band b are final once event b has completed: download band by band on a second stream
    side = torch.cuda.Stream()
    host = torch.empty((h, w, 3), dtype=torch.float32).pin_memory()
    out2 = engine.forward(pos, rad, opa, feat, bg, spec, gamma=0.1, tau=0.01, check=False, band_events=events)
    with torch.cuda.stream(side):
        for (r0, r1), e in zip(rows, events):
            side.wait_event(e)
            if r1 > r0:
                host[r0:r1].copy_(out2["image"][r0:r1], non_blocking=True)
    side.synchronize()
    assert np.array_equal(host.numpy(), ref["image"].cpu().numpy())


def test_host_session_multi_view_step_pipelined_equals_serial(engine):
    """A multi-view render_step with a staged upstream alternates views between two lanes (engines) on two compute
    streams.  Its gradients must equal the serial loop's (pixel counts exactly) and the sum over views of the
    engine's single-view backward; the image that comes back is the last view's."""
    import torch
    import paper_2004_07484_b200 as pk
    from paper_2004_07484_b200.host import HostRenderSession
    from paper_2004_07484_b200.synthetic import benchmark_scene, orbit_camera_vectors
    m, w, h = 30000, 160, 112
    pos, rad, opa, feat, bg, _ = benchmark_scene(m, w, h, seed=4)
    cams = [pk.CameraSpec.from_camera(pk.camera_from_vector(v, w, h)) for v in orbit_camera_vectors(64)[:5]]
    up = torch.sign(torch.rand((h, w, 3), generator=torch.Generator().manual_seed(1)) - 0.5)
    # reference: the engine, view by view
    want, last_image = None, None
    for cam in cams:
        f = engine.forward(pos, rad, opa, feat, bg, cam, gamma=0.1, tau=0.01)
        o = engine.backward(pos, rad, opa, feat, bg, cam, f, up.cuda(), gamma=0.1, eps=1e-2)
        got = {k: o[k].double().cpu().numpy() for k in ("d_pos", "d_rad", "d_opa", "d_feat", "pixel_count")}
        want = got if want is None else {k: want[k] + got[k] for k in got}
        last_image = f["image"].cpu().numpy()
    results = {}
    for mode in (True, False, True):
        sess = HostRenderSession(m, 3, w, h, 5, engine=engine)
        sess.set_scene(pos, rad, opa, feat, bg)
        sess.h_upstream.copy_(up)
        for _ in range(2):  # second step: buffers, lanes and events are reused
            image, g = sess.render_step(cams, gamma=0.1, eps=1e-2, tau=0.01, pipeline=mode)
        assert np.array_equal(image.numpy(), last_image)
        assert np.array_equal(g["pixel_count"].numpy(), want["pixel_count"].astype(np.int32))
        for k in ("d_pos", "d_rad", "d_opa", "d_feat"):
            grad_close(g[k].numpy(), want[k], f"multi-view session {k} (pipeline={mode})", rtol=5e-5)
        results[mode] = {k: g[k].numpy().copy() for k in ("d_pos", "d_feat")}
        # compact download after a pipelined step
        image, cg = sess.render_step(cams, gamma=0.1, eps=1e-2, tau=0.01, pipeline=mode, compact=True)
        touched = np.flatnonzero(want["pixel_count"] > 0)
        assert cg["count"] == touched.size and np.array_equal(cg["index"].numpy(), touched)
