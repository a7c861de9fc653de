"""GPU: the reference's plug-in seam end to end.

`SoftsphereAdapter` is the `renderer=` object of the reference's fit loop (optim.py:265-278).  The first
tests drive it with this package's own host types against the golden fixtures (outputs of the reference).
The last ones run the UNMODIFIED reference package (installed by the build hook into the git-ignored
baseline/_ref) with the adapter plugged in: its own `fit`, and the acceptance checks of its own test-suite
restated here against its own oracle (`testkit.oracle_render`) -- skipped where baseline/_ref is absent.
"""
import numpy as np
import pytest

from helpers import (FWD_ATOL, FWD_RTOL, assert_close, grad_close, load_golden, make_random_scene,
                     reference_package)

pytestmark = pytest.mark.gpu


def _scene_obj(mod, pos, rad, opa, feat, bg):
    """SphereScene of `mod` (this package or the reference) with float64 columns."""
    s = mod.new_scene(bg.shape[0], bg.astype(np.float64))
    s.positions, s.radii = pos.astype(np.float64), rad.astype(np.float64)
    s.opacities, s.features = opa.astype(np.float64), feat.astype(np.float64)
    return s


def test_adapter_forward_backward_golden_c1(engine):
    import paper_2004_07484_b200 as pk
    g = load_golden("c1_bench1k_64")
    scene = _scene_obj(pk, g["pos"], g["rad"], g["opa"], g["feat"], g["bg"])
    cam = pk.camera_from_vector(g["cam_vec"], g["width"], g["height"])
    params = pk.BlendParams(gamma=g["gamma"], epsilon=g["eps"], tau=g["tau"], top_k=g["top_k"])
    r = pk.SoftsphereAdapter(normalize=g["normalize"], gate=g["gate"], engine=engine)
    image, buffer, stats = r.forward(scene, cam, params)
    assert image.data.dtype == np.float64 and image.background_weight.dtype == np.float64
    assert image.data.flags.writeable and image.data.flags.c_contiguous
    assert_close(image.data, g["image"], FWD_RTOL, FWD_ATOL, "image")
    assert_close(image.background_weight, g["bg_weight"], FWD_RTOL, FWD_ATOL, "bg_weight")
    assert np.array_equal(buffer.ids, g["ids"]) and buffer.z.dtype == np.float64
    assert_close(buffer.z, g["z"], FWD_RTOL, FWD_ATOL, "z")
    assert stats.hits_blended == int(g["stats"][3])
    # photometric-style host upstream, as the fit loop forms it (optim.py:87-97)
    target = np.clip(g["image"] + 0.05, 0, 1)
    upstream = np.sign(image.data - target) / image.data.size
    grads, cg = r.backward(scene, cam, params, buffer, upstream)
    for a in (grads.d_position, grads.d_radius, grads.d_opacity, grads.d_feature):
        assert a.dtype == np.float64 and a.flags.writeable
    assert grads.pixel_count.dtype == np.int64 and np.array_equal(grads.pixel_count, g["pixel_count"])
    grads.d_position += 1.0  # the fit loop adds the regulariser in place (optim.py:305-306)
    # the same upstream through the golden's upstream: compare values on the fixture's own upstream
    grads, cg = r.backward(scene, cam, params, buffer, g["upstream"])
    grad_close(grads.d_position, g["d_position"], "d_position")
    grad_close(grads.d_radius, g["d_radius"], "d_radius")
    grad_close(grads.d_opacity, g["d_opacity"], "d_opacity")
    grad_close(grads.d_feature, g["d_feature"], "d_feature")
    want = np.concatenate([g["d_translation"], g["d_rotation"], [g["d_focal"], g["d_sensor_width"]]])
    grad_close(np.concatenate([cg.d_translation, cg.d_rotation, [cg.d_focal, cg.d_sensor_width]]), want, "camera")


def test_forward_dtype_argument_like_reference(engine):
    """raster.py:443, :462-474: the arrays of the result carry render_forward's dtype."""
    import paper_2004_07484_b200 as pk
    g = load_golden("c1_bench1k_64")
    scene = _scene_obj(pk, g["pos"], g["rad"], g["opa"], g["feat"], g["bg"])
    cam = pk.camera_from_vector(g["cam_vec"], g["width"], g["height"])
    params = pk.BlendParams(gamma=g["gamma"], epsilon=g["eps"], tau=g["tau"], top_k=g["top_k"])
    i32, b32, _ = pk.render_forward(scene, cam, params, dtype=np.float32, engine=engine)
    i64, b64, _ = pk.render_forward(scene, cam, params, dtype=np.float64, engine=engine)
    assert i32.data.dtype == np.float32 and b32.z.dtype == np.float32 and b32.ids.dtype == np.int32
    assert i64.data.dtype == np.float64 and np.array_equal(i32.data.astype(np.float64), i64.data)
    with pytest.raises(pk.ConfigurationError):
        pk.render_forward(scene, cam, params, dtype=np.int32, engine=engine)


def test_backward_shares_the_forward_upload_only_for_the_same_scene(engine):
    """render_backward re-uses the device scene of its buffer's forward call for the SAME scene object with the
    same column arrays; a different scene (finite-difference style: forward(scene + eps), backward(scene, buf0)),
    replaced columns or a bulk in-place edit are uploaded again, like the reference re-reads its argument."""
    import paper_2004_07484_b200 as pk
    from paper_2004_07484_b200 import api
    rng = np.random.default_rng(4)
    pos, rad, opa, feat, bg = make_random_scene(rng, 200)
    scene = _scene_obj(pk, pos, rad, opa, feat, bg)
    cam = pk.camera_from_vector([0, 0, 0, 0, 0, 0, 5.0, 2.0], 48, 48)
    params = pk.BlendParams(gamma=0.1, tau=0.0)
    up = rng.normal(size=(48, 48, 3))
    _, buf0, _ = pk.render_forward(scene, cam, params, engine=engine)
    assert api._same_scene(buf0, api._scene_columns(scene))
    g0, _ = pk.render_backward(scene, cam, params, buf0, up, engine=engine)
    g0b, _ = pk.render_backward(scene, cam, params, buf0, up, engine=engine, reuse_upload=False)
    grad_close(g0.d_position, g0b.d_position, "shared vs fresh upload", rtol=2e-5)
    # another forward in between (different scene), then the first buffer with the first scene
    moved = scene.copy()
    moved.positions = moved.positions + 0.01
    _, buf1, _ = pk.render_forward(moved, cam, params, engine=engine)
    g0c, _ = pk.render_backward(scene, cam, params, buf0, up, engine=engine)
    grad_close(g0c.d_position, g0.d_position, "backward after an unrelated forward", rtol=2e-5)
    # stale buffer with ANOTHER scene object: the scene argument wins (grad.py:213)
    assert not api._same_scene(buf0, api._scene_columns(moved))
    gm, _ = pk.render_backward(moved, cam, params, buf0, up, engine=engine)
    gm_ref, _ = pk.render_backward(moved, cam, params, buf0, up, engine=engine, reuse_upload=False)
    grad_close(gm.d_position, gm_ref.d_position, "other scene object", rtol=2e-5)
    assert np.abs(gm.d_position - g0.d_position).max() > 1e-3 * np.abs(g0.d_position).max()
    # bulk in-place edit of the very same arrays
    scene.positions += 0.01
    assert not api._same_scene(buf0, api._scene_columns(scene))
    ge, _ = pk.render_backward(scene, cam, params, buf0, up, engine=engine)
    grad_close(ge.d_position, gm_ref.d_position, "in-place edited scene", rtol=2e-5)


def test_fit_accepts_the_adapter_as_renderer(engine):
    """fit(scene, observations, config, renderer=SoftsphereAdapter(...)) -- the reference call shape -- runs the
    device loop with the adapter's engine and flags; other plug-ins are refused with a clear error."""
    import paper_2004_07484_b200 as pk
    rng = np.random.default_rng(8)
    pos, rad, opa, feat, bg = make_random_scene(rng, 40)
    scene = _scene_obj(pk, pos, rad, opa, feat, bg)
    cam = pk.camera_from_vector([0, 0, 0, 0, 0, 0, 5.0, 2.0], 32, 32)
    target, _, _ = pk.render_forward(scene, cam, pk.BlendParams(gamma=0.1, tau=0.0), engine=engine)
    start = scene.copy()
    start.features = np.clip(start.features + rng.normal(scale=0.2, size=start.features.shape), 0, 1)
    cfg = pk.FitConfig(steps=12, lr_position=0.0, lr_radius=0.0, lr_opacity=0.0, lr_feature=0.05, gamma_start=0.1,
                       gamma_end=0.1, tau=0.0, workers=3)
    obs = [pk.Observation(image=target.data, camera=cam)]
    a = pk.fit(start, obs, cfg, renderer=pk.SoftsphereAdapter(engine=engine))
    b = pk.fit(start, obs, cfg)
    assert np.allclose(a.trace, b.trace, rtol=1e-5, atol=1e-9) and a.trace[-1] < 0.7 * a.trace[0]

    class Other:
        def forward(self, *a):
            raise AssertionError

    with pytest.raises(pk.ConfigurationError):
        pk.fit(start, obs, cfg, renderer=Other())


# ---------------------------------------------------------------------- the unmodified reference + adapter
@pytest.fixture(scope="module")
def ref():
    mod = reference_package()
    if mod is None:
        pytest.skip("baseline/_ref (the reference package) is not installed on this box")
    return mod


def test_reference_fit_loop_with_the_adapter_plugged_in(engine, ref):
    """softsphere.fit(..., renderer=SoftsphereAdapter()) -- the reference's OWN loop, Adam and scene types,
    rendering through the B200 path -- against the same call without a renderer (pure reference)."""
    import paper_2004_07484_b200 as pk
    rng = np.random.default_rng(21)
    pos, rad, opa, feat, bg = make_random_scene(rng, 60)
    truth = _scene_obj(ref, pos, rad, opa, feat, bg)
    cams = [ref.camera_from_vector(v, 40, 40) for v in ([0, 0, 0, 0, 0, 0, 5.0, 2.0], [0.4, 0.1, 0, 0, 0.02, 0, 5.0, 2.0])]
    params = ref.BlendParams(gamma=0.1, tau=0.0)
    obs = [ref.Observation(image=ref.render_forward(truth, c, params)[0].data, camera=c) for c in cams]
    start = truth.copy()
    start.features = np.clip(start.features + rng.normal(scale=0.2, size=start.features.shape), 0, 1)
    start.positions = start.positions + rng.normal(scale=0.05, size=start.positions.shape)
    cfg = ref.FitConfig(steps=10, lr_position=2e-3, lr_radius=1e-3, lr_opacity=1e-2, lr_feature=2e-2, lr_camera=1e-4,
                        gamma_start=0.1, gamma_end=0.05, tau=0.0, top_k=5, lambda_od=0.01, seed=3)
    want = ref.fit(start, obs, cfg)
    got = ref.fit(start, obs, cfg, renderer=pk.SoftsphereAdapter(normalize=cfg.normalize_grads, gate=cfg.gate,
                                                                 engine=engine))
    assert got.trace[-1] < got.trace[0]
    assert np.allclose(got.trace, want.trace, rtol=2e-4, atol=1e-7), (got.trace, want.trace)
    assert np.allclose(got.scene.features, want.scene.features, atol=2e-3)
    assert np.allclose(got.scene.positions, want.scene.positions, atol=2e-3)


def test_reference_acceptance_checks_through_the_adapter(engine, ref):
    """The reference's own acceptance criteria, evaluated with the reference's own oracle and
    types on the adapter's output: forward == brute-force oracle_render (tests/test_raster.py:234-242, bar 1e-5
    for the float32 blend), input-order invariance (:271-283), zero upstream => zero gradients
    (tests/test_grad.py:59-67), gradients == the reference's render_backward on its own buffer."""
    import paper_2004_07484_b200 as pk
    rng = np.random.default_rng(33)
    pos, rad, opa, feat, bg = make_random_scene(rng, 80)
    scene = _scene_obj(ref, pos, rad, opa, feat, bg)
    cam = ref.camera_from_vector([0.2, -0.1, 0.3, 0.01, 0.02, -0.01, 5.0, 2.0], 48, 40)
    params = ref.BlendParams(gamma=0.1, tau=0.0, top_k=5)
    r = pk.SoftsphereAdapter(engine=engine)
    image, buffer, stats = r.forward(scene, cam, params)
    big_k = ref.BlendParams(gamma=0.1, tau=0.0, top_k=64)
    brute = ref.oracle_render(scene, cam, big_k)
    assert_close(image.data, brute.data, FWD_RTOL, FWD_ATOL, "adapter image vs reference oracle_render")
    ref_image, ref_buffer, ref_stats = ref.render_forward(scene, cam, params)
    assert np.array_equal(buffer.ids, ref_buffer.ids)
    assert (stats.candidates_tested, stats.hits_blended) == (ref_stats.candidates_tested, ref_stats.hits_blended)
    perm = rng.permutation(len(scene))
    shuffled = _scene_obj(ref, pos[perm], rad[perm], opa[perm], feat[perm], bg)
    image_p, _, _ = r.forward(shuffled, cam, params)
    assert_close(image_p.data, image.data, 1e-6, 1e-7, "input-order invariance")
    g0, c0 = r.backward(scene, cam, params, buffer, np.zeros_like(image.data))
    assert not g0.d_position.any() and not g0.d_feature.any() and not c0.d_translation.any()
    up = rng.normal(size=image.data.shape)
    got, got_c = r.backward(scene, cam, params, buffer, up)
    want, want_c = ref.render_backward(scene, cam, params, ref_buffer, up)
    assert np.array_equal(got.pixel_count, want.pixel_count)
    grad_close(got.d_position, want.d_position, "d_position vs reference")
    grad_close(got.d_radius, want.d_radius, "d_radius vs reference")
    grad_close(got.d_opacity, want.d_opacity, "d_opacity vs reference")
    grad_close(got.d_feature, want.d_feature, "d_feature vs reference")
    grad_close(got_c.d_translation, want_c.d_translation, "d_translation vs reference")
    grad_close(got_c.d_rotation, want_c.d_rotation, "d_rotation vs reference")
    # the adapter's buffer is accepted by the reference's own backward (same layout and meaning) ...
    cross, _ = ref.render_backward(scene, cam, params, buffer, up)
    grad_close(cross.d_feature, want.d_feature, "reference backward on the adapter's buffer")
    # ... and the reference's own buffer (NumPy, (H, W, K)) by the adapter's backward
    mixed, mixed_c = r.backward(scene, cam, params, ref_buffer, up)
    assert np.array_equal(mixed.pixel_count, want.pixel_count)
    grad_close(mixed.d_position, want.d_position, "adapter backward on the reference's buffer")
    grad_close(mixed.d_feature, want.d_feature, "adapter backward on the reference's buffer (features)")
    grad_close(mixed_c.d_translation, want_c.d_translation, "adapter backward on the reference's buffer (camera)")


def test_plugin_forward_survives_a_workspace_regrowth():
    """render_forward downloads the image band by band from a hook that runs before the status read; when the
    pair capacity overflows, the engine regrows its workspace and renders again (the hook runs a second time):
    the image that comes back must be the second, complete one."""
    import paper_2004_07484_b200 as pk
    from oracle import oracle as orc
    eng = pk.RenderEngine("cuda", pair_factor=1.0, min_pairs=8)
    pos = np.array([[0, 0, 3.0], [0.5, 0.2, 20.0], [0, 0, 10.0]], np.float32)
    rad = np.array([2.9, 1.0, 30.0], np.float32)  # third: camera inside the sphere -> every tile
    opa = np.array([0.6, 0.9, 0.3], np.float32)
    feat, bg = np.eye(3, dtype=np.float32), np.zeros(3, np.float32)
    vec = [0, 0, 0, 0, 0, 0, 5.0, 2.0]
    scene = _scene_obj(pk, pos, rad, opa, feat, bg)
    cam = pk.camera_from_vector(vec, 72, 100)  # 7 tile rows: uneven bands
    params = pk.BlendParams(gamma=0.2, epsilon=1e-2, tau=0.0, top_k=5)
    image, buffer, stats = pk.render_forward(scene, cam, params, engine=eng)
    ref = orc.render_forward(pos, rad, opa, feat, bg, orc.camera_from_vector(vec, 72, 100), gamma=0.2, tau=0.0)
    assert stats.candidates_tested == ref["stats"]["candidates_tested"] > 8
    assert_close(image.data, ref["image"], FWD_RTOL, FWD_ATOL, "image after regrowth")
    assert_close(image.background_weight, ref["bg_weight"], FWD_RTOL, FWD_ATOL, "bg_weight after regrowth")
    assert np.array_equal(buffer.ids, ref["ids"])
