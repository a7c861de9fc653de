"""GPU: SURVEY 8(f) rank 1 -- photometric loss, Adam and the fused fit step against the oracle's
restatement of softsphere/optim.py and against golden vectors produced by the reference."""
import os

import numpy as np
import pytest

from helpers import GOLDEN_DIR, assert_close, make_random_scene

pytestmark = pytest.mark.gpu

CFG = dict(lr_position=2e-3, lr_radius=1e-3, lr_opacity=1e-2, lr_feature=2e-2, beta1=0.9, beta2=0.999,
           adam_eps=1e-8, gamma=0.2, epsilon=1e-2, tau=0.0, top_k=5, lambda_od=0.05, radius_min=1e-6,
           normalize_grads=True, gate=True)


def test_photometric_loss_reference_signature(engine):
    import paper_2004_07484_b200 as pk
    from oracle import oracle as orc
    g = np.load(os.path.join(GOLDEN_DIR, "fit_step.npz"))
    loss, up = pk.photometric_loss(g["pm_a"], g["pm_b"])
    want_loss, want_up = orc.photometric_loss(g["pm_a"], g["pm_b"])
    assert abs(loss - want_loss) < 1e-6 * want_loss
    assert up.shape == want_up.shape and up[0, 0, 0] == 0.0  # ties give 0
    assert_close(up, want_up, 1e-6, 0.0, "upstream")
    with pytest.raises(pk.ValidationError):
        pk.photometric_loss(np.zeros((4, 4, 3)), np.zeros((4, 5, 3)))
    # ragged size (not a multiple of 4) and a larger image
    rng = np.random.default_rng(0)
    a, b = rng.uniform(0, 1, (257, 131, 3)).astype(np.float32), rng.uniform(0, 1, (257, 131, 3)).astype(np.float32)
    loss, up = pk.photometric_loss(a, b)
    want_loss, want_up = orc.photometric_loss(a, b)
    assert abs(loss - want_loss) < 1e-6 * want_loss
    assert_close(up, want_up, 1e-6, 0.0, "upstream (large)")


def test_adam_step_reference_signature(engine):
    import paper_2004_07484_b200 as pk
    from oracle import oracle as orc
    rng = np.random.default_rng(1)
    p = rng.normal(size=(37, 3)).astype(np.float32).astype(np.float64)
    st = pk.AdamState.like(p)
    cfg = pk.FitConfig()
    po, mo, vo, to = p.copy(), np.zeros_like(p), np.zeros_like(p), 0
    for _ in range(4):
        g = rng.normal(size=p.shape).astype(np.float32).astype(np.float64)
        p = pk.adam_step(p, g, st, 3e-3, cfg)
        po, mo, vo, to = orc.adam_step(po, g, mo, vo, to, 3e-3)
    assert st.t == 4
    # float32 moments on the device vs float64 in the reference: a few float32 roundings per step
    assert_close(p, po, 1e-5, 1e-6, "adam params")
    assert_close(st.m, mo, 1e-5, 1e-7, "adam m")
    assert_close(st.v, vo, 1e-5, 1e-9, "adam v")
    with pytest.raises(pk.ValidationError):
        pk.adam_step(np.zeros(3), np.zeros(4), pk.AdamState.like(np.zeros(3)), 1e-3, cfg)


def test_device_fit_matches_reference_golden(engine):
    """Three iterations of the reference's fit-loop body; golden outputs are the reference's own."""
    import torch
    import paper_2004_07484_b200 as pk
    g = np.load(os.path.join(GOLDEN_DIR, "fit_step.npz"))
    w, h = int(g["width"]), int(g["height"])
    spec = pk.CameraSpec.from_camera(pk.camera_from_vector(g["cam_vec"], w, h))
    cfg = pk.FitConfig(lr_position=2e-3, lr_radius=1e-3, lr_opacity=1e-2, lr_feature=2e-2, gamma=0.2, tau=0.0,
                       top_k=5, lambda_od=0.05)
    fit = pk.DeviceFit(g["pos"], g["rad"], g["opa"], g["feat"], g["bg"], cfg, engine=engine)
    target = torch.from_numpy(g["target"]).cuda()
    for want in g["losses"]:
        loss = fit.step(target, spec)
        assert abs(float(loss.item()) - want) < 2e-5 * abs(want)
    assert_close(fit.pos.cpu().numpy(), g["pos_out"], 2e-5, 2e-6, "positions after 3 steps")
    assert_close(fit.rad.cpu().numpy(), g["rad_out"], 2e-5, 1e-6, "radii after 3 steps")
    assert_close(fit.opa.cpu().numpy(), g["opa_out"], 2e-5, 2e-6, "opacities after 3 steps")
    assert_close(fit.feat.cpu().numpy(), g["feat_out"], 2e-5, 2e-6, "features after 3 steps")
    assert int(fit.visibility.sum()) > 0 and fit.steps == [3, 3, 3, 3]


def test_fused_fit_step_vs_oracle(engine):
    """One fused update on a 20K-sphere scene: regulariser + visibility + Adam + radius floor + frozen group."""
    import torch
    import paper_2004_07484_b200 as pk
    from oracle import oracle as orc
    from paper_2004_07484_b200.synthetic import benchmark_scene
    pos, rad, opa, feat, bg, vec = benchmark_scene(20000, 128, 128, seed=5)
    rad[:50] = 2e-6  # will be pushed below the floor
    rng = np.random.default_rng(4)
    target = rng.uniform(0, 1, (128, 128, 3)).astype(np.float32)
    cfg = dict(CFG, lr_opacity=0.0, radius_min=1.9e-6, gamma=0.1)  # opacity group frozen
    ocam = orc.camera_from_vector(vec, 128, 128)
    scene = dict(pos=pos.astype(np.float64), rad=rad.astype(np.float64), opa=opa.astype(np.float64),
                 feat=feat.astype(np.float64), bg=bg.astype(np.float64))
    state = {k: (np.zeros_like(scene[k]), np.zeros_like(scene[k]), 0) for k in ("pos", "rad", "opa", "feat")}
    o_loss, o_scene, o_state, o_g = orc.fit_step(scene, ocam, target.astype(np.float64), state, cfg, threads=4)
    fc = pk.FitConfig(lr_position=2e-3, lr_radius=1e-3, lr_opacity=0.0, lr_feature=2e-2, gamma=0.1, tau=0.0, top_k=5,
                      lambda_od=0.05, radius_min=1.9e-6)
    fit = pk.DeviceFit(pos, rad, opa, feat, bg, fc, engine=engine)
    spec = pk.CameraSpec.from_camera(pk.camera_from_vector(vec, 128, 128))
    loss = fit.step(torch.from_numpy(target).cuda(), spec)
    assert abs(float(loss.item()) - o_loss) < 2e-5 * abs(o_loss)
    assert_close(fit.pos.cpu().numpy(), o_scene["pos"], 1e-6, 1e-6, "positions")
    assert_close(fit.rad.cpu().numpy(), o_scene["rad"], 1e-5, 1e-9, "radii")
    assert np.array_equal(fit.opa.cpu().numpy(), opa)  # frozen group untouched
    assert_close(fit.feat.cpu().numpy(), o_scene["feat"], 1e-5, 1e-6, "features")
    assert float(fit.rad.min()) >= np.float32(1.9e-6)
    assert np.array_equal(fit.visibility.cpu().numpy(), o_g["pixel_count"])
    assert fit.steps == [1, 1, 0, 1]
