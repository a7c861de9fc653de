"""CPU: host-side mirror of the reference interface (types, camera math, error behaviour)."""
import numpy as np
import pytest

import paper_2004_07484_b200 as pk
from oracle import oracle as orc


def test_blend_params_clamp_and_validate():
    assert pk.BlendParams(gamma=5.0).gamma == 1.0 and pk.BlendParams(gamma=1e-9).gamma == 1e-5
    with pytest.raises(pk.ValidationError):
        pk.BlendParams(epsilon=0.0)
    with pytest.raises(pk.ValidationError):
        pk.BlendParams(tau=1.0)
    with pytest.raises(pk.ValidationError):
        pk.BlendParams(top_k=0)


def test_camera_vector_layouts():
    c8 = pk.camera_from_vector([1, 2, 3, 0.1, 0.2, 0.3, 5.0, 2.0], 64, 48)
    assert c8.rotation_type == pk.AXIS_ANGLE and c8.focal_length == 5.0 and c8.sensor_width == 2.0
    c11 = pk.camera_from_vector([1, 2, 3, 1, 0, 0, 0, 1, 0, 4.0, 3.0], 64, 48)
    assert c11.rotation_type == pk.SIX_D and np.allclose(c11.rotation, np.eye(3))
    assert np.allclose(pk.camera_to_vector(c8), [1, 2, 3, 0.1, 0.2, 0.3, 5.0, 2.0])
    with pytest.raises(pk.ConfigurationError):
        pk.camera_from_vector([0] * 9, 8, 8)
    with pytest.raises(pk.ConfigurationError):
        pk.camera_from_vector([0, 0, 0, 0, 0, 0, -1.0, 2.0], 8, 8)
    with pytest.raises(pk.ConfigurationError):
        pk.camera_from_vector([0, 0, 0, 0, 0, 0, 5.0, 2.0], 8, 8, near=2.0, far=1.0)
    with pytest.raises(pk.ConfigurationError):
        pk.camera_from_vector([0, 0, 0, 0, 0, 0, 0, 0, 0, 5.0, 2.0], 8, 8)  # degenerate 6d


@pytest.mark.parametrize("v", [[0.02, -0.03, 0.01], [1.2, -0.7, 2.1], [0, 0, 0], [1e-9, 0, 0]])
def test_axis_angle_matrix_and_vjp(v):
    r = pk.axis_angle_to_matrix(v)
    assert np.allclose(r @ r.T, np.eye(3), atol=1e-12) and np.isclose(np.linalg.det(r), 1.0)
    assert np.allclose(r, orc.axis_angle_to_matrix(v), atol=1e-15)
    rng = np.random.default_rng(0)
    g = rng.normal(size=(3, 3))
    fd = np.zeros(3)
    for i in range(3):
        e = np.zeros(3)
        e[i] = 1e-6
        fd[i] = np.sum(g * (pk.axis_angle_to_matrix(np.add(v, e)) - pk.axis_angle_to_matrix(np.subtract(v, e)))) / 2e-6
    assert np.allclose(pk.axis_angle_vjp(v, g), fd, atol=1e-6)
    assert np.allclose(pk.axis_angle_vjp(v, g), orc.axis_angle_vjp(v, g), atol=1e-12)


def test_rotation_6d_and_vjp():
    a = np.array([1.0, 0.01, 0.02, -0.02, 1.0, 0.03])
    r = pk.rotation_from_6d(a)
    assert np.allclose(r.T @ r, np.eye(3), atol=1e-12)
    assert np.allclose(r, pk.rotation_from_6d(np.concatenate([3.0 * a[:3], 0.5 * a[3:]])))  # scale invariant
    g = np.random.default_rng(1).normal(size=(3, 3))
    fd = np.zeros(6)
    for i in range(6):
        e = np.zeros(6)
        e[i] = 1e-6
        fd[i] = np.sum(g * (pk.rotation_from_6d(a + e) - pk.rotation_from_6d(a - e))) / 2e-6
    assert np.allclose(pk.rotation_6d_vjp(a, g), fd, atol=1e-6)
    assert np.allclose(pk.rotation_6d_vjp(a, g), orc.rotation_6d_vjp(a, g), atol=1e-12)


def test_scene_validation_errors():
    s = pk.new_scene(3, [0, 0, 0])
    pk.add_sphere_arrays(s, [[0, 0, 10.0]], [1.0], [0.5], [[1, 0, 0]])
    s.validate()
    bad = s.copy()
    bad.radii = np.array([0.0])
    with pytest.raises(pk.ValidationError):
        bad.validate()
    bad = s.copy()
    bad.positions = np.array([[np.nan, 0, 1.0]])
    with pytest.raises(pk.ValidationError):
        bad.validate()
    with pytest.raises(pk.ValidationError):
        pk.add_sphere_arrays(s, [[0, 0, 1.0]], [1.0], [0.5], [[1, 0]])  # feature dim mismatch
    with pytest.raises(pk.ConfigurationError):
        pk.new_scene(0, [])


def test_world_to_camera_convention():
    cam = pk.camera_from_vector([0.3, -0.2, 0.5, 0.02, -0.03, 0.01, 5.0, 2.0], 32, 32)
    p = np.random.default_rng(2).normal(size=(5, 3))
    assert np.allclose(cam.world_to_camera(p), (cam.rotation @ (p - cam.translation).T).T)
    assert np.allclose(cam.camera_to_world(cam.world_to_camera(p)), p)


def test_render_fails_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(pk._lib.NativeLibraryError):
        pk.RenderEngine("cuda")
    scene = pk.new_scene(3, [0, 0, 0])
    cam = pk.camera_from_vector([0, 0, 0, 0, 0, 0, 5.0, 2.0], 16, 16)
    with pytest.raises(pk._lib.NativeLibraryError):
        pk.render_forward(scene, cam, pk.BlendParams())


def test_product_never_imports_the_oracle():
    import os
    import re
    root = os.path.dirname(pk.__file__)
    for dirpath, _, files in os.walk(root):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", src, flags=re.M), f
                assert "ss_oracle" not in src, f
