"""CPU: SURVEY 8(f) ranks 2-4 -- the NumPy restatement (oracle/extras.py) against golden vectors written by
the reference (oracle/pin_extras_against_reference.py), plus the host-side logic of the product (PLY text
parsing, PSC1 / PSK1 header handling, FitConfig schedule).  No GPU calls."""
import os
import struct

import numpy as np
import pytest

from helpers import GOLDEN_DIR, assert_close


@pytest.fixture(scope="module")
def g():
    z = np.load(os.path.join(GOLDEN_DIR, "extras.npz"))
    return {k: z[k] for k in z.files}


@pytest.mark.parametrize("tag", ["a", "b"])
def test_oracle_prune_matches_reference(g, tag):
    from oracle import extras as ex
    p = f"prune_{tag}_"
    pos, rad, opa, feat, keep = ex.prune(g[p + "pos"], g[p + "rad"], g[p + "opa"], g[p + "feat"], g[p + "bg"],
                                         g[p + "vis"], *g[p + "cfg"])
    assert np.array_equal(keep, g[p + "keep"]) and 0 < keep.sum() < keep.size
    assert np.array_equal(pos, g[p + "out_pos"]) and np.array_equal(feat, g[p + "out_feat"])


def test_oracle_subdivide_matches_reference(g):
    from oracle import extras as ex
    pos, rad, opa, feat = ex.subdivide(g["sub_pos"], g["sub_rad"], g["sub_opa"], g["sub_feat"], float(g["sub_scale"]))
    assert_close(pos, g["sub_out_pos"], 1e-14, 0, "children")
    assert_close(rad, g["sub_out_rad"], 1e-14, 0, "radii")
    assert np.array_equal(opa, g["sub_out_opa"]) and np.array_equal(feat, g["sub_out_feat"])
    # known answers of the reference's tests (test_optim.py:166-188): 12 children at distance r
    d = np.linalg.norm(pos.reshape(-1, 12, 3) - g["sub_pos"][:, None, :], axis=2)
    assert_close(d, np.repeat(g["sub_rad"][:, None], 12, 1), 1e-12, 0, "equidistant")


@pytest.mark.parametrize("tag", ["d3", "d15", "empty"])
def test_oracle_psc1_matches_reference_bytes(g, tag):
    from oracle import extras as ex
    p = f"psc1_{tag}_"
    blob = g[p + "blob"].tobytes()
    pos, rad, opa, feat, bg = ex.psc1_decode(blob)
    for a, n in ((pos, "pos"), (rad, "rad"), (opa, "opa"), (feat, "feat"), (bg, "bg")):
        assert np.array_equal(a, g[p + n]), n
    assert ex.psc1_encode(pos, rad, opa, feat, bg) == blob
    with pytest.raises(ValueError):
        ex.psc1_decode(b"XXXX" + blob[4:])
    if len(pos):
        with pytest.raises(ValueError):
            ex.psc1_decode(blob[:-4])


def test_oracle_shaders_match_reference(g):
    from oracle import extras as ex
    assert_close(ex.shade_identity(g["id_f"]), g["id_out"], 0, 0, "identity")
    assert_close(ex.shade_identity_backward(g["id_f"], g["id_up"]), g["id_bwd"], 0, 0, "identity bwd")
    lights = [(r[:3], r[3], r[4]) for r in g["df_lights"]]
    assert_close(ex.shade_diffuse(g["df_f"], lights), g["df_out"], 1e-13, 1e-15, "diffuse")
    assert_close(ex.shade_diffuse_backward(g["df_f"], lights, g["df_up"]), g["df_bwd"], 1e-12, 1e-14, "diffuse bwd")
    w, h, f, s = g["vd_cam"]
    assert_close(ex.view_direction_plane(int(w), int(h), f, s), g["vd_out"], 1e-14, 0, "view dirs")
    for tag in ("plain", "view"):
        p = f"lin_{tag}_"
        v = g.get(p + "v")
        assert_close(ex.shade_linear(g[p + "f"], g[p + "w"], g[p + "b"], v), g[p + "out"], 1e-13, 1e-15, "linear")
        d_f, d_w, d_b = ex.shade_linear_backward(g[p + "f"], g[p + "w"], g[p + "b"], g[p + "up"], v)
        assert_close(d_f, g[p + "df"], 1e-12, 1e-14, "d_f")
        assert_close(d_w, g[p + "dw"], 1e-12, 1e-13, "d_w")
        assert_close(d_b, g[p + "db"], 1e-12, 1e-13, "d_b")


def test_ply_import_host_parser(g, tmp_path):
    import paper_2004_07484_b200 as pk
    sc = pk.import_point_cloud(os.path.join(GOLDEN_DIR, "cloud.ply"), 0.05, 0.8)
    assert np.array_equal(sc.positions, g["ply_pos"]) and np.array_equal(sc.features, g["ply_feat"])
    assert np.array_equal(sc.radii, g["ply_rad"]) and np.array_equal(sc.opacities, g["ply_opa"])
    # error behaviour of scene.py:242-326
    with pytest.raises(pk.ValidationError):
        pk.import_point_cloud(os.path.join(GOLDEN_DIR, "cloud.ply"), 0.0, 0.8)
    text = open(os.path.join(GOLDEN_DIR, "cloud.ply")).read().splitlines()
    bad = tmp_path / "t.ply"
    bad.write_text("\n".join(text[:-2]) + "\n")  # truncated
    with pytest.raises(pk.FormatError, match="expected 5 vertices"):
        pk.import_point_cloud(str(bad), 0.05, 0.8)
    bad.write_text("\n".join(l for l in text if "property float y" not in l) + "\n")
    with pytest.raises(pk.FormatError, match="lacks 'y'"):
        pk.import_point_cloud(str(bad), 0.05, 0.8)
    bad.write_text("\n".join(text).replace("format ascii 1.0", "format binary_little_endian 1.0") + "\n")
    with pytest.raises(pk.FormatError, match="only ascii"):
        pk.import_point_cloud(str(bad), 0.05, 0.8)
    bad.write_text("plx\n")
    with pytest.raises(pk.FormatError, match="not a PLY"):
        pk.import_point_cloud(str(bad), 0.05, 0.8)
    # without colours every feature equals the black background
    bad.write_text("ply\nformat ascii 1.0\nelement vertex 2\nproperty float x\nproperty float y\nproperty float z\n"
                   "end_header\n0 0 5\n1 1 6\n")
    sc = pk.import_point_cloud(str(bad), 0.1, 1.0)
    assert len(sc) == 2 and not sc.features.any()


def test_psc1_header_errors_and_schedule(g):
    import paper_2004_07484_b200 as pk
    from paper_2004_07484_b200 import sceneio
    blob = g["psc1_d3_blob"].tobytes()
    d, m, bg, off = sceneio.parse_psc1_header(blob)
    assert (d, m, off) == (3, 257, 28) and np.array_equal(bg.astype(np.float64), g["psc1_d3_bg"])
    with pytest.raises(pk.FormatError, match="bad magic"):
        sceneio.parse_psc1_header(b"PSC2" + blob[4:])
    with pytest.raises(pk.FormatError, match="truncated header"):
        sceneio.parse_psc1_header(blob[:10])
    with pytest.raises(pk.FormatError, match="truncated scene data"):
        sceneio.parse_psc1_header(blob[:-1])
    with pytest.raises(pk.FormatError, match="invalid feature_dim"):
        sceneio.parse_psc1_header(b"PSC1" + struct.pack("<IQ", 0, 0))
    cfg = pk.FitConfig(steps=11, gamma_start=0.1, gamma_end=1e-3)
    assert cfg.gamma_at(0) == pytest.approx(0.1) and cfg.gamma_at(10) == pytest.approx(1e-3)
    assert cfg.gamma_at(5) == pytest.approx(1e-2)
    with pytest.raises(pk.ConfigurationError):
        pk.FitConfig(gamma_end=1e-6)
    with pytest.raises(pk.ValidationError):
        pk.DirectionalLight([0, 0, 0])
    with pytest.raises(pk.ValidationError):
        pk.LinearShader(np.zeros((4, 2)), np.zeros(3))
