"""CPU oracle: NumPy restatement of the reference's scene surgery, PSC1 / PSK1
byte formats and shading stage.

TEST INFRASTRUCTURE ONLY (same rule as oracle/oracle.py): imported by tests/ only; nothing under
paper_2004_07484_b200/ imports this module.

Each function cites the reference lines it follows (paths relative to /root/reference/pkg/src/softsphere/).
Parity is pinned: oracle/pin_extras_against_reference.py checks every function here against the imported
reference (exactly for masks / bytes / integer outputs, 1e-12 for floats) and writes the reference's own
outputs to tests/golden/extras.npz.
"""
from __future__ import annotations

import json
import struct

import numpy as np

FCC_DIRS = np.array([[1, 1, 0], [1, -1, 0], [-1, 1, 0], [-1, -1, 0], [1, 0, 1], [1, 0, -1],
                     [-1, 0, 1], [-1, 0, -1], [0, 1, 1], [0, 1, -1], [0, -1, 1], [0, -1, -1]], dtype=np.float64)


# ------------------------------------------------------------------ rank 2: scene surgery (optim.py:161-213)
def prune_mask(opa, feat, bg, visibility, opacity_min, background_dist):
    """optim.py:169-175."""
    opa = np.asarray(opa, np.float64)
    keep = np.clip(opa, 0.0, 1.0) >= opacity_min
    if background_dist > 0:
        diff = np.asarray(feat, np.float64) - np.asarray(bg, np.float64)
        keep &= np.sqrt((diff * diff).sum(axis=1)) >= background_dist
    keep &= np.asarray(visibility).reshape(-1) > 0
    return keep


def prune(pos, rad, opa, feat, bg, visibility, opacity_min, background_dist):
    """optim.py:161-183: (pos', rad', opa', feat', keep)."""
    keep = prune_mask(opa, feat, bg, visibility, opacity_min, background_dist)
    return (np.asarray(pos)[keep], np.asarray(rad)[keep], np.asarray(opa)[keep], np.asarray(feat)[keep], keep)


def subdivide(pos, rad, opa, feat, scale):
    """optim.py:197-213: 12 children per sphere at parent + r/sqrt(2) * dir; child c of parent p at 12 p + c."""
    pos, rad = np.asarray(pos, np.float64), np.asarray(rad, np.float64)
    m = pos.shape[0]
    off = (rad / np.sqrt(2.0))[:, None, None] * FCC_DIRS[None, :, :]
    return ((pos[:, None, :] + off).reshape(m * 12, 3), np.repeat(rad * scale, 12),
            np.repeat(np.asarray(opa, np.float64), 12), np.repeat(np.asarray(feat, np.float64), 12, axis=0))


# ------------------------------------------------------------------ rank 3: PSC1 / PSK1 (scene.py:179-227, optim.py:375-466)
def psc1_encode(pos, rad, opa, feat, bg) -> bytes:
    """scene.py:179-200 (validation left to the caller)."""
    pos = np.asarray(pos)
    m, d = pos.shape[0], np.asarray(bg).size
    rec = np.empty((m, 5 + d), dtype="<f4")
    rec[:, 0:3] = pos
    rec[:, 3] = rad
    rec[:, 4] = opa
    rec[:, 5:] = np.asarray(feat).reshape(m, d)
    return b"".join([b"PSC1", struct.pack("<IQ", d, m), np.asarray(bg).astype("<f4").tobytes(), rec.tobytes()])


def psc1_decode(blob: bytes):
    """scene.py:203-227: (pos, rad, opa, feat, bg) as float64, or ValueError on a malformed blob."""
    if blob[:4] != b"PSC1":
        raise ValueError("bad magic")
    if len(blob) < 16:
        raise ValueError("truncated header")
    d, m = struct.unpack("<IQ", blob[4:16])
    if d < 1:
        raise ValueError("invalid feature_dim")
    need = 16 + 4 * d + 4 * m * (5 + d)
    if len(blob) < need:
        raise ValueError("truncated scene data")
    bg = np.frombuffer(blob[16:16 + 4 * d], dtype="<f4").astype(np.float64)
    rec = np.frombuffer(blob[16 + 4 * d:need], dtype="<f4").reshape(m, 5 + d).astype(np.float64)
    return rec[:, 0:3].copy(), rec[:, 3].copy(), rec[:, 4].copy(), rec[:, 5:].copy(), bg


def psk1_encode(scene_blob: bytes, camera_vectors, camera_meta, states, meta=None) -> bytes:
    """optim.py:382-425.  camera_vectors: list of float64 vectors; camera_meta: list of dicts with width,
    height, near, far, mode; states: {name: (m, v, t)}."""
    blobs = [("scene", scene_blob, {"kind": "psc1"})]
    for i, vec in enumerate(camera_vectors):
        vec = np.asarray(vec).astype("<f8")
        blobs.append((f"camera_{i}", vec.tobytes(), {"kind": "f8", "shape": [vec.size]}))
    for name, (m, v, t) in (states or {}).items():
        for part, arr in (("m", m), ("v", v)):
            arr = np.ascontiguousarray(arr, dtype="<f8")
            blobs.append((f"adam.{name}.{part}", arr.tobytes(), {"kind": "f8", "shape": list(arr.shape), "t": t}))
    header = {"version": 1, "cameras": list(camera_meta), "meta": meta or {},
              "blobs": [{"name": n, "nbytes": len(b), **info} for n, b, info in blobs]}
    hdr = json.dumps(header, sort_keys=True).encode("utf-8")
    return b"".join([b"PSK1", struct.pack("<IQ", 1, len(hdr)), hdr] + [b for _, b, _ in blobs])


# ------------------------------------------------------------------ rank 4: shading (shade.py)
def _mask01(x):
    return (x >= 0.0) & (x <= 1.0)


def shade_identity(f):
    """shade.py:66-71."""
    return np.clip(np.asarray(f, np.float64), 0.0, 1.0)


def shade_identity_backward(f, up):
    """shade.py:74-77."""
    return np.asarray(up, np.float64) * _mask01(np.asarray(f, np.float64))


def _diffuse_parts(f, lights):
    """shade.py:84-101; lights: list of (unit direction, intensity, ambient)."""
    albedo, raw_n = f[..., :3], f[..., 3:]
    norm = np.sqrt((raw_n * raw_n).sum(axis=-1, keepdims=True))
    ok = norm[..., 0] > 1e-12
    n_hat = np.where(ok[..., None], raw_n / np.where(ok[..., None], norm, 1.0), 0.0)
    shade = np.zeros(f.shape[:-1])
    for direction, intensity, ambient in lights:
        shade = shade + ambient + intensity * np.maximum(0.0, n_hat @ (-np.asarray(direction, np.float64)))
    return albedo, raw_n, norm, ok, n_hat, shade


def shade_diffuse(f, lights):
    """shade.py:104-110."""
    albedo, _, _, _, _, shade = _diffuse_parts(np.asarray(f, np.float64), lights)
    return np.clip(albedo * shade[..., None], 0.0, 1.0)


def shade_diffuse_backward(f, lights, up):
    """shade.py:113-131."""
    f = np.asarray(f, np.float64)
    albedo, raw_n, norm, ok, n_hat, shade = _diffuse_parts(f, lights)
    up = np.asarray(up, np.float64) * _mask01(albedo * shade[..., None])
    d_albedo = up * shade[..., None]
    d_shade = (up * albedo).sum(axis=-1)
    d_nhat = np.zeros_like(raw_n)
    for direction, intensity, _ in lights:
        nd = -np.asarray(direction, np.float64)
        lit = (n_hat @ nd) > 0.0
        d_nhat += (d_shade * intensity * lit)[..., None] * nd
    safe = np.where(ok[..., None], norm, 1.0)
    d_n = (d_nhat - (d_nhat * n_hat).sum(-1, keepdims=True) * n_hat) / safe
    d_n = np.where(ok[..., None], d_n, 0.0)
    return np.concatenate([d_albedo, d_n], axis=-1)


def view_direction_plane(width, height, focal, sensor_w, pinhole=True):
    """shade.py:138-142 with camera.py:181-192 (sensor coords) and :332-357 (rays)."""
    pix = sensor_w / width
    xs = ((np.arange(width) + 0.5) - width / 2.0) * pix
    ys = ((np.arange(height) + 0.5) - height / 2.0) * pix
    out = np.zeros((height, width, 3))
    if not pinhole:
        out[..., 2] = 1.0
        return out
    gx, gy = np.meshgrid(xs, ys)
    v = np.stack([gx, gy, np.full_like(gx, focal)], axis=-1)
    return v / np.sqrt((v * v).sum(axis=-1, keepdims=True))


def _linear_input(f, view_dirs):
    return f if view_dirs is None else np.concatenate([f, np.asarray(view_dirs, np.float64)], axis=-1)


def shade_linear(f, weight, bias, view_dirs=None):
    """shade.py:148-157."""
    x = _linear_input(np.asarray(f, np.float64), view_dirs)
    return np.clip(x @ np.asarray(weight, np.float64) + np.asarray(bias, np.float64), 0.0, 1.0)


def shade_linear_backward(f, weight, bias, up, view_dirs=None):
    """shade.py:160-171: (d_features, d_weight, d_bias)."""
    f = np.asarray(f, np.float64)
    weight = np.asarray(weight, np.float64)
    x = _linear_input(f, view_dirs)
    pre = x @ weight + np.asarray(bias, np.float64)
    up = np.asarray(up, np.float64) * _mask01(pre)
    d_x = up @ weight.T
    return (d_x[..., :f.shape[-1]], x.reshape(-1, x.shape[-1]).T @ up.reshape(-1, 3), up.reshape(-1, 3).sum(axis=0))
