"""the on-disk formats of the path's inputs, straight into / out of the device SoA
columns (reference softsphere/scene.py:179-326 and softsphere/optim.py:375-466).

  scene_to_bytes / scene_from_bytes / save_scene / load_scene   PSC1 (reference signatures, SphereScene)
  scene_from_bytes_device / scene_to_bytes_device               PSC1 <-> device tensors (pos, rad, opa, feat, bg)
  save_checkpoint / load_checkpoint                             PSK1: PSC1 blob + camera vectors + Adam moments
  import_point_cloud                                            ASCII PLY -> SphereScene (host text parsing)

Byte layouts are the reference's, bit for bit (golden blobs in tests/golden/formats.npz were written by the
reference).  The record block is (de)interleaved by k_psc1_unpack / k_psc1_pack and the <f8 moment blobs are
converted by k_cvt_* on the device (csrc/ss_scene.cu); header parsing, JSON and text parsing are host work.
"""
from __future__ import annotations

import ctypes as C
import json
import struct

import numpy as np
import torch

from . import _lib
from .engine import _ptr, _raise_for, default_engine
from .types import (FormatError, SphereScene, ValidationError, add_sphere_arrays, camera_from_vector,
                    camera_to_vector, new_scene)

_MAGIC = b"PSC1"
_CKPT_MAGIC = b"PSK1"
_CKPT_VERSION = 1


def _stream(dev):
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _check(rc):
    if rc != _lib.SS_OK:
        _raise_for(rc)


# ----------------------------------------------------------------------------------------------- PSC1
def parse_psc1_header(blob: bytes):
    """(d, m, background float32 array, offset of the record block); FormatError like scene.py:205-219."""
    if blob[:4] != _MAGIC:
        raise FormatError(f"bad magic {blob[:4]!r}, expected {_MAGIC!r}")
    if len(blob) < 16:
        raise FormatError("truncated header")
    d, m = struct.unpack("<IQ", blob[4:16])
    if d < 1:
        raise FormatError(f"invalid feature_dim {d}")
    need = 16 + 4 * d + 4 * m * (5 + d)
    if len(blob) < need:
        raise FormatError(f"truncated scene data: {len(blob)} bytes, need {need}")
    bg = np.frombuffer(blob[16:16 + 4 * d], dtype="<f4")
    return int(d), int(m), bg, 16 + 4 * d


def scene_from_bytes_device(blob: bytes, device="cuda"):
    """PSC1 bytes -> dict(pos, rad, opa, feat, bg) of float32 device tensors (k_psc1_unpack)."""
    lib = _lib.load()
    d, m, bg, off = parse_psc1_header(blob)
    if d > _lib.MAX_FEATURE_DIM:
        raise FormatError(f"feature_dim {d} exceeds the device limit {_lib.MAX_FEATURE_DIM}")
    dev = default_engine(device).device
    rec_host = np.frombuffer(blob, dtype=np.uint8, count=4 * m * (5 + d), offset=off)
    rec = torch.from_numpy(rec_host.copy()).to(dev)
    pos = torch.empty((m, 3), dtype=torch.float32, device=dev)
    rad = torch.empty(m, dtype=torch.float32, device=dev)
    opa = torch.empty(m, dtype=torch.float32, device=dev)
    feat = torch.empty((m, d), dtype=torch.float32, device=dev)
    _check(lib.ss_psc1_unpack(_ptr(rec), m, d, _ptr(pos), _ptr(rad), _ptr(opa), _ptr(feat), _stream(dev)))
    return {"pos": pos, "rad": rad, "opa": opa, "feat": feat,
            "bg": torch.from_numpy(bg.astype(np.float32)).to(dev), "feature_dim": d}


def scene_to_bytes_device(pos, rad, opa, feat, bg) -> bytes:
    """Device tensors -> PSC1 bytes (k_psc1_pack); no validation (see scene_to_bytes)."""
    lib = _lib.load()
    m, d = int(pos.shape[0]), int(feat.shape[1])
    dev = pos.device
    rec = torch.empty(max(m * (5 + d), 1), dtype=torch.float32, device=dev)
    _check(lib.ss_psc1_pack(_ptr(pos.contiguous()), _ptr(rad.contiguous()), _ptr(opa.contiguous()),
                            _ptr(feat.contiguous()), m, d, _ptr(rec), _stream(dev)))
    body = rec[:m * (5 + d)].cpu().numpy().astype("<f4").tobytes()
    bg_b = bg.detach().cpu().numpy().astype("<f4").tobytes() if isinstance(bg, torch.Tensor) else \
        np.asarray(bg).astype("<f4").tobytes()
    return b"".join([_MAGIC, struct.pack("<IQ", d, m), bg_b, body])


def scene_to_bytes(scene: SphereScene, device="cuda") -> bytes:
    """Reference signature (scene.py:179): validates, then encodes PSC1."""
    scene.validate()
    dev = default_engine(device).device
    d = scene.feature_dim
    f32 = lambda a, shape: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).reshape(shape).to(dev)
    return scene_to_bytes_device(f32(scene.positions, (-1, 3)), f32(scene.radii, (-1,)), f32(scene.opacities, (-1,)),
                                 f32(scene.features, (-1, d)), scene.background)


def scene_from_bytes(blob: bytes, device="cuda") -> SphereScene:
    """Reference signature (scene.py:203): float64 SphereScene (values are the stored float32)."""
    t = scene_from_bytes_device(blob, device)
    f64 = lambda x: np.ascontiguousarray(x.cpu().numpy().astype(np.float64))
    scene = SphereScene(feature_dim=t["feature_dim"], background=f64(t["bg"]))
    scene.positions, scene.radii = f64(t["pos"]), f64(t["rad"])
    scene.opacities, scene.features = f64(t["opa"]), f64(t["feat"])
    return scene


def save_scene(scene: SphereScene, path, device="cuda") -> None:
    with open(path, "wb") as f:
        f.write(scene_to_bytes(scene, device))


def load_scene(path, device="cuda") -> SphereScene:
    with open(path, "rb") as f:
        return scene_from_bytes(f.read(), device)


# ----------------------------------------------------------------------------------------------- PSK1
def _f64_blob(t: torch.Tensor) -> bytes:
    """float32 device tensor -> little-endian float64 bytes (k_cvt_f32_f64)."""
    lib = _lib.load()
    t = t.contiguous()
    out = torch.empty(t.shape, dtype=torch.float64, device=t.device)
    _check(lib.ss_convert_f32_f64(_ptr(t), _ptr(out), t.numel(), _stream(t.device)))
    return out.cpu().numpy().astype("<f8").tobytes()


def _f32_from_f64_blob(buf: bytes, shape, dev) -> torch.Tensor:
    lib = _lib.load()
    src = torch.from_numpy(np.frombuffer(buf, dtype="<f8").astype(np.float64)).to(dev)
    out = torch.empty(src.shape, dtype=torch.float32, device=dev)
    _check(lib.ss_convert_f64_f32(_ptr(src), _ptr(out), src.numel(), _stream(dev)))
    return out.reshape(shape)


def _write_checkpoint(path, scene_blob: bytes, cameras, state_blobs, meta):
    """The reference's byte layout (optim.py:382-425): magic, version u32, header length u64, sorted-key
    JSON header describing the blobs, then the blobs in header order."""
    blobs = [("scene", scene_blob, {"kind": "psc1"})]
    cam_meta = []
    for i, cam in enumerate(cameras):
        vec = camera_to_vector(cam).astype("<f8")
        blobs.append((f"camera_{i}", vec.tobytes(), {"kind": "f8", "shape": [vec.size]}))
        cam_meta.append({"width": cam.width, "height": cam.height, "near": cam.near, "far": cam.far,
                         "mode": cam.mode})
    blobs.extend(state_blobs)
    header = {"version": _CKPT_VERSION, "cameras": cam_meta, "meta": meta or {},
              "blobs": [{"name": n, "nbytes": len(b), **info} for n, b, info in blobs]}
    hdr = json.dumps(header, sort_keys=True).encode("utf-8")
    with open(path, "wb") as f:
        f.write(_CKPT_MAGIC)
        f.write(struct.pack("<IQ", _CKPT_VERSION, len(hdr)))
        f.write(hdr)
        for _, b, _info in blobs:
            f.write(b)


def save_checkpoint(path, scene: SphereScene, cameras, states=None, meta=None, device="cuda"):
    """Reference signature (optim.py:382): states is {name: AdamState-like with .m, .v (float64), .t}."""
    state_blobs = []
    if states:
        for name, st in states.items():
            for part in ("m", "v"):
                arr = np.ascontiguousarray(getattr(st, part), dtype="<f8")
                state_blobs.append((f"adam.{name}.{part}", arr.tobytes(),
                                    {"kind": "f8", "shape": list(arr.shape), "t": st.t}))
    _write_checkpoint(path, scene_to_bytes(scene, device), cameras, state_blobs, meta)


def save_checkpoint_device(path, fit, cameras, meta=None):
    """Checkpoint of a DeviceFit: parameters packed and moments widened to <f8 on the device."""
    names = (("position", "pos"), ("radius", "rad"), ("opacity", "opa"), ("feature", "feat"))
    state_blobs = []
    for g, (name, key) in enumerate(names):
        m, v = fit.moments[key]
        for part, t in (("m", m), ("v", v)):
            state_blobs.append((f"adam.{name}.{part}", _f64_blob(t),
                                {"kind": "f8", "shape": list(t.shape), "t": int(fit.steps[g])}))
    blob = scene_to_bytes_device(fit.pos, fit.rad, fit.opa, fit.feat, fit.bg)
    _write_checkpoint(path, blob, cameras, state_blobs, meta)


def _read_checkpoint(path):
    with open(path, "rb") as f:
        data = f.read()
    if data[:4] != _CKPT_MAGIC:
        raise FormatError(f"bad checkpoint magic {data[:4]!r}")
    version, hdr_len = struct.unpack("<IQ", data[4:16])
    if version != _CKPT_VERSION:
        raise FormatError(f"unsupported checkpoint version {version}")
    header = json.loads(data[16:16 + hdr_len].decode("utf-8"))
    offset = 16 + hdr_len
    raw = {}
    for blob in header["blobs"]:
        raw[blob["name"]] = (data[offset:offset + blob["nbytes"]], blob)
        offset += blob["nbytes"]
    cameras = []
    for i, cmeta in enumerate(header["cameras"]):
        vec = np.frombuffer(raw[f"camera_{i}"][0], dtype="<f8")
        cameras.append(camera_from_vector(vec, cmeta["width"], cmeta["height"], near=cmeta["near"],
                                          far=cmeta["far"], mode=cmeta["mode"]))
    return raw, cameras, header.get("meta", {})


def load_checkpoint(path, device="cuda"):
    """Reference signature (optim.py:428): (scene, cameras, states, meta); states hold float64 arrays."""
    from .optim import AdamState
    raw, cameras, meta = _read_checkpoint(path)
    scene = scene_from_bytes(raw["scene"][0], device)
    states = {}
    for name in ("position", "radius", "opacity", "feature"):
        key = f"adam.{name}.m"
        if key in raw:
            m_buf, m_blob = raw[key]
            v_buf, _ = raw[f"adam.{name}.v"]
            shape = tuple(m_blob["shape"])
            states[name] = AdamState(m=np.frombuffer(m_buf, dtype="<f8").reshape(shape).copy(),
                                     v=np.frombuffer(v_buf, dtype="<f8").reshape(shape).copy(),
                                     t=int(m_blob.get("t", 0)))
    return scene, cameras, states, meta


def load_checkpoint_device(path, config=None, engine=None, device="cuda"):
    """(DeviceFit, cameras, meta): scene unpacked and moments narrowed to float32 on the device."""
    from .optim import DeviceFit
    raw, cameras, meta = _read_checkpoint(path)
    t = scene_from_bytes_device(raw["scene"][0], device)
    fit = DeviceFit.from_device(t["pos"], t["rad"], t["opa"], t["feat"], t["bg"], config=config, engine=engine)
    names = (("position", "pos"), ("radius", "rad"), ("opacity", "opa"), ("feature", "feat"))
    for g, (name, key) in enumerate(names):
        mk = f"adam.{name}.m"
        if mk in raw:
            shape = tuple(raw[mk][1]["shape"])
            fit.moments[key] = (_f32_from_f64_blob(raw[mk][0], shape, fit.pos.device),
                                _f32_from_f64_blob(raw[f"adam.{name}.v"][0], shape, fit.pos.device))
            fit.steps[g] = int(raw[mk][1].get("t", 0))
    return fit, cameras, meta


# ----------------------------------------------------------------------------------------------- PLY
def import_point_cloud(path, default_radius: float, default_opacity: float) -> SphereScene:
    """ASCII PLY point cloud -> scene, one sphere per point (scene.py:242-326): red/green/blue (uchar
    0..255 or float) become a 3-channel feature, otherwise every feature equals the black background."""
    if default_radius <= 0:
        raise ValidationError("default_radius must be positive")
    with open(path, "r", encoding="ascii", errors="replace") as f:
        lines = f.readlines()

    def fail(lineno, msg):
        raise FormatError(f"{path}:{lineno + 1}: {msg}")

    if not lines or lines[0].strip() != "ply":
        fail(0, "not a PLY file (missing 'ply' header)")
    count, props, in_vertex, end = None, [], False, None
    for i in range(1, len(lines)):
        tok = lines[i].strip().split()
        if not tok:
            continue
        key = tok[0]
        if key == "format":
            if len(tok) < 2 or tok[1] != "ascii":
                fail(i, f"unsupported PLY format {' '.join(tok[1:])!r}; only ascii")
        elif key == "element":
            in_vertex = tok[1] == "vertex"
            if in_vertex:
                try:
                    count = int(tok[2])
                except (IndexError, ValueError):
                    fail(i, "malformed vertex element line")
        elif key == "property" and in_vertex:
            if len(tok) < 3:
                fail(i, "malformed property line")
            props.append((tok[1], tok[2]))
        elif key == "end_header":
            end = i
            break
    if end is None:
        fail(len(lines) - 1, "missing end_header")
    if count is None:
        fail(end, "missing vertex element")
    names = [n for _, n in props]
    for axis in "xyz":
        if axis not in names:
            fail(end, f"vertex element lacks '{axis}' coordinate")
    col = {n: names.index(n) for n in names}
    colored = all(c in names for c in ("red", "green", "blue"))
    byte_color = colored and props[col["red"]][0] in ("uchar", "uint8", "char")

    scene = new_scene(3, [0.0, 0.0, 0.0])
    pts = np.zeros((count, 3))
    feats = np.tile(scene.background, (count, 1))
    row = 0
    for i in range(end + 1, len(lines)):
        tok = lines[i].split()
        if not tok:
            continue
        if row >= count:
            break
        if len(tok) < len(props):
            fail(i, f"expected {len(props)} values, got {len(tok)}")
        try:
            vals = [float(t) for t in tok[:len(props)]]
        except ValueError:
            fail(i, "non-numeric vertex value")
        pts[row] = (vals[col["x"]], vals[col["y"]], vals[col["z"]])
        if colored:
            rgb = np.array([vals[col["red"]], vals[col["green"]], vals[col["blue"]]])
            feats[row] = rgb / 255.0 if byte_color else rgb
        row += 1
    if row < count:
        fail(len(lines) - 1, f"expected {count} vertices, file ends after {row}")
    add_sphere_arrays(scene, pts, np.full(count, float(default_radius)), np.full(count, float(default_opacity)),
                      feats)
    return scene
