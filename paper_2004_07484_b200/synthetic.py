"""Synthetic inputs of the headline benchmark (BASELINE.json configs): the reference benchmark's
`uniform` / `occluded` sphere clouds (softsphere/cli.py:323-356) for the identity camera
cam_vec = [0,0,0, 0,0,0, 5, 2], drawn from numpy.random.default_rng(seed) in the reference's
draw order and snapped to float32, plus the small-baseline camera orbit of config 4."""
from __future__ import annotations

import numpy as np

FOCAL, SENSOR = 5.0, 2.0


def benchmark_scene(count: int, width: int, height: int, seed: int = 0, d: int = 3, profile: str = "uniform",
                    aspect_fill: bool = False):
    """Returns (pos (M,3), rad (M), opa (M), feat (M,d), bg (d), cam_vec (8,)) as float32 (+ float64 cam)."""
    rng = np.random.default_rng(seed)
    px = SENSOR / width
    blocks = []
    if profile == "occluded":  # opaque 16x16 wall at depth 5, `count` spheres hidden behind it
        side = 16
        half = 5.0 * (SENSOR / 2.0) / FOCAL
        gx, gy = np.meshgrid(np.linspace(-half, half, side), np.linspace(-half, half, side))
        wall = np.column_stack([gx.ravel(), gy.ravel(), np.full(side * side, 5.0)])
        blocks.append((wall, np.full(side * side, 2.2 * 2 * half / side), np.ones(side * side),
                       rng.uniform(0.2, 1.0, (side * side, d))))
        depth = rng.uniform(30.0, 43.0, count)
    elif profile == "uniform":
        depth = rng.uniform(6.0, 43.0, count)
    else:
        raise ValueError(f"unknown profile {profile!r}")
    half_w = depth * (SENSOR / 2.0) / FOCAL
    x = rng.uniform(-1, 1, count) * half_w
    y = rng.uniform(-1, 1, count) * half_w * ((height / width) if aspect_fill else 1.0)
    radius = 3.0 * depth * px / FOCAL  # 3 px projected
    blocks.append((np.column_stack([x, y, depth]), radius, rng.uniform(0.5, 1.0, count),
                   rng.uniform(0, 1, (count, d))))
    f32 = np.float32
    pos = np.concatenate([b[0] for b in blocks]).astype(f32)
    rad = np.concatenate([b[1] for b in blocks]).astype(f32)
    opa = np.concatenate([b[2] for b in blocks]).astype(f32)
    feat = np.concatenate([b[3] for b in blocks]).astype(f32)
    return pos, rad, opa, feat, np.zeros(d, f32), np.array([0, 0, 0, 0, 0, 0, FOCAL, SENSOR], np.float64)


def orbit_camera_vectors(num_views: int = 64):
    """Config 4: cam_vec_v = [0.3 cos th, 0.3 sin th, 0, 0, 0.02 sin th, 0, 5, 2], th = 2 pi v / V."""
    out = []
    for v in range(num_views):
        th = 2.0 * np.pi * v / num_views
        out.append(np.array([0.3 * np.cos(th), 0.3 * np.sin(th), 0.0, 0.0, 0.02 * np.sin(th), 0.0, FOCAL, SENSOR]))
    return out
