"""Synthetic scenes and ground-truth views for the large configurations
(SURVEY §8f row 1): the parameter distribution of generate_synthetic
(reference dataset.hpp:178-250) drawn with numpy, the reference camera ring
(:207-219, look_at :161-172), and GT images rendered by the GPU forward path
(K1-K6) then quantised through 8 bits as the PNG round trip does
(png_io.cpp:64, 97-98).

Extensions recorded in DESIGN.md: non-square images with
fx = fy = 1.1 * H * 2.6, and a scale multiplier (500 / N)^(1/3) for N >= 100K
so per-pixel depth complexity stays finite.
"""
from __future__ import annotations

import math

import numpy as np

SH_C0 = 0.28209479177387814


def n_components(deg: int) -> int:
    return 11 + 3 * (deg + 1) ** 2


def scale_multiplier(n: int) -> float:
    return (500.0 / n) ** (1.0 / 3.0) if n >= 100_000 else 1.0


def gaussians(n: int, seed: int = 1, sh_degree: int = 3, scale_mult: float | None = None) -> np.ndarray:
    """GT scene (sh_degree 1 content, padded to `sh_degree`), planar [C][n] float32."""
    rng = np.random.default_rng(seed)
    mult = scale_multiplier(n) if scale_mult is None else scale_mult
    p = np.zeros((n_components(sh_degree), n), np.float32)
    p[0:3] = rng.uniform(-0.5, 0.5, (3, n))
    q = rng.normal(size=(4, n))
    nq = np.linalg.norm(q, axis=0)
    q = np.where(nq > 1e-6, q / np.maximum(nq, 1e-12), np.array([[1], [0], [0], [0]]))
    p[3:7] = q
    p[7:10] = np.log(rng.uniform(0.02, 0.075, (3, n)) * mult)
    op = rng.uniform(0.25, 0.95, n)
    p[10] = np.log(op / (1.0 - op))
    p[11:14] = (rng.uniform(0.05, 0.95, (3, n)) - 0.5) / SH_C0
    if sh_degree >= 1:
        p[14:23] = rng.uniform(-0.1, 0.1, (9, n))
    return p


def look_at(eye, target=(0.0, 0.0, 0.0), up=(0.0, 0.0, 1.0)) -> np.ndarray:
    eye = np.asarray(eye, np.float64)
    z = np.asarray(target, np.float64) - eye
    z /= np.linalg.norm(z)
    x = np.cross(z, up)
    x /= np.linalg.norm(x)
    y = np.cross(z, x)
    m = np.eye(4)
    m[0, :3], m[1, :3], m[2, :3] = x, y, z
    m[:3, 3] = -(m[:3, :3] @ eye)
    return m


def ring_camera(view: int, n_views: int, width: int, height: int, focal: float | None = None, camera_fn=None):
    """Camera `view` of the reference ring (radius 2.4, height 1.0, look-at origin).
    camera_fn builds the struct (default: this package's sk_camera; the
    benchmark's reference arm passes the oracle's)."""
    if camera_fn is None:
        from . import camera as camera_fn
    camera = camera_fn
    angle = 2.0 * math.pi * view / n_views
    eye = (2.4 * math.cos(angle), 2.4 * math.sin(angle), 1.0)
    f = focal if focal is not None else 1.1 * height * 2.6
    return camera(width, height, f, f, (width - 1) / 2.0, (height - 1) / 2.0, look_at(eye), 0.2)


def ring_extent(n_views: int = 64) -> float:
    """scene_extent (dataset.hpp:56-66) of the camera ring: 1.1 x max distance
    of the camera centres from their mean."""
    return 1.1 * 2.4


def quantize_u8(img: np.ndarray) -> np.ndarray:
    """lround(clamp(v, 0, 1) * 255) (png_io.cpp:97-98)."""
    prod = np.clip(img.astype(np.float32), np.float32(0.0), np.float32(1.0)) * np.float32(255.0)
    return np.floor(prod.astype(np.float64) + 0.5).astype(np.uint8)  # lround, half away from zero


def render_gt_u8(ctx, params: np.ndarray, sh_degree: int, cam) -> np.ndarray:
    """GT view rendered by the GPU forward path, as 8-bit HWC."""
    scene = ctx.scene(params, sh_degree)
    ctx.preprocess(scene, cam)
    ctx.build_tile_grid()
    img = ctx.blend_forward().image
    scene.close()
    return quantize_u8(img)


def perturb_positions(params: np.ndarray, sigma: float, seed: int = 2) -> np.ndarray:
    rng = np.random.default_rng(seed)
    q = params.copy()
    q[0:3] += (sigma * rng.normal(size=(3, params.shape[1]))).astype(np.float32)
    return q
