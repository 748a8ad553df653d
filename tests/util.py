"""Shared test helpers: random scenes/cameras (numpy RNG) and comparison utilities."""
import math

import numpy as np


def random_scene(rng, n, sh_degree=2, max_opacity=0.8, z=(2.0, 5.0), xy=0.6):
    """Same distribution as tests/helpers.hpp:100-118 (random_scene), planar layout."""
    from oracle.oracle import n_components
    p = np.zeros((n_components(sh_degree), n), np.float32)
    p[0] = rng.uniform(-xy, xy, n)
    p[1] = rng.uniform(-xy, xy, n)
    p[2] = rng.uniform(z[0], z[1], n)
    q = rng.normal(size=(4, n))
    p[3:7] = q / np.linalg.norm(q, axis=0)
    p[7:10] = np.log(rng.uniform(0.03, 0.15, (3, n)))
    op = rng.uniform(0.1, max_opacity, n)
    p[10] = np.log(op / (1 - op))
    nsh = (sh_degree + 1) ** 2
    for k in range(nsh):
        for c in range(3):
            p[11 + 3 * k + c] = rng.uniform(-0.3, 0.3, n) + (rng.uniform(0.2, 1.2, n) if k == 0 else 0)
    return p


def look_at(eye, target=(0.0, 0.0, 0.0), up=(0.0, 0.0, 1.0)):
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


def ring_camera(orc, width, height, angle=0.0, focal=None, radius=2.4, height_z=1.0):
    f = focal if focal is not None else 1.1 * height
    eye = (radius * math.cos(angle), radius * math.sin(angle), height_z)
    return orc.camera(width, height, f, f, (width - 1) / 2.0, (height - 1) / 2.0, look_at(eye), 0.2)


def synthetic_scene(n, deg=3, seed=1, scale_mult=None):
    """Unit-cube scene like generate_synthetic (dataset.hpp:187-201), numpy RNG, padded to `deg`."""
    rng = np.random.default_rng(seed)
    from oracle.oracle import n_components
    if scale_mult is None:
        scale_mult = (500.0 / n) ** (1.0 / 3.0) if n >= 100_000 else 1.0
    p = np.zeros((n_components(deg), n), np.float32)
    p[0:3] = rng.uniform(-0.5, 0.5, (3, n))
    q = rng.normal(size=(4, n))
    p[3:7] = q / np.linalg.norm(q, axis=0)
    p[7:10] = np.log(rng.uniform(0.02, 0.075, (3, n)) * scale_mult)
    op = rng.uniform(0.25, 0.95, n)
    p[10] = np.log(op / (1 - op))
    p[11:14] = (rng.uniform(0.05, 0.95, (3, n)) - 0.5) / 0.28209479177387814
    if deg >= 1:
        p[14:23] = rng.uniform(-0.1, 0.1, (9, n))
    return p


def rel_err_vec(a, b, floor_frac=1e-3):
    """Elementwise |a-b| / max(|a|, |b|, floor), floor = floor_frac * max|b| (atomic-order tolerance)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    floor = max(floor_frac * np.abs(b).max(), 1e-12)
    return np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)


def unfloored_report(name, got, ref, floor_frac=1e-3):
    """Distribution of the elementwise relative error WITHOUT a floor
    (|a-b| / max(|a|, |b|), elements where both are exactly zero excluded),
    next to the floored maximum the assertions use. Appended as one JSON line
    to $SK_PARITY_REPORT when that is set (the round's parity evidence)."""
    import json
    import os
    a = np.asarray(got, np.float64).ravel()
    b = np.asarray(ref, np.float64).ravel()
    den = np.maximum(np.abs(a), np.abs(b))
    nz = den > 0
    e = np.abs(a - b)[nz] / den[nz]
    rep = {"name": name, "elements": int(a.size), "nonzero": int(nz.sum()),
           "floored_max": float(rel_err_vec(a, b, floor_frac).max()) if a.size else 0.0,
           "unfloored_p50": float(np.percentile(e, 50)) if e.size else 0.0,
           "unfloored_p99": float(np.percentile(e, 99)) if e.size else 0.0,
           "unfloored_p999": float(np.percentile(e, 99.9)) if e.size else 0.0,
           "unfloored_max": float(e.max()) if e.size else 0.0,
           "frac_unfloored_gt_1e-3": float((e > 1e-3).mean()) if e.size else 0.0,
           "max_abs_err": float(np.abs(a - b).max()) if a.size else 0.0,
           "max_abs_ref": float(np.abs(b).max()) if b.size else 0.0}
    path = os.environ.get("SK_PARITY_REPORT")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rep) + "\n")
    return rep
