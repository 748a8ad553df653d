"""Generates tests/golden/*.json: frozen outputs of the CPU oracle (the
restated reference) on small seeded scenes, as SHA-256 digests of the exact
little-endian array bytes plus a few scalars. The reference itself cannot be
built in this image (Eigen3 / libpng / doctest absent), so these
fixtures freeze the oracle after it was pinned by the reference's own
known-answer tests (tests/test_oracle_kats.py); tests/test_golden.py checks
that the oracle still reproduces them (CPU) and that the GPU path matches
them bit for bit where the contract is bit-exact (GPU).

    python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as orc  # noqa: E402
from tests.util import ring_camera, synthetic_scene  # noqa: E402

# (name, n, deg, seed, width, height, ring angle, binning mode, beta)
CASES = [
    ("ring_aabb_deg3", 2500, 3, 11, 160, 120, 0.3, "aabb", 1.0),
    ("ring_compact_deg1", 1800, 1, 12, 128, 96, 2.0, "compact", 0.8),
    ("ring_aabb_deg0_tile8", 1200, 0, 13, 96, 64, 4.1, "aabb", 1.0),
]


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.astype(a.dtype.newbyteorder("<"), copy=False).tobytes()).hexdigest()


def build(name, n, deg, seed, w, h, angle, mode, beta):
    tile = 8 if name.endswith("tile8") else 16
    p = synthetic_scene(n, deg=deg, seed=seed)
    cam = ring_camera(orc, w, h, angle)
    b = orc.binning(mode, beta=beta, tile_size=tile)
    r = orc.render_scene(p, deg, cam, b)
    visited = orc.last_pge_visited()
    gt = np.clip(r.image[::-1, ::-1] * 0.9 + 0.05, 0, 1).astype(np.float32)  # a deterministic "target"
    loss, l1, ssim, d_image = orc.training_loss(r.image, gt, 0.2)
    return {
        "inputs": {"n": n, "sh_degree": deg, "seed": seed, "width": w, "height": h, "angle": angle,
                   "bin_mode": mode, "beta": beta, "tile_size": tile,
                   "scene": "tests/util.py:synthetic_scene", "camera": "tests/util.py:ring_camera",
                   "target": "clip(image[::-1, ::-1] * 0.9 + 0.05, 0, 1)"},
        "pairs": int(r.pairs),
        "pge_visited": int(visited),
        "pge_contributing": int(r.contrib.astype(np.int64).sum()),
        "sha256": {"image": digest(r.image), "transmittance": digest(r.transmittance),
                   "contrib": digest(r.contrib), "tile_values": digest(r.values)},
        "image_sum": float(np.float64(r.image).sum()),
        "loss": {"loss": float(loss), "l1": float(l1), "ssim": float(ssim)},
    }


def main():
    orc.build()
    for c in CASES:
        out = build(*c)
        with open(os.path.join(HERE, c[0] + ".json"), "w") as f:
            json.dump(out, f, indent=1, sort_keys=True)
            f.write("\n")
        print(c[0], out["pairs"], out["sha256"]["image"][:16])


if __name__ == "__main__":
    main()
