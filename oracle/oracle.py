"""TEST INFRASTRUCTURE ONLY — ctypes binding of the CPU oracle.

The oracle (splat_oracle.hpp) restates the reference splatkit hot path
(/root/reference/proj/include/splatkit/*.hpp) operation by operation. Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
arm may import this module, and only as the checker. The product path never
touches it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")


class SkCamera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("world_to_cam", C.c_float * 16),
                ("near_plane", C.c_float)]


class SkBinning(C.Structure):
    _fields_ = [("mode", C.c_int32), ("beta", C.c_float), ("tau_alpha", C.c_float), ("tile_size", C.c_int32)]


class OrTable(C.Structure):
    _fields_ = [("s_d", C.c_void_p), ("s_p", C.c_void_p), ("grad_norm_acc", C.c_void_p),
                ("abs_grad_acc", C.c_void_p), ("grad3d_acc", C.c_void_p), ("views_seen", C.c_void_p),
                ("max_radius2d", C.c_void_p)]


class OrTrainConfig(C.Structure):
    _fields_ = [("iterations", C.c_int), ("k", C.c_int), ("lambda_", C.c_double), ("tau", C.c_double),
                ("tau_d", C.c_double), ("tau_p", C.c_double), ("beta", C.c_double), ("tau_alpha", C.c_double),
                ("densify_from", C.c_int), ("densify_until", C.c_int), ("densify_every", C.c_int),
                ("prune_every_early", C.c_int), ("prune_every_late", C.c_int),
                ("grad_threshold", C.c_double), ("percent_dense", C.c_double),
                ("lr_position", C.c_double), ("lr_position_final", C.c_double), ("lr_sh_dc", C.c_double),
                ("lr_sh_rest", C.c_double), ("lr_opacity", C.c_double), ("lr_scale", C.c_double),
                ("lr_rotation", C.c_double), ("opacity_reset_every", C.c_int), ("lazy_opt_enabled", C.c_int),
                ("lazy_opt_interval_15k", C.c_int), ("lazy_opt_interval_20k", C.c_int), ("seed", C.c_uint64),
                ("tile_size", C.c_int), ("workers", C.c_int), ("sh_degree", C.c_int), ("compact", C.c_int),
                ("vcd", C.c_int), ("vcp", C.c_int), ("prune_min_opacity", C.c_double),
                ("prune_opacity_late", C.c_double), ("prune_world_size_frac", C.c_double),
                ("prune_screen_size", C.c_double), ("size_prune_from", C.c_int), ("schedule_dry_run", C.c_int)]


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-C", HERE, "-s"], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
        _lib.or_last_error.restype = C.c_char_p
        _lib.or_expf.restype = C.c_float
        _lib.or_expf.argtypes = [C.c_float]
        _lib.or_logf.restype = C.c_float
        _lib.or_logf.argtypes = [C.c_float]
        _lib.or_compact_threshold_d.restype = C.c_double
        _lib.or_compact_threshold_d.argtypes = [C.c_double] * 3
        _lib.or_expon_lr_f.restype = C.c_double
        _lib.or_expon_lr_f.argtypes = [C.c_float, C.c_float, C.c_int, C.c_int]
        _lib.or_synth_create.restype = C.c_void_p
        _lib.or_synth_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_double,
                                         C.c_double, C.c_int]
        _lib.or_dataset_extent.restype = C.c_float
        _lib.or_dataset_extent.argtypes = [C.c_void_p]
        for f in ("or_dataset_num_views", "or_dataset_num_points", "or_dataset_destroy"):
            getattr(_lib, f).argtypes = [C.c_void_p]
        _lib.or_trainer_create.restype = C.c_void_p
        _lib.or_trainer_size.restype = C.c_int64
        _lib.or_trainer_size.argtypes = [C.c_void_p]
        _lib.or_trainer_num_events.argtypes = [C.c_void_p]
        _lib.or_trainer_destroy.argtypes = [C.c_void_p]
    return _lib


def ptr(a):
    """Raw pointer of a contiguous numpy array (or None)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "array must be contiguous"
    return C.c_void_p(a.ctypes.data)


def check(rc: int):
    if rc != 0:
        msg = lib().or_last_error().decode()
        if rc == 1:
            raise ValueError(msg)
        raise RuntimeError(msg)


def set_detmath(on: bool):
    lib().or_set_detmath(1 if on else 0)


# ---------------------------------------------------------------------------
# cameras / binning
# ---------------------------------------------------------------------------

def camera(width, height, fx, fy, cx, cy, world_to_cam=None, near=0.2) -> SkCamera:
    c = SkCamera()
    c.width, c.height = int(width), int(height)
    c.fx, c.fy, c.cx, c.cy = float(fx), float(fy), float(cx), float(cy)
    w = np.eye(4, dtype=np.float64) if world_to_cam is None else np.asarray(world_to_cam, np.float64)
    for i, v in enumerate(w.reshape(-1)):
        c.world_to_cam[i] = float(v)
    c.near_plane = float(near)
    return c


def default_camera(width=32, height=32) -> SkCamera:
    """tests/helpers.hpp:121-131."""
    return camera(width, height, np.float32(0.9) * width, np.float32(0.9) * width,
                  (width - 1) / 2.0, (height - 1) / 2.0)


def binning(mode="aabb", beta=1.0, tau_alpha=1.0 / 255, tile_size=16) -> SkBinning:
    b = SkBinning()
    b.mode = 1 if mode in ("compact", 1) else 0
    b.beta = float(beta)
    b.tau_alpha = float(tau_alpha)
    b.tile_size = int(tile_size)
    return b


# ---------------------------------------------------------------------------
# host RNG (rng.hpp) — pure-python mt19937_64 via numpy is not bit-compatible,
# so random scenes for tests come from numpy's own generator; the oracle Rng
# is exercised through the trainer / synthetic generator.
# ---------------------------------------------------------------------------

def n_components(deg: int) -> int:
    return 11 + 3 * (deg + 1) ** 2


@dataclass
class Projected:
    visible: np.ndarray
    mu2d: np.ndarray
    cov2d: np.ndarray
    conic: np.ndarray
    depth: np.ndarray
    color: np.ndarray
    opacity: np.ndarray
    tiles_touched: np.ndarray


def project_scene(params: np.ndarray, deg: int, cam: SkCamera, bin_: SkBinning | None = None,
                  dtype=np.float32) -> Projected:
    p = np.ascontiguousarray(params, dtype)
    n = p.shape[1]
    out = Projected(np.zeros(n, np.int32), np.zeros((n, 2), dtype), np.zeros((n, 4), dtype),
                    np.zeros((n, 4), dtype), np.zeros(n, dtype), np.zeros((n, 3), dtype), np.zeros(n, dtype),
                    np.zeros(n, np.int32))
    fn = lib().or_project_scene_f if dtype == np.float32 else lib().or_project_scene_d
    check(fn(ptr(p), C.c_int64(n), C.c_int(deg), C.byref(cam), C.byref(bin_ or binning()), ptr(out.visible),
             ptr(out.mu2d), ptr(out.cov2d), ptr(out.conic), ptr(out.depth), ptr(out.color), ptr(out.opacity),
             ptr(out.tiles_touched)))
    return out


@dataclass
class Render:
    image: np.ndarray
    transmittance: np.ndarray
    contrib: np.ndarray
    ranges: np.ndarray
    values: np.ndarray
    pairs: int
    counts: np.ndarray | None = None


def _tiles(w, h, ts):
    return ((w + ts - 1) // ts) * ((h + ts - 1) // ts)


def render_scene(params, deg, cam: SkCamera, bin_: SkBinning | None = None, mask=None, workers=1,
                 values_cap=None) -> Render:
    bin_ = bin_ or binning()
    p = np.ascontiguousarray(params, np.float32)
    n = p.shape[1]
    w, h = cam.width, cam.height
    img = np.zeros((h, w, 3), np.float32)
    tr = np.zeros((h, w), np.float32)
    cc = np.zeros((h, w), np.int32)
    ranges = np.zeros((_tiles(w, h, bin_.tile_size), 2), np.int32)
    cap = values_cap if values_cap is not None else max(1, 64 * n)
    vals = np.zeros(cap, np.int32)
    pairs = C.c_int64(0)
    counts = None
    m = None
    if mask is not None:
        m = np.ascontiguousarray(mask, np.uint8)
        counts = np.zeros(n, np.int32)
    check(lib().or_render_scene_f(ptr(p), C.c_int64(n), C.c_int(deg), C.byref(cam), C.byref(bin_), ptr(m),
                                  ptr(counts), C.c_int(workers), ptr(img), ptr(tr), ptr(cc), ptr(ranges),
                                  ptr(vals), C.c_int64(cap), C.byref(pairs)))
    assert pairs.value <= cap, "values_cap too small"
    return Render(img, tr, cc, ranges, vals[: pairs.value].copy(), pairs.value, counts)


def rng_normals(seed: int, count: int) -> np.ndarray:
    """count successive Rng::normal() draws (rng.hpp:36-49) as float32."""
    out = np.zeros(max(1, count), np.float32)
    check(lib().or_rng_normals(C.c_uint64(seed), C.c_int64(count), ptr(out)))
    return out[:count]


def last_pge_visited() -> int:
    """Pixel-Gaussian evaluations the reference loop visited in the last
    render_scene / render_pg call on this thread (RenderOutputs::pge_visited)."""
    f = lib().or_last_pge_visited
    f.restype = C.c_int64
    return int(f())


@dataclass
class PG:
    """Projected Gaussians (camera.hpp:60-68) in projected order."""
    mu2d: np.ndarray
    cov2d: np.ndarray
    conic: np.ndarray
    depth: np.ndarray
    color: np.ndarray
    opacity: np.ndarray

    @property
    def n(self):
        return self.mu2d.shape[0]

    def astype(self, dtype):
        return PG(*(np.array(getattr(self, f), dtype, copy=True, order="C") for f in
                    ("mu2d", "cov2d", "conic", "depth", "color", "opacity")))


def random_projected(rng: np.random.Generator, n, width, height, max_opacity=0.34, min_opacity=0.05,
                     dtype=np.float64) -> PG:
    """Same distribution as tests/helpers.hpp:72-96 (numpy RNG instead of Rng)."""
    mu = np.stack([rng.uniform(-2.0, width + 2.0, n), rng.uniform(-2.0, height + 2.0, n)], 1)
    a = rng.uniform(-2, 2, (n, 2, 2))
    a = a.astype(dtype)
    cov = a @ np.transpose(a, (0, 2, 1))
    cov[:, 0, 0] += dtype(0.3)
    cov[:, 1, 1] += dtype(0.3)
    det = cov[:, 0, 0] * cov[:, 1, 1] - cov[:, 0, 1] * cov[:, 1, 0]
    inv = np.stack([cov[:, 1, 1] / det, -cov[:, 0, 1] / det, -cov[:, 1, 0] / det, cov[:, 0, 0] / det], 1)
    depth = rng.uniform(0.5, 10.0, n)
    color = rng.uniform(0, 1, (n, 3))
    op = rng.uniform(min_opacity, max_opacity, n)
    return PG(mu.astype(dtype), cov.reshape(n, 4).astype(dtype), inv.astype(dtype), depth.astype(dtype),
              color.astype(dtype), op.astype(dtype))


def _pg_args(pg: PG, dtype):
    pg = pg.astype(dtype)
    return pg, [ptr(pg.mu2d), ptr(pg.cov2d), ptr(pg.conic), ptr(pg.depth), ptr(pg.color), ptr(pg.opacity)]


def render_pg(pg: PG, width, height, bin_: SkBinning | None = None, mask=None, workers=1, dtype=np.float32,
              values_cap=None) -> Render:
    bin_ = bin_ or binning()
    pg, args = _pg_args(pg, dtype)
    n = pg.n
    img = np.zeros((height, width, 3), dtype)
    tr = np.zeros((height, width), dtype)
    cc = np.zeros((height, width), np.int32)
    ranges = np.zeros((_tiles(width, height, bin_.tile_size), 2), np.int32)
    cap = values_cap if values_cap is not None else max(1, 4 * n * _tiles(width, height, bin_.tile_size))
    vals = np.zeros(cap, np.int32)
    pairs = C.c_int64(0)
    counts = None
    m = None
    if mask is not None:
        m = np.ascontiguousarray(mask, np.uint8)
        counts = np.zeros(n, np.int32)
    fn = lib().or_render_pg_f if dtype == np.float32 else lib().or_render_pg_d
    check(fn(*args, C.c_int64(n), C.c_int(width), C.c_int(height), C.byref(bin_), ptr(m), ptr(counts),
             C.c_int(workers), ptr(img), ptr(tr), ptr(cc), ptr(ranges), ptr(vals), C.c_int64(cap), C.byref(pairs)))
    return Render(img, tr, cc, ranges, vals[: pairs.value].copy(), pairs.value, counts)


def brute_render_pg(pg: PG, width, height, mask=None, dtype=np.float32):
    pg, args = _pg_args(pg, dtype)
    img = np.zeros((height, width, 3), dtype)
    tr = np.zeros((height, width), dtype)
    cc = np.zeros((height, width), np.int32)
    counts = None
    m = None
    if mask is not None:
        m = np.ascontiguousarray(mask, np.uint8)
        counts = np.zeros(pg.n, np.int32)
    fn = lib().or_brute_render_pg_f if dtype == np.float32 else lib().or_brute_render_pg_d
    check(fn(*args, C.c_int64(pg.n), C.c_int(width), C.c_int(height), ptr(m), ptr(counts), ptr(img), ptr(tr),
             ptr(cc)))
    return img, tr, cc, counts


@dataclass
class BlendGrads:
    d_mu2d: np.ndarray
    d_conic: np.ndarray
    d_color: np.ndarray
    d_opacity: np.ndarray
    abs_grad: np.ndarray


def blend_backward_pg(pg: PG, width, height, d_image, bin_: SkBinning | None = None, workers=1,
                      dtype=np.float32) -> BlendGrads:
    bin_ = bin_ or binning()
    pg, args = _pg_args(pg, dtype)
    n = pg.n
    g = BlendGrads(np.zeros((n, 2), dtype), np.zeros((n, 4), dtype), np.zeros((n, 3), dtype), np.zeros(n, dtype),
                   np.zeros((n, 2), dtype))
    di = np.ascontiguousarray(d_image, dtype)
    fn = lib().or_blend_backward_pg_f if dtype == np.float32 else lib().or_blend_backward_pg_d
    check(fn(*args, C.c_int64(n), C.c_int(width), C.c_int(height), C.byref(bin_), ptr(di), C.c_int(workers),
             ptr(g.d_mu2d), ptr(g.d_conic), ptr(g.d_color), ptr(g.d_opacity), ptr(g.abs_grad)))
    return g


def training_loss(rendered, gt, lam=0.2, dtype=np.float32):
    r = np.ascontiguousarray(rendered, dtype)
    g = np.ascontiguousarray(gt, dtype)
    h, w = r.shape[:2]
    ct = C.c_float if dtype == np.float32 else C.c_double
    loss, l1, ss = ct(), ct(), ct()
    d = np.zeros_like(r)
    fn = lib().or_training_loss_f if dtype == np.float32 else lib().or_training_loss_d
    check(fn(ptr(r), ptr(g), C.c_int(w), C.c_int(h), ct(lam), C.byref(loss), C.byref(l1), C.byref(ss), ptr(d)))
    return loss.value, l1.value, ss.value, d


def ssim(a, b, dtype=np.float32):
    a = np.ascontiguousarray(a, dtype)
    b = np.ascontiguousarray(b, dtype)
    h, w = a.shape[:2]
    ct = C.c_float if dtype == np.float32 else C.c_double
    out = ct()
    fn = lib().or_ssim_f if dtype == np.float32 else lib().or_ssim_d
    check(fn(ptr(a), ptr(b), C.c_int(w), C.c_int(h), C.byref(out)))
    return out.value


def psnr(a, b, dtype=np.float32):
    a = np.ascontiguousarray(a, dtype)
    b = np.ascontiguousarray(b, dtype)
    h, w = a.shape[:2]
    out = C.c_double()
    fn = lib().or_psnr_f if dtype == np.float32 else lib().or_psnr_d
    check(fn(ptr(a), ptr(b), C.c_int(w), C.c_int(h), C.byref(out)))
    return out.value


def error_maps(r, g, tau=0.5, lam=0.2, dtype=np.float64):
    r = np.ascontiguousarray(r, dtype)
    g = np.ascontiguousarray(g, dtype)
    h, w = r.shape[:2]
    raw = np.zeros((h, w), dtype)
    nrm = np.zeros((h, w), dtype)
    mask = np.zeros((h, w), np.uint8)
    ct = C.c_double if dtype == np.float64 else C.c_float
    ph = ct()
    fn = lib().or_error_maps_d if dtype == np.float64 else lib().or_error_maps_f
    check(fn(ptr(r), ptr(g), C.c_int(w), C.c_int(h), ct(tau), ct(lam), ptr(raw), ptr(nrm), ptr(mask), C.byref(ph)))
    return raw, nrm, mask, ph.value


def project_backward(params, deg, cam, d_mu2d, d_conic, d_color, d_opacity, dtype=np.float32):
    p = np.ascontiguousarray(params, dtype)
    out = np.zeros_like(p)
    args = [np.ascontiguousarray(a, dtype) for a in (d_mu2d, d_conic, d_color, d_opacity)]
    fn = lib().or_project_backward_f if dtype == np.float32 else lib().or_project_backward_d
    check(fn(ptr(p), C.c_int64(p.shape[1]), C.c_int(deg), C.byref(cam), *[ptr(a) for a in args], ptr(out)))
    return out


def covariance_3d(rot, scale):
    r = np.ascontiguousarray(rot, np.float64)
    s = np.ascontiguousarray(scale, np.float64)
    out = np.zeros((3, 3))
    check(lib().or_covariance_3d_d(ptr(r), ptr(s), ptr(out)))
    return out


def evaluate_sh(sh, deg, direction):
    sh = np.ascontiguousarray(sh, np.float64)
    d = np.ascontiguousarray(direction, np.float64)
    out = np.zeros(3)
    check(lib().or_evaluate_sh_d(ptr(sh), C.c_int(deg), ptr(d), ptr(out)))
    return out


def bin_one(mu2d, cov2d, conic, opacity, width, height, bin_: SkBinning):
    mu = np.ascontiguousarray(mu2d, np.float64)
    cv = np.ascontiguousarray(cov2d, np.float64).reshape(4)
    cn = np.ascontiguousarray(conic, np.float64).reshape(4)
    tiles = np.zeros(4096, np.int32)
    cnt = C.c_int()
    check(lib().or_bin_one_d(ptr(mu), ptr(cv), ptr(cn), C.c_double(opacity), C.c_int(width), C.c_int(height),
                             C.byref(bin_), ptr(tiles), C.c_int(4096), C.byref(cnt)))
    return tiles[: cnt.value].tolist()


def compact_threshold(sigma, tau_alpha, beta):
    return lib().or_compact_threshold_d(sigma, tau_alpha, beta)


def scores_from_counts(counts, photometric):
    c = np.ascontiguousarray(counts, np.int32)
    ph = np.ascontiguousarray(photometric, np.float32)
    k, n = c.shape
    s_d = np.zeros(n, np.float32)
    s_p_raw = np.zeros(n, np.float32)
    s_p = np.zeros(n, np.float32)
    check(lib().or_scores_from_counts_f(ptr(c), ptr(ph), C.c_int(k), C.c_int64(n), ptr(s_d), ptr(s_p_raw),
                                        ptr(s_p)))
    return s_d, s_p_raw, s_p


def make_table(n, **fields):
    arrs = {}
    t = OrTable()
    for name, dt in (("s_d", np.float32), ("s_p", np.float32), ("grad_norm_acc", np.float32),
                     ("abs_grad_acc", np.float32), ("grad3d_acc", np.float32), ("views_seen", np.int32),
                     ("max_radius2d", np.float32)):
        if name in fields and fields[name] is not None:
            a = np.ascontiguousarray(fields[name], dt)
            arrs[name] = a
            setattr(t, name, a.ctypes.data)
    t._keep = arrs
    return t


def select_densify(params, deg, table: OrTable, tau_d=5.0, grad_threshold=2e-4, percent_dense=0.01,
                   use_vcd=True, extent=1.0):
    p = np.ascontiguousarray(params, np.float32)
    n = p.shape[1]
    clone = np.zeros(n, np.uint8)
    split = np.zeros(n, np.uint8)
    check(lib().or_select_densify_f(ptr(p), C.c_int64(n), C.c_int(deg), C.byref(table), C.c_float(tau_d),
                                    C.c_float(grad_threshold), C.c_float(percent_dense), C.c_int(int(use_vcd)),
                                    C.c_float(extent), ptr(clone), ptr(split)))
    return clone, split


def select_prune(params, deg, table: OrTable, iteration, tau_p=0.9, min_opacity=0.005, opacity_late=0.1,
                 world_size_frac=0.1, screen_size=20.0, size_prune_from=3000, densify_until=15000, use_vcp=True,
                 extent=1.0):
    p = np.ascontiguousarray(params, np.float32)
    n = p.shape[1]
    prune = np.zeros(n, np.uint8)
    check(lib().or_select_prune_f(ptr(p), C.c_int64(n), C.c_int(deg), C.byref(table), C.c_int(iteration),
                                  C.c_float(tau_p), C.c_float(min_opacity), C.c_float(opacity_late),
                                  C.c_float(world_size_frac), C.c_float(screen_size), C.c_int(size_prune_from),
                                  C.c_int(densify_until), C.c_int(int(use_vcp)), C.c_float(extent), ptr(prune)))
    return prune


def default_config() -> OrTrainConfig:
    c = OrTrainConfig()
    lib().or_default_config(C.byref(c))
    return c


class Dataset:
    """generate_synthetic (dataset.hpp:178-250), in memory."""

    def __init__(self, n_gaussians=500, n_views=64, width=128, height=None, seed=1, scale_mult=1.0, focal=-1.0,
                 render=True):
        height = width if height is None else height
        self.h = lib().or_synth_create(n_gaussians, n_views, width, height, seed, scale_mult, focal,
                                       1 if render else 0)
        if not self.h:
            raise ValueError(lib().or_last_error().decode())
        self.n_gaussians = n_gaussians
        self.width, self.height = width, height

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_dataset_destroy(self.h)
            self.h = None

    @property
    def num_views(self):
        return lib().or_dataset_num_views(self.h)

    @property
    def extent(self):
        return lib().or_dataset_extent(self.h)

    def camera(self, v) -> SkCamera:
        c = SkCamera()
        lib().or_dataset_camera(C.c_void_p(self.h), C.c_int(v), C.byref(c))
        return c

    def image_u8(self, v):
        out = np.zeros((self.height, self.width, 3), np.uint8)
        check(lib().or_dataset_image_u8(C.c_void_p(self.h), C.c_int(v), ptr(out)))
        return out

    def set_image_u8(self, v, img):
        img = np.ascontiguousarray(img, np.uint8)
        check(lib().or_dataset_set_image_u8(C.c_void_p(self.h), C.c_int(v), ptr(img)))

    def points(self):
        n = lib().or_dataset_num_points(self.h)
        xyz = np.zeros((n, 3), np.float32)
        rgb = np.zeros((n, 3), np.float32)
        lib().or_dataset_points(C.c_void_p(self.h), ptr(xyz), ptr(rgb))
        return xyz, rgb

    def train_indices(self):
        cnt = C.c_int()
        lib().or_dataset_train_indices(C.c_void_p(self.h), None, C.byref(cnt))
        out = np.zeros(cnt.value, np.int32)
        lib().or_dataset_train_indices(C.c_void_p(self.h), ptr(out), C.byref(cnt))
        return out

    def gt_scene(self):
        p = np.zeros((n_components(1), self.n_gaussians), np.float32)
        lib().or_dataset_gt_scene(C.c_void_p(self.h), ptr(p))
        return p


def init_from_points(xyz, rgb, deg):
    xyz = np.ascontiguousarray(xyz, np.float32)
    rgb = np.ascontiguousarray(rgb, np.float32)
    n = xyz.shape[0]
    out = np.zeros((n_components(deg), n), np.float32)
    check(lib().or_init_from_points(ptr(xyz), ptr(rgb), C.c_int64(n), C.c_int(deg), ptr(out)))
    return out


class Trainer:
    """Trainer (trainer.hpp:70-261) on an oracle Dataset."""

    def __init__(self, params, deg, dataset: Dataset, cfg: OrTrainConfig):
        p = np.ascontiguousarray(params, np.float32)
        self.deg = deg
        self.dataset = dataset  # keep alive: the trainer borrows it
        self.h = lib().or_trainer_create(ptr(p), C.c_int64(p.shape[1]), C.c_int(deg), C.c_void_p(dataset.h),
                                         C.byref(cfg))
        if not self.h:
            raise ValueError(lib().or_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_trainer_destroy(self.h)
            self.h = None

    def run(self, iters):
        rows = np.zeros((iters, 4), np.float64)
        secs = C.c_double()
        check(lib().or_trainer_run(C.c_void_p(self.h), C.c_int(iters), ptr(rows), C.byref(secs)))
        return rows, secs.value

    def set_iteration(self, it):
        lib().or_trainer_set_iteration(C.c_void_p(self.h), C.c_int(it))

    def scene(self):
        n = lib().or_trainer_size(self.h)
        p = np.zeros((n_components(self.deg), n), np.float32)
        lib().or_trainer_scene(C.c_void_p(self.h), ptr(p))
        return p

    def events(self):
        out = []
        for e in range(lib().or_trainer_num_events(self.h)):
            hdr = np.zeros(7, np.int32)
            lib().or_trainer_event(C.c_void_p(self.h), C.c_int(e), ptr(hdr), None, None, None, None, None)
            clone = np.zeros(max(1, hdr[3]), np.int32)
            split = np.zeros(max(1, hdr[4]), np.int32)
            prune = np.zeros(max(1, hdr[5]), np.int32)
            sampled = np.zeros(max(1, hdr[6]), np.int32)
            photo = np.zeros(max(1, hdr[6]), np.float32)
            lib().or_trainer_event(C.c_void_p(self.h), C.c_int(e), ptr(hdr), ptr(clone), ptr(split), ptr(prune),
                                   ptr(sampled), ptr(photo))
            out.append(dict(iteration=int(hdr[0]), n_before=int(hdr[1]), n_after=int(hdr[2]),
                            clone=clone[: hdr[3]], split=split[: hdr[4]], prune=prune[: hdr[5]],
                            sampled=sampled[: hdr[6]], photometric=photo[: hdr[6]]))
        return out


def train_step_view(params, deg, cam, gt_hwc, cfg: OrTrainConfig, extent, iteration, workers=1):
    """One train_iteration (trainer.hpp:124-175) on one explicit view."""
    p = np.ascontiguousarray(params, np.float32)
    n = p.shape[1]
    out = np.zeros_like(p)
    lp = np.zeros(2, np.float64)
    pairs = C.c_int64()
    gn = np.zeros(n, np.float32)
    ag = np.zeros(n, np.float32)
    g3 = np.zeros((n, 3), np.float32)
    vs = np.zeros(n, np.int32)
    mr = np.zeros(n, np.float32)
    gt = np.ascontiguousarray(gt_hwc, np.float32)
    check(lib().or_train_step_view(ptr(p), C.c_int64(n), C.c_int(deg), C.byref(cam), ptr(gt), C.byref(cfg),
                                   C.c_float(extent), C.c_int(iteration), C.c_int(workers), ptr(out), ptr(lp),
                                   C.byref(pairs), ptr(gn), ptr(ag), ptr(g3), ptr(vs), ptr(mr)))
    return dict(params=out, loss=lp[0], psnr=lp[1], pairs=pairs.value, grad_norm_acc=gn, abs_grad_acc=ag,
                grad3d_acc=g3, views_seen=vs, max_radius2d=mr)


def accumulate_scores(params, deg, cams, images, tau=0.5, lam=0.2, bin_=None, workers=1):
    """accumulate_scores (adc.hpp:91-115) over explicit views; images float HWC."""
    p = np.ascontiguousarray(params, np.float32)
    n = p.shape[1]
    k = len(cams)
    arr = (SkCamera * k)(*[SkCamera.from_buffer_copy(bytes(c)) for c in cams])
    imgs = np.ascontiguousarray(np.concatenate([np.asarray(i, np.float32).reshape(-1) for i in images]))
    counts = np.zeros((k, n), np.int32)
    photo = np.zeros(k, np.float32)
    s_d = np.zeros(n, np.float32)
    s_p_raw = np.zeros(n, np.float32)
    s_p = np.zeros(n, np.float32)
    check(lib().or_accumulate_scores_f(ptr(p), C.c_int64(n), C.c_int(deg), C.c_int(k), arr, ptr(imgs),
                                       C.c_float(tau), C.c_float(lam), C.byref(bin_ or binning()), C.c_int(workers),
                                       ptr(counts), ptr(photo), ptr(s_d), ptr(s_p_raw), ptr(s_p)))
    return counts, photo, s_d, s_p_raw, s_p


def apply_prune_densify(params, deg, prune, clone, split, grad3d, views_seen, clone_lr, eps, m=None, v=None):
    """Trainer::density_event compaction (trainer.hpp:203-233) with explicit split normals."""
    p = np.ascontiguousarray(params, np.float32)
    n = p.shape[1]
    cap = n + int(np.sum(clone)) + 2 * int(np.sum(split))
    out = np.zeros((p.shape[0], cap), np.float32)
    mo = np.zeros_like(out)
    vo = np.zeros_like(out)
    nn = C.c_int64()
    o2n = np.zeros(n, np.int32)
    args = [np.ascontiguousarray(a, np.uint8) for a in (prune, clone, split)]
    g3 = np.ascontiguousarray(grad3d, np.float32)
    vs = np.ascontiguousarray(views_seen, np.int32)
    e = np.ascontiguousarray(eps, np.float32) if len(eps) else np.zeros(1, np.float32)
    mi = None if m is None else np.ascontiguousarray(m, np.float32)
    vi = None if v is None else np.ascontiguousarray(v, np.float32)
    check(lib().or_apply_prune_densify_f(ptr(p), C.c_int64(n), C.c_int(deg), *[ptr(a) for a in args], ptr(g3),
                                         ptr(vs), C.c_float(clone_lr), ptr(e), ptr(mi), ptr(vi), ptr(out), ptr(mo),
                                         ptr(vo), C.byref(nn), ptr(o2n)))
    k = nn.value
    # scene_to_planar wrote [C][k] contiguously at the start of each buffer
    flat = out.reshape(-1)[: p.shape[0] * k].reshape(p.shape[0], k)
    mflat = mo.reshape(-1)[: p.shape[0] * k].reshape(p.shape[0], k)
    vflat = vo.reshape(-1)[: p.shape[0] * k].reshape(p.shape[0], k)
    return flat.copy(), mflat.copy(), vflat.copy(), o2n


class ViewTrainer(Trainer):
    """Trainer over a one-view dataset (camera + 8-bit GT) — the CPU baseline of
    the config-2 training step."""

    def __init__(self, params, deg, cam, gt_u8, cfg, extent):
        p = np.ascontiguousarray(params, np.float32)
        g = np.ascontiguousarray(gt_u8, np.uint8)
        self.deg = deg
        self.dataset = None
        f = lib().or_view_trainer_create
        f.restype = C.c_void_p
        self.h = f(ptr(p), C.c_int64(p.shape[1]), C.c_int(deg), C.byref(SkCamera.from_buffer_copy(bytes(cam))),
                   ptr(g), C.byref(cfg), C.c_float(extent))
        if not self.h:
            raise ValueError(lib().or_last_error().decode())


def view_grads(params, deg, cam, gt_hwc, lam=0.2, workers=1):
    """Parameter gradients of one view (trainer.hpp:128-147), planar [C][n]."""
    p = np.ascontiguousarray(params, np.float32)
    g = np.zeros_like(p)
    gt = np.ascontiguousarray(gt_hwc, np.float32)
    loss = C.c_double()
    check(lib().or_view_grads_f(ptr(p), C.c_int64(p.shape[1]), C.c_int(deg),
                                C.byref(SkCamera.from_buffer_copy(bytes(cam))), ptr(gt), C.c_float(lam),
                                C.c_int(workers), ptr(g), C.byref(loss)))
    return g, loss.value


def trainer_force_events(trainer: Trainer, events):
    """Follow mode: replay another run's per-event decisions (flags over the
    pre-event indices) so both runs consume the shared Rng identically."""
    for i, e in enumerate(events):
        n = int(e["n_before"])
        args = [np.ascontiguousarray(e[k][:n], np.uint8) for k in ("clone", "split", "prune")]
        check(lib().or_trainer_force_event(C.c_void_p(trainer.h), C.c_int(i), C.c_int(n), *[ptr(a) for a in args]))
