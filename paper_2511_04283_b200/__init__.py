"""splatkit_b200: B200-native (sm_100a) 3DGS training hot path.

Python host mirror of the reference's splat:: API over the C ABI in
include/splatkit_b200.h (libsplatkit_b200.so, built in-tree by build.py).
There is no CPU fallback: every compute call goes through the CUDA library,
and importing the package fails loudly if the library is missing.

Reference interface mirrored (proj/include/splatkit/):
  project_scene      camera.hpp:137     -> Context.project_scene
  build_tile_grid    raster.hpp:157     -> Context.build_tile_grid
  blend_forward      raster.hpp:194     -> Context.blend_forward
  blend_backward     raster.hpp:281     -> Context.blend_backward
  training_loss      loss.hpp:21        -> Context.training_loss
  ssim / psnr        metrics.hpp:83,126 -> Context.ssim
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsplatkit_b200.so")

SK_OK = 0
SK_ERR_INVALID_ARGUMENT = 1
SK_ERR_RUNTIME = 2
SK_ERR_CUDA = 3
SK_ERR_OUT_OF_MEMORY = 4


class SkCamera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("world_to_cam", C.c_float * 16),
                ("near_plane", C.c_float)]


class SkBinning(C.Structure):
    _fields_ = [("mode", C.c_int32), ("beta", C.c_float), ("tau_alpha", C.c_float), ("tile_size", C.c_int32)]


class SkProjected(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("visible", "mu2d", "cov2d", "conic", "depth", "color", "opacity",
                                          "tiles_touched")]


class SkBlendGrads(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("d_mu2d", "d_conic", "d_color", "d_opacity", "abs_grad")]


class SkLossValues(C.Structure):
    _fields_ = [("loss", C.c_double), ("l1", C.c_double), ("ssim", C.c_double), ("psnr", C.c_double)]


_lib = None


def lib():
    """Loads libsplatkit_b200.so. Raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run paper_2511_04283_b200.build() (no CPU fallback)")
        _lib = C.CDLL(LIB_PATH)
        _lib.sk_last_error.restype = C.c_char_p
        _lib.sk_last_error.argtypes = [C.c_void_p]
        _lib.sk_version.restype = C.c_char_p
    return _lib


def build(verbose=False, force=False):
    from . import builder as _b
    return _b.build(verbose=verbose, force=force)


def _p(a):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return C.c_void_p(a.ctypes.data)


class SplatError(RuntimeError):
    pass


def camera(width, height, fx, fy, cx, cy, world_to_cam=None, near=0.2) -> SkCamera:
    c = SkCamera()
    c.width, c.height = int(width), int(height)
    c.fx, c.fy, c.cx, c.cy = float(fx), float(fy), float(cx), float(cy)
    w = np.eye(4) if world_to_cam is None else np.asarray(world_to_cam, np.float64)
    for i, v in enumerate(w.reshape(-1)):
        c.world_to_cam[i] = float(v)
    c.near_plane = float(near)
    return c


def binning(mode="aabb", beta=1.0, tau_alpha=1.0 / 255, tile_size=16) -> SkBinning:
    b = SkBinning()
    b.mode = 1 if mode in ("compact", 1) else 0
    b.beta = float(beta)
    b.tau_alpha = float(tau_alpha)
    b.tile_size = int(tile_size)
    return b


def as_camera(cam) -> SkCamera:
    """Accepts any ctypes struct with the sk_camera layout (e.g. the oracle's)."""
    if isinstance(cam, SkCamera):
        return cam
    return SkCamera.from_buffer_copy(bytes(cam))


def as_binning(b) -> SkBinning:
    if b is None:
        return binning()
    if isinstance(b, SkBinning):
        return b
    return SkBinning.from_buffer_copy(bytes(b))


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


@dataclass
class TileLists:
    ranges: np.ndarray  # [tiles][2]
    values: np.ndarray  # [pairs] projected (== source) indices
    pairs: int


@dataclass
class Render:
    image: np.ndarray          # [H][W][3]
    transmittance: np.ndarray  # [H][W]
    contrib: np.ndarray        # [H][W]
    counts: np.ndarray | None = None


@dataclass
class BlendGrads:
    d_mu2d: np.ndarray
    d_conic: np.ndarray
    d_color: np.ndarray
    d_opacity: np.ndarray
    abs_grad: np.ndarray


class Context:
    """One CUDA device + stream (sk_ctx). Not thread-safe."""

    def __init__(self, device: int = 0):
        self._lib = lib()
        h = C.c_void_p()
        rc = self._lib.sk_ctx_create(C.c_int(device), C.byref(h))
        if rc != SK_OK:
            raise SplatError(f"sk_ctx_create failed ({rc})")
        self.h = h
        self._frame = self._new_frame()

    def close(self):
        if getattr(self, "h", None):
            if getattr(self, "_frame", None):
                self._lib.sk_frame_destroy(self._frame)
                self._frame = None
            self._lib.sk_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc):
        if rc != SK_OK:
            msg = self._lib.sk_last_error(self.h).decode()
            if rc == SK_ERR_INVALID_ARGUMENT:
                raise ValueError(msg)
            raise SplatError(msg)

    def _new_frame(self):
        f = C.c_void_p()
        self.check(self._lib.sk_frame_create(self.h, C.byref(f)))
        return f

    def synchronize(self):
        self.check(self._lib.sk_ctx_synchronize(self.h))

    def launch_count(self) -> int:
        v = C.c_int64()
        self._lib.sk_ctx_launch_count(self.h, C.byref(v))
        return v.value

    # ---- scene ----------------------------------------------------------
    def scene(self, params: np.ndarray, sh_degree: int, capacity: int | None = None) -> "Scene":
        return Scene(self, params, sh_degree, capacity)

    # ---- frame-level pipeline (reference free functions) -------------------
    def project_scene(self, scene: "Scene", cam, bin_=None, frame=None) -> Projected:
        frame = frame or self._frame
        self.check(self._lib.sk_preprocess(self.h, scene.h, C.byref(as_camera(cam)), C.byref(as_binning(bin_)),
                                           frame))
        return self.get_projected(frame)

    def preprocess(self, scene: "Scene", cam, bin_=None, frame=None):
        frame = frame or self._frame
        self.check(self._lib.sk_preprocess(self.h, scene.h, C.byref(as_camera(cam)), C.byref(as_binning(bin_)),
                                           frame))

    def set_projected(self, pg, width, height, bin_=None, frame=None):
        """pg: object with mu2d [n,2], cov2d [n,4], conic [n,4], depth, color [n,3], opacity (float32)."""
        frame = frame or self._frame
        arrs = [np.ascontiguousarray(getattr(pg, f), np.float32) for f in
                ("mu2d", "cov2d", "conic", "depth", "color", "opacity")]
        s = SkProjected()
        s.mu2d, s.cov2d, s.conic, s.depth, s.color, s.opacity = [a.ctypes.data for a in arrs]
        self.check(self._lib.sk_frame_set_projected(self.h, frame, C.byref(s), C.c_int64(arrs[0].shape[0]),
                                                    C.c_int(width), C.c_int(height), C.byref(as_binning(bin_))))

    def get_projected(self, frame=None) -> Projected:
        frame = frame or self._frame
        n = C.c_int64()
        self._lib.sk_frame_num_projected(frame, C.byref(n))
        n = n.value
        out = Projected(np.zeros(n, np.int32), np.zeros((n, 2), np.float32), np.zeros((n, 4), np.float32),
                        np.zeros((n, 4), np.float32), np.zeros(n, np.float32), np.zeros((n, 3), np.float32),
                        np.zeros(n, np.float32), np.zeros(n, np.int32))
        s = SkProjected()
        for f in ("visible", "mu2d", "cov2d", "conic", "depth", "color", "opacity", "tiles_touched"):
            setattr(s, f, getattr(out, f).ctypes.data)
        self.check(self._lib.sk_frame_get_projected(self.h, frame, C.byref(s)))
        return out

    def build_tile_grid(self, frame=None) -> int:
        frame = frame or self._frame
        pairs = C.c_int64()
        self.check(self._lib.sk_bin_sort(self.h, frame, C.byref(pairs)))
        return pairs.value

    def tile_lists(self, frame=None) -> TileLists:
        frame = frame or self._frame
        tx, ty = C.c_int(), C.c_int()
        self._lib.sk_frame_num_tiles(frame, C.byref(tx), C.byref(ty))
        ranges = np.zeros((tx.value * ty.value, 2), np.int32)
        self.check(self._lib.sk_frame_get_tile_lists(self.h, frame, _p(ranges), None))
        total = int(ranges[:, 1].max()) if ranges.size else 0
        values = np.zeros(max(total, 1), np.int32)
        self.check(self._lib.sk_frame_get_tile_lists(self.h, frame, _p(ranges), _p(values)))
        return TileLists(ranges, values[:total], total)

    def blend_forward(self, mask=None, frame=None, counts_len=None) -> Render:
        frame = frame or self._frame
        counts = None
        m = None
        if mask is not None:
            m = np.ascontiguousarray(mask, np.uint8)
            n = C.c_int64()
            self._lib.sk_frame_num_projected(frame, C.byref(n))
            counts = np.zeros(counts_len or n.value, np.int32)
        self.check(self._lib.sk_render_forward(self.h, frame, _p(m), _p(counts)))
        return self.get_render(frame, counts)

    def pge_counts(self, frame=None):
        """(visited, contributing) pixel-Gaussian evaluations of the last
        forward render, in the reference loop's terms (sk_frame_pge_counts)."""
        frame = frame or self._frame
        v, c = C.c_int64(), C.c_int64()
        self.check(self._lib.sk_frame_pge_counts(self.h, frame, C.byref(v), C.byref(c)))
        return v.value, c.value

    def get_render(self, frame=None, counts=None) -> Render:
        frame = frame or self._frame
        w, h = self._frame_dims(frame)
        img = np.zeros((h, w, 3), np.float32)
        tr = np.zeros((h, w), np.float32)
        cc = np.zeros((h, w), np.int32)
        self.check(self._lib.sk_frame_get_image(self.h, frame, _p(img)))
        self.check(self._lib.sk_frame_get_transmittance(self.h, frame, _p(tr)))
        self.check(self._lib.sk_frame_get_contrib_count(self.h, frame, _p(cc)))
        return Render(img, tr, cc, counts)

    def _frame_dims(self, frame):
        w, h = C.c_int(), C.c_int()
        self._lib.sk_frame_dims(frame, C.byref(w), C.byref(h))
        return w.value, h.value

    def training_loss(self, gt, lam=0.2, frame=None):
        frame = frame or self._frame
        v = SkLossValues()
        if gt.dtype == np.uint8:
            g = np.ascontiguousarray(gt, np.uint8)
            self.check(self._lib.sk_loss_u8(self.h, frame, _p(g), C.c_float(lam), C.byref(v)))
        else:
            g = np.ascontiguousarray(gt, np.float32)
            self.check(self._lib.sk_loss(self.h, frame, _p(g), C.c_float(lam), C.byref(v)))
        return v

    def get_dimage(self, frame=None):
        frame = frame or self._frame
        w, h = self._frame_dims(frame)
        d = np.zeros((h, w, 3), np.float32)
        self.check(self._lib.sk_frame_get_dimage(self.h, frame, _p(d)))
        return d

    def set_dimage(self, d, frame=None):
        frame = frame or self._frame
        d = np.ascontiguousarray(d, np.float32)
        self.check(self._lib.sk_frame_set_dimage(self.h, frame, _p(d)))

    def blend_backward(self, d_image=None, frame=None) -> BlendGrads:
        frame = frame or self._frame
        if d_image is not None:
            self.set_dimage(d_image, frame)
        self.check(self._lib.sk_render_backward(self.h, frame))
        n = C.c_int64()
        self._lib.sk_frame_num_projected(frame, C.byref(n))
        n = n.value
        g = BlendGrads(np.zeros((n, 2), np.float32), np.zeros((n, 4), np.float32), np.zeros((n, 3), np.float32),
                       np.zeros(n, np.float32), np.zeros((n, 2), np.float32))
        s = SkBlendGrads()
        for f in ("d_mu2d", "d_conic", "d_color", "d_opacity", "abs_grad"):
            setattr(s, f, getattr(g, f).ctypes.data)
        self.check(self._lib.sk_frame_get_blend_grads(self.h, frame, C.byref(s)))
        return g

    def ssim(self, a, b):
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        h, w = a.shape[:2]
        s, p = C.c_double(), C.c_double()
        self.check(self._lib.sk_ssim(self.h, _p(a), _p(b), C.c_int(w), C.c_int(h), C.byref(s), C.byref(p)))
        return s.value, p.value

    def fp64_render_loss(self, params, sh_degree, cam, gt=None, lam=0.2, bin_=None):
        """float64 project -> blend_forward -> training_loss on the device (the
        reference's double instantiation, for finite-difference checks).
        Returns (image [H][W][3] float64, (loss, l1, ssim) or None)."""
        p = np.ascontiguousarray(params, np.float64)
        cam = as_camera(cam)
        img = np.zeros((cam.height, cam.width, 3), np.float64)
        out = np.zeros(3, np.float64)
        g = None if gt is None else np.ascontiguousarray(gt, np.float64)
        self.check(self._lib.sk_fp64_render_loss(
            self.h, _p(p), C.c_int64(p.shape[1]), C.c_int(sh_degree), C.byref(cam), C.byref(as_binning(bin_)),
            _p(g) if g is not None else None, C.c_double(lam), _p(img), _p(out) if g is not None else None))
        return img, (tuple(float(v) for v in out) if g is not None else None)


class Scene:
    """Device-resident Scene<T> (scene.hpp:30-52), planar [C][n] parameters."""

    def __init__(self, ctx: Context, params: np.ndarray, sh_degree: int, capacity=None):
        self.ctx = ctx
        self.sh_degree = sh_degree
        p = np.ascontiguousarray(params, np.float32)
        assert p.shape[0] == n_components(sh_degree)
        h = C.c_void_p()
        ctx.check(ctx._lib.sk_scene_create(ctx.h, C.c_int(sh_degree), C.c_int64(capacity or p.shape[1]),
                                           C.byref(h)))
        self.h = h
        ctx.check(ctx._lib.sk_scene_upload(ctx.h, h, _p(p), C.c_int64(p.shape[1])))

    @classmethod
    def _wrap(cls, ctx: Context, handle, sh_degree: int) -> "Scene":
        s = cls.__new__(cls)
        s.ctx, s.sh_degree, s.h = ctx, sh_degree, handle
        return s

    @classmethod
    def from_points(cls, ctx: Context, xyz, rgb, sh_degree: int, capacity=None) -> "Scene":
        """init_from_points (scene.hpp:117-141); 3-NN distances on the GPU."""
        xyz = np.ascontiguousarray(xyz, np.float32).reshape(-1, 3)
        rgb = np.ascontiguousarray(rgb, np.float32).reshape(-1, 3)
        h = C.c_void_p()
        ctx.check(ctx._lib.sk_init_from_points(ctx.h, C.c_int64(xyz.shape[0]), _p(xyz), _p(rgb), C.c_int(sh_degree),
                                               C.c_int64(capacity or xyz.shape[0]), C.byref(h)))
        return cls._wrap(ctx, h, sh_degree)

    @classmethod
    def load_checkpoint(cls, ctx: Context, path, capacity=None) -> "Scene":
        """load_checkpoint (ply.hpp:251-315) straight into HBM."""
        h = C.c_void_p()
        ctx.check(ctx._lib.sk_checkpoint_load(ctx.h, os.fsencode(path), C.c_int64(capacity or 0), C.byref(h)))
        deg = C.c_int()
        ctx._lib.sk_scene_sh_degree(h, C.byref(deg))
        return cls._wrap(ctx, h, deg.value)

    def save_checkpoint(self, path):
        """save_checkpoint (ply.hpp:217-248)."""
        self.ctx.check(self.ctx._lib.sk_checkpoint_save(self.ctx.h, self.h, os.fsencode(path)))

    @property
    def size(self) -> int:
        n = C.c_int64()
        self.ctx._lib.sk_scene_size(self.h, C.byref(n))
        return n.value

    def download(self) -> np.ndarray:
        out = np.zeros((n_components(self.sh_degree), self.size), np.float32)
        self.ctx.check(self.ctx._lib.sk_scene_download(self.ctx.h, self.h, _p(out)))
        return out

    def close(self):
        if getattr(self, "h", None):
            self.ctx._lib.sk_scene_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# optimizer, score table, density control, trainer
# ---------------------------------------------------------------------------

class SkLearningRates(C.Structure):
    _fields_ = [(n, C.c_float) for n in ("position", "position_final", "sh_dc", "sh_rest", "opacity", "scale",
                                         "rotation")]


class SkScoreTable(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("s_d", "s_p_raw", "s_p", "grad_norm_acc", "abs_grad_acc", "grad3d_acc",
                                          "views_seen", "max_radius2d")]


class SkTrainConfig(C.Structure):
    """TrainConfig (config.hpp:20-61); same layout as the oracle's or_train_config."""
    _fields_ = [("iterations", C.c_int32), ("k", C.c_int32), ("lambda_", C.c_double), ("tau", C.c_double),
                ("tau_d", C.c_double), ("tau_p", C.c_double), ("beta", C.c_double), ("tau_alpha", C.c_double),
                ("densify_from", C.c_int32), ("densify_until", C.c_int32), ("densify_every", C.c_int32),
                ("prune_every_early", C.c_int32), ("prune_every_late", C.c_int32),
                ("grad_threshold", C.c_double), ("percent_dense", C.c_double),
                ("lr_position", C.c_double), ("lr_position_final", C.c_double), ("lr_sh_dc", C.c_double),
                ("lr_sh_rest", C.c_double), ("lr_opacity", C.c_double), ("lr_scale", C.c_double),
                ("lr_rotation", C.c_double), ("opacity_reset_every", C.c_int32), ("lazy_opt_enabled", C.c_int32),
                ("lazy_opt_interval_15k", C.c_int32), ("lazy_opt_interval_20k", C.c_int32), ("seed", C.c_uint64),
                ("tile_size", C.c_int32), ("workers", C.c_int32), ("sh_degree", C.c_int32), ("compact", C.c_int32),
                ("vcd", C.c_int32), ("vcp", C.c_int32), ("prune_min_opacity", C.c_double),
                ("prune_opacity_late", C.c_double), ("prune_world_size_frac", C.c_double),
                ("prune_screen_size", C.c_double), ("size_prune_from", C.c_int32), ("schedule_dry_run", C.c_int32)]


class SkPruneParams(C.Structure):
    _fields_ = [("tau_p", C.c_float), ("min_opacity", C.c_float), ("opacity_late", C.c_float),
                ("world_size_frac", C.c_float), ("screen_size", C.c_float), ("size_prune_from", C.c_int32),
                ("densify_until", C.c_int32), ("use_vcp", C.c_int32)]


class SkLogRow(C.Structure):
    _fields_ = [("iteration", C.c_int32), ("gaussians", C.c_int32), ("tile_pairs", C.c_int64), ("loss", C.c_double),
                ("psnr", C.c_double), ("elapsed_ms", C.c_double), ("view", C.c_int32), ("event", C.c_int32)]


def default_config() -> SkTrainConfig:
    c = SkTrainConfig()
    lib().sk_default_config(C.byref(c))
    return c


def load_config_file(path, cfg: SkTrainConfig | None = None) -> SkTrainConfig:
    """load_config_file (config.hpp:167-196) onto cfg (default: defaults)."""
    cfg = cfg if cfg is not None else default_config()
    rc = lib().sk_config_load_file(None, C.byref(cfg), os.fsencode(path))
    _io_check(rc, f"config file {path}")
    return cfg


def set_config_value(cfg: SkTrainConfig, key: str, value: str):
    """set_config_value (config.hpp:139-163)."""
    rc = lib().sk_config_set(None, C.byref(cfg), key.encode(), str(value).encode())
    _io_check(rc, f"config: key '{key}' = '{value}'")


def validate_config(cfg: SkTrainConfig):
    """TrainConfig::validate (config.hpp:63-80)."""
    _io_check(lib().sk_validate_config(None, C.byref(cfg)), "config: invalid")


def as_config(cfg) -> SkTrainConfig:
    if isinstance(cfg, SkTrainConfig):
        return cfg
    return SkTrainConfig.from_buffer_copy(bytes(cfg))


def default_learning_rates() -> SkLearningRates:
    l = SkLearningRates()
    lib().sk_default_learning_rates(C.byref(l))
    return l


def default_prune_params() -> SkPruneParams:
    p = SkPruneParams()
    lib().sk_default_prune_params(C.byref(p))
    return p


def expon_lr(lr_init, lr_final, step, max_steps) -> float:
    f = lib().sk_expon_lr
    f.restype = C.c_float
    f.argtypes = [C.c_float, C.c_float, C.c_int, C.c_int]
    return f(lr_init, lr_final, step, max_steps)


@dataclass
class ScoreTable:
    s_d: np.ndarray
    s_p_raw: np.ndarray
    s_p: np.ndarray
    grad_norm_acc: np.ndarray
    abs_grad_acc: np.ndarray
    grad3d_acc: np.ndarray
    views_seen: np.ndarray
    max_radius2d: np.ndarray


def _score_struct(t: ScoreTable) -> SkScoreTable:
    s = SkScoreTable()
    for f in ("s_d", "s_p_raw", "s_p", "grad_norm_acc", "abs_grad_acc", "grad3d_acc", "views_seen", "max_radius2d"):
        a = getattr(t, f)
        setattr(s, f, a.ctypes.data if a is not None else None)
    return s


def _scene_methods():
    def score_table(self) -> ScoreTable:
        n = self.size
        t = ScoreTable(np.zeros(n, np.float32), np.zeros(n, np.float32), np.zeros(n, np.float32),
                       np.zeros(n, np.float32), np.zeros(n, np.float32), np.zeros((n, 3), np.float32),
                       np.zeros(n, np.int32), np.zeros(n, np.float32))
        self.ctx.check(self.ctx._lib.sk_scene_get_score_table(self.ctx.h, self.h, C.byref(_score_struct(t))))
        return t

    def set_score_table(self, **fields):
        n = self.size
        full = {}
        for f, dt, shape in (("s_d", np.float32, (n,)), ("s_p_raw", np.float32, (n,)), ("s_p", np.float32, (n,)),
                             ("grad_norm_acc", np.float32, (n,)), ("abs_grad_acc", np.float32, (n,)),
                             ("grad3d_acc", np.float32, (n, 3)), ("views_seen", np.int32, (n,)),
                             ("max_radius2d", np.float32, (n,))):
            v = fields.get(f)
            full[f] = None if v is None else np.ascontiguousarray(np.broadcast_to(v, shape), dt)
        t = ScoreTable(**full)
        self.ctx.check(self.ctx._lib.sk_scene_set_score_table(self.ctx.h, self.h, C.byref(_score_struct(t))))

    def reset_score_table(self):
        self.ctx.check(self.ctx._lib.sk_scene_reset_score_table(self.ctx.h, self.h))

    def set_grads(self, g):
        g = np.ascontiguousarray(g, np.float32)
        self.ctx.check(self.ctx._lib.sk_scene_set_grads(self.ctx.h, self.h, _p(g)))

    def adam_state(self):
        n = self.size
        m = np.zeros((n_components(self.sh_degree), n), np.float32)
        v = np.zeros_like(m)
        t = np.zeros(6, np.int64)
        self.ctx.check(self.ctx._lib.sk_scene_get_adam(self.ctx.h, self.h, _p(m), _p(v), _p(t)))
        return m, v, t

    Scene.score_table = score_table
    Scene.set_score_table = set_score_table
    Scene.reset_score_table = reset_score_table
    Scene.set_grads = set_grads
    Scene.adam_state = adam_state


_scene_methods()


def _ctx_methods():
    def project_backward(self, scene, stats=True, frame=None):
        frame = frame or self._frame
        g = np.zeros((n_components(scene.sh_degree), scene.size), np.float32)
        self.check(self._lib.sk_project_backward(self.h, scene.h, frame, C.c_int(int(stats)), _p(g)))
        return g

    def adam_step(self, scene, lrs=None, position_lr=None, update_sh_rest=True):
        lrs = lrs or default_learning_rates()
        plr = lrs.position if position_lr is None else position_lr
        self.check(self._lib.sk_adam_step(self.h, scene.h, C.byref(lrs), C.c_float(plr), C.c_int(int(update_sh_rest))))

    def project_backward_adam(self, scene, lrs=None, position_lr=None, update_sh_rest=True, stats=True, frame=None):
        frame = frame or self._frame
        lrs = lrs or default_learning_rates()
        plr = lrs.position if position_lr is None else position_lr
        self.check(self._lib.sk_project_backward_adam(self.h, scene.h, frame, C.byref(lrs), C.c_float(plr),
                                                      C.c_int(int(update_sh_rest)), C.c_int(int(stats))))

    def accumulate_scores(self, scene, cams, images, tau=0.5, lam=0.2, bin_=None):
        k = len(cams)
        arr = (SkCamera * k)(*[as_camera(c) for c in cams])
        imgs = np.ascontiguousarray(np.concatenate([np.asarray(i, np.float32).reshape(-1) for i in images]))
        counts = np.zeros((k, scene.size), np.int32)
        photo = np.zeros(k, np.float32)
        self.check(self._lib.sk_accumulate_scores(self.h, scene.h, C.c_int(k), arr, _p(imgs), C.c_float(tau),
                                                  C.c_float(lam), C.byref(as_binning(bin_)), _p(counts), _p(photo)))
        return counts, photo

    def select_densify(self, scene, tau_d=5.0, grad_threshold=2e-4, percent_dense=0.01, use_vcd=True, extent=1.0):
        n = scene.size
        clone = np.zeros(n, np.uint8)
        split = np.zeros(n, np.uint8)
        self.check(self._lib.sk_select_densify(self.h, scene.h, C.c_float(tau_d), C.c_float(grad_threshold),
                                               C.c_float(percent_dense), C.c_int(int(use_vcd)), C.c_float(extent),
                                               _p(clone), _p(split)))
        return clone, split

    def select_prune(self, scene, iteration, params=None, extent=1.0, **kw):
        p = params or default_prune_params()
        for k, v in kw.items():
            setattr(p, k, v)
        prune = np.zeros(scene.size, np.uint8)
        self.check(self._lib.sk_select_prune(self.h, scene.h, C.c_int(iteration), C.byref(p), C.c_float(extent),
                                             _p(prune)))
        return prune

    def apply_prune_densify(self, scene, prune=None, clone=None, split=None, clone_step_lr=0.0, eps=None):
        n = scene.size
        arrs = [None if a is None else np.ascontiguousarray(a, np.uint8) for a in (prune, clone, split)]
        e = None if eps is None else np.ascontiguousarray(eps, np.float32)
        o2n = np.zeros(n, np.int32)
        new = C.c_int64()
        self.check(self._lib.sk_apply_prune_densify(self.h, scene.h, *[_p(a) for a in arrs], C.c_float(clone_step_lr),
                                                    _p(e), _p(o2n), C.byref(new)))
        return o2n, new.value

    Context.project_backward = project_backward
    Context.adam_step = adam_step
    Context.project_backward_adam = project_backward_adam
    Context.accumulate_scores = accumulate_scores
    Context.select_densify = select_densify
    Context.select_prune = select_prune
    Context.apply_prune_densify = apply_prune_densify


_ctx_methods()


class SkSynthSpec(C.Structure):
    _fields_ = [("n_gaussians", C.c_int32), ("n_views", C.c_int32), ("width", C.c_int32), ("height", C.c_int32),
                ("seed", C.c_uint64), ("scale_mult", C.c_double), ("focal", C.c_double)]


class Dataset:
    """Dataset<T> (dataset.hpp:24-32) resident in HBM (8-bit GT images)."""

    @classmethod
    def synthetic(cls, ctx: Context, n_gaussians=500, n_views=64, width=128, height=None, seed=1, scale_mult=1.0,
                  focal=-1.0):
        """generate_synthetic (dataset.hpp:178-250) with the GT views rendered
        on the GPU. Returns (dataset, gt_scene (SH degree 1), init_xyz,
        init_rgb)."""
        height = width if height is None else height
        spec = SkSynthSpec(n_gaussians, n_views, width, height, seed, scale_mult, focal)
        xyz = np.zeros((n_gaussians, 3), np.float32)
        rgb = np.zeros((n_gaussians, 3), np.float32)
        ext = C.c_float()
        g, d = C.c_void_p(), C.c_void_p()
        ctx.check(ctx._lib.sk_synthetic_create(ctx.h, C.byref(spec), C.byref(g), C.byref(d), _p(xyz), _p(rgb),
                                               C.byref(ext)))
        ds = cls.__new__(cls)
        ds.ctx, ds.h = ctx, d
        return ds, Scene._wrap(ctx, g, 1), xyz, rgb

    @classmethod
    def load(cls, ctx: Context, directory: str) -> "Dataset":
        """load_dataset (dataset.hpp:73-125): cameras.json + images/%05d.png +
        points3d.ply into HBM."""
        d = C.c_void_p()
        ctx.check(ctx._lib.sk_dataset_load(ctx.h, os.fsencode(directory), C.byref(d)))
        ds = cls.__new__(cls)
        ds.ctx, ds.h = ctx, d
        return ds

    def save(self, directory: str):
        """The files generate_synthetic writes (dataset.hpp:221-247)."""
        self.ctx.check(self.ctx._lib.sk_dataset_save(self.ctx.h, self.h, os.fsencode(directory)))

    def init_points(self):
        n = C.c_int64()
        self.ctx._lib.sk_dataset_init_points(self.h, None, None, C.byref(n))
        xyz = np.zeros((n.value, 3), np.float32)
        rgb = np.zeros((n.value, 3), np.float32)
        if n.value:
            self.ctx.check(self.ctx._lib.sk_dataset_init_points(self.h, _p(xyz), _p(rgb), C.byref(n)))
        return xyz, rgb

    @property
    def num_views(self) -> int:
        n = C.c_int()
        self.ctx._lib.sk_dataset_num_views(self.h, C.byref(n))
        return n.value

    @property
    def extent(self) -> float:
        e = C.c_float()
        self.ctx._lib.sk_dataset_extent(self.h, C.byref(e))
        return e.value

    def camera(self, v) -> "SkCamera":
        c = SkCamera()
        self.ctx.check(self.ctx._lib.sk_dataset_camera(self.h, C.c_int(v), C.byref(c)))
        return c

    def image_u8(self, v) -> np.ndarray:
        c = self.camera(v)
        out = np.zeros((c.height, c.width, 3), np.uint8)
        self.ctx.check(self.ctx._lib.sk_dataset_image_u8(self.ctx.h, self.h, C.c_int(v), _p(out)))
        return out

    def set_train_indices(self, idx):
        idx = np.ascontiguousarray(idx, np.int32)
        rc = self.ctx._lib.sk_dataset_set_train_indices(self.h, _p(idx), C.c_int(len(idx)))
        if rc != SK_OK:
            raise ValueError("dataset: train index out of range")

    def train_indices(self) -> np.ndarray:
        cnt = C.c_int()
        self.ctx._lib.sk_dataset_train_indices(self.h, None, C.byref(cnt))
        out = np.zeros(cnt.value, np.int32)
        self.ctx._lib.sk_dataset_train_indices(self.h, _p(out), C.byref(cnt))
        return out

    def __init__(self, ctx: Context, cams, images_u8, train_indices=None, extent=1.0):
        self.ctx = ctx
        k = len(cams)
        arr = (SkCamera * k)(*[as_camera(c) for c in cams])
        imgs = np.ascontiguousarray(np.concatenate([np.asarray(i, np.uint8).reshape(-1) for i in images_u8]))
        tr = None if train_indices is None else np.ascontiguousarray(train_indices, np.int32)
        h = C.c_void_p()
        ctx.check(ctx._lib.sk_dataset_create(ctx.h, C.c_int(k), arr, _p(imgs), _p(tr),
                                             C.c_int(0 if tr is None else len(tr)), C.c_float(extent), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.ctx._lib.sk_dataset_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Trainer:
    """Trainer (trainer.hpp:70-261) on the GPU; borrows scene and dataset."""

    def __init__(self, ctx: Context, scene: Scene, data: Dataset, cfg, record_events=False):
        self.ctx, self.scene, self.data = ctx, scene, data
        self.cfg = as_config(cfg)
        h = C.c_void_p()
        ctx.check(ctx._lib.sk_trainer_create(ctx.h, scene.h, data.h, C.byref(self.cfg), C.byref(h)))
        self.h = h
        if record_events:
            ctx._lib.sk_trainer_record_events(h, C.c_int(1))

    def set_iteration(self, it):
        self.ctx.check(self.ctx._lib.sk_trainer_set_iteration(self.h, C.c_int(it)))

    def density_event(self, iteration, densify=True, prune=True):
        """Trainer::density_event (trainer.hpp:177-243) outside the schedule."""
        self.ctx.check(self.ctx._lib.sk_trainer_density_event(self.h, C.c_int(iteration), C.c_int(int(densify)),
                                                              C.c_int(int(prune))))

    def run(self, iterations):
        rows = (SkLogRow * max(1, iterations))()
        self.ctx.check(self.ctx._lib.sk_trainer_run(self.h, C.c_int(iterations), rows))
        return [dict(iteration=r.iteration, gaussians=r.gaussians, tile_pairs=r.tile_pairs, loss=r.loss,
                     psnr=r.psnr, elapsed_ms=r.elapsed_ms, view=r.view, event=r.event) for r in rows[:iterations]]

    def events(self):
        n = C.c_int()
        self.ctx._lib.sk_trainer_num_events(self.h, C.byref(n))
        out = []
        for e in range(n.value):
            hdr = np.zeros(7, np.int32)
            self.ctx._lib.sk_trainer_event(self.h, C.c_int(e), _p(hdr), None, None, None, None, None)
            nb, k = int(hdr[1]), int(hdr[6])
            clone, split, prune = (np.zeros(max(nb, 1), np.uint8) for _ in range(3))
            sampled = np.zeros(max(k, 1), np.int32)
            photo = np.zeros(max(k, 1), np.float32)
            self.ctx._lib.sk_trainer_event(self.h, C.c_int(e), _p(hdr), _p(clone), _p(split), _p(prune),
                                           _p(sampled), _p(photo))
            out.append(dict(iteration=int(hdr[0]), n_before=nb, n_after=int(hdr[2]), n_clone=int(hdr[3]),
                            n_split=int(hdr[4]), n_prune=int(hdr[5]), clone=clone[:nb], split=split[:nb],
                            prune=prune[:nb], sampled=sampled[:k], photometric=photo[:k]))
        return out

    def close(self):
        if getattr(self, "h", None):
            self.ctx._lib.sk_trainer_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- on-disk formats; host-only, no GPU needed ----------

def _io_check(rc, what):
    if rc != SK_OK:
        raise (ValueError if rc == SK_ERR_INVALID_ARGUMENT else SplatError)(f"{what} failed (status {rc})")


def _io_call(ctx, fn, *args, what=""):
    """Runs a file-format entry point; with a Context the library's message is
    raised, without one the status."""
    rc = fn(ctx.h if ctx is not None else None, *args)
    if ctx is not None:
        ctx.check(rc)
    else:
        _io_check(rc, what)


def read_points_ply(path, ctx: Context | None = None):
    """read_points_ply (ply.hpp:179-196) -> (xyz [n,3], rgb [n,3]) float32."""
    L = lib()
    n = C.c_int64()
    _io_call(ctx, L.sk_points_read, os.fsencode(path), None, None, C.byref(n), what=f"ply read {path}")
    xyz = np.zeros((n.value, 3), np.float32)
    rgb = np.zeros((n.value, 3), np.float32)
    _io_call(ctx, L.sk_points_read, os.fsencode(path), _p(xyz), _p(rgb), C.byref(n), what=f"ply read {path}")
    return xyz, rgb


def write_points_ply(path, xyz, rgb, ctx: Context | None = None):
    xyz = np.ascontiguousarray(xyz, np.float32)
    rgb = np.ascontiguousarray(rgb, np.float32)
    _io_call(ctx, lib().sk_points_write, os.fsencode(path), _p(xyz), _p(rgb), C.c_int64(xyz.shape[0]),
             what=f"ply write {path}")


def read_png(path, ctx: Context | None = None) -> np.ndarray:
    """read_png (png_io.cpp:25-72) as uint8 [H][W][3]; the reference's float
    image is this / 255.0f."""
    L = lib()
    w, h = C.c_int(), C.c_int()
    _io_call(ctx, L.sk_png_read, os.fsencode(path), None, C.byref(w), C.byref(h), what=f"png read {path}")
    img = np.zeros((h.value, w.value, 3), np.uint8)
    _io_call(ctx, L.sk_png_read, os.fsencode(path), _p(img), C.byref(w), C.byref(h), what=f"png read {path}")
    return img


def write_png(path, image, ctx: Context | None = None):
    """write_png (png_io.cpp:74-104): float [H][W][3] quantised with
    lround(clamp(v)·255), or uint8 written as is."""
    L = lib()
    if image.dtype == np.uint8:
        img = np.ascontiguousarray(image)
        fn = L.sk_png_write_u8
    else:
        img = np.ascontiguousarray(image, np.float32)
        fn = L.sk_png_write
    _io_call(ctx, fn, os.fsencode(path), _p(img), C.c_int(img.shape[1]), C.c_int(img.shape[0]),
             what=f"png write {path}")


def read_cameras_json(path, ctx: Context | None = None):
    """cameras.json records (dataset.hpp:80-100) -> (list of SkCamera, ids)."""
    L = lib()
    n = C.c_int()
    _io_call(ctx, L.sk_cameras_read, os.fsencode(path), None, None, C.byref(n), what=f"cameras read {path}")
    cams = (SkCamera * max(1, n.value))()
    ids = np.zeros(max(1, n.value), np.int32)
    _io_call(ctx, L.sk_cameras_read, os.fsencode(path), cams, _p(ids), C.byref(n), what=f"cameras read {path}")
    return [cams[i] for i in range(n.value)], ids[: n.value]


def write_cameras_json(path, cams, ids=None, ctx: Context | None = None):
    """save_cameras_json (dataset.hpp:127-150)."""
    arr = (SkCamera * max(1, len(cams)))(*[as_camera(c) for c in cams])
    ids = np.ascontiguousarray(np.arange(len(cams)) if ids is None else ids, np.int32)
    _io_call(ctx, lib().sk_cameras_write, os.fsencode(path), arr, _p(ids), C.c_int(len(cams)),
             what=f"cameras write {path}")


def train_step_host(ctx: Context, scene: Scene, cam, gt_u8, cfg, extent, iteration, frame=None) -> dict:
    """One train_iteration with the GT in host memory (the end-to-end entry point)."""
    frame = frame or ctx._frame
    g = np.ascontiguousarray(gt_u8, np.uint8)
    row = SkLogRow()
    ctx.check(ctx._lib.sk_train_step_host(ctx.h, scene.h, frame, C.byref(as_camera(cam)), _p(g),
                                          C.byref(as_config(cfg)), C.c_float(extent), C.c_int(iteration),
                                          C.byref(row)))
    return dict(loss=row.loss, psnr=row.psnr, tile_pairs=row.tile_pairs, gaussians=row.gaussians)


class HostStepPipeline:
    """Pipelined end-to-end steps (sk_train_step_host_async): the GT upload of
    each step overlaps the previous step on a copy stream and each step's
    loss is read back when the next step is issued (or at flush()). Rows are
    kept alive here until they are filled."""

    def __init__(self, ctx: Context, frame=None, comm=None):
        self.ctx = ctx
        self.frame = frame or ctx._frame
        self.comm = comm
        self.rows = []

    def step(self, scene: Scene, cam, gt_u8_pinned: np.ndarray, cfg, extent, iteration):
        row = SkLogRow()
        self.rows.append(row)
        self.ctx.check(self.ctx._lib.sk_train_step_host_async(
            self.ctx.h, scene.h, self.frame, C.byref(as_camera(cam)), _p(gt_u8_pinned), C.byref(as_config(cfg)),
            C.c_float(extent), C.c_int(iteration), C.byref(row), self.comm.h if self.comm is not None else None))

    def flush(self):
        self.ctx.check(self.ctx._lib.sk_train_step_host_flush(self.ctx.h, self.frame))
        out = [dict(iteration=r.iteration, loss=r.loss, psnr=r.psnr, tile_pairs=r.tile_pairs) for r in self.rows]
        self.rows = []
        return out


# ---------------------------------------------------------------------------
# multi-GPU: NCCL communicator (view sharding)
# ---------------------------------------------------------------------------

COMM_ID_BYTES = 128


def comm_unique_id() -> bytes:
    buf = (C.c_uint8 * COMM_ID_BYTES)()
    rc = lib().sk_comm_unique_id(buf)
    if rc != SK_OK:
        raise SplatError("sk_comm_unique_id failed")
    return bytes(buf)


def share_comm_id(dist, rank: int) -> bytes:
    """Rank 0 draws the NCCL id; every rank receives it over torch.distributed
    (works with the gloo and nccl backends)."""
    obj = [comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


class Comm:
    """sk_comm: one rank of the NCCL communicator used by the trainer."""

    def __init__(self, ctx: Context, uid: bytes, world: int, rank: int):
        self.ctx = ctx
        buf = (C.c_uint8 * COMM_ID_BYTES).from_buffer_copy(uid)
        h = C.c_void_p()
        ctx.check(ctx._lib.sk_comm_create(ctx.h, buf, C.c_int(world), C.c_int(rank), C.byref(h)))
        self.h = h
        self.rank, self.world = rank, world

    @classmethod
    def from_torch(cls, ctx: Context, dist, rank: int, world: int) -> "Comm":
        return cls(ctx, share_comm_id(dist, rank), world, rank)

    def close(self):
        if getattr(self, "h", None):
            self.ctx._lib.sk_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_AR = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int)
_RS = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int)
_AG = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int)


class SkCommHostOps(C.Structure):
    _fields_ = [("user", C.c_void_p), ("all_reduce", _AR), ("reduce_scatter", _RS), ("all_gather", _AG)]


class HostComm(Comm):
    """sk_comm over torch.distributed collectives on host memory
    (sk_comm_create_host): the library's own C1 / C2 / C3 code with any
    torch.distributed backend (gloo on CPU; several ranks may share one GPU,
    which NCCL refuses)."""

    def __init__(self, ctx: Context, dist, rank: int, world: int):
        import torch
        self.ctx = ctx
        self.rank, self.world = rank, world

        def view(ptr, count, dtype):
            ct = C.c_float if dtype == 0 else C.c_int32
            return torch.from_numpy(np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ct)), shape=(count,)))

        def op_of(op):
            return dist.ReduceOp.SUM if op == 0 else dist.ReduceOp.MAX

        def all_reduce(_, buf, count, dtype, op):
            try:
                dist.all_reduce(view(buf, count, dtype), op=op_of(op))
                return 0
            except Exception:
                return 1

        def reduce_scatter(_, send, recv, count, dtype, op):
            try:
                t = view(send, count * world, dtype)
                dist.all_reduce(t, op=op_of(op))  # gloo has no reduce_scatter
                view(recv, count, dtype).copy_(t[rank * count:(rank + 1) * count])
                return 0
            except Exception:
                return 1

        def all_gather(_, send, recv, count, dtype):
            try:
                out = view(recv, count * world, dtype)
                dist.all_gather(list(out.split(count)), view(send, count, dtype).clone())
                return 0
            except Exception:
                return 1

        self._ops = SkCommHostOps(None, _AR(all_reduce), _RS(reduce_scatter), _AG(all_gather))
        h = C.c_void_p()
        ctx.check(ctx._lib.sk_comm_create_host(ctx.h, C.c_int(world), C.c_int(rank), C.byref(self._ops),
                                               C.byref(h)))
        self.h = h


def shard_assign(n_items: int, world: int, rank: int) -> list:
    """Round-robin ownership of the K scored views (C3 sharding)."""
    out = (C.c_int32 * max(1, n_items))()
    n = C.c_int()
    rc = lib().sk_shard_assign(C.c_int(n_items), C.c_int(world), C.c_int(rank), out, C.byref(n))
    if rc != SK_OK:
        raise ValueError("sk_shard_assign: bad arguments")
    return list(out[: n.value])


def _trainer_set_comm(self, comm: Comm):
    self.comm = comm
    self.ctx.check(self.ctx._lib.sk_trainer_set_comm(self.h, comm.h))


Trainer.set_comm = _trainer_set_comm
