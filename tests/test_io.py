"""On-disk formats — the host-side file functions of the C
ABI, which need no GPU: points PLY, PNG and cameras.json. Ports the
reference's tests/test_dataset.cpp cases for these formats; checkpoint and
dataset-directory round trips (device scenes / images) are in
tests/test_gpu_io.py."""
import json
import struct
import zlib

import numpy as np
import pytest

import paper_2511_04283_b200 as sk


@pytest.fixture(scope="module", autouse=True)
def _lib():
    sk.build()


def test_points_ply_round_trip(tmp_path):
    """test_dataset.cpp:64-84: positions exact, colours within 0.5/255."""
    rng = np.random.default_rng(101)
    xyz = rng.uniform(-2, 2, (100, 3)).astype(np.float32)
    rgb = rng.uniform(0, 1, (100, 3)).astype(np.float32)
    path = tmp_path / "points3d.ply"
    sk.write_points_ply(path, xyz, rgb)
    bx, brgb = sk.read_points_ply(path)
    assert np.array_equal(bx, xyz)
    assert np.abs(brgb - rgb).max() <= 0.5 / 255 + 1e-6
    # the body is 15 bytes per point after the reference's header
    data = path.read_bytes()
    head, body = data.split(b"end_header\n", 1)
    assert b"element vertex 100" in head and len(body) == 15 * 100
    assert np.array_equal(np.frombuffer(body, np.uint8).reshape(100, 15)[:, 12:],
                          np.round(np.clip(rgb.astype(np.float64), 0, 1) * 255).astype(np.uint8))


def test_ascii_ply_with_extra_properties(tmp_path):
    """test_dataset.cpp:86-107."""
    path = tmp_path / "pts.ply"
    path.write_text("ply\nformat ascii 1.0\ncomment hand-written\nelement vertex 2\n"
                    "property float x\nproperty float y\nproperty float z\nproperty float nx\n"
                    "property uchar red\nproperty uchar green\nproperty uchar blue\nend_header\n"
                    "0.5 1.5 -2 0 255 0 128\n1 2 3 0 0 255 64\n")
    xyz, rgb = sk.read_points_ply(path)
    assert xyz.tolist() == [[0.5, 1.5, -2.0], [1.0, 2.0, 3.0]]
    assert rgb[0, 0] == pytest.approx(1.0)
    assert rgb[0, 2] == pytest.approx(128.0 / 255)
    assert rgb[1, 1] == pytest.approx(1.0)


def test_ply_float_colours_and_errors(tmp_path):
    path = tmp_path / "f.ply"
    body = struct.pack("<6f", 1, 2, 3, 0.25, 0.5, 0.75)
    path.write_bytes(b"ply\nformat binary_little_endian 1.0\nelement vertex 1\n"
                     b"property float x\nproperty float y\nproperty float z\n"
                     b"property float red\nproperty float green\nproperty float blue\nend_header\n" + body)
    xyz, rgb = sk.read_points_ply(path)
    assert rgb.tolist() == [[0.25, 0.5, 0.75]]  # float colours are not rescaled
    bad = tmp_path / "bad.ply"
    bad.write_bytes(b"PLY\n")
    with pytest.raises(sk.SplatError):
        sk.read_points_ply(bad)
    trunc = tmp_path / "trunc.ply"
    trunc.write_bytes(b"ply\nformat binary_little_endian 1.0\nelement vertex 2\n"
                      b"property float x\nproperty float y\nproperty float z\n"
                      b"property uchar red\nproperty uchar green\nproperty uchar blue\nend_header\n" + b"\0" * 20)
    with pytest.raises(sk.SplatError):
        sk.read_points_ply(trunc)


def test_png_round_trip_exact_at_8_bit(tmp_path):
    """test_dataset.cpp:182-197, plus the exact quantisation of png_io.cpp:97-98."""
    rng = np.random.default_rng(105)
    img = rng.uniform(0, 1, (14, 20, 3)).astype(np.float32)
    img[0, 0] = [-0.5, 1.5, 0.5 / 255]  # clamp and round-half-away
    path = tmp_path / "img.png"
    sk.write_png(path, img)
    back = sk.read_png(path)
    assert back.shape == (14, 20, 3)
    expect = np.array([[int(np.floor(min(max(float(v), 0.0), 1.0) * np.float32(255) + 0.5)) for v in px]
                       for px in img.reshape(-1, 3)], np.uint8).reshape(back.shape)
    assert np.array_equal(back, expect)
    assert np.abs(back / np.float32(255) - img.clip(0, 1)).max() <= 0.5 / 255 + 1e-6


def _png(width, height, ctype, depth, rows, filters, palette=None):
    """Minimal PNG encoder with explicit per-row filter types (0-4)."""
    ch = {0: 1, 2: 3, 3: 1, 4: 2, 6: 4}[ctype]
    bpp = max(1, ch * depth // 8)
    raw = bytearray()
    prev = bytes(len(rows[0]))
    for y, row in enumerate(rows):
        ft = filters[y % len(filters)]
        out = bytearray()
        for i, x in enumerate(row):
            a = row[i - bpp] if i >= bpp else 0
            b = prev[i]
            c = prev[i - bpp] if i >= bpp else 0
            if ft == 0:
                p = 0
            elif ft == 1:
                p = a
            elif ft == 2:
                p = b
            elif ft == 3:
                p = (a + b) // 2
            else:
                pa, pb, pc = abs(b - c), abs(a - c), abs(a + b - 2 * c)
                p = a if pa <= pb and pa <= pc else (b if pb <= pc else c)
            out.append((x - p) & 255)
        raw += bytes([ft]) + out
        prev = bytes(row)

    def chunk(t, d):
        return struct.pack(">I", len(d)) + t + d + struct.pack(">I", zlib.crc32(t + d) & 0xffffffff)

    data = b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", width, height, depth, ctype, 0, 0, 0))
    if palette is not None:
        data += chunk(b"PLTE", bytes(palette))
    return data + chunk(b"IDAT", zlib.compress(bytes(raw))) + chunk(b"IEND", b"")


@pytest.mark.parametrize("filters", [[0], [1], [2], [3], [4], [0, 1, 2, 3, 4]])
def test_png_decoder_filters_rgb8(tmp_path, filters):
    rng = np.random.default_rng(7 + len(filters) + filters[0])
    img = rng.integers(0, 256, (9, 13, 3), dtype=np.uint8)
    path = tmp_path / "f.png"
    path.write_bytes(_png(13, 9, 2, 8, [img[y].tobytes() for y in range(9)], filters))
    assert np.array_equal(sk.read_png(path), img)


def test_png_decoder_colour_types(tmp_path):
    """The reference's libpng transforms (png_io.cpp:43-51): strip 16-bit to
    the high byte, expand low-depth gray, palette to RGB, gray to RGB, strip
    alpha."""
    rng = np.random.default_rng(11)
    w, h = 11, 7
    # 16-bit RGBA
    v = rng.integers(0, 65536, (h, w, 4), dtype=np.uint16)
    p = tmp_path / "rgba16.png"
    p.write_bytes(_png(w, h, 6, 16, [v[y].astype(">u2").tobytes() for y in range(h)], [4, 1]))
    assert np.array_equal(sk.read_png(p), (v[..., :3] >> 8).astype(np.uint8))
    # 8-bit gray + alpha
    g = rng.integers(0, 256, (h, w, 2), dtype=np.uint8)
    p = tmp_path / "la.png"
    p.write_bytes(_png(w, h, 4, 8, [g[y].tobytes() for y in range(h)], [3]))
    assert np.array_equal(sk.read_png(p), np.repeat(g[..., :1], 3, axis=2))
    # 2-bit gray (expanded x85)
    q = rng.integers(0, 4, (h, w), dtype=np.uint8)
    rows = []
    for y in range(h):
        bits = "".join(format(int(x), "02b") for x in q[y]).ljust(((2 * w + 7) // 8) * 8, "0")
        rows.append(bytes(int(bits[i:i + 8], 2) for i in range(0, len(bits), 8)))
    p = tmp_path / "g2.png"
    p.write_bytes(_png(w, h, 0, 2, rows, [0, 2]))
    assert np.array_equal(sk.read_png(p), np.repeat((q * 85)[..., None], 3, axis=2))
    # 4-bit palette
    pal = rng.integers(0, 256, (16, 3), dtype=np.uint8)
    idx = rng.integers(0, 16, (h, w), dtype=np.uint8)
    rows = []
    for y in range(h):
        bits = "".join(format(int(x), "04b") for x in idx[y]).ljust(((4 * w + 7) // 8) * 8, "0")
        rows.append(bytes(int(bits[i:i + 8], 2) for i in range(0, len(bits), 8)))
    p = tmp_path / "p4.png"
    p.write_bytes(_png(w, h, 3, 4, rows, [1], palette=pal.reshape(-1).tolist()))
    assert np.array_equal(sk.read_png(p), pal[idx])


def test_png_decodes_pil_output(tmp_path):
    PIL = pytest.importorskip("PIL.Image")
    rng = np.random.default_rng(3)
    img = rng.integers(0, 256, (31, 17, 3), dtype=np.uint8)
    p = tmp_path / "pil.png"
    PIL.fromarray(img).save(p, optimize=True)
    assert np.array_equal(sk.read_png(p), img)
    ours = tmp_path / "ours.png"
    sk.write_png(ours, img)
    assert np.array_equal(np.asarray(PIL.open(ours).convert("RGB")), img)


def test_png_errors(tmp_path):
    p = tmp_path / "x.png"
    p.write_bytes(b"not a png")
    with pytest.raises(sk.SplatError):
        sk.read_png(p)
    with pytest.raises(sk.SplatError):
        sk.read_png(tmp_path / "missing.png")


def _cam(w, h, angle):
    from tests.util import look_at
    m = look_at((2.4 * np.cos(angle), 2.4 * np.sin(angle), 1.0))
    return sk.camera(w, h, 1.1 * w, 1.1 * w, (w - 1) / 2.0, (h - 1) / 2.0, m)


def test_cameras_json_round_trip_and_layout(tmp_path):
    cams = [_cam(48, 32, a) for a in np.linspace(0, 6, 5)]
    path = tmp_path / "cameras.json"
    sk.write_cameras_json(path, cams, ids=[3, 1, 4, 1, 5])
    back, ids = sk.read_cameras_json(path)
    assert ids.tolist() == [3, 1, 4, 1, 5]
    for a, b in zip(cams, back):
        assert (a.width, a.height, a.fx, a.fy, a.cx, a.cy) == (b.width, b.height, b.fx, b.fy, b.cx, b.cy)
        assert list(a.world_to_cam) == list(b.world_to_cam)
    # the reference's json: an array of records with these keys, doubles
    doc = json.loads(path.read_text())
    assert [sorted(r) for r in doc] == [["cx", "cy", "fx", "fy", "height", "id", "width", "world_to_cam"]] * 5
    assert doc[0]["fx"] == pytest.approx(1.1 * 48) and len(doc[0]["world_to_cam"]) == 16
    text = path.read_text()
    assert text.startswith('[\n  {\n    "cx": 23.5,\n') and '"height": 32,' in text


def test_cameras_json_errors(tmp_path):
    p = tmp_path / "c.json"
    p.write_text('[{"id": 0, "width": 4, "height": 4, "fx": 1, "fy": 1, "cx": 1}]')
    with pytest.raises(sk.SplatError):
        sk.read_cameras_json(p)
    p.write_text("[")
    with pytest.raises(sk.SplatError):
        sk.read_cameras_json(p)
    p.write_text('[{"id": 0, "width": 4, "height": 4, "fx": 1, "fy": 1, "cx": 1, "cy": 1, '
                 '"world_to_cam": [2,0,0,0, 0,1,0,0, 0,0,1,0, 0,0,0,1]}]')
    with pytest.raises(sk.SplatError):  # not orthonormal (Camera::validate)
        sk.read_cameras_json(p)
    p.write_text('[{"id": 0, "width": 4, "height": 4, "fx": 1, "fy": 1, "cx": 1, "cy": 1, '
                 '"world_to_cam": [1,0,0,0, 0,1,0,0, 0,0,1,0, 0,0,0,1]}]')
    cams, ids = sk.read_cameras_json(p)
    assert len(cams) == 1 and ids.tolist() == [0]


def test_config_files_parse_override_and_reject_unknown_keys(tmp_path):
    """test_dataset.cpp:253-285 (load_config_file, config.hpp:139-196)."""
    p = tmp_path / "train.cfg"
    p.write_text("# comment line\niterations = 1234\ntau = 0.25\nbin_mode = compact\nvcd = false\n")
    cfg = sk.load_config_file(p)
    assert cfg.iterations == 1234 and cfg.tau == pytest.approx(0.25)
    assert cfg.compact == 1 and cfg.vcd == 0 and cfg.k == 10  # untouched keys keep their defaults
    bad = tmp_path / "bad.cfg"
    bad.write_text("not_a_real_key = 3\n")
    with pytest.raises(sk.SplatError):
        sk.load_config_file(bad)
    rc = sk.lib().sk_config_set(None, sk.C.byref(cfg), b"vcp", b"maybe")
    assert rc != 0
    for k, v in (("seed", "18446744073709551615"), ("lambda", "0.3"), ("lazy_opt_enabled", "1"),
                 ("bin_mode", "aabb")):
        sk.set_config_value(cfg, k, v)
    assert cfg.seed == 2 ** 64 - 1 and cfg.lambda_ == pytest.approx(0.3)
    assert cfg.lazy_opt_enabled == 1 and cfg.compact == 0
    with pytest.raises(sk.SplatError):
        sk.set_config_value(cfg, "iterations", "many")
    malformed = tmp_path / "m.cfg"
    malformed.write_text("iterations 5\n")
    with pytest.raises(sk.SplatError):
        sk.load_config_file(malformed)
    invalid = sk.default_config()
    invalid.densify_every = 600  # does not divide 14500
    with pytest.raises((sk.SplatError, ValueError)):
        sk.validate_config(invalid)


def test_rng_normals_match_reference_stream(orc):
    """The split noise (adc.hpp:190-197) comes from the reference Rng's
    normal() stream; the library's batched draw (parallel Box-Muller) must be
    bit-identical to sequential draws, across chunk boundaries (odd chunks
    carry the cached spare) and for large batches (worker threads)."""
    chunks = [3, 4, 1, 0, 5, 100001, 6]
    total = sum(chunks)
    ref = orc.rng_normals(17, total)
    arr = (sk.C.c_int64 * len(chunks))(*chunks)
    out = np.zeros(total, np.float32)
    assert sk.lib().sk_rng_normals(sk.C.c_uint64(17), arr, len(chunks), sk._p(out)) == 0
    assert np.array_equal(out, ref)
