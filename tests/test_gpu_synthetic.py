"""GPU scene construction against the CPU oracle.

sk_synthetic_create restates generate_synthetic (dataset.hpp:178-250): same
Rng draw order on the host, GT views rendered by the bit-exact K1-K6 path on
the GPU and quantised through 8 bits. sk_init_from_points restates
init_from_points (scene.hpp:117-141) with a GPU all-pairs 3-NN. Everything is
compared bit for bit with the oracle.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2511_04283_b200 as sk
    sk.build()
    c = sk.Context(0)
    yield c
    c.close()


def _cam_tuple(c):
    return (c.width, c.height, c.fx, c.fy, c.cx, c.cy, tuple(c.world_to_cam), c.near_plane)


@pytest.mark.parametrize("n,views,w,h,seed", [(600, 9, 64, 64, 1), (1500, 10, 80, 48, 7)])
def test_synthetic_dataset_bit_exact(ctx, orc, n, views, w, h, seed):
    import paper_2511_04283_b200 as sk
    ref = orc.Dataset(n_gaussians=n, n_views=views, width=w, height=h, seed=seed)
    ds, gt, xyz, rgb = sk.Dataset.synthetic(ctx, n_gaussians=n, n_views=views, width=w, height=h, seed=seed)
    assert ds.num_views == ref.num_views == views
    assert np.array_equal(gt.download(), ref.gt_scene())
    for v in range(views):
        assert _cam_tuple(ds.camera(v)) == _cam_tuple(ref.camera(v)), v
        assert np.array_equal(ds.image_u8(v), ref.image_u8(v)), v
    rx, rc = ref.points()
    assert np.array_equal(xyz, rx)
    assert np.array_equal(rgb, rc)
    assert np.array_equal(ds.train_indices(), ref.train_indices())
    assert ds.extent == ref.extent


@pytest.mark.parametrize("n", [2, 3, 4, 700])
def test_init_from_points_bit_exact(ctx, orc, n):
    import paper_2511_04283_b200 as sk
    rng = np.random.default_rng(50 + n)
    xyz = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    if n > 4:
        xyz[5] = xyz[3]  # a duplicate point: zero distance, clamped to 1e-7
    rgb = rng.uniform(0, 1, (n, 3)).astype(np.float32)
    for deg in (0, 3):
        got = sk.Scene.from_points(ctx, xyz, rgb, deg)
        assert np.array_equal(got.download(), orc.init_from_points(xyz, rgb, deg))


def test_init_from_points_empty(ctx):
    import paper_2511_04283_b200 as sk
    with pytest.raises(ValueError, match="init_from_points: empty point cloud"):  # std::invalid_argument
        sk.Scene.from_points(ctx, np.zeros((0, 3), np.float32), np.zeros((0, 3), np.float32), 3)


def test_synthetic_trains(ctx):
    """The generated dataset and point-cloud init drive the GPU trainer."""
    import paper_2511_04283_b200 as sk
    ds, gt, xyz, rgb = sk.Dataset.synthetic(ctx, n_gaussians=800, n_views=8, width=64, seed=3)
    scene = sk.Scene.from_points(ctx, xyz, rgb, 3)
    cfg = sk.default_config()
    cfg.iterations = 60
    cfg.densify_from = cfg.densify_until = 1 << 30
    tr = sk.Trainer(ctx, scene, ds, cfg)
    rows = tr.run(60)
    assert len(rows) == 60
    assert rows[-1]["loss"] < rows[0]["loss"]
