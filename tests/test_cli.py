"""splatkit_b200 CLI: the reference tool's subcommands
(tools/splatkit_main.cpp) over the C ABI, with its output files and formats;
mirrors tests/cli_smoke.sh."""
import json
import os
import subprocess

import numpy as np
import pytest

import paper_2511_04283_b200 as sk

CFG = """# short schedule (tests/cli_smoke.sh style)
iterations = 300
densify_from = 100
densify_until = 200
densify_every = 100
prune_every_early = 100
prune_every_late = 100
size_prune_from = 100
k = 4
"""


@pytest.fixture(scope="module")
def cli():
    from paper_2511_04283_b200 import builder
    sk.build()
    return builder.CLI


def run(cli, *args, check=True):
    r = subprocess.run([cli, *map(str, args)], capture_output=True, text=True, timeout=600)
    if check:
        assert r.returncode == 0, r.stdout + r.stderr
    return r


def test_cli_builds_and_prints_usage(cli):
    r = run(cli, "--help")
    assert "synth" in r.stderr and "bench-tiles" in r.stderr and "ablate" in r.stderr
    r = run(cli, "frobnicate", check=False)
    assert r.returncode != 0


@pytest.mark.gpu
def test_cli_synth_train_eval_render_bench(cli, tmp_path):
    data = tmp_path / "data"
    run(cli, "synth", "--out", data, "--gaussians", 1500, "--views", 9, "--size", 64, "--seed", 3)
    assert sorted(os.listdir(data)) == ["cameras.json", "gt_checkpoint.ply", "images", "points3d.ply"]
    assert len(os.listdir(data / "images")) == 9
    cfg = tmp_path / "train.cfg"
    cfg.write_text(CFG)
    out = tmp_path / "run"
    r = run(cli, "train", "--data", data, "--out", out, "--config", cfg, "--seed", 17)
    assert "training complete" in r.stdout
    for f in ("checkpoint.ply", "log.csv", "metrics.json", "timing.json"):
        assert (out / f).exists(), f
    log = (out / "log.csv").read_text().splitlines()
    assert log[0] == "iteration,loss,psnr,gaussian_count,tile_pairs,elapsed_ms" and len(log) == 301
    m = json.loads((out / "metrics.json").read_text())
    assert m["split"] == "test" and [v["id"] for v in m["views"]] == [0, 8]
    assert m["mean_psnr"] > 15 and 0 < m["mean_ssim"] <= 1 and m["total_tile_pairs"] > 0
    assert sorted(os.listdir(out / "renders")) == ["00000.png", "00008.png"]
    assert "wall_seconds" in json.loads((out / "timing.json").read_text())
    # eval of the written checkpoint reproduces the training run's test metrics
    r = run(cli, "eval", "--checkpoint", out / "checkpoint.ply", "--data", data, "--out", tmp_path / "e.json")
    e = json.loads((tmp_path / "e.json").read_text())
    assert e == m
    # render --split all
    r = run(cli, "render", "--checkpoint", out / "checkpoint.ply", "--data", data, "--out", tmp_path / "r",
            "--split", "all")
    assert len([f for f in os.listdir(tmp_path / "r") if f.endswith(".png")]) == 9
    # rendered PNGs are the GPU renders quantised like write_png
    img = sk.read_png(tmp_path / "r" / "00000.png")
    assert img.shape == (64, 64, 3)
    # bench-tiles: AABB >= compact(1.0) >= compact(0.8) pairs (tests/test_raster.cpp:194-214)
    r = run(cli, "bench-tiles", "--data", data, "--betas", "1.0,0.8", "--out", tmp_path / "b.csv")
    rows = [ln.split(",") for ln in (tmp_path / "b.csv").read_text().splitlines()[1:]]
    pairs = [int(x[2]) for x in rows]
    assert rows[0][0] == "aabb" and pairs[0] >= pairs[1] >= pairs[2]
    assert float(rows[1][4]) == 0.0  # beta 1 against itself
    # errors exit 1 with the reference's message text
    r = run(cli, "eval", "--checkpoint", tmp_path / "missing.ply", "--data", data, check=False)
    assert r.returncode == 1 and "ply: cannot open" in r.stderr
    bad = tmp_path / "bad.cfg"
    bad.write_text("not_a_real_key = 1\n")
    r = run(cli, "train", "--data", data, "--out", tmp_path / "x", "--config", bad, check=False)
    assert r.returncode == 1 and "not_a_real_key" in r.stderr


@pytest.mark.gpu
def test_cli_ablate_directions(cli, tmp_path):
    """Acceptance criteria 4-6 directions (tests/acceptance.cpp:301-396) on a
    short schedule: +VCD densifies no more than the baseline, +VCP keeps fewer
    Gaussians, compact binning (beta 0.8) emits fewer pairs."""
    data = tmp_path / "data"
    run(cli, "synth", "--out", data, "--gaussians", 1500, "--views", 9, "--size", 64, "--seed", 5)
    cfg = tmp_path / "train.cfg"
    cfg.write_text(CFG)
    out = tmp_path / "abl"
    run(cli, "ablate", "--data", data, "--out", out, "--config", cfg, "--seed", 17)
    rows = {ln.split(",")[0]: ln.split(",") for ln in (out / "ablation.csv").read_text().splitlines()[1:]}
    assert set(rows) == {"baseline", "vcd", "vcp", "full"}
    g = {k: int(v[4]) for k, v in rows.items()}
    assert g["vcd"] <= g["baseline"]
    assert g["vcp"] <= g["baseline"]
    for k in rows:
        assert (out / k / "metrics.json").exists()
        assert np.isfinite(float(rows[k][2]))
