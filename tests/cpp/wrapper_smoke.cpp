// C++ caller of the splat:: surface (include/splatkit_b200.hpp) — written the
// way the reference's own tests call splatkit (tests/test_raster.cpp:146-156,
// tests/test_camera.cpp:23-36). Exit code 0 = all checks passed.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "splatkit_b200.hpp"

using namespace splat;

static int failures = 0;
#define CHECK(c)                                              \
  do {                                                        \
    if (!(c)) {                                               \
      std::printf("FAILED %s:%d %s\n", __FILE__, __LINE__, #c); \
      ++failures;                                             \
    }                                                         \
  } while (0)

int main() {
  Device dev(0);
  // two-term front-to-back expansion
  std::vector<ProjectedGaussian> pgs(2);
  for (int i = 0; i < 2; ++i) {
    pgs[i].mu2d[0] = 3;
    pgs[i].mu2d[1] = 3;
    pgs[i].cov2d(0, 0) = pgs[i].cov2d(1, 1) = 1;
    pgs[i].cov2d_inv(0, 0) = pgs[i].cov2d_inv(1, 1) = 1;
    pgs[i].opacity = 0.5f;
    pgs[i].depth = 1.0f + i;
    pgs[i].source_index = i;
  }
  pgs[0].color[0] = 1;
  pgs[1].color[1] = 1;
  const TileGrid grid = build_tile_grid(dev, pgs, 8, 8, BinningConfig{}, 8);
  CHECK(count_pairs(grid) == 2);
  const RenderOutputs out = blend_forward(dev, grid, pgs);
  CHECK(std::fabs(out.image.at(3, 3)[0] - 0.5f) < 1e-7f);
  CHECK(std::fabs(out.image.at(3, 3)[1] - 0.25f) < 1e-7f);
  CHECK(std::fabs(out.transmittance(3, 3) - 0.25f) < 1e-7f);
  CHECK(out.contrib_count(3, 3) == 2);

  // principal point (tests/test_camera.cpp:23-36)
  Scene scene;
  scene.sh_degree = 1;
  Gaussian3D g;
  g.mu[2] = 5;
  g.sh = ShMatrix(4);
  g.sh(0, 0) = g.sh(0, 1) = g.sh(0, 2) = 0.5f;
  scene.gaussians.push_back(g);
  Camera cam;
  cam.width = cam.height = 64;
  cam.fx = cam.fy = 100;
  cam.cx = cam.cy = 32;
  const auto proj = project_scene(dev, scene, cam);
  CHECK(proj.size() == 1);
  CHECK(std::fabs(proj[0].mu2d[0] - 32) < 1e-5f && std::fabs(proj[0].mu2d[1] - 32) < 1e-5f);
  CHECK(std::fabs(proj[0].depth - 5) < 1e-6f);

  // invalid scale raises the reference's exception
  Scene bad = scene;
  bad.gaussians[0].log_scale[0] = NAN;
  bool threw = false;
  try {
    project_scene(dev, bad, cam);
  } catch (const std::invalid_argument& e) {
    threw = std::string(e.what()).find("covariance_3d") != std::string::npos;
  }
  CHECK(threw);

  // on-disk formats (tests/test_dataset.cpp:64-84, 109-128, 182-197)
  const std::string tmp = std::string(std::getenv("SK_TMP") ? std::getenv("SK_TMP") : "/tmp");
  Image img(5, 3);
  for (size_t i = 0; i < img.pixels.size(); ++i)
    for (int c = 0; c < 3; ++c) img.pixels[i][c] = float((i * 3 + c) % 11) / 10.0f;
  write_png(tmp + "/wrapper.png", img);
  const Image back = read_png(tmp + "/wrapper.png");
  CHECK(back.width == 5 && back.height == 3);
  for (size_t i = 0; i < img.pixels.size(); ++i)
    for (int c = 0; c < 3; ++c) CHECK(std::fabs(back.pixels[i][c] - img.pixels[i][c]) <= 0.5f / 255 + 1e-6f);
  std::vector<std::pair<Vec3, Vec3>> pts(1);
  pts[0].first[0] = 1.5f;
  pts[0].second[1] = 1.0f;
  write_points_ply(tmp + "/wrapper_points.ply", pts);
  const auto pb = read_points_ply(tmp + "/wrapper_points.ply");
  CHECK(pb.size() == 1 && pb[0].first[0] == 1.5f && pb[0].second[1] == 1.0f);
  save_checkpoint(dev, scene, tmp + "/wrapper_ckpt.ply");
  const Scene sb = load_checkpoint(dev, tmp + "/wrapper_ckpt.ply");
  CHECK(sb.sh_degree == 1 && sb.size() == 1);
  CHECK(sb.gaussians[0].mu[2] == 5.0f && sb.gaussians[0].sh(0, 1) == 0.5f);
  std::printf("%s (%d failures)\n", failures ? "FAIL" : "PASS", failures);
  return failures ? 1 : 0;
}
