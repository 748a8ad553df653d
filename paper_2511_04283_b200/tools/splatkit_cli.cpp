// splatkit_b200 command-line tool: the reference CLI's
// subcommands (tools/splatkit_main.cpp: synth, train, render, eval,
// bench-tiles, ablate) driving the B200 hot path through the C ABI only.
// Outputs keep the reference's file names and formats: checkpoint.ply,
// log.csv, renders/%05d.png, metrics.json (nlohmann dump(2) layout, wall time
// kept out so seeded reruns are byte-identical), timing.json, ablation.csv,
// the bench-tiles CSV. Every view is rendered and scored on the GPU; the
// scene, dataset images and all frame buffers stay in HBM.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "splatkit_b200.h"

namespace fs = std::filesystem;

namespace {

sk_ctx* g_ctx = nullptr;

void check(int rc) {
  if (rc != SK_OK) throw std::runtime_error(g_ctx ? sk_last_error(g_ctx) : "splatkit_b200: call failed");
}

// ---- argument parsing ------------------------------------------------------

struct Args {
  std::map<std::string, std::string> opts;
  std::vector<std::string> flags;
  bool has(const std::string& k) const { return opts.count(k) > 0; }
  bool flag(const std::string& k) const { return std::find(flags.begin(), flags.end(), k) != flags.end(); }
  std::string get(const std::string& k, const std::string& dflt = "") const {
    auto it = opts.find(k);
    return it == opts.end() ? dflt : it->second;
  }
  std::string need(const std::string& k) const {
    if (!has(k)) throw std::runtime_error(k + " is required");
    return opts.at(k);
  }
};

const char* const kBoolFlags[] = {"--plot", "--float64"};

Args parse(int argc, char** argv, int first) {
  Args a;
  for (int i = first; i < argc; ++i) {
    std::string k = argv[i];
    if (k.rfind("--", 0) != 0) throw std::runtime_error("unexpected argument '" + k + "'");
    const auto eq = k.find('=');
    if (eq != std::string::npos) {
      a.opts[k.substr(0, eq)] = k.substr(eq + 1);
      continue;
    }
    if (std::find(std::begin(kBoolFlags), std::end(kBoolFlags), k) != std::end(kBoolFlags)) {
      a.flags.push_back(k);
      continue;
    }
    if (i + 1 >= argc) throw std::runtime_error(k + " needs a value");
    a.opts[k] = argv[++i];
  }
  return a;
}

// build_config (splatkit_main.cpp:62-75): config file, then CLI overrides.
sk_train_config build_config(const Args& a) {
  sk_train_config cfg;
  sk_default_config(&cfg);
  if (a.has("--config")) check(sk_config_load_file(g_ctx, &cfg, a.get("--config").c_str()));
  const std::pair<const char*, const char*> overrides[] = {{"--seed", "seed"},   {"--workers", "workers"},
                                                           {"--beta", "beta"},   {"--tau", "tau"},
                                                           {"--tau-d", "tau_d"}, {"--tau-p", "tau_p"},
                                                           {"--iters", "iterations"}};
  for (const auto& [flag, key] : overrides)
    if (a.has(flag)) check(sk_config_set(g_ctx, &cfg, key, a.get(flag).c_str()));
  check(sk_validate_config(g_ctx, &cfg));
  if (a.flag("--float64"))
    throw std::runtime_error("--float64: the B200 path trains in fp32; the float64 value path (sk_fp64_render_loss) serves the finite-difference checks");
  if (a.flag("--plot")) std::fprintf(stderr, "note: --plot charts are not produced by splatkit_b200\n");
  return cfg;
}

// ---- JSON output in nlohmann::json::dump(2) layout --------------------------

std::string jnum(double v) {
  if (!std::isfinite(v)) return "null";
  char buf[64];
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof(buf), "%.*g", prec, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  std::string s(buf);
  if (s.find_first_of(".eE") == std::string::npos) s += ".0";
  return s;
}

struct ViewMetric {
  int id;
  double psnr, ssim;
};

struct Metrics {
  std::string split;
  int64_t gaussians = 0;
  std::vector<ViewMetric> views;
  double mean_psnr = 0, mean_ssim = 0;
  int64_t total_pairs = 0;

  std::string dump() const {  // keys in nlohmann's sorted order
    std::ostringstream o;
    o << "{\n  \"gaussian_count\": " << gaussians << ",\n  \"mean_psnr\": " << jnum(mean_psnr)
      << ",\n  \"mean_ssim\": " << jnum(mean_ssim) << ",\n  \"split\": \"" << split
      << "\",\n  \"total_tile_pairs\": " << total_pairs << ",\n  \"views\": ";
    if (views.empty()) {
      o << "[]";
    } else {
      o << "[";
      for (size_t i = 0; i < views.size(); ++i)
        o << (i ? ",\n" : "\n") << "    {\n      \"id\": " << views[i].id << ",\n      \"psnr\": "
          << jnum(views[i].psnr) << ",\n      \"ssim\": " << jnum(views[i].ssim) << "\n    }";
      o << "\n  ]";
    }
    o << "\n}";
    return o.str();
  }
};

void write_text(const fs::path& p, const std::string& s) {
  std::ofstream out(p, std::ios::binary);
  if (!out.good()) throw std::runtime_error("cannot write " + p.string());
  out << s;
}

// ---- device helpers --------------------------------------------------------

struct Handles {
  sk_frame* frame = nullptr;
  ~Handles() {
    if (frame) sk_frame_destroy(frame);
  }
};

struct DatasetInfo {
  sk_dataset* d = nullptr;
  std::vector<int> ids, train, test;
  int views = 0;
  ~DatasetInfo() {
    if (d) sk_dataset_destroy(d);
  }
};

std::unique_ptr<DatasetInfo> load_dataset(const std::string& dir) {
  auto info = std::make_unique<DatasetInfo>();
  check(sk_dataset_load(g_ctx, dir.c_str(), &info->d));
  check(sk_dataset_num_views(info->d, &info->views));
  int cnt = 0;
  check(sk_dataset_train_indices(info->d, nullptr, &cnt));
  std::vector<int32_t> tr(static_cast<size_t>(cnt));
  check(sk_dataset_train_indices(info->d, tr.data(), &cnt));
  info->train.assign(tr.begin(), tr.end());
  for (int v = 0; v < info->views; ++v)
    if (std::find(tr.begin(), tr.end(), v) == tr.end()) info->test.push_back(v);
  std::vector<sk_camera> cams(static_cast<size_t>(info->views));
  std::vector<int32_t> ids(static_cast<size_t>(info->views));
  int n = info->views;
  check(sk_cameras_read(g_ctx, (fs::path(dir) / "cameras.json").c_str(), cams.data(), ids.data(), &n));
  info->ids.assign(ids.begin(), ids.end());
  return info;
}

sk_binning binning_of(const sk_train_config& cfg) {
  return sk_binning{cfg.compact, (float)cfg.beta, (float)cfg.tau_alpha, cfg.tile_size};
}

// render_view (splatkit_main.cpp:84-94) into `frame`; returns the pair count.
int64_t render_view(sk_scene* scene, const sk_camera& cam, const sk_binning& b, sk_frame* frame) {
  check(sk_preprocess(g_ctx, scene, &cam, &b, frame));
  int64_t pairs = 0;
  check(sk_bin_sort(g_ctx, frame, &pairs));
  check(sk_render_forward(g_ctx, frame, nullptr, nullptr));
  return pairs;
}

std::vector<float> frame_image(sk_frame* frame, const sk_camera& cam) {
  std::vector<float> img(static_cast<size_t>(cam.width) * cam.height * 3);
  check(sk_frame_get_image(g_ctx, frame, img.data()));
  return img;
}

// evaluation_metrics (splatkit_main.cpp:99-130): PSNR / SSIM of each view's
// render against its 8-bit GT, scored on the GPU.
Metrics evaluate(sk_scene* scene, const DatasetInfo& data, const std::vector<int>& views, const std::string& split,
                 const sk_train_config& cfg, const std::string& render_dir) {
  Metrics m;
  m.split = split;
  check(sk_scene_size(scene, &m.gaussians));
  Handles h;
  check(sk_frame_create(g_ctx, &h.frame));
  const sk_binning b = binning_of(cfg);
  double ps = 0, ss = 0;
  for (const int v : views) {
    sk_camera cam;
    check(sk_dataset_camera(data.d, v, &cam));
    m.total_pairs += render_view(scene, cam, b, h.frame);
    std::vector<uint8_t> gt(static_cast<size_t>(cam.width) * cam.height * 3);
    check(sk_dataset_image_u8(g_ctx, data.d, v, gt.data()));
    sk_loss_values lv;
    check(sk_loss_u8(g_ctx, h.frame, gt.data(), (float)cfg.lambda, &lv));
    m.views.push_back({data.ids[v], lv.psnr, lv.ssim});
    ps += lv.psnr;
    ss += lv.ssim;
    if (!render_dir.empty()) {
      char name[32];
      std::snprintf(name, sizeof(name), "%05d.png", data.ids[v]);
      const auto img = frame_image(h.frame, cam);
      check(sk_png_write(g_ctx, (fs::path(render_dir) / name).c_str(), img.data(), cam.width, cam.height));
    }
  }
  m.mean_psnr = views.empty() ? 0.0 : ps / views.size();
  m.mean_ssim = views.empty() ? 0.0 : ss / views.size();
  return m;
}

struct SceneGuard {
  sk_scene* s = nullptr;
  ~SceneGuard() {
    if (s) sk_scene_destroy(s);
  }
};

sk_scene* load_checkpoint(const std::string& path) {
  sk_scene* s = nullptr;
  check(sk_checkpoint_load(g_ctx, path.c_str(), 0, &s));
  return s;
}

struct TrainOutputs {
  Metrics metrics;
  double wall = 0;
  int64_t final_count = 0;
};

// train_pipeline (splatkit_main.cpp:147-196)
TrainOutputs train_pipeline(const DatasetInfo& data, const sk_train_config& cfg, const fs::path& out_dir) {
  fs::create_directories(out_dir);
  int64_t np = 0;
  check(sk_dataset_init_points(data.d, nullptr, nullptr, &np));
  std::vector<float> xyz(static_cast<size_t>(np) * 3), rgb(static_cast<size_t>(np) * 3);
  check(sk_dataset_init_points(data.d, xyz.data(), rgb.data(), &np));
  SceneGuard scene;
  check(sk_init_from_points(g_ctx, np, xyz.data(), rgb.data(), cfg.sh_degree, 0, &scene.s));
  sk_trainer* t = nullptr;
  check(sk_trainer_create(g_ctx, scene.s, data.d, &cfg, &t));
  std::unique_ptr<sk_trainer, int (*)(sk_trainer*)> tguard(t, sk_trainer_destroy);
  std::vector<sk_log_row> rows(static_cast<size_t>(std::max(cfg.iterations, 1)));
  const auto start = std::chrono::steady_clock::now();
  check(sk_trainer_run(t, cfg.iterations, rows.data()));
  check(sk_ctx_synchronize(g_ctx));
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();

  check(sk_checkpoint_save(g_ctx, scene.s, (out_dir / "checkpoint.ply").c_str()));
  {  // write_log_csv (splatkit_main.cpp:132-142)
    std::ostringstream o;
    o << "iteration,loss,psnr,gaussian_count,tile_pairs,elapsed_ms\n";
    char buf[160];
    for (int i = 0; i < cfg.iterations; ++i) {
      const sk_log_row& r = rows[i];
      std::snprintf(buf, sizeof(buf), "%d,%.9g,%.9g,%d,%lld,%.3f\n", r.iteration, r.loss, r.psnr, r.gaussians,
                    static_cast<long long>(r.tile_pairs), r.elapsed_ms);
      o << buf;
    }
    write_text(out_dir / "log.csv", o.str());
  }
  const bool have_test = !data.test.empty();
  fs::create_directories(out_dir / "renders");
  TrainOutputs out;
  out.metrics = evaluate(scene.s, data, have_test ? data.test : data.train, have_test ? "test" : "train", cfg,
                         (out_dir / "renders").string());
  write_text(out_dir / "metrics.json", out.metrics.dump() + "\n");
  write_text(out_dir / "timing.json", "{\n  \"wall_seconds\": " + jnum(wall) + "\n}\n");
  out.wall = wall;
  check(sk_scene_size(scene.s, &out.final_count));
  return out;
}

// ---- subcommands -----------------------------------------------------------

int cmd_synth(const Args& a) {
  sk_synth_spec spec{};
  spec.n_gaussians = std::stoi(a.get("--gaussians", "500"));
  spec.n_views = std::stoi(a.get("--views", "64"));
  const int size = std::stoi(a.get("--size", "128"));
  spec.width = std::stoi(a.get("--width", std::to_string(size)));
  spec.height = std::stoi(a.get("--height", std::to_string(size)));
  spec.seed = std::stoull(a.get("--seed", "1"));
  spec.scale_mult = std::stod(a.get("--scale-mult", "1"));
  spec.focal = std::stod(a.get("--focal", "-1"));
  const std::string out = a.need("--out");
  sk_scene* gt = nullptr;
  sk_dataset* d = nullptr;
  check(sk_synthetic_create(g_ctx, &spec, &gt, &d, nullptr, nullptr, nullptr));
  SceneGuard gguard{gt};
  std::unique_ptr<sk_dataset, int (*)(sk_dataset*)> dguard(d, sk_dataset_destroy);
  check(sk_dataset_save(g_ctx, d, out.c_str()));
  check(sk_checkpoint_save(g_ctx, gt, (fs::path(out) / "gt_checkpoint.ply").c_str()));
  std::printf("synthetic dataset written to %s\n", out.c_str());
  return 0;
}

int cmd_train(const Args& a) {
  const sk_train_config cfg = build_config(a);
  const auto data = load_dataset(a.need("--data"));
  const std::string out = a.get("--out", "run");
  train_pipeline(*data, cfg, out);
  std::printf("training complete; outputs in %s\n", out.c_str());
  return 0;
}

int cmd_render(const Args& a) {
  const sk_train_config cfg = build_config(a);
  const auto data = load_dataset(a.need("--data"));
  SceneGuard scene{load_checkpoint(a.need("--checkpoint"))};
  const std::string split = a.get("--split", "test");
  std::vector<int> views;
  if (split == "train")
    views = data->train;
  else if (split == "test")
    views = data->test;
  else
    for (int v = 0; v < data->views; ++v) views.push_back(v);
  if (views.empty()) throw std::runtime_error("render: selected split '" + split + "' is empty");
  const std::string out = a.get("--out", "renders");
  fs::create_directories(out);
  const Metrics m = evaluate(scene.s, *data, views, split, cfg, out);
  write_text(fs::path(out) / "metrics.json", m.dump() + "\n");
  std::printf("%s\n", m.dump().c_str());
  return 0;
}

int cmd_eval(const Args& a) {
  const sk_train_config cfg = build_config(a);
  const auto data = load_dataset(a.need("--data"));
  SceneGuard scene{load_checkpoint(a.need("--checkpoint"))};
  if (data->test.empty()) throw std::runtime_error("eval: dataset has an empty test split");
  const Metrics m = evaluate(scene.s, *data, data->test, "test", cfg, "");
  if (a.has("--out")) write_text(a.get("--out"), m.dump() + "\n");
  std::printf("%s\n", m.dump().c_str());
  return 0;
}

// cmd_bench_tiles (splatkit_main.cpp:226-297): pair counts, render time and
// the mean |difference| against the beta = 1 compact-box renders.
int cmd_bench_tiles(const Args& a) {
  const sk_train_config cfg = build_config(a);
  const std::string dir = a.need("--data");
  const auto data = load_dataset(dir);
  SceneGuard scene{load_checkpoint(a.get("--checkpoint", (fs::path(dir) / "gt_checkpoint.ply").string()))};
  std::vector<double> betas;
  {
    std::stringstream ss(a.get("--betas", "1.0,0.9,0.8"));
    std::string tok;
    while (std::getline(ss, tok, ',')) betas.push_back(std::stod(tok));
  }
  if (betas.empty()) throw std::runtime_error("bench-tiles: empty beta list");
  Handles h;
  check(sk_frame_create(g_ctx, &h.frame));
  std::vector<sk_camera> cams(static_cast<size_t>(data->views));
  for (int v = 0; v < data->views; ++v) check(sk_dataset_camera(data->d, v, &cams[v]));
  std::vector<std::vector<float>> reference;
  const sk_binning ref{1, 1.0f, (float)cfg.tau_alpha, cfg.tile_size};
  for (int v = 0; v < data->views; ++v) {
    render_view(scene.s, cams[v], ref, h.frame);
    reference.push_back(frame_image(h.frame, cams[v]));
  }
  auto run_mode = [&](const sk_binning& b, double& ms, int64_t& pairs, double& mean_diff) {
    ms = 0;
    pairs = 0;
    double diff = 0;
    int64_t cnt = 0;
    for (int v = 0; v < data->views; ++v) {
      check(sk_ctx_synchronize(g_ctx));
      const auto t0 = std::chrono::steady_clock::now();
      pairs += render_view(scene.s, cams[v], b, h.frame);
      check(sk_ctx_synchronize(g_ctx));
      ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      const auto img = frame_image(h.frame, cams[v]);
      for (size_t i = 0; i < img.size(); ++i) diff += std::fabs((double)img[i] - (double)reference[v][i]);
      cnt += (int64_t)img.size();
    }
    mean_diff = diff / (double)cnt;
  };
  std::ostringstream csv;
  csv << "binning,beta,pairs,render_ms,mean_abs_diff_vs_beta1\n";
  char buf[160];
  double ms, diff;
  int64_t pairs;
  run_mode(sk_binning{0, 1.0f, (float)cfg.tau_alpha, cfg.tile_size}, ms, pairs, diff);
  std::snprintf(buf, sizeof(buf), "aabb,,%lld,%.3f,%.9g\n", static_cast<long long>(pairs), ms, diff);
  csv << buf;
  for (const double beta : betas) {
    run_mode(sk_binning{1, (float)beta, (float)cfg.tau_alpha, cfg.tile_size}, ms, pairs, diff);
    std::snprintf(buf, sizeof(buf), "compact,%.4g,%lld,%.3f,%.9g\n", beta, static_cast<long long>(pairs), ms, diff);
    csv << buf;
  }
  if (a.has("--out")) write_text(a.get("--out"), csv.str());
  std::printf("%s", csv.str().c_str());
  return 0;
}

// cmd_ablate (splatkit_main.cpp:299-337): baseline / +VCD / +VCP / full.
int cmd_ablate(const Args& a) {
  const sk_train_config base = build_config(a);
  const auto data = load_dataset(a.need("--data"));
  const fs::path out = a.get("--out", "ablation");
  fs::create_directories(out);
  struct Row {
    const char* name;
    bool vcd, vcp, cb;
  };
  const Row rows[4] = {{"baseline", false, false, false},
                       {"vcd", true, false, false},
                       {"vcp", false, true, false},
                       {"full", true, true, true}};
  std::ostringstream csv;
  csv << "config,wall_s,mean_psnr,mean_ssim,gaussians,total_tile_pairs\n";
  for (const Row& row : rows) {
    sk_train_config cfg = base;
    cfg.vcd = row.vcd;
    cfg.vcp = row.vcp;
    cfg.compact = row.cb;
    if (row.cb && cfg.beta >= 1.0) cfg.beta = 0.8;
    const TrainOutputs o = train_pipeline(*data, cfg, out / row.name);
    char buf[200];
    std::snprintf(buf, sizeof(buf), "%s,%.3f,%.6f,%.6f,%lld,%lld\n", row.name, o.wall, o.metrics.mean_psnr,
                  o.metrics.mean_ssim, static_cast<long long>(o.final_count),
                  static_cast<long long>(o.metrics.total_pairs));
    csv << buf;
    std::printf("%s", buf);
    std::fflush(stdout);
  }
  write_text(out / "ablation.csv", csv.str());
  return 0;
}

void usage() {
  std::fprintf(stderr,
               "splatkit_b200: 3D Gaussian splatting on the B200 with multi-view consistent density control\n"
               "usage: splatkit_b200 <synth|train|render|eval|bench-tiles|ablate> [options]\n"
               "  synth       --out DIR [--gaussians N] [--views V] [--size S | --width W --height H] [--seed S]\n"
               "  train       --data DIR [--out DIR]\n"
               "  render      --checkpoint PLY --data DIR [--out DIR] [--split test|train|all]\n"
               "  eval        --checkpoint PLY --data DIR [--out JSON]\n"
               "  bench-tiles --data DIR [--checkpoint PLY] [--betas 1.0,0.9,0.8] [--out CSV]\n"
               "  ablate      --data DIR [--out DIR]\n"
               "common: --config FILE --seed --workers --beta --tau --tau-d --tau-p --iters --device N\n");
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    usage();
    return 1;
  }
  const std::string cmd = argv[1];
  if (cmd == "-h" || cmd == "--help") {
    usage();
    return 0;
  }
  try {
    const Args a = parse(argc, argv, 2);
    check(sk_ctx_create(std::stoi(a.get("--device", "0")), &g_ctx));
    int rc = 1;
    if (cmd == "synth")
      rc = cmd_synth(a);
    else if (cmd == "train")
      rc = cmd_train(a);
    else if (cmd == "render")
      rc = cmd_render(a);
    else if (cmd == "eval")
      rc = cmd_eval(a);
    else if (cmd == "bench-tiles")
      rc = cmd_bench_tiles(a);
    else if (cmd == "ablate")
      rc = cmd_ablate(a);
    else {
      usage();
      rc = 1;
    }
    sk_ctx_destroy(g_ctx);
    return rc;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    if (g_ctx) sk_ctx_destroy(g_ctx);
    return 1;
  }
}
