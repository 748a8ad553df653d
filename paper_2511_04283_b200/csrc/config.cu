// Flat `key = value` training configs (reference config.hpp:83-198):
// set_config_value / load_config_file over sk_train_config, with the
// reference's key names, value parsing (istream >> for numbers, true/false/1/0
// for booleans, "aabb"/"compact" for bin_mode) and error messages. Host code.
#include <cstddef>
#include <fstream>
#include <vector>
#include <sstream>
#include <string>

#include "abi_util.h"

namespace sk {
namespace {

enum class Kind { I32, F64, Bool, U64, BinMode };
struct Field {
  const char* key;
  Kind kind;
  size_t off;
};

#define SKF(name, kind) {#name, Kind::kind, offsetof(sk_train_config, name)}
// config.hpp:89-129, same keys and order
const Field kFields[] = {
    SKF(iterations, I32),
    SKF(k, I32),
    SKF(lambda, F64),
    SKF(tau, F64),
    SKF(tau_d, F64),
    SKF(tau_p, F64),
    SKF(beta, F64),
    SKF(tau_alpha, F64),
    SKF(densify_from, I32),
    SKF(densify_until, I32),
    SKF(densify_every, I32),
    SKF(prune_every_early, I32),
    SKF(prune_every_late, I32),
    SKF(grad_threshold, F64),
    SKF(percent_dense, F64),
    SKF(lr_position, F64),
    SKF(lr_position_final, F64),
    SKF(lr_sh_dc, F64),
    SKF(lr_sh_rest, F64),
    SKF(lr_opacity, F64),
    SKF(lr_scale, F64),
    SKF(lr_rotation, F64),
    SKF(opacity_reset_every, I32),
    SKF(lazy_opt_enabled, Bool),
    SKF(lazy_opt_interval_15k, I32),
    SKF(lazy_opt_interval_20k, I32),
    SKF(seed, U64),
    SKF(tile_size, I32),
    SKF(workers, I32),
    SKF(sh_degree, I32),
    {"bin_mode", Kind::BinMode, offsetof(sk_train_config, compact)},
    SKF(vcd, Bool),
    SKF(vcp, Bool),
    SKF(prune_min_opacity, F64),
    SKF(prune_opacity_late, F64),
    SKF(prune_world_size_frac, F64),
    SKF(prune_screen_size, F64),
    SKF(size_prune_from, I32),
    SKF(schedule_dry_run, Bool),
};
#undef SKF

template <typename M>
void parse_number(const std::string& key, const std::string& value, void* dst) {
  std::istringstream in(value);
  M parsed{};
  in >> parsed;
  require(!in.fail(), "config: cannot parse value '" + value + "' for key '" + key + "'");
  *static_cast<M*>(dst) = parsed;
}

// set_config_value (config.hpp:139-163)
void set_value(sk_train_config& cfg, const std::string& key, const std::string& value) {
  const Field* f = nullptr;
  for (const Field& x : kFields)
    if (key == x.key) f = &x;
  require(f != nullptr, "config: unknown key '" + key + "'");
  void* dst = reinterpret_cast<char*>(&cfg) + f->off;
  switch (f->kind) {
    case Kind::I32: {
      int v = 0;
      parse_number<int>(key, value, &v);
      *static_cast<int32_t*>(dst) = v;
      break;
    }
    case Kind::F64: parse_number<double>(key, value, dst); break;
    case Kind::U64: {
      uint64_t v = 0;
      parse_number<uint64_t>(key, value, &v);
      *static_cast<uint64_t*>(dst) = v;
      break;
    }
    case Kind::Bool:
      if (value == "true" || value == "1")
        *static_cast<int32_t*>(dst) = 1;
      else if (value == "false" || value == "0")
        *static_cast<int32_t*>(dst) = 0;
      else
        throw std::runtime_error("config: key '" + key + "' expects a boolean, got '" + value + "'");
      break;
    case Kind::BinMode:
      // config.hpp:78-79 validates the string; the C struct stores the mode
      require(value == "aabb" || value == "compact", "config: bin_mode must be 'aabb' or 'compact'");
      *static_cast<int32_t*>(dst) = value == "compact" ? 1 : 0;
      break;
  }
}

std::string trim(const std::string& s) {
  const auto b = s.find_first_not_of(" \t\r");
  const auto e = s.find_last_not_of(" \t\r");
  return b == std::string::npos ? std::string() : s.substr(b, e - b + 1);
}

// load_config_file (config.hpp:162-188): a flat "key = value" file; '#'
// starts a comment; blank lines are skipped; any other line without '=' is
// an error naming its 1-based line number. The whole file is read first and
// then applied line by line.
void load_file(sk_train_config& cfg, const std::string& path) {
  std::ifstream file(path);
  require(file.good(), "config: cannot open '" + path + "'");
  std::vector<std::string> lines;
  for (std::string l; std::getline(file, l);) lines.push_back(std::move(l));
  for (size_t i = 0; i < lines.size(); ++i) {
    const std::string body = trim(lines[i].substr(0, lines[i].find('#')));
    if (body.empty()) continue;
    const size_t sep = body.find('=');
    require(sep != std::string::npos, "config: malformed line " + std::to_string(i + 1) + " (expected key = value)");
    set_value(cfg, trim(body.substr(0, sep)), trim(body.substr(sep + 1)));
  }
}

}  // namespace
}  // namespace sk

using namespace sk;

extern "C" {

int sk_config_set(sk_ctx* ctx, sk_train_config* cfg, const char* key, const char* value) {
  return guarded(ctx, [&] {
    arg(cfg && key && value, "config: null argument");
    set_value(*cfg, key, value);
  });
}

int sk_config_load_file(sk_ctx* ctx, sk_train_config* cfg, const char* path) {
  return guarded(ctx, [&] {
    arg(cfg && path, "config: null argument");
    load_file(*cfg, path);
  });
}

}  // extern "C"
