// On-disk formats of the reference, so GPU-trained scenes
// and GPU-generated datasets are interchangeable with the reference tooling:
//
// * PLY vertex tables (ply.hpp:19-175): ASCII or binary little-endian, scalar
//   properties only, vertex element first; points3d.ply (x y z + 8-bit rgb,
//   ply.hpp:179-212) and the splatting checkpoint layout (ply.hpp:217-315).
//   A checkpoint moves between the planar device scene ([C][capacity]) and
//   the row-major file body ([n][P] float32) with one gather kernel on the
//   GPU and a single bulk host<->device copy, instead of the reference's
//   per-Gaussian heap rows.
// * PNG (png_io.cpp:25-104), written directly over zlib (libpng is absent):
//   8-bit RGB out with lround(clamp(v)·255); in: 1/2/4/8/16-bit gray, RGB,
//   palette, gray+alpha, RGBA, non-interlaced, with the reference's
//   libpng transforms (strip 16 to the high byte, expand low-depth gray,
//   palette to RGB, gray to RGB, strip alpha).
// * cameras.json (dataset.hpp:73-150): a small JSON reader for the record
//   schema (id, width, height, fx, fy, cx, cy, world_to_cam[16]) and a writer
//   in nlohmann's dump(2) layout (sorted keys, shortest round-trip doubles).
// * load_dataset / the file side of generate_synthetic: cameras.json +
//   images/%05d.png + points3d.ply into a device-resident sk_dataset.
//
// Host code only except the two checkpoint gather kernels.
#include <zlib.h>

#include <algorithm>
#include <thread>
#include <atomic>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "abi_util.h"
#include "trainer.h"

namespace sk {
namespace io {

namespace fs = std::filesystem;

// ---------------------------------------------------------------------------
// PLY
// ---------------------------------------------------------------------------

// Scalar property types a vertex element may carry, keyed by every spelling
// the PLY format allows (ply.hpp:49-72 accepts the same set).
enum class PlyScalar { I8, U8, I16, U16, I32, U32, F32, F64 };

struct PlyProp {
  std::string name;
  PlyScalar kind = PlyScalar::F32;
  int size = 4;                 // bytes in a binary row
  bool integer = false;         // integer-typed (points3d colours are then rescaled by 1/255)
};

PlyProp make_prop(const std::string& type, const std::string& name) {
  static const std::pair<const char*, PlyScalar> kTypes[] = {
      {"char", PlyScalar::I8},    {"int8", PlyScalar::I8},     {"uchar", PlyScalar::U8},
      {"uint8", PlyScalar::U8},   {"short", PlyScalar::I16},   {"int16", PlyScalar::I16},
      {"ushort", PlyScalar::U16}, {"uint16", PlyScalar::U16},  {"int", PlyScalar::I32},
      {"int32", PlyScalar::I32},  {"uint", PlyScalar::U32},    {"uint32", PlyScalar::U32},
      {"float", PlyScalar::F32},  {"float32", PlyScalar::F32}, {"double", PlyScalar::F64},
      {"float64", PlyScalar::F64}};
  static const int kSize[] = {1, 1, 2, 2, 4, 4, 4, 8};
  for (const auto& [spelling, kind] : kTypes)
    if (type == spelling) {
      PlyProp p;
      p.name = name;
      p.kind = kind;
      p.size = kSize[static_cast<int>(kind)];
      p.integer = kind != PlyScalar::F32 && kind != PlyScalar::F64;
      return p;
    }
  throw std::runtime_error("ply: unsupported property type '" + type + "'");
}

// One little-endian binary value of the given type, widened to double.
template <typename V>
double load_as(const char* p) {
  V v;
  std::memcpy(&v, p, sizeof(V));
  return static_cast<double>(v);
}
double decode_value(const char* p, PlyScalar kind) {
  switch (kind) {
    case PlyScalar::I8: return load_as<int8_t>(p);
    case PlyScalar::U8: return load_as<uint8_t>(p);
    case PlyScalar::I16: return load_as<int16_t>(p);
    case PlyScalar::U16: return load_as<uint16_t>(p);
    case PlyScalar::I32: return load_as<int32_t>(p);
    case PlyScalar::U32: return load_as<uint32_t>(p);
    case PlyScalar::F32: return load_as<float>(p);
    default: return load_as<double>(p);
  }
}

// The vertex table of a PLY file (PlyVertexTable, ply.hpp:19-40). When the
// file is binary and every vertex property is float32, the body is kept as
// raw rows (`raw`, [count][props]) and `columns` stays empty: the checkpoint
// path gathers it on the GPU.
struct PlyTable {
  int64_t count = 0;
  std::vector<PlyProp> props;
  std::vector<std::vector<double>> columns;
  std::vector<float> raw;
  bool raw_f32 = false;

  int find(const std::string& name) const {
    const auto it = std::find_if(props.begin(), props.end(), [&](const PlyProp& p) { return p.name == name; });
    return it == props.end() ? -1 : int(it - props.begin());
  }
  int need(const std::string& name, const std::string& context) const {
    const int i = find(name);
    require(i >= 0, context + ": missing property '" + name + "'");
    return i;
  }
  double value(int col, int64_t row) const {
    return raw_f32 ? (double)raw[(size_t)row * props.size() + col] : columns[col][row];
  }
};

// Header state: which element the property lines belong to, the body
// encoding and the vertex element's declaration.
struct PlyHeader {
  bool have_format = false, binary = false;
  int64_t vertices = -1;     // count of the vertex element once declared
  bool reading_vertex = false;
  std::vector<PlyProp> props;
};

// The header grammar of read_ply_vertices (ply.hpp:103-175): magic line,
// format (ascii | binary_little_endian), the vertex element first, scalar
// vertex properties, properties of later elements ignored, end_header.
PlyHeader parse_ply_header(std::istream& in, const std::string& path) {
  std::string line;
  require(std::getline(in, line) && (line == "ply" || line == "ply\r"),
          "ply: '" + path + "' does not start with a ply magic line");
  PlyHeader h;
  const auto where = " in '" + path + "'";
  while (std::getline(in, line)) {
    if (!line.empty() && line.back() == '\r') line.pop_back();
    std::istringstream words(line);
    std::string key;
    words >> key;
    if (key.empty() || key == "comment" || key == "obj_info") continue;
    if (key == "end_header") break;
    if (key == "format") {
      std::string enc;
      words >> enc;
      if (enc != "ascii" && enc != "binary_little_endian")
        throw std::runtime_error("ply: unsupported format '" + enc + "'" + where);
      h.binary = enc == "binary_little_endian";
      h.have_format = true;
    } else if (key == "element") {
      std::string what;
      int64_t n = 0;
      words >> what >> n;
      const bool vertex = what == "vertex";
      require(vertex ? h.props.empty() : h.vertices >= 0, "ply: vertex element must come first" + where);
      if (vertex) h.vertices = n;
      h.reading_vertex = vertex;
    } else if (key == "property") {
      if (!h.reading_vertex) continue;
      std::string type, name;
      words >> type;
      require(type != "list", "ply: list properties are not supported on vertices");
      words >> name;
      h.props.push_back(make_prop(type, name));
    } else {
      throw std::runtime_error("ply: unexpected header token '" + key + "'" + where);
    }
  }
  require(h.have_format, "ply: missing format line" + where);
  require(h.vertices >= 0, "ply: missing vertex element" + where);
  return h;
}

// read_ply_vertices (ply.hpp:103-175): the header, then the vertex rows as
// columns of doubles (or as raw float32 rows, see PlyTable).
PlyTable read_ply(const std::string& path, bool keep_raw_f32) {
  std::ifstream in(path, std::ios::binary);
  require(in.good(), "ply: cannot open '" + path + "'");
  PlyHeader h = parse_ply_header(in, path);
  PlyTable t;
  t.count = h.vertices;
  t.props = std::move(h.props);
  const size_t np = t.props.size();
  const std::string truncated = "ply: truncated vertex data in '" + path + "'";
  size_t row_bytes = 0;
  for (const auto& p : t.props) row_bytes += (size_t)p.size;
  const bool f32_rows = h.binary && np > 0 && row_bytes == 4 * np &&
                        std::all_of(t.props.begin(), t.props.end(),
                                    [](const PlyProp& p) { return p.kind == PlyScalar::F32; });
  if (f32_rows && keep_raw_f32) {
    t.raw_f32 = true;
    t.raw.resize((size_t)t.count * np);
    const auto bytes = (std::streamsize)(t.raw.size() * sizeof(float));
    in.read(reinterpret_cast<char*>(t.raw.data()), bytes);
    require(in.gcount() == bytes, truncated);
    return t;
  }
  t.columns.assign(np, std::vector<double>((size_t)t.count));
  if (h.binary) {
    std::vector<char> body((size_t)t.count * row_bytes);
    in.read(body.data(), (std::streamsize)body.size());
    require(in.gcount() == (std::streamsize)body.size(), truncated);
    const char* row = body.data();
    for (int64_t v = 0; v < t.count; ++v)
      for (size_t i = 0; i < np; row += t.props[i].size, ++i) t.columns[i][v] = decode_value(row, t.props[i].kind);
  } else {
    for (int64_t v = 0; v < t.count; ++v)
      for (size_t i = 0; i < np; ++i) require(static_cast<bool>(in >> t.columns[i][v]), truncated);
  }
  return t;
}

int sh_coeff_count(int deg) { return (deg + 1) * (deg + 1); }

// Column of checkpoint property `j` (ply.hpp:227-236 order) for planar
// component c: x y z, nx ny nz (no component), f_dc_c = sh(0,c), f_rest
// channel-major (c, m) = sh(m, c), opacity, scale_0..2, rot_0..3.
// Returns the planar component, or -1 for the zero normals.
int ckpt_prop_component(int j, int deg) {
  const int n_sh = sh_coeff_count(deg);
  const int n_rest = 3 * (n_sh - 1);
  if (j < 3) return SK_COMP_MU + j;
  if (j < 6) return -1;
  j -= 6;
  if (j < 3) return SK_COMP_SH + j;  // sh(0, c)
  j -= 3;
  if (j < n_rest) {
    const int c = j / (n_sh - 1), m = 1 + j % (n_sh - 1);
    return SK_COMP_SH + 3 * m + c;
  }
  j -= n_rest;
  if (j == 0) return SK_COMP_OPACITY;
  j -= 1;
  if (j < 3) return SK_COMP_LOG_SCALE + j;
  j -= 3;
  return SK_COMP_ROT + j;
}

// rows[i][j] = planar[comp(j)][i] (0 for the normals); one thread per cell,
// consecutive threads walk a row so the row-major writes coalesce.
__global__ void planar_to_rows_kernel(const float* __restrict__ planar, int64_t stride, int64_t n, int props,
                                      const int* __restrict__ comp_of, float* __restrict__ rows) {
  const int64_t cells = n * props;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < cells; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / props;
    const int j = (int)(e - i * props);
    const int c = comp_of[j];
    rows[e] = c < 0 ? 0.0f : planar[(size_t)c * stride + i];
  }
}

// planar[c][i] = rows[i][col_of[c]]; one thread per planar cell (coalesced
// planar writes; the row reads of one component hit the same cache lines
// across the components of a row).
__global__ void rows_to_planar_kernel(const float* __restrict__ rows, int64_t n, int props,
                                      const int* __restrict__ col_of, int comps, float* __restrict__ planar,
                                      int64_t stride) {
  const int64_t cells = (int64_t)comps * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < cells; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e / n);
    const int64_t i = e - (int64_t)c * n;
    planar[(size_t)c * stride + i] = rows[(size_t)i * props + col_of[c]];
  }
}

unsigned grid_for(int64_t cells) { return (unsigned)std::min<int64_t>((cells + 255) / 256, 148 * 16); }

// save_checkpoint (ply.hpp:217-248): header, then n rows of P float32.
void save_checkpoint(sk_ctx* ctx, const sk_scene* s, const std::string& path) {
  const int deg = s->sh_degree;
  const int n_sh = sh_coeff_count(deg);
  const int n_rest = 3 * (n_sh - 1);
  const int props = 6 + 3 + n_rest + 1 + 3 + 4;
  std::ofstream out(path, std::ios::binary);
  require(out.good(), "checkpoint: cannot open '" + path + "' for writing");
  out << "ply\nformat binary_little_endian 1.0\nelement vertex " << s->n << "\n";
  for (const char* f : {"x", "y", "z", "nx", "ny", "nz"}) out << "property float " << f << "\n";
  for (int i = 0; i < 3; ++i) out << "property float f_dc_" << i << "\n";
  for (int i = 0; i < n_rest; ++i) out << "property float f_rest_" << i << "\n";
  out << "property float opacity\n";
  for (int i = 0; i < 3; ++i) out << "property float scale_" << i << "\n";
  for (int i = 0; i < 4; ++i) out << "property float rot_" << i << "\n";
  out << "end_header\n";
  if (s->n > 0) {
    std::vector<int> comp_of(props);
    for (int j = 0; j < props; ++j) comp_of[j] = ckpt_prop_component(j, deg);
    DevBuf d_map, d_rows;
    int* dm = ensure<int>(d_map, props);
    float* dr = ensure<float>(d_rows, (size_t)s->n * props);
    h2d(ctx, dm, comp_of.data(), props);
    planar_to_rows_kernel<<<grid_for(s->n * props), 256, 0, ctx->stream>>>(s->params.as<float>(), s->capacity, s->n,
                                                                          props, dm, dr);
    note_launch();
    SK_CUDA(cudaGetLastError());
    std::vector<float> rows((size_t)s->n * props);
    d2h(ctx, rows.data(), dr, rows.size());
    sync(ctx);
    out.write(reinterpret_cast<const char*>(rows.data()), (std::streamsize)(rows.size() * sizeof(float)));
  }
  require(out.good(), "checkpoint: write failed for '" + path + "'");
}

// load_checkpoint (ply.hpp:251-315): SH degree from the f_rest count, every
// field required by name.
sk_scene* load_checkpoint(sk_ctx* ctx, const std::string& path, int64_t capacity) {
  const PlyTable t = read_ply(path, true);
  int n_rest = 0;
  while (t.find("f_rest_" + std::to_string(n_rest)) >= 0) ++n_rest;
  require(n_rest % 3 == 0, "checkpoint: f_rest count must be divisible by 3");
  const int rest_coeffs = n_rest / 3;
  int degree = -1;
  for (int d = 0; d <= 3; ++d)
    if (sh_coeff_count(d) - 1 == rest_coeffs) degree = d;
  require(degree >= 0,
          "checkpoint: f_rest count " + std::to_string(n_rest) + " does not match any SH degree 0..3");
  const int comps = SK_COMP_COUNT(degree);
  const int n_sh = sh_coeff_count(degree);
  // planar component -> file column, resolved in the reference's lookup order
  std::vector<int> col_of(comps, -1);
  const char* xyz[3] = {"x", "y", "z"};
  for (int d = 0; d < 3; ++d) col_of[SK_COMP_MU + d] = t.need(xyz[d], "checkpoint");
  const int op = t.need("opacity", "checkpoint");
  for (int c = 0; c < 3; ++c) col_of[SK_COMP_SH + c] = t.need("f_dc_" + std::to_string(c), "checkpoint");
  for (int d = 0; d < 3; ++d) col_of[SK_COMP_LOG_SCALE + d] = t.need("scale_" + std::to_string(d), "checkpoint");
  for (int d = 0; d < 4; ++d) col_of[SK_COMP_ROT + d] = t.need("rot_" + std::to_string(d), "checkpoint");
  for (int c = 0; c < 3; ++c)
    for (int m = 1; m < n_sh; ++m)
      col_of[SK_COMP_SH + 3 * m + c] = t.need("f_rest_" + std::to_string(c * (n_sh - 1) + (m - 1)), "checkpoint");
  col_of[SK_COMP_OPACITY] = op;

  auto s = std::make_unique<sk_scene>();
  s->sh_degree = degree;
  s->comps = comps;
  s->capacity = round_capacity(std::max<int64_t>(capacity, t.count));
  ensure<float>(s->params, (size_t)comps * s->capacity);
  s->n = t.count;
  if (t.count > 0) {
    if (t.raw_f32) {
      const int props = (int)t.props.size();
      DevBuf d_map, d_rows;
      int* dm = ensure<int>(d_map, comps);
      float* dr = ensure<float>(d_rows, t.raw.size());
      h2d(ctx, dm, col_of.data(), comps);
      h2d(ctx, dr, t.raw.data(), t.raw.size());
      rows_to_planar_kernel<<<grid_for((int64_t)comps * t.count), 256, 0, ctx->stream>>>(
          dr, t.count, props, dm, comps, s->params.as<float>(), s->capacity);
      note_launch();
      SK_CUDA(cudaGetLastError());
      sync(ctx);
    } else {
      // generic columns (ASCII or mixed types): T(double) per value as the reference
      std::vector<float> planar((size_t)comps * t.count);
      for (int c = 0; c < comps; ++c)
        for (int64_t i = 0; i < t.count; ++i) planar[(size_t)c * t.count + i] = (float)t.columns[col_of[c]][i];
      SK_CUDA(cudaMemcpy2DAsync(s->params.ptr, sizeof(float) * s->capacity, planar.data(), sizeof(float) * t.count,
                                sizeof(float) * t.count, comps, cudaMemcpyHostToDevice, ctx->stream));
      sync(ctx);
    }
  }
  return s.release();
}

// read_points_ply (ply.hpp:179-196): colours rescaled from 0..255 when the
// red column is integer-typed.
void read_points(const std::string& path, std::vector<float>& xyz, std::vector<float>& rgb) {
  const PlyTable t = read_ply(path, false);
  const int cx = t.need("x", "points3d"), cy = t.need("y", "points3d"), cz = t.need("z", "points3d");
  const int cr = t.need("red", "points3d"), cg = t.need("green", "points3d"), cb = t.need("blue", "points3d");
  const double scale = t.props[cr].integer ? 1.0 / 255 : 1.0;
  xyz.resize((size_t)t.count * 3);
  rgb.resize((size_t)t.count * 3);
  for (int64_t i = 0; i < t.count; ++i) {
    xyz[3 * i + 0] = (float)t.value(cx, i);
    xyz[3 * i + 1] = (float)t.value(cy, i);
    xyz[3 * i + 2] = (float)t.value(cz, i);
    rgb[3 * i + 0] = (float)(t.value(cr, i) * scale);
    rgb[3 * i + 1] = (float)(t.value(cg, i) * scale);
    rgb[3 * i + 2] = (float)(t.value(cb, i) * scale);
  }
}

// write_points_ply (ply.hpp:198-212)
void write_points(const std::string& path, const float* xyz, const float* rgb, int64_t n) {
  std::ofstream out(path, std::ios::binary);
  require(out.good(), "ply: cannot open '" + path + "' for writing");
  out << "ply\nformat binary_little_endian 1.0\nelement vertex " << n << "\n"
      << "property float x\nproperty float y\nproperty float z\n"
      << "property uchar red\nproperty uchar green\nproperty uchar blue\nend_header\n";
  std::vector<char> body((size_t)n * 15);
  for (int64_t i = 0; i < n; ++i) {
    char* r = body.data() + 15 * i;
    std::memcpy(r, xyz + 3 * i, 12);
    for (int c = 0; c < 3; ++c) {
      const double v = std::clamp((double)rgb[3 * i + c], 0.0, 1.0);
      r[12 + c] = (char)(uint8_t)std::lround(v * 255.0);
    }
  }
  out.write(body.data(), (std::streamsize)body.size());
  require(out.good(), "ply: write failed for '" + path + "'");
}

// ---------------------------------------------------------------------------
// PNG over zlib
// ---------------------------------------------------------------------------

void put_be32(std::vector<uint8_t>& v, uint32_t x) {
  v.push_back((uint8_t)(x >> 24));
  v.push_back((uint8_t)(x >> 16));
  v.push_back((uint8_t)(x >> 8));
  v.push_back((uint8_t)x);
}
uint32_t get_be32(const uint8_t* p) {
  return ((uint32_t)p[0] << 24) | ((uint32_t)p[1] << 16) | ((uint32_t)p[2] << 8) | p[3];
}

void png_chunk(std::vector<uint8_t>& out, const char* type, const uint8_t* data, size_t len) {
  put_be32(out, (uint32_t)len);
  const size_t start = out.size();
  out.insert(out.end(), type, type + 4);
  if (len) out.insert(out.end(), data, data + len);
  const uLong crc = crc32(0L, out.data() + start, (uInt)(len + 4));
  put_be32(out, (uint32_t)crc);
}

// write_png (png_io.cpp:74-104) from 8-bit RGB rows: filter byte 0 per row,
// zlib default compression.
void write_png_u8(const std::string& path, const uint8_t* rgb, int w, int h) {
  require(w > 0 && h > 0, "png: failed to encode '" + path + "'");
  std::vector<uint8_t> raw((size_t)h * (3 * (size_t)w + 1));
  for (int y = 0; y < h; ++y) {
    uint8_t* r = raw.data() + (size_t)y * (3 * (size_t)w + 1);
    r[0] = 0;
    std::memcpy(r + 1, rgb + (size_t)y * 3 * w, 3 * (size_t)w);
  }
  uLongf zlen = compressBound((uLong)raw.size());
  std::vector<uint8_t> z(zlen);
  require(compress2(z.data(), &zlen, raw.data(), (uLong)raw.size(), Z_DEFAULT_COMPRESSION) == Z_OK,
          "png: failed to encode '" + path + "'");
  std::vector<uint8_t> out = {0x89, 'P', 'N', 'G', '\r', '\n', 0x1a, '\n'};
  std::vector<uint8_t> ihdr;
  put_be32(ihdr, (uint32_t)w);
  put_be32(ihdr, (uint32_t)h);
  ihdr.insert(ihdr.end(), {8, 2, 0, 0, 0});  // 8-bit RGB, deflate, adaptive filtering, no interlace
  png_chunk(out, "IHDR", ihdr.data(), ihdr.size());
  png_chunk(out, "IDAT", z.data(), zlen);
  png_chunk(out, "IEND", nullptr, 0);
  std::FILE* f = std::fopen(path.c_str(), "wb");
  require(f != nullptr, "png: cannot open '" + path + "' for writing");
  const size_t wr = std::fwrite(out.data(), 1, out.size(), f);
  std::fclose(f);
  require(wr == out.size(), "png: failed to encode '" + path + "'");
}

int paeth(int a, int b, int c) {
  const int p = a + b - c;
  const int pa = std::abs(p - a), pb = std::abs(p - b), pc = std::abs(p - c);
  if (pa <= pb && pa <= pc) return a;
  if (pb <= pc) return b;
  return c;
}

// read_png (png_io.cpp:25-72) to 8-bit RGB; the float image is byte / 255.0f.
void read_png_u8(const std::string& path, std::vector<uint8_t>& rgb, int& w, int& h) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  require(f != nullptr, "png: cannot open '" + path + "'");
  std::vector<uint8_t> file;
  {
    uint8_t buf[1 << 16];
    size_t got;
    while ((got = std::fread(buf, 1, sizeof(buf), f)) > 0) file.insert(file.end(), buf, buf + got);
    std::fclose(f);
  }
  const std::string bad = "png: failed to decode '" + path + "'";
  static const uint8_t sig[8] = {0x89, 'P', 'N', 'G', '\r', '\n', 0x1a, '\n'};
  require(file.size() >= 8 && std::memcmp(file.data(), sig, 8) == 0, bad);
  size_t pos = 8;
  int depth = 0, ctype = -1, interlace = 0;
  std::vector<uint8_t> idat, palette;
  w = h = 0;
  while (pos + 12 <= file.size()) {
    const uint32_t len = get_be32(&file[pos]);
    require(pos + 12 + (size_t)len <= file.size(), bad);
    const char* type = reinterpret_cast<const char*>(&file[pos + 4]);
    const uint8_t* data = &file[pos + 8];
    if (!std::memcmp(type, "IHDR", 4)) {
      require(len >= 13, bad);
      w = (int)get_be32(data);
      h = (int)get_be32(data + 4);
      depth = data[8];
      ctype = data[9];
      interlace = data[12];
    } else if (!std::memcmp(type, "PLTE", 4)) {
      palette.assign(data, data + len);
    } else if (!std::memcmp(type, "IDAT", 4)) {
      idat.insert(idat.end(), data, data + len);
    } else if (!std::memcmp(type, "IEND", 4)) {
      break;
    }
    pos += 12 + len;
  }
  require(w > 0 && h > 0 && ctype >= 0, bad);
  require(interlace == 0, "png: interlaced images are not supported: '" + path + "'");
  int channels = 0;
  switch (ctype) {
    case 0: channels = 1; break;
    case 2: channels = 3; break;
    case 3: channels = 1; break;
    case 4: channels = 2; break;
    case 6: channels = 4; break;
    default: throw std::runtime_error(bad);
  }
  require(depth == 1 || depth == 2 || depth == 4 || depth == 8 || depth == 16, bad);
  require(ctype != 3 || !palette.empty(), bad);
  const size_t bpp_bits = (size_t)channels * depth;
  const size_t row_bytes = ((size_t)w * bpp_bits + 7) / 8;
  const size_t bpp = std::max<size_t>(1, bpp_bits / 8);
  std::vector<uint8_t> raw((size_t)h * (row_bytes + 1));
  uLongf rlen = (uLongf)raw.size();
  require(uncompress(raw.data(), &rlen, idat.data(), (uLong)idat.size()) == Z_OK && rlen == raw.size(), bad);
  // unfilter in place
  std::vector<uint8_t> prev(row_bytes, 0), cur(row_bytes);
  rgb.assign((size_t)w * h * 3, 0);
  for (int y = 0; y < h; ++y) {
    const uint8_t* src = raw.data() + (size_t)y * (row_bytes + 1);
    const int ft = src[0];
    for (size_t i = 0; i < row_bytes; ++i) {
      const int a = i >= bpp ? cur[i - bpp] : 0, b = prev[i], c = i >= bpp ? prev[i - bpp] : 0;
      int x = src[1 + i];
      switch (ft) {
        case 0: break;
        case 1: x += a; break;
        case 2: x += b; break;
        case 3: x += (a + b) / 2; break;
        case 4: x += paeth(a, b, c); break;
        default: throw std::runtime_error(bad);
      }
      cur[i] = (uint8_t)x;
    }
    // sample k of this row (channel-interleaved), reduced to 8 bits the way
    // the reference's libpng transforms do
    auto sample = [&](size_t k) -> int {
      if (depth == 8) return cur[k];
      if (depth == 16) return cur[2 * k];  // png_set_strip_16: high byte
      const size_t bit = k * depth;
      const int v = (cur[bit / 8] >> (8 - depth - (int)(bit % 8))) & ((1 << depth) - 1);
      return v;
    };
    uint8_t* dst = rgb.data() + (size_t)y * w * 3;
    for (int x = 0; x < w; ++x) {
      int r, g, b;
      if (ctype == 3) {
        const int idx = sample((size_t)x);
        require((size_t)(3 * idx + 2) < palette.size(), bad);
        r = palette[3 * idx];
        g = palette[3 * idx + 1];
        b = palette[3 * idx + 2];
      } else if (ctype == 0 || ctype == 4) {
        int v = sample((size_t)x * channels);
        if (depth < 8) v = v * (255 / ((1 << depth) - 1));  // png_set_expand_gray_1_2_4_to_8
        r = g = b = v;
      } else {
        r = sample((size_t)x * channels);
        g = sample((size_t)x * channels + 1);
        b = sample((size_t)x * channels + 2);
      }
      dst[3 * x] = (uint8_t)r;
      dst[3 * x + 1] = (uint8_t)g;
      dst[3 * x + 2] = (uint8_t)b;
    }
    std::swap(prev, cur);
  }
}

// ---------------------------------------------------------------------------
// cameras.json
// ---------------------------------------------------------------------------

struct Json {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  double num = 0.0;
  bool is_int = false;
  bool b = false;
  std::string str;
  std::vector<Json> arr;
  std::map<std::string, Json> obj;
};

struct JsonParser {
  const std::string& s;
  size_t p = 0;
  explicit JsonParser(const std::string& src) : s(src) {}
  [[noreturn]] void fail(const std::string& what) {
    throw std::runtime_error("dataset: malformed cameras.json: " + what + " at offset " + std::to_string(p));
  }
  void ws() {
    while (p < s.size() && (s[p] == ' ' || s[p] == '\n' || s[p] == '\r' || s[p] == '\t')) ++p;
  }
  bool lit(const char* w) {
    const size_t n = std::strlen(w);
    if (s.compare(p, n, w) == 0) {
      p += n;
      return true;
    }
    return false;
  }
  Json value() {
    ws();
    if (p >= s.size()) fail("unexpected end of input");
    Json j;
    const char c = s[p];
    if (c == '{') {
      j.kind = Json::Obj;
      ++p;
      ws();
      if (p < s.size() && s[p] == '}') {
        ++p;
        return j;
      }
      for (;;) {
        ws();
        if (p >= s.size() || s[p] != '"') fail("expected a key");
        std::string key = string();
        ws();
        if (p >= s.size() || s[p] != ':') fail("expected ':'");
        ++p;
        j.obj[key] = value();
        ws();
        if (p < s.size() && s[p] == ',') {
          ++p;
          continue;
        }
        if (p < s.size() && s[p] == '}') {
          ++p;
          return j;
        }
        fail("expected ',' or '}'");
      }
    }
    if (c == '[') {
      j.kind = Json::Arr;
      ++p;
      ws();
      if (p < s.size() && s[p] == ']') {
        ++p;
        return j;
      }
      for (;;) {
        j.arr.push_back(value());
        ws();
        if (p < s.size() && s[p] == ',') {
          ++p;
          continue;
        }
        if (p < s.size() && s[p] == ']') {
          ++p;
          return j;
        }
        fail("expected ',' or ']'");
      }
    }
    if (c == '"') {
      j.kind = Json::Str;
      j.str = string();
      return j;
    }
    if (lit("true")) {
      j.kind = Json::Bool;
      j.b = true;
      return j;
    }
    if (lit("false")) {
      j.kind = Json::Bool;
      return j;
    }
    if (lit("null")) return j;
    // number
    const size_t start = p;
    if (s[p] == '-') ++p;
    bool frac = false;
    while (p < s.size() && (std::isdigit((unsigned char)s[p]) || s[p] == '.' || s[p] == 'e' || s[p] == 'E' ||
                            s[p] == '+' || s[p] == '-')) {
      frac = frac || s[p] == '.' || s[p] == 'e' || s[p] == 'E';
      ++p;
    }
    if (p == start) fail("unexpected character");
    j.kind = Json::Num;
    j.is_int = !frac;
    char* end = nullptr;
    const std::string tok = s.substr(start, p - start);
    j.num = std::strtod(tok.c_str(), &end);
    if (end != tok.c_str() + tok.size()) fail("bad number '" + tok + "'");
    return j;
  }
  std::string string() {
    ++p;  // opening quote
    std::string out;
    while (p < s.size() && s[p] != '"') {
      if (s[p] == '\\') {
        ++p;
        if (p >= s.size()) fail("bad escape");
        const char e = s[p];
        out.push_back(e == 'n' ? '\n' : e == 't' ? '\t' : e == 'r' ? '\r' : e == 'b' ? '\b' : e == 'f' ? '\f' : e);
        if (e == 'u') fail("unicode escapes are not supported");
      } else {
        out.push_back(s[p]);
      }
      ++p;
    }
    if (p >= s.size()) fail("unterminated string");
    ++p;
    return out;
  }
};

// Camera::validate (camera.hpp:34-42) in float, Frobenius norm of R R^T - I.
void validate_camera(const sk_camera& c) {
  require(c.fx > 0.0f && c.fy > 0.0f, "camera: focal lengths must be positive");
  require(c.width > 0 && c.height > 0, "camera: empty image");
  float r[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r[3 * i + j] = c.world_to_cam[4 * i + j];
  float fro = 0.0f;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      float d = r[3 * i] * r[3 * j];
      d = d + r[3 * i + 1] * r[3 * j + 1];
      d = d + r[3 * i + 2] * r[3 * j + 2];
      d = d - (i == j ? 1.0f : 0.0f);
      fro = fro + d * d;
    }
  require(std::sqrt(fro) < 1e-6f, "camera: world_to_cam rotation block is not orthonormal");
  const float det = r[0] * (r[4] * r[8] - r[5] * r[7]) - r[1] * (r[3] * r[8] - r[5] * r[6]) +
                    r[2] * (r[3] * r[7] - r[4] * r[6]);
  require(std::fabs(det - 1.0f) < 1e-6f, "camera: world_to_cam rotation block must have det +1");
}

// load side of load_dataset (dataset.hpp:80-107)
void read_cameras(const std::string& path, std::vector<sk_camera>& cams, std::vector<int>& ids) {
  std::ifstream in(path, std::ios::binary);
  require(in.good(), "dataset: cannot read " + path);
  const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  JsonParser jp(text);
  const Json doc = jp.value();
  require(doc.kind == Json::Arr, "dataset: cameras.json must be an array of camera records");
  for (const Json& rec : doc.arr) {
    for (const char* key : {"id", "width", "height", "fx", "fy", "cx", "cy", "world_to_cam"})
      require(rec.kind == Json::Obj && rec.obj.count(key),
              std::string("dataset: camera record missing key '") + key + "'");
    auto num = [&](const char* key) {
      const Json& v = rec.obj.at(key);
      require(v.kind == Json::Num, std::string("dataset: malformed cameras.json: '") + key + "' is not a number");
      return v.num;
    };
    sk_camera c{};
    c.width = (int)num("width");
    c.height = (int)num("height");
    c.fx = (float)num("fx");
    c.fy = (float)num("fy");
    c.cx = (float)num("cx");
    c.cy = (float)num("cy");
    c.near_plane = 0.2f;
    const Json& m = rec.obj.at("world_to_cam");
    require(m.kind == Json::Arr && m.arr.size() == 16, "dataset: world_to_cam must hold 16 floats");
    for (int i = 0; i < 16; ++i) {
      require(m.arr[i].kind == Json::Num, "dataset: world_to_cam must hold 16 floats");
      c.world_to_cam[i] = (float)m.arr[i].num;
    }
    validate_camera(c);
    cams.push_back(c);
    ids.push_back((int)num("id"));
  }
  require(!cams.empty(), "dataset: cameras.json contains no cameras");
}

// Shortest decimal that round-trips the double, with a ".0" on integral
// values — the way nlohmann::json::dump prints floating-point numbers.
std::string json_double(double v) {
  char buf[64];
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof(buf), "%.*g", prec, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  std::string s(buf);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

// save_cameras_json (dataset.hpp:127-150) in dump(2) layout with the keys in
// nlohmann's (sorted) object order.
void write_cameras(const std::string& path, const sk_camera* cams, const int* ids, int n) {
  std::ofstream out(path, std::ios::binary);
  require(out.good(), "dataset: cannot write " + path);
  out << "[";
  for (int i = 0; i < n; ++i) {
    const sk_camera& c = cams[i];
    out << (i ? ",\n" : "\n") << "  {\n";
    out << "    \"cx\": " << json_double((double)c.cx) << ",\n";
    out << "    \"cy\": " << json_double((double)c.cy) << ",\n";
    out << "    \"fx\": " << json_double((double)c.fx) << ",\n";
    out << "    \"fy\": " << json_double((double)c.fy) << ",\n";
    out << "    \"height\": " << c.height << ",\n";
    out << "    \"id\": " << ids[i] << ",\n";
    out << "    \"width\": " << c.width << ",\n";
    out << "    \"world_to_cam\": [";
    for (int k = 0; k < 16; ++k)
      out << (k ? ",\n" : "\n") << "      " << json_double((double)c.world_to_cam[k]);
    out << "\n    ]\n  }";
  }
  out << (n ? "\n]" : "]") << "\n";
  require(out.good(), "dataset: cannot write " + path);
}

std::string image_name(int id) {
  char buf[32];
  std::snprintf(buf, sizeof(buf), "%05d.png", id);
  return buf;
}

// scene_extent (dataset.hpp:57-69) in float: centre = mean camera centre,
// radius = 1.1 x the largest distance of a camera centre or point to it.
float scene_extent(const std::vector<sk_camera>& cams, const std::vector<float>& xyz) {
  float cen[3] = {0.0f, 0.0f, 0.0f};
  std::vector<CamParams> cp;
  for (const auto& c : cams) cp.push_back(make_cam_params(c));
  for (const auto& p : cp)
    for (int d = 0; d < 3; ++d) cen[d] = cen[d] + p.center[d];
  if (!cams.empty())
    for (int d = 0; d < 3; ++d) cen[d] = cen[d] / (float)cams.size();
  auto dist = [&](const float* q) {
    float s = 0.0f;
    for (int d = 0; d < 3; ++d) s = s + (q[d] - cen[d]) * (q[d] - cen[d]);
    return std::sqrt(s);
  };
  float radius = 0.0f;
  for (const auto& p : cp) radius = std::max(radius, dist(p.center));
  for (size_t i = 0; i + 2 < xyz.size(); i += 3) radius = std::max(radius, dist(&xyz[i]));
  radius = radius * 1.1f;
  return radius > 1e-9f ? radius : 1.0f;
}

}  // namespace io
}  // namespace sk

using namespace sk;

extern "C" {

int sk_checkpoint_save(sk_ctx* ctx, const sk_scene* scene, const char* path) {
  return guarded(ctx, [&] {
    arg(scene && path, "checkpoint: null argument");
    SK_CUDA(cudaSetDevice(ctx->device));
    io::save_checkpoint(ctx, scene, path);
  });
}

int sk_checkpoint_load(sk_ctx* ctx, const char* path, int64_t capacity, sk_scene** out) {
  return guarded(ctx, [&] {
    arg(path && out, "checkpoint: null argument");
    SK_CUDA(cudaSetDevice(ctx->device));
    *out = io::load_checkpoint(ctx, path, capacity);
  });
}

int sk_points_read(sk_ctx* ctx, const char* path, float* xyz, float* rgb, int64_t* count) {
  return guarded(ctx, [&] {
    arg(path && count, "ply: null argument");
    std::vector<float> p, c;
    io::read_points(path, p, c);
    const int64_t n = (int64_t)(p.size() / 3);
    if (xyz && rgb) {
      arg(*count >= n, "ply: output buffer too small");
      std::copy(p.begin(), p.end(), xyz);
      std::copy(c.begin(), c.end(), rgb);
    }
    *count = n;
  });
}

int sk_points_write(sk_ctx* ctx, const char* path, const float* xyz, const float* rgb, int64_t n) {
  return guarded(ctx, [&] {
    arg(path && n >= 0 && (n == 0 || (xyz && rgb)), "ply: null argument");
    io::write_points(path, xyz, rgb, n);
  });
}

int sk_png_read(sk_ctx* ctx, const char* path, uint8_t* rgb, int* width, int* height) {
  return guarded(ctx, [&] {
    arg(path && width && height, "png: null argument");
    std::vector<uint8_t> img;
    int w = 0, h = 0;
    io::read_png_u8(path, img, w, h);
    if (rgb) {
      arg(*width == w && *height == h, "png: output buffer size differs from the image");
      std::copy(img.begin(), img.end(), rgb);
    }
    *width = w;
    *height = h;
  });
}

int sk_png_write(sk_ctx* ctx, const char* path, const float* rgb, int width, int height) {
  return guarded(ctx, [&] {
    arg(path && rgb && width > 0 && height > 0, "png: null argument");
    std::vector<uint8_t> q((size_t)width * height * 3);
    for (size_t i = 0; i < q.size(); ++i)
      q[i] = (uint8_t)std::lround(std::clamp(rgb[i], 0.0f, 1.0f) * 255.0f);  // png_io.cpp:97-98
    io::write_png_u8(path, q.data(), width, height);
  });
}

int sk_png_write_u8(sk_ctx* ctx, const char* path, const uint8_t* rgb, int width, int height) {
  return guarded(ctx, [&] {
    arg(path && rgb && width > 0 && height > 0, "png: null argument");
    io::write_png_u8(path, rgb, width, height);
  });
}

int sk_cameras_read(sk_ctx* ctx, const char* path, sk_camera* cams, int32_t* ids, int* count) {
  return guarded(ctx, [&] {
    arg(path && count, "dataset: null argument");
    std::vector<sk_camera> cv;
    std::vector<int> iv;
    io::read_cameras(path, cv, iv);
    if (cams) {
      arg(*count >= (int)cv.size(), "dataset: output buffer too small");
      std::copy(cv.begin(), cv.end(), cams);
      if (ids) std::copy(iv.begin(), iv.end(), ids);
    }
    *count = (int)cv.size();
  });
}

int sk_cameras_write(sk_ctx* ctx, const char* path, const sk_camera* cams, const int32_t* ids, int n) {
  return guarded(ctx, [&] {
    arg(path && n >= 0 && (n == 0 || (cams && ids)), "dataset: null argument");
    io::write_cameras(path, cams, ids, n);
  });
}

int sk_dataset_load(sk_ctx* ctx, const char* dir, sk_dataset** out) {
  return guarded(ctx, [&] {
    arg(dir && out, "dataset: null argument");
    SK_CUDA(cudaSetDevice(ctx->device));
    const io::fs::path root(dir);
    require(io::fs::exists(root / "cameras.json"), "dataset: missing " + (root / "cameras.json").string());
    require(io::fs::exists(root / "points3d.ply"), "dataset: missing " + (root / "points3d.ply").string());
    std::vector<sk_camera> cams;
    std::vector<int> ids;
    io::read_cameras((root / "cameras.json").string(), cams, ids);
    auto d = std::make_unique<sk_dataset>();
    // decode the PNGs on host worker threads (independent files), then upload
    // in view order; errors are reported for the first failing view, as the
    // reference's sequential loop would
    const size_t nv = cams.size();
    std::vector<std::vector<uint8_t>> rgb(nv);
    std::vector<std::string> errs(nv);
    std::atomic<size_t> next{0};
    auto worker = [&] {
      for (size_t v; (v = next.fetch_add(1)) < nv;) {
        try {
          const io::fs::path img = root / "images" / io::image_name(ids[v]);
          require(io::fs::exists(img), "dataset: missing image " + img.string());
          int w = 0, h = 0;
          io::read_png_u8(img.string(), rgb[v], w, h);
          require(w == cams[v].width && h == cams[v].height,
                  "dataset: image " + img.string() + " is " + std::to_string(w) + "x" + std::to_string(h) +
                      " but camera " + std::to_string(ids[v]) + " expects " + std::to_string(cams[v].width) + "x" +
                      std::to_string(cams[v].height));
        } catch (const std::exception& e) {
          errs[v] = e.what();
        }
      }
    };
    const size_t nt = std::min<size_t>(nv, std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
    std::vector<std::thread> pool;
    for (size_t t = 1; t < nt; ++t) pool.emplace_back(worker);
    worker();
    for (auto& t : pool) t.join();
    for (size_t v = 0; v < nv; ++v) require(errs[v].empty(), errs[v]);
    for (size_t v = 0; v < nv; ++v) {
      auto buf = std::make_unique<DevBuf>();
      buf->ensure(rgb[v].size());
      h2d(ctx, buf->ptr, rgb[v].data(), rgb[v].size());
      d->cams.push_back(cams[v]);
      d->images.push_back(std::move(buf));
    }
    sync(ctx);  // the host images are pageable temporaries
    io::read_points((root / "points3d.ply").string(), d->init_xyz, d->init_rgb);
    d->ids = ids;
    // split_views (dataset.hpp:44-53)
    const int n = (int)cams.size();
    for (int i = 0; i < n; ++i)
      if (i % 8 != 0) d->train.push_back(i);
    if (d->train.empty())
      for (int i = 0; i < n; ++i) d->train.push_back(i);
    d->extent = io::scene_extent(cams, d->init_xyz);
    *out = d.release();
  });
}

int sk_dataset_init_points(const sk_dataset* d, float* xyz, float* rgb, int64_t* count) {
  if (!d || !count) return SK_ERR_INVALID_ARGUMENT;
  const int64_t n = (int64_t)(d->init_xyz.size() / 3);
  if (xyz && rgb) {
    if (*count < n) return SK_ERR_INVALID_ARGUMENT;
    std::copy(d->init_xyz.begin(), d->init_xyz.end(), xyz);
    std::copy(d->init_rgb.begin(), d->init_rgb.end(), rgb);
  }
  *count = n;
  return SK_OK;
}

int sk_dataset_save(sk_ctx* ctx, const sk_dataset* d, const char* dir) {
  return guarded(ctx, [&] {
    arg(d && dir, "dataset: null argument");
    SK_CUDA(cudaSetDevice(ctx->device));
    const io::fs::path root(dir);
    io::fs::create_directories(root / "images");
    std::vector<int> ids = d->ids;
    if (ids.size() != d->cams.size()) {
      ids.resize(d->cams.size());
      for (size_t v = 0; v < ids.size(); ++v) ids[v] = (int)v;
    }
    io::write_cameras((root / "cameras.json").string(), d->cams.data(), ids.data(), (int)d->cams.size());
    for (size_t v = 0; v < d->cams.size(); ++v) {
      const sk_camera& c = d->cams[v];
      std::vector<uint8_t> rgb((size_t)c.width * c.height * 3);
      d2h(ctx, rgb.data(), d->images[v]->ptr, rgb.size());
      sync(ctx);
      io::write_png_u8((root / "images" / io::image_name(ids[v])).string(), rgb.data(), c.width, c.height);
    }
    io::write_points((root / "points3d.ply").string(), d->init_xyz.data(), d->init_rgb.data(),
                     (int64_t)(d->init_xyz.size() / 3));
  });
}

}  // extern "C"
