// ply.cu — native reader for 3DGS binary PLY scenes (SPEC.md:51-59
// load_splat_ply).  Host code only.
//
// Layout (the de-facto 3DGS format): element vertex with properties
// x,y,z, [nx,ny,nz], f_dc_0..2, f_rest_0..(3*((d+1)^2-1)-1), opacity,
// scale_0..2, rot_0..3; binary_little_endian.  Activations:
// scale = exp(scale_i), opacity = sigmoid(opacity), quaternion (w,x,y,z) =
// rot_0..3 (normalised by gg_load_scene).  f_rest is stored channel-major
// (f_rest[c*(K-1) + k-1] is coefficient k of channel c); the output SH array
// is [n, K, 3] coefficient-major.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "gg.h"

namespace {

struct Prop {
  std::string name;
  int type;      // 0 f32, 1 f64, 2 u8, 3 i8, 4 u16, 5 i16, 6 u32, 7 i32
  int offset;
};

int type_of(const std::string& t, int* size) {
  static const std::map<std::string, std::pair<int, int>> m = {
      {"float", {0, 4}}, {"float32", {0, 4}}, {"double", {1, 8}}, {"float64", {1, 8}},
      {"uchar", {2, 1}}, {"uint8", {2, 1}}, {"char", {3, 1}}, {"int8", {3, 1}},
      {"ushort", {4, 2}}, {"uint16", {4, 2}}, {"short", {5, 2}}, {"int16", {5, 2}},
      {"uint", {6, 4}}, {"uint32", {6, 4}}, {"int", {7, 4}}, {"int32", {7, 4}}};
  auto it = m.find(t);
  if (it == m.end()) return -1;
  *size = it->second.second;
  return it->second.first;
}

double read_as(const unsigned char* p, int type) {
  switch (type) {
    case 0: { float v; std::memcpy(&v, p, 4); return v; }
    case 1: { double v; std::memcpy(&v, p, 8); return v; }
    case 2: return *p;
    case 3: return (signed char)*p;
    case 4: { uint16_t v; std::memcpy(&v, p, 2); return v; }
    case 5: { int16_t v; std::memcpy(&v, p, 2); return v; }
    case 6: { uint32_t v; std::memcpy(&v, p, 4); return v; }
    case 7: { int32_t v; std::memcpy(&v, p, 4); return v; }
  }
  return 0.0;
}

thread_local std::string g_ply_err;

gg_status perr(const char* fmt, const char* a = "", long long b = 0) {
  char buf[512];
  snprintf(buf, sizeof buf, fmt, a, b);
  g_ply_err = buf;
  return GG_E_INVALID;
}

}  // namespace

extern "C" {

const char* gg_ply_error(void) { return g_ply_err.c_str(); }

gg_status gg_read_ply(const char* path, int64_t* out_n, int32_t* out_degree, float* means, float* scales,
                      float* quats, float* opacities, float* sh) {
  if (!path || !out_n || !out_degree) return perr("gg_read_ply: null argument%s", "");
  std::ifstream f(path, std::ios::binary);
  if (!f) return perr("gg_read_ply: cannot open %s", path);
  std::string line;
  std::getline(f, line);
  if (line.rfind("ply", 0) != 0) return perr("gg_read_ply: %s is not a PLY file", path);
  bool in_vertex = false, seen_vertex = false;
  long long nv = -1;
  int stride = 0;
  std::vector<Prop> props;
  std::string format;
  while (std::getline(f, line)) {
    if (!line.empty() && line.back() == '\r') line.pop_back();
    std::istringstream ss(line);
    std::string kw;
    ss >> kw;
    if (kw == "format") {
      ss >> format;
    } else if (kw == "element") {
      std::string name;
      long long cnt;
      ss >> name >> cnt;
      in_vertex = name == "vertex";
      if (in_vertex) { nv = cnt; seen_vertex = true; }
      else if (!seen_vertex) return perr("gg_read_ply: element '%s' before vertex is not supported", name.c_str());
    } else if (kw == "property" && in_vertex) {
      std::string t, name;
      ss >> t;
      if (t == "list") return perr("gg_read_ply: list property in vertex element%s", "");
      ss >> name;
      int sz = 0;
      const int ty = type_of(t, &sz);
      if (ty < 0) return perr("gg_read_ply: unknown property type %s", t.c_str());
      props.push_back({name, ty, stride});
      stride += sz;
    } else if (kw == "end_header") {
      break;
    }
  }
  if (format != "binary_little_endian") return perr("gg_read_ply: format '%s' unsupported (need binary_little_endian)", format.c_str());
  if (nv <= 0) return perr("gg_read_ply: empty file (%s)", path);   // SPEC.md:55 "empty file -> error"
  std::map<std::string, const Prop*> by;
  for (const auto& p : props) by[p.name] = &p;
  const char* req[] = {"x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2", "opacity", "scale_0", "scale_1", "scale_2",
                       "rot_0", "rot_1", "rot_2", "rot_3"};
  for (const char* r : req)
    if (!by.count(r)) return perr("gg_read_ply: missing property '%s'", r);
  int nrest = 0;
  while (by.count("f_rest_" + std::to_string(nrest))) ++nrest;
  int d = 0;
  while (d <= 3 && 3 * ((d + 1) * (d + 1) - 1) != nrest) ++d;
  if (d > 3) return perr("gg_read_ply: %s f_rest count does not match an SH degree 0..3", "", nrest);
  *out_n = nv;
  *out_degree = d;
  if (!means || !scales || !quats || !opacities || !sh) return GG_OK;   // size query
  const int K = (d + 1) * (d + 1);
  std::vector<unsigned char> rec((size_t)stride);
  auto get = [&](const char* name) { const Prop* p = by[name]; return read_as(rec.data() + p->offset, p->type); };
  std::vector<const Prop*> rest(nrest);
  for (int i = 0; i < nrest; ++i) rest[i] = by["f_rest_" + std::to_string(i)];
  for (long long i = 0; i < nv; ++i) {
    if (!f.read(reinterpret_cast<char*>(rec.data()), stride))
      return perr("gg_read_ply: truncated file at record %s%lld", "", i);
    double v[14];
    for (int k = 0; k < 14; ++k) v[k] = get(req[k]);
    for (int k = 0; k < 14; ++k)
      if (!std::isfinite(v[k])) return perr("gg_read_ply: non-finite value in record %s%lld", "", i);
    means[i * 3 + 0] = (float)v[0]; means[i * 3 + 1] = (float)v[1]; means[i * 3 + 2] = (float)v[2];
    sh[i * K * 3 + 0] = (float)v[3]; sh[i * K * 3 + 1] = (float)v[4]; sh[i * K * 3 + 2] = (float)v[5];
    opacities[i] = (float)(1.0 / (1.0 + std::exp(-v[6])));
    scales[i * 3 + 0] = (float)std::exp(v[7]);
    scales[i * 3 + 1] = (float)std::exp(v[8]);
    scales[i * 3 + 2] = (float)std::exp(v[9]);
    quats[i * 4 + 0] = (float)v[10]; quats[i * 4 + 1] = (float)v[11];
    quats[i * 4 + 2] = (float)v[12]; quats[i * 4 + 3] = (float)v[13];
    for (int c = 0; c < 3; ++c)
      for (int k = 1; k < K; ++k) {
        const double x = read_as(rec.data() + rest[c * (K - 1) + (k - 1)]->offset, rest[c * (K - 1) + (k - 1)]->type);
        if (!std::isfinite(x)) return perr("gg_read_ply: non-finite value in record %s%lld", "", i);
        sh[(i * K + k) * 3 + c] = (float)x;
      }
  }
  return GG_OK;
}

gg_status gg_load_ply(gg_context* ctx, const char* path, int32_t* out_scene_id) {
  int64_t n = 0;
  int32_t d = 0;
  gg_status s = gg_read_ply(path, &n, &d, nullptr, nullptr, nullptr, nullptr, nullptr);
  if (s != GG_OK) return s;
  const int K = (d + 1) * (d + 1);
  std::vector<float> m(n * 3), sc(n * 3), q(n * 4), o(n), sh((size_t)n * K * 3);
  s = gg_read_ply(path, &n, &d, m.data(), sc.data(), q.data(), o.data(), sh.data());
  if (s != GG_OK) return s;
  return gg_load_scene(ctx, n, d, m.data(), sc.data(), q.data(), o.data(), sh.data(), out_scene_id);
}

}  // extern "C"
