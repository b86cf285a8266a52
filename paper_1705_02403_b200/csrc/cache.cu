// cache.cu -- interop with the reference's binary graph cache ("GMTG" v1,
// graph.cpp:190-343) and its cache key (problem_key, problem.cpp:281-303),
// a graph built on the GPU can be handed to the
// reference's `--graph-cache` and a reference-built cache file can seed a
// device instance.  Host code: the format is bytes on disk.
//
// Layout (all little-endian): "GMTG", u32 version = 1, u64 problem key,
// u32 n, f64 radius, u8 model (1 = dubins_airplane), f64 rho, f64
// discretization_step (the raw field), u8 planar_cost_only, then per sample
// u: u32 count, count x (u32 target, f64 cost) with strictly increasing
// targets != u; nothing after.  Writes go to `file.tmp` and are renamed into
// place (graph.cpp:262-275).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "gmt_b200.h"
#include "internal.cuh"
#include "offline.cuh"

namespace gmtb {

namespace {

constexpr char kMagic[4] = {'G', 'M', 'T', 'G'};
constexpr uint32_t kVersion = 1;
// Euclidean SteeringModel defaults (steering.hpp:12-22): rho = 0.1, step()
// = rho / 10, planar_cost_only = false.
constexpr double kRho = 0.1;

uint64_t mix64(uint64_t x) {  // splitmix64 (rng.hpp:68-73)
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
uint64_t fold(uint64_t h, uint64_t x) { return mix64(mix64(h) ^ x); }  // mix64(a, b), rng.hpp:75
uint64_t fold_f(uint64_t h, double x) {
  uint64_t b;
  std::memcpy(&b, &x, 8);
  return fold(h, b);
}

void put_u32(std::string& b, uint32_t v) {
  for (int i = 0; i < 4; ++i) b.push_back(static_cast<char>((v >> (8 * i)) & 0xff));
}
void put_u64(std::string& b, uint64_t v) {
  for (int i = 0; i < 8; ++i) b.push_back(static_cast<char>((v >> (8 * i)) & 0xff));
}
void put_f64(std::string& b, double v) {
  uint64_t bits;
  std::memcpy(&bits, &v, 8);
  put_u64(b, bits);
}

struct Cursor {
  const unsigned char* p;
  size_t left;
  bool u8(uint8_t& v) {
    if (left < 1) return false;
    v = *p++;
    --left;
    return true;
  }
  bool u32(uint32_t& v) {
    if (left < 4) return false;
    v = 0;
    for (int i = 0; i < 4; ++i) v |= static_cast<uint32_t>(p[i]) << (8 * i);
    p += 4;
    left -= 4;
    return true;
  }
  bool u64(uint64_t& v) {
    if (left < 8) return false;
    v = 0;
    for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(p[i]) << (8 * i);
    p += 8;
    left -= 8;
    return true;
  }
  bool f64(double& v) {
    uint64_t b;
    if (!u64(b)) return false;
    std::memcpy(&v, &b, 8);
    return true;
  }
};

}  // namespace

CacheModel cache_model_of(const gmt_problem* p) {
  CacheModel m;
  if (p->steering == GMT_STEER_DUBINS_AIRPLANE) {
    m.dubins = 1;
    m.rho = p->dubins.rho;
    m.step_raw = p->dubins.discretization_step;
    m.planar = p->dubins.planar_cost_only != 0 ? 1 : 0;
  } else {
    m.rho = kRho;
  }
  return m;
}

int problem_key_of(const gmt_problem* p, uint64_t* out) {
  if (!p || !out) return set_error(GMT_E_INVALID_INPUT, "problem_key: null argument");
  if (p->steering != GMT_STEER_EUCLIDEAN && p->steering != GMT_STEER_DUBINS_AIRPLANE)
    return set_error(GMT_E_INVALID_INPUT,
                     "the graph cache covers the reference's steering models (Euclidean, Dubins airplane)");
  const CacheModel m = cache_model_of(p);
  const gmt_scene& s = p->scene;
  const int d = s.dim;
  uint64_t h = mix64(0x676d742d70726f62ULL);  // stable salt (problem.cpp:282)
  h = fold(h, static_cast<uint64_t>(d));
  h = fold(h, static_cast<uint64_t>(m.dubins));  // SteeringModel::Kind (steering.hpp:10)
  h = fold_f(h, m.rho);
  h = fold_f(h, m.step_raw > 0.0 ? m.step_raw : m.rho / 10.0);  // step() (steering.hpp:22)
  h = fold(h, static_cast<uint64_t>(m.planar));
  h = fold(h, static_cast<uint64_t>(s.num_boxes));
  for (int b = 0; b < s.num_boxes; ++b) {
    for (int k = 0; k < d; ++k) h = fold_f(h, s.box_lo[static_cast<size_t>(b) * d + k]);
    for (int k = 0; k < d; ++k) h = fold_f(h, s.box_hi[static_cast<size_t>(b) * d + k]);
  }
  for (int k = 0; k < d; ++k) h = fold_f(h, p->init[k]);
  h = fold_f(h, p->init_has_heading ? p->init_heading : -1.0);
  for (int k = 0; k < d; ++k) h = fold_f(h, s.goal_lo[k]);
  for (int k = 0; k < d; ++k) h = fold_f(h, s.goal_hi[k]);
  h = fold(h, static_cast<uint64_t>(static_cast<int64_t>(p->n)));
  h = fold(h, static_cast<uint64_t>(p->sampling.kind));
  h = fold(h, p->sampling.start_index);
  h = fold(h, p->sampling.seed);
  // load_problem sets with_heading exactly for Dubins problems (problem.cpp:197)
  h = fold(h, static_cast<uint64_t>(p->sampling.with_heading != 0 || m.dubins));
  *out = h;
  return GMT_OK;
}

int cache_write(const char* file, uint64_t key, int32_t n, double radius, const int64_t* ptr,
                const int32_t* col, const double* cost, const CacheModel& m) {
  if (!file) return set_error(GMT_E_INVALID_INPUT, "graph cache: null file name");
  std::string b;
  b.reserve(41 + static_cast<size_t>(n) * 4 + static_cast<size_t>(ptr[n]) * 12);
  b.append(kMagic, 4);
  put_u32(b, kVersion);
  put_u64(b, key);
  put_u32(b, static_cast<uint32_t>(n));
  put_f64(b, radius);
  b.push_back(static_cast<char>(m.dubins ? 1 : 0));
  put_f64(b, m.rho);
  put_f64(b, m.step_raw);  // the raw discretization_step field (0 = rho / 10), not step()
  b.push_back(static_cast<char>(m.planar ? 1 : 0));
  for (int32_t u = 0; u < n; ++u) {
    put_u32(b, static_cast<uint32_t>(ptr[u + 1] - ptr[u]));
    for (int64_t e = ptr[u]; e < ptr[u + 1]; ++e) {
      put_u32(b, static_cast<uint32_t>(col[e]));
      put_f64(b, cost[e]);
    }
  }
  const std::string tmp = std::string(file) + ".tmp";
  std::FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) return set_error(GMT_E_IO, std::string("graph cache: cannot open ") + tmp);
  bool ok = std::fwrite(b.data(), 1, b.size(), f) == b.size();
  ok = (std::fclose(f) == 0) && ok;
  if (!ok || std::rename(tmp.c_str(), file) != 0) {
    std::remove(tmp.c_str());
    return set_error(GMT_E_IO, std::string("graph cache: cannot write ") + file);
  }
  return GMT_OK;
}

int cache_read(const char* file, uint64_t key, int32_t n, double radius, std::vector<int64_t>& ptr,
               std::vector<int32_t>& col, std::vector<double>& cost, bool* hit, const CacheModel& m) {
  *hit = false;
  if (!file) return set_error(GMT_E_INVALID_INPUT, "graph cache: null file name");
  std::FILE* f = std::fopen(file, "rb");
  if (!f) return GMT_OK;  // a missing file is a miss (graph.cpp:281-282)
  std::string data;
  char chunk[1 << 16];
  size_t got;
  while ((got = std::fread(chunk, 1, sizeof(chunk), f)) > 0) data.append(chunk, got);
  std::fclose(f);
  Cursor r{reinterpret_cast<const unsigned char*>(data.data()), data.size()};
  if (r.left < 4 || std::memcmp(r.p, kMagic, 4) != 0) return GMT_OK;
  r.p += 4;
  r.left -= 4;
  uint32_t version, nn;
  uint64_t k;
  double rad, rho, step;
  uint8_t kind, planar;
  if (!r.u32(version) || version != kVersion) return GMT_OK;
  if (!r.u64(k) || k != key) return GMT_OK;
  if (!r.u32(nn) || nn != static_cast<uint32_t>(n)) return GMT_OK;
  if (!r.f64(rad) || rad != radius) return GMT_OK;
  if (!r.u8(kind) || (kind == 1) != (m.dubins != 0)) return GMT_OK;  // the model kind must match
  if (!r.f64(rho) || !r.f64(step) || !r.u8(planar)) return GMT_OK;
  if (m.dubins && (rho != m.rho || step != m.step_raw || (planar != 0) != (m.planar != 0)))
    return GMT_OK;  // graph.cpp:317-320
  ptr.assign(static_cast<size_t>(n) + 1, 0);
  col.clear();
  cost.clear();
  for (uint32_t u = 0; u < nn; ++u) {
    uint32_t cnt;
    if (!r.u32(cnt)) return GMT_OK;
    int64_t prev = -1;
    for (uint32_t j = 0; j < cnt; ++j) {
      uint32_t t;
      double c;
      if (!r.u32(t) || !r.f64(c)) return GMT_OK;
      if (t >= nn || static_cast<int64_t>(t) <= prev || t == u) return GMT_OK;
      prev = t;
      col.push_back(static_cast<int32_t>(t));
      cost.push_back(c);
    }
    ptr[u + 1] = static_cast<int64_t>(col.size());
  }
  if (r.left != 0) return GMT_OK;
  *hit = true;
  return GMT_OK;
}

}  // namespace gmtb

using namespace gmtb;

extern "C" int gmt_problem_key(const gmt_problem* problem, uint64_t* key_out) {
  return problem_key_of(problem, key_out);
}

extern "C" int gmt_graph_cache_save(const char* file, uint64_t key, int32_t n, double radius,
                                    const int64_t* row_ptr, const int32_t* col, const double* cost) {
  if (n < 0 || !row_ptr || (row_ptr[n] > 0 && (!col || !cost)))
    return set_error(GMT_E_INVALID_INPUT, "graph cache: invalid graph arrays");
  return cache_write(file, key, n, radius, row_ptr, col, cost);
}

extern "C" int gmt_graph_cache_load(const char* file, uint64_t key, int32_t n, double radius,
                                    int32_t* hit, int64_t* num_edges, int64_t edge_capacity,
                                    int64_t* row_ptr, int32_t* col, double* cost) {
  std::vector<int64_t> p;
  std::vector<int32_t> c;
  std::vector<double> w;
  bool h = false;
  int rc = cache_read(file, key, n, radius, p, c, w, &h);
  if (rc) return rc;
  *hit = h ? 1 : 0;
  *num_edges = h ? static_cast<int64_t>(c.size()) : 0;
  if (h && row_ptr) {
    // The file may have been replaced since the caller sized its buffers
    // (the reference renames files into place): never write past them.
    if (static_cast<int64_t>(c.size()) > edge_capacity)
      return set_error(GMT_E_INVALID_INPUT, "graph cache: the file holds " + std::to_string(c.size()) +
                                                " edges, more than the " + std::to_string(edge_capacity) +
                                                " the buffers hold");
    std::memcpy(row_ptr, p.data(), sizeof(int64_t) * p.size());
    if (!c.empty()) {
      std::memcpy(col, c.data(), sizeof(int32_t) * c.size());
      std::memcpy(cost, w.data(), sizeof(double) * w.size());
    }
  }
  return GMT_OK;
}

extern "C" int gmt_instance_cache_save(gmt_ctx* ctx, const gmt_instance* inst, const char* file,
                                       uint64_t key) {
  gmtb::AllocScope alloc_scope_(ctx);
  const DevInstance& D = inst->desc;
  if (D.directed && D.steering != GMT_STEER_DUBINS_AIRPLANE)
    return set_error(GMT_E_INVALID_INPUT,
                     "the graph cache covers the reference's steering models (Euclidean, Dubins airplane)");
  const int n = D.n;
  std::vector<int64_t> p(static_cast<size_t>(n) + 1);
  cudaStream_t s = ctx->stream;
  cudaError_t e = cudaMemcpyAsync(p.data(), D.out_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_error(e, "graph cache download");
  const size_t E = static_cast<size_t>(p[n]);
  std::vector<int32_t> c(E);
  std::vector<double> w(E);
  if (E) {
    e = cudaMemcpyAsync(c.data(), D.out_col, sizeof(int32_t) * E, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(w.data(), D.out_cost, sizeof(double) * E, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_error(e, "graph cache download");
  }
  return cache_write(file, key, n, D.radius, p.data(), c.data(), w.data(), inst->cache_model);
}
