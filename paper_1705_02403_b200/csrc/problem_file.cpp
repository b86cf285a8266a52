// problem_file.cpp -- the gmt-problem/1 scene format on the host (the C ABI's
// gmt_problem_parse / gmt_problem_load): parse_problem and load_problem of
// the reference (problem.cpp:102-231) -- the same strict validation (unknown
// keys rejected, every error named by its field path, the Dubins-only fields,
// the free start state) and the same defaults (problem.hpp:17-29,
// steering.hpp:9-23, sampling.hpp:20-29), so a scene loads identically on
// either side of the drop-in.  The reference reads JSON with nlohmann/json
// (ordered_json); the parser below is a small strict RFC 8259 reader with
// its number model: integer literals are signed (negative) or unsigned
// (non-negative) 64-bit values unless they overflow, everything else is a
// double converted by strtod; a repeated key keeps the last value.
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

#include "gmt_b200.h"

namespace gmtb {
int set_error(int code, const std::string& msg);
}

namespace {

struct Json {
  enum Kind { Null, Bool, Int, Uint, Float, String, Array, Object } kind = Null;
  bool b = false;
  int64_t i = 0;
  uint64_t u = 0;
  double f = 0.0;
  std::string s;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;  // insertion order, last value kept for repeats

  bool is_number() const { return kind == Int || kind == Uint || kind == Float; }
  bool is_integer() const { return kind == Int || kind == Uint; }
  double as_double() const { return kind == Int ? static_cast<double>(i) : kind == Uint ? static_cast<double>(u) : f; }
  long long as_ll() const { return kind == Int ? i : static_cast<long long>(u); }
  const Json* find(const char* key) const {
    for (const auto& kv : obj)
      if (kv.first == key) return &kv.second;
    return nullptr;
  }
};

struct ParseError {
  std::string what;
};

class Reader {
 public:
  Reader(const char* p, size_t n) : p_(p), end_(p + n), begin_(p) {}

  Json document() {
    Json v = value();
    ws();
    if (p_ != end_) error("syntax error: unexpected content after the JSON value");
    return v;
  }

 private:
  const char* p_;
  const char* end_;
  const char* begin_;

  [[noreturn]] void error(const std::string& what) {
    throw ParseError{what + " at byte " + std::to_string(p_ - begin_)};
  }
  void ws() {
    while (p_ != end_ && (*p_ == ' ' || *p_ == '\t' || *p_ == '\n' || *p_ == '\r')) ++p_;
  }
  bool literal(const char* lit) {
    const size_t n = std::strlen(lit);
    if (static_cast<size_t>(end_ - p_) >= n && std::memcmp(p_, lit, n) == 0) {
      p_ += n;
      return true;
    }
    return false;
  }
  Json value() {
    ws();
    if (p_ == end_) error("syntax error: unexpected end of input");
    Json v;
    switch (*p_) {
      case '{': object(v); break;
      case '[': array(v); break;
      case '"':
        v.kind = Json::String;
        v.s = string();
        break;
      case 't':
        if (!literal("true")) error("syntax error: invalid literal");
        v.kind = Json::Bool;
        v.b = true;
        break;
      case 'f':
        if (!literal("false")) error("syntax error: invalid literal");
        v.kind = Json::Bool;
        break;
      case 'n':
        if (!literal("null")) error("syntax error: invalid literal");
        break;
      default: number(v);
    }
    return v;
  }
  void object(Json& v) {
    v.kind = Json::Object;
    ++p_;
    ws();
    if (p_ != end_ && *p_ == '}') {
      ++p_;
      return;
    }
    for (;;) {
      ws();
      if (p_ == end_ || *p_ != '"') error("syntax error: expected a string key");
      std::string key = string();
      ws();
      if (p_ == end_ || *p_ != ':') error("syntax error: expected ':'");
      ++p_;
      Json item = value();
      bool repeated = false;
      for (auto& kv : v.obj)
        if (kv.first == key) {
          kv.second = std::move(item);
          repeated = true;
          break;
        }
      if (!repeated) v.obj.emplace_back(std::move(key), std::move(item));
      ws();
      if (p_ == end_) error("syntax error: unexpected end of input");
      if (*p_ == ',') {
        ++p_;
        continue;
      }
      if (*p_ == '}') {
        ++p_;
        return;
      }
      error("syntax error: expected ',' or '}'");
    }
  }
  void array(Json& v) {
    v.kind = Json::Array;
    ++p_;
    ws();
    if (p_ != end_ && *p_ == ']') {
      ++p_;
      return;
    }
    for (;;) {
      v.arr.push_back(value());
      ws();
      if (p_ == end_) error("syntax error: unexpected end of input");
      if (*p_ == ',') {
        ++p_;
        continue;
      }
      if (*p_ == ']') {
        ++p_;
        return;
      }
      error("syntax error: expected ',' or ']'");
    }
  }
  static void utf8(std::string& out, uint32_t cp) {
    if (cp < 0x80) {
      out += static_cast<char>(cp);
    } else if (cp < 0x800) {
      out += static_cast<char>(0xC0 | (cp >> 6));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      out += static_cast<char>(0xE0 | (cp >> 12));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else {
      out += static_cast<char>(0xF0 | (cp >> 18));
      out += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    }
  }
  uint32_t hex4() {
    if (end_ - p_ < 4) error("syntax error: incomplete \\u escape");
    uint32_t v = 0;
    for (int k = 0; k < 4; ++k) {
      const char c = *p_++;
      v <<= 4;
      if (c >= '0' && c <= '9') v |= static_cast<uint32_t>(c - '0');
      else if (c >= 'a' && c <= 'f') v |= static_cast<uint32_t>(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= static_cast<uint32_t>(c - 'A' + 10);
      else error("syntax error: invalid \\u escape");
    }
    return v;
  }
  std::string string() {
    ++p_;  // opening quote
    std::string out;
    for (;;) {
      if (p_ == end_) error("syntax error: unterminated string");
      const unsigned char c = static_cast<unsigned char>(*p_++);
      if (c == '"') return out;
      if (c < 0x20) error("syntax error: control character in a string");
      if (c != '\\') {
        out += static_cast<char>(c);
        continue;
      }
      if (p_ == end_) error("syntax error: unterminated string");
      const char e = *p_++;
      switch (e) {
        case '"': out += '"'; break;
        case '\\': out += '\\'; break;
        case '/': out += '/'; break;
        case 'b': out += '\b'; break;
        case 'f': out += '\f'; break;
        case 'n': out += '\n'; break;
        case 'r': out += '\r'; break;
        case 't': out += '\t'; break;
        case 'u': {
          uint32_t cp = hex4();
          if (cp >= 0xD800 && cp <= 0xDBFF) {
            if (end_ - p_ < 6 || p_[0] != '\\' || p_[1] != 'u') error("syntax error: unpaired surrogate");
            p_ += 2;
            const uint32_t lo = hex4();
            if (lo < 0xDC00 || lo > 0xDFFF) error("syntax error: unpaired surrogate");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
            error("syntax error: unpaired surrogate");
          }
          utf8(out, cp);
          break;
        }
        default: error("syntax error: invalid escape");
      }
    }
  }
  void number(Json& v) {
    const char* s = p_;
    bool neg = false, integral = true;
    if (p_ != end_ && *p_ == '-') {
      neg = true;
      ++p_;
    }
    if (p_ == end_ || !(*p_ >= '0' && *p_ <= '9')) error("syntax error: invalid literal");
    if (*p_ == '0') {
      ++p_;
    } else {
      while (p_ != end_ && *p_ >= '0' && *p_ <= '9') ++p_;
    }
    if (p_ != end_ && *p_ == '.') {
      integral = false;
      ++p_;
      if (p_ == end_ || !(*p_ >= '0' && *p_ <= '9')) error("syntax error: invalid number");
      while (p_ != end_ && *p_ >= '0' && *p_ <= '9') ++p_;
    }
    if (p_ != end_ && (*p_ == 'e' || *p_ == 'E')) {
      integral = false;
      ++p_;
      if (p_ != end_ && (*p_ == '+' || *p_ == '-')) ++p_;
      if (p_ == end_ || !(*p_ >= '0' && *p_ <= '9')) error("syntax error: invalid number");
      while (p_ != end_ && *p_ >= '0' && *p_ <= '9') ++p_;
    }
    const std::string lit(s, p_);
    if (integral) {
      errno = 0;
      if (neg) {
        const long long x = std::strtoll(lit.c_str(), nullptr, 10);
        if (errno == 0) {
          v.kind = Json::Int;
          v.i = x;
          return;
        }
      } else {
        const unsigned long long x = std::strtoull(lit.c_str(), nullptr, 10);
        if (errno == 0) {
          v.kind = Json::Uint;
          v.u = x;
          return;
        }
      }
    }
    v.kind = Json::Float;
    v.f = std::strtod(lit.c_str(), nullptr);
  }
};

// ---- parse_problem (problem.cpp:102-223) ---------------------------------------
struct Fail {
  std::string msg;
};
[[noreturn]] void fail(const std::string& path, const std::string& what) { throw Fail{path + ": " + what}; }
std::string join(const std::string& path, const char* key) { return path.empty() ? key : path + "." + key; }

void reject_unknown(const Json& obj, const std::string& path, std::initializer_list<const char*> allowed) {
  for (const auto& kv : obj.obj) {
    bool known = false;
    for (const char* key : allowed)
      if (kv.first == key) known = true;
    if (!known) fail(path.empty() ? kv.first : path + "." + kv.first, "unknown field");
  }
}
const Json& member(const Json& obj, const std::string& path, const char* key) {
  const Json* v = obj.find(key);
  if (!v) fail(join(path, key), "required field is missing");
  return *v;
}
double as_double(const Json& v, const std::string& path) {
  if (!v.is_number()) fail(path, "expected a number");
  return v.as_double();
}
long long as_int(const Json& v, const std::string& path) {
  if (!v.is_integer()) fail(path, "expected an integer");
  return v.as_ll();
}
uint64_t as_u64(const Json& v, const std::string& path) {
  if (v.kind == Json::Uint) return v.u;
  if (v.kind == Json::Int && v.i >= 0) return static_cast<uint64_t>(v.i);
  fail(path, "expected a non-negative integer");
}
std::string as_string(const Json& v, const std::string& path) {
  if (v.kind != Json::String) fail(path, "expected a string");
  return v.s;
}
std::vector<double> as_vector(const Json& v, const std::string& path, int dim) {
  if (v.kind != Json::Array) fail(path, "expected an array of numbers");
  if (static_cast<int>(v.arr.size()) != dim)
    fail(path, "expected " + std::to_string(dim) + " coordinates, got " + std::to_string(v.arr.size()));
  std::vector<double> out(v.arr.size());
  for (size_t k = 0; k < v.arr.size(); ++k) out[k] = as_double(v.arr[k], path + "[" + std::to_string(k) + "]");
  return out;
}
void parse_box(const Json& v, const std::string& path, int dim, std::vector<double>& lo, std::vector<double>& hi) {
  if (v.kind != Json::Object) fail(path, "expected an object with lo and hi");
  reject_unknown(v, path, {"lo", "hi"});
  const std::vector<double> l = as_vector(member(v, path, "lo"), path + ".lo", dim);
  const std::vector<double> h = as_vector(member(v, path, "hi"), path + ".hi", dim);
  for (int k = 0; k < dim; ++k)
    if (l[k] > h[k]) fail(path, "lo exceeds hi on axis " + std::to_string(k));
  lo.insert(lo.end(), l.begin(), l.end());
  hi.insert(hi.end(), h.begin(), h.end());
}

}  // namespace

// The parsed file: owns every array its flat gmt_problem view points to.
struct gmt_problem_file {
  int dim = 0;
  std::vector<double> box_lo, box_hi, goal_lo, goal_hi, init;
  gmt_problem view{};
  std::string notes;
};

namespace {

void parse_into(const Json& doc, gmt_problem_file& f) {
  if (doc.kind != Json::Object) throw Fail{"top level: expected a JSON object"};
  reject_unknown(doc, "",
                 {"schema", "dimension", "steering", "obstacles", "init", "goal", "n", "lambda", "eta",
                  "radius_override", "sampling", "notes"});
  if (as_string(member(doc, "", "schema"), "schema") != "gmt-problem/1")
    fail("schema", "expected \"gmt-problem/1\"");
  gmt_problem& p = f.view;
  std::memset(&p, 0, sizeof(p));
  const long long dim = as_int(member(doc, "", "dimension"), "dimension");
  if (dim < 1) fail("dimension", "must be at least 1");
  f.dim = static_cast<int>(dim);
  const int d = f.dim;

  const Json& steering = member(doc, "", "steering");
  if (steering.kind != Json::Object) fail("steering", "expected an object");
  reject_unknown(steering, "steering", {"model", "rho", "discretization_step", "planar_cost_only"});
  const std::string model = as_string(member(steering, "steering", "model"), "steering.model");
  p.dubins.rho = 0.1;  // steering.hpp:17-22 defaults
  p.dubins.discretization_step = 0.0;
  p.dubins.planar_cost_only = 0;
  bool dubins = false;
  if (model == "euclidean") {
    p.steering = GMT_STEER_EUCLIDEAN;
    for (const char* key : {"rho", "discretization_step", "planar_cost_only"})
      if (steering.find(key)) fail(join("steering", key), "only the dubins_airplane model uses this field");
  } else if (model == "dubins_airplane") {
    p.steering = GMT_STEER_DUBINS_AIRPLANE;
    dubins = true;
    if (d != 2 && d != 3) fail("dimension", "dubins_airplane needs dimension 2 or 3");
    if (const Json* v = steering.find("rho")) {
      p.dubins.rho = as_double(*v, "steering.rho");
      if (!(p.dubins.rho > 0.0)) fail("steering.rho", "must be positive");
    }
    if (const Json* v = steering.find("discretization_step")) {
      p.dubins.discretization_step = as_double(*v, "steering.discretization_step");
      if (p.dubins.discretization_step < 0.0) fail("steering.discretization_step", "must be non-negative");
    }
    if (const Json* v = steering.find("planar_cost_only")) {
      if (v->kind != Json::Bool) fail("steering.planar_cost_only", "expected a boolean");
      p.dubins.planar_cost_only = v->b ? 1 : 0;
    }
  } else {
    fail("steering.model", "expected \"euclidean\" or \"dubins_airplane\"");
  }

  const Json& obstacles = member(doc, "", "obstacles");
  if (obstacles.kind != Json::Array) fail("obstacles", "expected an array of boxes");
  for (size_t k = 0; k < obstacles.arr.size(); ++k)
    parse_box(obstacles.arr[k], "obstacles[" + std::to_string(k) + "]", d, f.box_lo, f.box_hi);

  const Json& init = member(doc, "", "init");
  if (init.kind != Json::Object) fail("init", "expected an object with coords");
  reject_unknown(init, "init", {"coords", "heading"});
  f.init = as_vector(member(init, "init", "coords"), "init.coords", d);
  if (const Json* h = init.find("heading")) {
    if (!dubins) fail("init.heading", "only the dubins_airplane model uses a heading");
    p.init_has_heading = 1;
    p.init_heading = as_double(*h, "init.heading");
  } else if (dubins) {
    fail("init.heading", "required field is missing");
  }
  // point_free (space.cpp:47-54): inside the closed unit cube, outside every closed box
  bool free = true;
  for (int k = 0; k < d; ++k)
    if (f.init[k] < 0.0 || f.init[k] > 1.0) free = false;
  const size_t nb = f.box_lo.size() / static_cast<size_t>(d);
  for (size_t b = 0; b < nb && free; ++b) {
    bool in = true;
    for (int k = 0; k < d; ++k)
      if (f.init[k] < f.box_lo[b * d + k] || f.init[k] > f.box_hi[b * d + k]) in = false;
    if (in) free = false;
  }
  if (!free) fail("init", "start state is not in free space");

  parse_box(member(doc, "", "goal"), "goal", d, f.goal_lo, f.goal_hi);

  const long long n = as_int(member(doc, "", "n"), "n");
  if (n < 1) fail("n", "must be at least 1");
  p.n = static_cast<int32_t>(n);
  p.lambda = 1.0;
  if (const Json* v = doc.find("lambda")) {
    p.lambda = as_double(*v, "lambda");
    if (!(p.lambda > 0.0) || p.lambda > 1.0) fail("lambda", "must be in (0, 1]");
  }
  if (const Json* v = doc.find("eta")) {
    p.eta = as_double(*v, "eta");
    if (p.eta < 0.0) fail("eta", "must be non-negative");
  }
  p.radius_override = 0.0;  // (<= 0: none)
  if (const Json* v = doc.find("radius_override")) {
    const double r = as_double(*v, "radius_override");
    if (!(r > 0.0)) fail("radius_override", "must be positive");
    p.radius_override = r;
  }
  p.sampling.kind = GMT_SAMPLE_HALTON;
  p.sampling.start_index = 1;
  p.sampling.seed = 0;
  p.sampling.with_heading = dubins ? 1 : 0;
  if (const Json* sp = doc.find("sampling")) {
    const Json& sampling = *sp;
    if (sampling.kind != Json::Object) fail("sampling", "expected an object");
    reject_unknown(sampling, "sampling", {"kind", "start_index", "seed"});
    const std::string kind = as_string(member(sampling, "sampling", "kind"), "sampling.kind");
    if (kind == "halton") {
      if (sampling.find("seed")) fail("sampling.seed", "only uniform sampling takes a seed");
      if (const Json* v = sampling.find("start_index")) {
        p.sampling.start_index = as_u64(*v, "sampling.start_index");
        if (p.sampling.start_index == 0) fail("sampling.start_index", "must be at least 1");
      }
    } else if (kind == "uniform") {
      p.sampling.kind = GMT_SAMPLE_UNIFORM;
      if (sampling.find("start_index")) fail("sampling.start_index", "only halton sampling takes a start index");
      if (const Json* v = sampling.find("seed")) p.sampling.seed = as_u64(*v, "sampling.seed");
    } else {
      fail("sampling.kind", "expected \"halton\" or \"uniform\"");
    }
  }
  if (const Json* v = doc.find("notes")) f.notes = as_string(*v, "notes");
  // the flat view
  p.scene.dim = d;
  p.scene.num_boxes = static_cast<int32_t>(nb);
  p.scene.box_lo = f.box_lo.data();
  p.scene.box_hi = f.box_hi.data();
  p.scene.goal_lo = f.goal_lo.data();
  p.scene.goal_hi = f.goal_hi.data();
  p.init = f.init.data();
}

}  // namespace

extern "C" int gmt_problem_parse(const char* json_text, size_t length, gmt_problem_file** out) {
  if (!out) return gmtb::set_error(GMT_E_INVALID_INPUT, "output handle is null");
  *out = nullptr;
  if (!json_text) return gmtb::set_error(GMT_E_INVALID_INPUT, "invalid JSON: null text");
  auto f = std::make_unique<gmt_problem_file>();
  try {
    const Json doc = Reader(json_text, length).document();
    parse_into(doc, *f);
  } catch (const ParseError& e) {
    return gmtb::set_error(GMT_E_INVALID_INPUT, "invalid JSON: " + e.what);
  } catch (const Fail& e) {
    return gmtb::set_error(GMT_E_INVALID_INPUT, e.msg);
  }
  *out = f.release();
  return GMT_OK;
}

extern "C" int gmt_problem_load(const char* path, gmt_problem_file** out) {
  if (!out) return gmtb::set_error(GMT_E_INVALID_INPUT, "output handle is null");
  *out = nullptr;
  const std::string p = path ? path : "";
  std::ifstream in(p, std::ios::binary);  // load_problem (problem.cpp:225-231)
  if (!in) return gmtb::set_error(GMT_E_INVALID_INPUT, p + ": cannot open file");
  std::ostringstream buf;
  buf << in.rdbuf();
  const std::string text = buf.str();
  return gmt_problem_parse(text.data(), text.size(), out);
}

extern "C" int gmt_problem_file_view(const gmt_problem_file* f, gmt_problem* view, const char** notes) {
  if (!f || !view) return gmtb::set_error(GMT_E_INVALID_INPUT, "problem file is null");
  *view = f->view;
  if (notes) *notes = f->notes.c_str();
  return GMT_OK;
}

extern "C" void gmt_problem_file_destroy(gmt_problem_file* f) { delete f; }
