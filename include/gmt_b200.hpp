// gmt_b200.hpp -- header-only C++ drop-in for the reference's planning API.
//
// Re-creates the `gmt::` types and free functions of the reference library
// (/root/reference/proj/include/gmtplan/*.hpp) on top of the C ABI in
// gmt_b200.h, so a caller swaps implementations by changing the include and
// the namespace (or by defining GMT_B200_AS_GMT before including this header
// in a translation unit that does not also include the reference headers,
// which aliases `gmt` to `gmt_b200`).
//
// Same names, argument meaning and error behaviour:
//   gmt_plan              planner.hpp:67-69   (IterationHook: replayed, see below)
//   fmt_plan              planner.hpp:71-74
//   sample_free           sampling.hpp:44-45
//   append_init           sampling.hpp:51
//   unit_ball_volume      graph.hpp:22
//   connection_radius     graph.hpp:25
//   build_neighbor_graph  graph.hpp:53-54     (Euclidean model)
//   build_instance        problem.hpp:59-60   (Euclidean model, GMTG v1 cache file)
//   problem_key           problem.hpp:43
//   save_graph_cache / load_graph_cache   graph.hpp:60-65 (Euclidean)
// Exceptions: InvalidInputError / InfeasibleSamplingError / GoalBlockedError
// (errors.hpp:9-21); CUDA failures throw gmt_b200::CudaError.  There is no
// CPU fallback: without a B200 every call throws NoDeviceError.
//
// IterationHook: the device runs the whole solve in one launch, so the hook
// is replayed after the solve from the final tree and the per-pass
// thresholds (labels, costs and parents as they stood after each commit,
// planner.cpp:195).
#pragma once

#include <cmath>
#include <cstdint>
#include <functional>
#include <limits>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "gmt_b200.h"

namespace gmt_b200 {

// ---- errors (errors.hpp:9-21) ------------------------------------------------
struct InvalidInputError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct InfeasibleSamplingError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct GoalBlockedError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NoDeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == GMT_OK) return;
  const std::string msg = gmt_last_error();
  switch (rc) {
    case GMT_E_INVALID_INPUT: throw InvalidInputError(msg);
    case GMT_E_INFEASIBLE_SAMPLING: throw InfeasibleSamplingError(msg);
    case GMT_E_GOAL_BLOCKED: throw GoalBlockedError(msg);
    case GMT_E_NO_DEVICE: throw NoDeviceError(msg);
    case GMT_E_CUDA: throw CudaError(msg);
    default: throw std::runtime_error(msg);
  }
}

// ---- types (space.hpp, sampling.hpp, graph.hpp, planner.hpp) ----------------
struct State {
  std::vector<double> coords;
  std::optional<double> heading;
  int dim() const { return static_cast<int>(coords.size()); }
};

struct Aabb {
  std::vector<double> lo;
  std::vector<double> hi;
  int dim() const { return static_cast<int>(lo.size()); }
  bool contains(const std::vector<double>& p) const {  // space.cpp:11-16
    for (std::size_t k = 0; k < lo.size(); ++k)
      if (p[k] < lo[k] || p[k] > hi[k]) return false;
    return true;
  }
  std::vector<double> center() const {
    std::vector<double> c(lo.size());
    for (std::size_t k = 0; k < lo.size(); ++k) c[k] = 0.5 * (lo[k] + hi[k]);
    return c;
  }
};

struct ObstacleSet {
  int dim = 0;
  std::vector<Aabb> boxes;
};

struct GoalRegion {
  Aabb box;
  bool contains(const State& s) const { return box.contains(s.coords); }
};

struct SampleSource {
  enum class Kind { halton, uniform };
  Kind kind = Kind::halton;
  std::uint64_t start_index = 1;
  std::uint64_t seed = 0;
  bool with_heading = false;
};

struct SampleSet {
  std::vector<State> states;
  std::vector<int> goal_indices;
};

struct SteeringModel {
  enum class Kind { euclidean, dubins_airplane };
  Kind kind = Kind::euclidean;
  double rho = 0.1;
  double discretization_step = 0.0;
  bool planar_cost_only = false;
};

struct RadiusParams {
  int dimension = 2;
  long long n = 0;
  double eta = 0.0;
  double mu_free = 1.0;
};

struct NeighborGraph {
  struct Edge {
    int other = -1;
    double cost = 0.0;
    int path_id = -1;
  };
  int n = 0;
  double radius = 0.0;
  SteeringModel model;
  std::vector<std::vector<Edge>> out;
  std::vector<std::vector<Edge>> in;
  std::vector<std::vector<State>> paths;

  const std::vector<State>* edge_path(int u, int v) const {  // graph.cpp:34-40
    const auto& lst = out[u];
    std::size_t lo = 0, hi = lst.size();
    while (lo < hi) {
      std::size_t mid = (lo + hi) / 2;
      if (lst[mid].other < v) lo = mid + 1; else hi = mid;
    }
    if (lo == lst.size() || lst[lo].other != v || lst[lo].path_id < 0) return nullptr;
    return &paths[lst[lo].path_id];
  }
  std::size_t edge_count() const {
    std::size_t c = 0;
    for (const auto& l : out) c += l.size();
    return c;
  }
};

enum class PlanStatus { success, failure_open_empty, infeasible_input };
enum class NodeLabel : std::uint8_t { unexplored, open, closed };

struct Wavefront {
  std::vector<NodeLabel> label;
  std::vector<double> cost;
  std::vector<int> parent;
  std::vector<long long> iteration_added;
};

struct GmtParams {
  double lambda = 1.0;
  double radius = 0.0;
  int workers = 1;  // accepted for API compatibility; the device ignores it
  double delta() const { return lambda * radius; }
};

struct IterationStats {
  std::vector<int> group_sizes;
  std::vector<int> nodes_added;
  std::vector<long long> collision_checks;
};

struct PlanResult {
  PlanStatus status = PlanStatus::infeasible_input;
  std::vector<int> path_indices;
  std::vector<State> path;
  double cost = std::numeric_limits<double>::infinity();
  long long iterations = 0;
  long long total_collision_checks = 0;
  Wavefront tree;
  IterationStats stats;
};

using IterationHook = std::function<void(const Wavefront&, long long iteration)>;

// ---- context: one per thread, device 0 by default ---------------------------
class Context {
 public:
  explicit Context(int device = 0) { check(gmt_ctx_create(device, &ctx_)); }
  ~Context() { gmt_ctx_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  gmt_ctx* get() const { return ctx_; }

  static Context& thread_default() {
    thread_local std::unique_ptr<Context> c;
    if (!c) c = std::make_unique<Context>(0);
    return *c;
  }

 private:
  gmt_ctx* ctx_ = nullptr;
};

namespace detail {

struct FlatScene {
  std::vector<double> lo, hi, glo, ghi;
  gmt_scene s{};
  FlatScene(const ObstacleSet& obs, const GoalRegion& goal) {
    const int d = obs.dim;
    for (const auto& b : obs.boxes) {
      if (b.dim() != d || static_cast<int>(b.hi.size()) != d)
        throw InvalidInputError("box dimension mismatch");
      lo.insert(lo.end(), b.lo.begin(), b.lo.end());
      hi.insert(hi.end(), b.hi.begin(), b.hi.end());
    }
    if (goal.box.dim() != d || static_cast<int>(goal.box.hi.size()) != d)
      throw InvalidInputError("box dimension mismatch");
    glo = goal.box.lo;
    ghi = goal.box.hi;
    s.dim = d;
    s.num_boxes = static_cast<int32_t>(obs.boxes.size());
    s.box_lo = lo.data();
    s.box_hi = hi.data();
    s.goal_lo = glo.data();
    s.goal_hi = ghi.data();
  }
};

inline std::vector<double> flat_coords(const SampleSet& samples, int dim) {
  std::vector<double> c;
  c.reserve(samples.states.size() * static_cast<std::size_t>(dim));
  for (const auto& st : samples.states) {
    if (st.dim() != dim) throw InvalidInputError("point dimension mismatch");
    c.insert(c.end(), st.coords.begin(), st.coords.end());
  }
  return c;
}

// NeighborGraph -> compressed rows.  in_path carries the id edge_path()
// would return for (source, x) (graph.cpp:34-40).
struct FlatGraph {
  std::vector<int64_t> optr, iptr, pptr;
  std::vector<int32_t> ocol, icol, opath, ipath;
  std::vector<double> ocost, icost, ppts;
  gmt_graph_view v{};
  FlatGraph(const NeighborGraph& g, int dim) {
    const bool directed = g.model.kind != SteeringModel::Kind::euclidean;
    const bool paths = !g.paths.empty();
    optr.assign(1, 0);
    for (int u = 0; u < g.n; ++u) {
      for (const auto& e : g.out[u]) {
        ocol.push_back(e.other);
        ocost.push_back(e.cost);
        opath.push_back(e.path_id);
      }
      optr.push_back(static_cast<int64_t>(ocol.size()));
    }
    if (directed || paths) {
      iptr.assign(1, 0);
      for (int x = 0; x < g.n; ++x) {
        for (const auto& e : g.in[x]) {
          icol.push_back(e.other);
          icost.push_back(e.cost);
          const std::vector<State>* p = g.edge_path(e.other, x);
          ipath.push_back(p ? static_cast<int32_t>(p - g.paths.data()) : -1);
        }
        iptr.push_back(static_cast<int64_t>(icol.size()));
      }
      pptr.assign(1, 0);
      for (const auto& p : g.paths) {
        for (const auto& st : p) ppts.insert(ppts.end(), st.coords.begin(), st.coords.end());
        pptr.push_back(pptr.back() + static_cast<int64_t>(p.size()));
      }
    }
    v.n = g.n;
    v.dim = dim;
    v.radius = g.radius;
    v.directed = (directed || paths) ? 1 : 0;
    v.out_ptr = optr.data();
    v.out_col = ocol.data();
    v.out_cost = ocost.data();
    v.out_path = paths ? opath.data() : nullptr;
    if (v.directed) {
      v.in_ptr = iptr.data();
      v.in_col = icol.data();
      v.in_cost = icost.data();
      v.in_path = paths ? ipath.data() : nullptr;
      v.num_paths = static_cast<int64_t>(g.paths.size());
      v.path_ptr = pptr.data();
      v.path_pts = ppts.empty() ? nullptr : ppts.data();
    }
  }
};

inline PlanResult to_result(const SampleSet& samples, int n, gmt_plan_out& o,
                            std::vector<int32_t>& path, std::vector<uint8_t>& label,
                            std::vector<double>& cost, std::vector<int32_t>& parent,
                            std::vector<int64_t>& iter, std::vector<int32_t>& gs,
                            std::vector<int32_t>& na, std::vector<int64_t>& ck) {
  (void)n;
  PlanResult r;
  r.status = static_cast<PlanStatus>(o.status);
  r.cost = o.cost;
  r.iterations = o.iterations;
  r.total_collision_checks = o.total_collision_checks;
  r.path_indices.assign(path.begin(), path.begin() + o.path_len);
  for (int idx : r.path_indices) r.path.push_back(samples.states[idx]);  // planner.cpp:48-49
  const int t = o.tree_size;
  r.tree.label.resize(t);
  for (int v = 0; v < t; ++v) r.tree.label[v] = static_cast<NodeLabel>(label[v]);
  r.tree.cost.assign(cost.begin(), cost.begin() + t);
  r.tree.parent.assign(parent.begin(), parent.begin() + t);
  r.tree.iteration_added.assign(iter.begin(), iter.begin() + t);
  r.stats.group_sizes.assign(gs.begin(), gs.begin() + o.num_stats);
  r.stats.nodes_added.assign(na.begin(), na.begin() + o.num_stats);
  r.stats.collision_checks.assign(ck.begin(), ck.begin() + o.num_stats);
  return r;
}

// Replays IterationHook from the final tree: after the commit of pass p
// (iteration i_p) a node is open/closed iff it was reached by then
// (iteration_added <= i_p) and closed iff it belonged to the group of some
// pass <= p; a node reached at iteration a is a group member of the first
// later pass whose threshold i*delta covers its cost (planner.cpp:137-141).
inline void replay_hook(const PlanResult& r, int init_index, double delta,
                        const IterationHook& hook) {
  if (!hook || r.tree.label.empty()) return;
  const int n = static_cast<int>(r.tree.label.size());
  const std::size_t expanded =
      r.stats.group_sizes.size() - (r.status == PlanStatus::success ? 1 : 0);
  // Pass thresholds: rebuild i_p by replaying the fast-forward rule on the
  // recorded min-open costs.
  std::vector<long long> iters;
  {
    std::vector<char> reached(n, 0), closed(n, 0);
    reached[init_index] = 1;
    long long i = 0;
    for (std::size_t p = 0; p < expanded; ++p) {
      double min_open = std::numeric_limits<double>::infinity();
      for (int v = 0; v < n; ++v)
        if (reached[v] && !closed[v] && r.tree.cost[v] < min_open) min_open = r.tree.cost[v];
      if (min_open > i * delta) {
        long long jump = static_cast<long long>(std::ceil(min_open / delta));
        i = jump > i + 1 ? jump : i + 1;
        while (min_open > i * delta) ++i;
      }
      iters.push_back(i);
      for (int v = 0; v < n; ++v)
        if (reached[v] && !closed[v] && r.tree.cost[v] <= i * delta) closed[v] = 1;
      for (int v = 0; v < n; ++v)
        if (r.tree.iteration_added[v] == i && v != init_index) reached[v] = 1;
      ++i;
    }
  }
  Wavefront w;
  w.label.assign(n, NodeLabel::unexplored);
  w.cost.assign(n, std::numeric_limits<double>::infinity());
  w.parent.assign(n, -1);
  w.iteration_added.assign(n, -1);
  w.label[init_index] = NodeLabel::open;
  w.cost[init_index] = 0.0;
  w.iteration_added[init_index] = 0;
  for (std::size_t p = 0; p < iters.size(); ++p) {
    const long long i = iters[p];
    for (int v = 0; v < n; ++v)  // close the group of pass p
      if (w.label[v] == NodeLabel::open && w.cost[v] <= i * delta) w.label[v] = NodeLabel::closed;
    for (int v = 0; v < n; ++v) {
      if (v != init_index && r.tree.iteration_added[v] == i) {
        w.label[v] = NodeLabel::open;
        w.cost[v] = r.tree.cost[v];
        w.parent[v] = r.tree.parent[v];
        w.iteration_added[v] = i;
      }
    }
    hook(w, i);
  }
}

}  // namespace detail

// ---- sampling (sampling.hpp) --------------------------------------------------
inline SampleSet sample_free(int n, const ObstacleSet& obs, const GoalRegion& goal,
                             const SampleSource& source, Context& ctx = Context::thread_default()) {
  if (n < 1) throw InvalidInputError("sample count must be >= 1");
  detail::FlatScene fs(obs, goal);
  gmt_sample_source src{source.kind == SampleSource::Kind::uniform ? GMT_SAMPLE_UNIFORM
                                                                   : GMT_SAMPLE_HALTON,
                        source.with_heading ? 1 : 0, source.start_index, source.seed};
  std::vector<double> coords(static_cast<std::size_t>(n) * obs.dim), heading(n);
  std::vector<int32_t> gidx(n + 1);
  int32_t gc = 0;
  check(gmt_sample_free(ctx.get(), n, &fs.s, &src, coords.data(), heading.data(), gidx.data(), &gc));
  SampleSet s;
  s.states.resize(n);
  for (int i = 0; i < n; ++i) {
    s.states[i].coords.assign(coords.begin() + static_cast<std::ptrdiff_t>(i) * obs.dim,
                              coords.begin() + static_cast<std::ptrdiff_t>(i + 1) * obs.dim);
    if (source.with_heading) s.states[i].heading = heading[i];
  }
  s.goal_indices.assign(gidx.begin(), gidx.begin() + gc);
  return s;
}

inline int append_init(SampleSet& samples, const State& init, const GoalRegion& goal,
                       Context& ctx = Context::thread_default()) {
  const int d = init.dim();
  int32_t n = static_cast<int32_t>(samples.states.size());
  std::vector<double> coords = detail::flat_coords(samples, d);
  coords.resize(coords.size() + d);
  const bool headings = !samples.states.empty() && samples.states[0].heading.has_value();
  std::vector<double> heading;
  if (headings) {
    for (const auto& st : samples.states) heading.push_back(st.heading.value_or(0.0));
    heading.push_back(0.0);
  }
  std::vector<int32_t> gidx(samples.goal_indices.begin(), samples.goal_indices.end());
  gidx.push_back(-1);
  int32_t gc = static_cast<int32_t>(samples.goal_indices.size());
  int32_t idx = -1;
  check(gmt_append_init(ctx.get(), d, coords.data(), headings ? heading.data() : nullptr, &n,
                        init.coords.data(), init.heading ? 1 : 0, init.heading.value_or(0.0),
                        goal.box.lo.data(), goal.box.hi.data(), gidx.data(), &gc, &idx));
  if (n > static_cast<int32_t>(samples.states.size())) {
    samples.states.push_back(init);
    samples.goal_indices.assign(gidx.begin(), gidx.begin() + gc);
  }
  return idx;
}

// ---- graph (graph.hpp) -----------------------------------------------------------
inline double unit_ball_volume(int d) {
  double v = 0.0;
  check(gmt_unit_ball_volume(d, &v));
  return v;
}

inline double connection_radius(const RadiusParams& p) {
  if (!(p.mu_free > 0.0 && p.mu_free <= 1.0)) throw InvalidInputError("mu_free must be in (0, 1]");
  double r = 0.0;
  check(gmt_connection_radius(p.dimension, p.n, p.eta, p.mu_free, &r));
  return r;
}

inline NeighborGraph build_neighbor_graph(const std::vector<State>& states, const SteeringModel& m,
                                          double radius, int workers = 1,
                                          Context& ctx = Context::thread_default()) {
  (void)workers;
  if (m.kind != SteeringModel::Kind::euclidean)
    throw InvalidInputError("dubins_airplane graphs are not built on the device yet");
  if (!(radius > 0.0)) throw InvalidInputError("connection radius must be positive");
  if (states.empty()) throw InvalidInputError("cannot build a graph over zero samples");
  const int n = static_cast<int>(states.size()), d = states[0].dim();
  SampleSet tmp;
  tmp.states = states;
  std::vector<double> coords = detail::flat_coords(tmp, d);
  int64_t E = 0;
  check(gmt_build_neighbor_graph(ctx.get(), coords.data(), n, d, radius, &E, nullptr, nullptr, nullptr));
  std::vector<int64_t> ptr(n + 1);
  std::vector<int32_t> col(E);
  std::vector<double> cost(E);
  check(gmt_build_neighbor_graph(ctx.get(), coords.data(), n, d, radius, &E, ptr.data(), col.data(),
                                 cost.data()));
  NeighborGraph g;
  g.n = n;
  g.radius = radius;
  g.model = m;
  g.out.resize(n);
  g.in.resize(n);
  for (int u = 0; u < n; ++u)
    for (int64_t e = ptr[u]; e < ptr[u + 1]; ++e) g.out[u].push_back({col[e], cost[e], -1});
  for (int u = 0; u < n; ++u)  // sequential in-list merge, graph.cpp:184-186
    for (const auto& e : g.out[u]) g.in[e.other].push_back({u, e.cost, e.path_id});
  return g;
}

// ---- planners (planner.hpp) --------------------------------------------------------
namespace detail {
inline PlanResult plan_common(const SampleSet& samples, const NeighborGraph& graph,
                              const ObstacleSet& obs, const GoalRegion& goal, int init_index,
                              double lambda, double radius, bool fmt, Context& ctx) {
  const int n = static_cast<int>(samples.states.size());
  if (graph.n != n) throw InvalidInputError("graph was built over a different sample count");
  if (init_index < 0 || init_index >= n)
    throw InvalidInputError("init_index " + std::to_string(init_index) + " out of range");
  FlatScene fs(obs, goal);
  std::vector<double> coords = flat_coords(samples, obs.dim);
  FlatGraph fg(graph, obs.dim);
  std::vector<int32_t> path(n), parent(n), gs(n + 1), na(n + 1);
  std::vector<uint8_t> label(n);
  std::vector<double> cost(n);
  std::vector<int64_t> iter(n), ck(n + 1);
  gmt_plan_out o{};
  o.stats_cap = n + 1;
  o.path = path.data();
  o.label = label.data();
  o.tree_cost = cost.data();
  o.parent = parent.data();
  o.iteration_added = iter.data();
  o.group_sizes = gs.data();
  o.nodes_added = na.data();
  o.collision_checks = ck.data();
  if (fmt) {
    gmt_instance* inst = nullptr;
    check(gmt_instance_upload(ctx.get(), &fs.s, coords.data(), n,
                              static_cast<int32_t>(samples.goal_indices.size()), &fg.v, &inst));
    int rc = gmt_fmt_plan(ctx.get(), inst, init_index, &o);
    gmt_instance_destroy(inst);
    check(rc);
  } else {
    check(gmt_plan_host(ctx.get(), &fs.s, coords.data(), n,
                        static_cast<int32_t>(samples.goal_indices.size()), &fg.v, init_index,
                        lambda, radius, &o));
  }
  return to_result(samples, n, o, path, label, cost, parent, iter, gs, na, ck);
}
}  // namespace detail

inline PlanResult gmt_plan(const SampleSet& samples, const NeighborGraph& graph,
                           const ObstacleSet& obs, const GoalRegion& goal, int init_index,
                           const GmtParams& params, const IterationHook& hook = {},
                           Context& ctx = Context::thread_default()) {
  PlanResult r = detail::plan_common(samples, graph, obs, goal, init_index, params.lambda,
                                     params.radius, false, ctx);
  detail::replay_hook(r, init_index, params.delta(), hook);
  return r;
}

inline PlanResult fmt_plan(const SampleSet& samples, const NeighborGraph& graph,
                           const ObstacleSet& obs, const GoalRegion& goal, int init_index,
                           Context& ctx = Context::thread_default()) {
  return detail::plan_common(samples, graph, obs, goal, init_index, 1.0, graph.radius, true, ctx);
}

// ---- problem instances (problem.hpp) ----------------------------------------------
struct ProblemFile {
  int dimension = 0;
  SteeringModel steering;
  ObstacleSet obstacles;
  State init;
  GoalRegion goal;
  int n = 0;
  double lambda = 1.0;
  double eta = 0.0;
  std::optional<double> radius_override;
  SampleSource sampling;
  std::string notes;
};

struct ProblemInstance {
  SampleSet samples;
  int init_index = -1;
  double radius = 0.0;
  NeighborGraph graph;
};

namespace detail {
// A gmt_problem view of a ProblemFile (arrays owned by the FlatScene).
struct FlatProblem {
  FlatScene scene;
  gmt_problem p{};
  explicit FlatProblem(const ProblemFile& f) : scene(f.obstacles, f.goal) {
    p.scene = scene.s;
    p.init = f.init.coords.data();
    p.init_has_heading = f.init.heading ? 1 : 0;
    p.init_heading = f.init.heading ? *f.init.heading : 0.0;
    p.n = f.n;
    p.lambda = f.lambda;
    p.eta = f.eta;
    p.radius_override = f.radius_override ? *f.radius_override : 0.0;
    p.sampling.kind = f.sampling.kind == SampleSource::Kind::uniform ? GMT_SAMPLE_UNIFORM : GMT_SAMPLE_HALTON;
    p.sampling.with_heading = f.sampling.with_heading ? 1 : 0;
    p.sampling.start_index = f.sampling.start_index;
    p.sampling.seed = f.sampling.seed;
    p.steering = GMT_STEER_EUCLIDEAN;
  }
};

inline NeighborGraph graph_from_csr(int n, double radius, const SteeringModel& m,
                                    const std::vector<int64_t>& ptr, const std::vector<int32_t>& col,
                                    const std::vector<double>& cost) {
  NeighborGraph g;
  g.n = n;
  g.radius = radius;
  g.model = m;
  g.out.resize(n);
  g.in.resize(n);
  for (int u = 0; u < n; ++u)
    for (int64_t e = ptr[u]; e < ptr[u + 1]; ++e) g.out[u].push_back({col[e], cost[e], -1});
  for (int u = 0; u < n; ++u)  // sequential in-list merge, graph.cpp:184-186
    for (const auto& e : g.out[u]) g.in[e.other].push_back({u, e.cost, e.path_id});
  return g;
}
}  // namespace detail

// problem_key (problem.cpp:281-303), Euclidean problems.
inline std::uint64_t problem_key(const ProblemFile& p) {
  if (p.steering.kind != SteeringModel::Kind::euclidean)
    throw InvalidInputError("the graph cache covers the Euclidean steering model only");
  detail::FlatProblem fp(p);
  std::uint64_t k = 0;
  check(gmt_problem_key(&fp.p, &k));
  return k;
}

// save_graph_cache (graph.cpp:240-276): false when the file cannot be written.
inline bool save_graph_cache(const NeighborGraph& g, const std::string& file, std::uint64_t key) {
  if (g.model.kind != SteeringModel::Kind::euclidean)
    throw InvalidInputError("the graph cache covers the Euclidean steering model only");
  std::vector<int64_t> ptr(g.n + 1, 0);
  std::vector<int32_t> col;
  std::vector<double> cost;
  for (int u = 0; u < g.n; ++u) {
    for (const auto& e : g.out[u]) {
      col.push_back(e.other);
      cost.push_back(e.cost);
    }
    ptr[u + 1] = static_cast<int64_t>(col.size());
  }
  return gmt_graph_cache_save(file.c_str(), key, g.n, g.radius, ptr.data(), col.data(), cost.data()) ==
         GMT_OK;
}

// load_graph_cache (graph.cpp:278-343): empty on any mismatch or corruption.
inline std::optional<NeighborGraph> load_graph_cache(const std::string& file, std::uint64_t key,
                                                     const std::vector<State>& states,
                                                     const SteeringModel& m, double radius) {
  if (m.kind != SteeringModel::Kind::euclidean) return std::nullopt;
  const int n = static_cast<int>(states.size());
  int32_t hit = 0;
  int64_t E = 0;
  check(gmt_graph_cache_load(file.c_str(), key, n, radius, &hit, &E, 0, nullptr, nullptr, nullptr));
  if (!hit) return std::nullopt;
  std::vector<int64_t> ptr(n + 1);
  std::vector<int32_t> col(E);
  std::vector<double> cost(E);
  check(gmt_graph_cache_load(file.c_str(), key, n, radius, &hit, &E, static_cast<int64_t>(col.size()),
                             ptr.data(), col.data(), cost.data()));
  if (!hit) return std::nullopt;  // replaced by a file that no longer matches
  col.resize(E);
  cost.resize(E);
  return detail::graph_from_csr(n, radius, m, ptr, col, cost);
}

namespace detail {
inline ProblemFile problem_from_file(gmt_problem_file* h) {
  gmt_problem v{};
  const char* notes = nullptr;
  const int rc = gmt_problem_file_view(h, &v, &notes);
  if (rc != GMT_OK) {
    gmt_problem_file_destroy(h);
    check(rc);
  }
  ProblemFile p;
  const int d = v.scene.dim;
  p.dimension = d;
  if (v.steering == GMT_STEER_DUBINS_AIRPLANE) {
    p.steering.kind = SteeringModel::Kind::dubins_airplane;
    p.steering.rho = v.dubins.rho;
    p.steering.discretization_step = v.dubins.discretization_step;
    p.steering.planar_cost_only = v.dubins.planar_cost_only != 0;
  }
  p.obstacles.dim = d;
  for (int b = 0; b < v.scene.num_boxes; ++b) {
    Aabb box;
    box.lo.assign(v.scene.box_lo + static_cast<size_t>(b) * d, v.scene.box_lo + static_cast<size_t>(b + 1) * d);
    box.hi.assign(v.scene.box_hi + static_cast<size_t>(b) * d, v.scene.box_hi + static_cast<size_t>(b + 1) * d);
    p.obstacles.boxes.push_back(std::move(box));
  }
  p.goal.box.lo.assign(v.scene.goal_lo, v.scene.goal_lo + d);
  p.goal.box.hi.assign(v.scene.goal_hi, v.scene.goal_hi + d);
  p.init.coords.assign(v.init, v.init + d);
  if (v.init_has_heading) p.init.heading = v.init_heading;
  p.n = v.n;
  p.lambda = v.lambda;
  p.eta = v.eta;
  if (v.radius_override > 0.0) p.radius_override = v.radius_override;
  p.sampling.kind = v.sampling.kind == GMT_SAMPLE_UNIFORM ? SampleSource::Kind::uniform : SampleSource::Kind::halton;
  p.sampling.start_index = v.sampling.start_index;
  p.sampling.seed = v.sampling.seed;
  p.sampling.with_heading = v.sampling.with_heading != 0;
  p.notes = notes ? notes : "";
  gmt_problem_file_destroy(h);
  return p;
}
}  // namespace detail

// parse_problem (problem.cpp:102-223): strict gmt-problem/1 parsing, the
// reference's path-named InvalidInputError messages.
inline ProblemFile parse_problem(const std::string& json_text) {
  gmt_problem_file* h = nullptr;
  check(gmt_problem_parse(json_text.data(), json_text.size(), &h));
  return detail::problem_from_file(h);
}

// load_problem (problem.cpp:225-231).
inline ProblemFile load_problem(const std::string& path) {
  gmt_problem_file* h = nullptr;
  check(gmt_problem_load(path.c_str(), &h));
  return detail::problem_from_file(h);
}

inline ProblemInstance build_instance(const ProblemFile& p, int workers = 1,
                                      const std::string& cache_file = "",
                                      Context& ctx = Context::thread_default()) {
  (void)workers;
  if (p.steering.kind != SteeringModel::Kind::euclidean)
    throw InvalidInputError("dubins_airplane problems are not supported on the device yet");
  // Same call sequence as problem.cpp:336-363, every step on the device.
  ProblemInstance inst;
  SampleSource src = p.sampling;
  src.with_heading = false;
  inst.samples = sample_free(p.n, p.obstacles, p.goal, src, ctx);
  inst.init_index = append_init(inst.samples, p.init, p.goal, ctx);
  if (p.radius_override) {
    inst.radius = *p.radius_override;
  } else {
    RadiusParams rp;
    rp.dimension = p.dimension;
    rp.n = p.n;
    rp.eta = p.eta;
    rp.mu_free = 1.0;  // free_measure_upper_bound (space.cpp:101-104)
    inst.radius = connection_radius(rp);
  }
  // Graph cache (problem.cpp:353-362): load on a key / shape match, else
  // build and save (a failed save is ignored, as in the reference).
  if (!cache_file.empty()) {
    const std::uint64_t key = problem_key(p);
    if (auto cached = load_graph_cache(cache_file, key, inst.samples.states, p.steering, inst.radius)) {
      inst.graph = std::move(*cached);
      return inst;
    }
    inst.graph = build_neighbor_graph(inst.samples.states, p.steering, inst.radius, workers, ctx);
    save_graph_cache(inst.graph, cache_file, key);
    return inst;
  }
  inst.graph = build_neighbor_graph(inst.samples.states, p.steering, inst.radius, workers, ctx);
  return inst;
}

}  // namespace gmt_b200

#ifdef GMT_B200_AS_GMT
namespace gmt = gmt_b200;
#endif
