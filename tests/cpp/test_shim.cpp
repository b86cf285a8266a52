// test_shim.cpp -- the C++ drop-in (include/gmt_b200.hpp) exercised the way
// the reference's own doctest suites exercise gmt:: (test_planner.cpp,
// test_sampling.cpp, test_graph.cpp), with the B200 library underneath and
// the CPU oracle (oracle/liboracle.so, the C restatement) as the checker.
// Built by tests/cpp/build.py; run by tests/test_gpu_shim.py on a B200.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "gmt_b200.h"
#include "gmt_b200.hpp"

extern "C" {
int oracle_gmt_plan(const gmt_scene*, const double*, int32_t, int32_t, const gmt_graph_view*,
                    int32_t, double, double, int32_t, gmt_plan_out*);
int oracle_sample_free(int32_t, const gmt_scene*, const gmt_sample_source*, double*, double*,
                       int32_t*, int32_t*);
}

using namespace gmt_b200;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    ++g_checks;                                                            \
    if (!(cond)) {                                                         \
      ++g_fail;                                                            \
      std::printf("FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
    }                                                                      \
  } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static ObstacleSet no_obstacles(int dim) {
  ObstacleSet o;
  o.dim = dim;
  return o;
}

static GoalRegion goal_box(std::vector<double> lo, std::vector<double> hi) {
  return GoalRegion{Aabb{std::move(lo), std::move(hi)}};
}

struct Built {
  SampleSet samples;
  NeighborGraph graph;
  int init_index = -1;
  GmtParams params;
};

static Built build_problem(const ObstacleSet& obs, const GoalRegion& goal, const State& init,
                           int n, double lambda, std::uint64_t seed = 0) {
  Built b;
  SampleSource src;
  if (seed != 0) {
    src.kind = SampleSource::Kind::uniform;
    src.seed = seed;
  }
  b.samples = sample_free(n, obs, goal, src);
  b.init_index = append_init(b.samples, init, goal);
  RadiusParams rp;
  rp.dimension = obs.dim;
  rp.n = n;
  double r = connection_radius(rp);
  b.graph = build_neighbor_graph(b.samples.states, SteeringModel{}, r);
  b.params.lambda = lambda;
  b.params.radius = r;
  return b;
}

// Oracle plan on the same inputs (C restatement of planner.cpp).
static bool same_as_oracle(const Built& b, const ObstacleSet& obs, const GoalRegion& goal,
                           const PlanResult& got) {
  detail::FlatScene fs(obs, goal);
  std::vector<double> coords = detail::flat_coords(b.samples, obs.dim);
  detail::FlatGraph fg(b.graph, obs.dim);
  const int n = static_cast<int>(b.samples.states.size());
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
  if (oracle_gmt_plan(&fs.s, coords.data(), n, static_cast<int32_t>(b.samples.goal_indices.size()),
                      &fg.v, b.init_index, b.params.lambda, b.params.radius, 1, &o) != 0)
    return false;
  PlanResult want = detail::to_result(b.samples, n, o, path, label, cost, parent, iter, gs, na, ck);
  if (want.status != got.status || want.path_indices != got.path_indices) return false;
  if (want.tree.parent != got.tree.parent || want.tree.label != got.tree.label) return false;
  if (want.tree.iteration_added != got.tree.iteration_added) return false;
  if (want.tree.cost.size() != got.tree.cost.size() ||
      std::memcmp(want.tree.cost.data(), got.tree.cost.data(), want.tree.cost.size() * 8) != 0)
    return false;
  if (std::memcmp(&want.cost, &got.cost, 8) != 0) return false;
  return want.iterations == got.iterations &&
         want.total_collision_checks == got.total_collision_checks &&
         want.stats.group_sizes == got.stats.group_sizes &&
         want.stats.nodes_added == got.stats.nodes_added &&
         want.stats.collision_checks == got.stats.collision_checks;
}

// test_planner.cpp:63-87
static void open_field() {
  ObstacleSet obs = no_obstacles(2);
  GoalRegion goal = goal_box({0.9, 0.9}, {0.9, 0.9});
  State init{{0.1, 0.1}, std::nullopt};
  Built b = build_problem(obs, goal, init, 2000, 1.0);
  PlanResult res = gmt_plan(b.samples, b.graph, obs, goal, b.init_index, b.params);
  CHECK(res.status == PlanStatus::success);
  CHECK(res.cost >= 0.8 * std::sqrt(2.0) - 1e-12);
  CHECK(res.cost <= 1.31);
  CHECK(!res.path_indices.empty() && res.path_indices.front() == b.init_index);
  CHECK(goal.contains(b.samples.states[res.path_indices.back()]));
  CHECK(res.path.size() == res.path_indices.size());
  CHECK(res.path.front().coords == init.coords);
  CHECK(res.cost == res.tree.cost[res.path_indices.back()]);
  CHECK(same_as_oracle(b, obs, goal, res));
}

// test_planner.cpp:89-111
static void init_in_goal() {
  ObstacleSet obs = no_obstacles(2);
  GoalRegion goal = goal_box({0.4, 0.4}, {0.6, 0.6});
  State init{{0.5, 0.5}, std::nullopt};
  SampleSet samples = sample_free(1, obs, goal, SampleSource{});
  int init_index = append_init(samples, init, goal);
  NeighborGraph g = build_neighbor_graph(samples.states, SteeringModel{}, 0.3);
  GmtParams params;
  params.radius = 0.3;
  PlanResult res = gmt_plan(samples, g, obs, goal, init_index, params);
  CHECK(res.status == PlanStatus::success);
  CHECK(res.cost == 0.0);
  CHECK(res.iterations == 0);
  CHECK(res.path_indices == std::vector<int>{init_index});
  CHECK(res.total_collision_checks == 0);
  PlanResult f = fmt_plan(samples, g, obs, goal, init_index);
  CHECK(f.status == PlanStatus::success && f.cost == 0.0);
}

// test_planner.cpp:113-151
static void infeasible_and_sealed() {
  ObstacleSet obs = no_obstacles(2);
  obs.boxes.push_back(Aabb{{0.6, 0.6}, {1.0, 0.7}});
  obs.boxes.push_back(Aabb{{0.6, 0.6}, {0.7, 1.0}});
  GoalRegion goal = goal_box({0.8, 0.8}, {0.9, 0.9});
  State init{{0.1, 0.1}, std::nullopt};
  Built b = build_problem(obs, goal, init, 800, 1.0);
  PlanResult res = gmt_plan(b.samples, b.graph, obs, goal, b.init_index, b.params);
  CHECK(res.status == PlanStatus::failure_open_empty);
  CHECK(res.path_indices.empty());
  CHECK(res.cost == std::numeric_limits<double>::infinity());
  CHECK(res.iterations > 0);
  CHECK(same_as_oracle(b, obs, goal, res));

  ObstacleSet obs2 = no_obstacles(2);
  obs2.boxes.push_back(Aabb{{0.4, 0.4}, {0.6, 0.6}});
  SampleSet samples = sample_free(50, obs2, goal, SampleSource{});
  int ii = append_init(samples, State{{0.5, 0.5}, std::nullopt}, goal);
  NeighborGraph g = build_neighbor_graph(samples.states, SteeringModel{}, 0.3);
  GmtParams params;
  params.radius = 0.3;
  CHECK(gmt_plan(samples, g, obs2, goal, ii, params).status == PlanStatus::infeasible_input);
  CHECK(gmt_plan(samples, g, obs2, goal, ii, params).tree.label.empty());
}

// test_planner.cpp:153-172
static void parameter_validation() {
  ObstacleSet obs = no_obstacles(2);
  GoalRegion goal = goal_box({0.8, 0.8}, {0.9, 0.9});
  SampleSet samples = sample_free(20, obs, goal, SampleSource{});
  int ii = append_init(samples, State{{0.1, 0.1}, std::nullopt}, goal);
  NeighborGraph g = build_neighbor_graph(samples.states, SteeringModel{}, 0.3);
  GmtParams p;
  p.radius = 0.3;
  p.lambda = 0.0;
  CHECK(throws<InvalidInputError>([&] { gmt_plan(samples, g, obs, goal, ii, p); }));
  p.lambda = 1.5;
  CHECK(throws<InvalidInputError>([&] { gmt_plan(samples, g, obs, goal, ii, p); }));
  p.lambda = 1.0;
  p.radius = 0.25;
  CHECK(throws<InvalidInputError>([&] { gmt_plan(samples, g, obs, goal, ii, p); }));
  p.radius = 0.3;
  CHECK(throws<InvalidInputError>([&] { gmt_plan(samples, g, obs, goal, -1, p); }));
  CHECK(throws<InvalidInputError>([&] { gmt_plan(samples, g, obs, goal, g.n, p); }));
  // sampling errors (test_sampling.cpp:108-121)
  ObstacleSet blocked = no_obstacles(2);
  blocked.boxes.push_back(Aabb{{0.55, 0.55}, {0.95, 0.95}});
  CHECK(throws<GoalBlockedError>(
      [&] { sample_free(50, blocked, goal_box({0.6, 0.6}, {0.9, 0.9}), SampleSource{}); }));
  ObstacleSet full = no_obstacles(2);
  full.boxes.push_back(Aabb{{0.0, 0.0}, {1.0, 1.0}});
  CHECK(throws<InfeasibleSamplingError>([&] { sample_free(10, full, goal, SampleSource{}); }));
}

// test_planner.cpp:332-387: invariants after every iteration, via the hook.
static void wavefront_invariants() {
  ObstacleSet obs = no_obstacles(2);
  obs.boxes.push_back(Aabb{{0.3, 0.0}, {0.4, 0.7}});
  GoalRegion goal = goal_box({0.8, 0.1}, {0.9, 0.2});
  State init{{0.1, 0.1}, std::nullopt};
  Built b = build_problem(obs, goal, init, 400, 0.5, 4242);
  const double delta = b.params.delta();
  long long calls = 0;
  bool ok = true;
  auto hook = [&](const Wavefront& w, long long iter) {
    ++calls;
    for (int v = 0; v < static_cast<int>(w.label.size()); ++v) {
      switch (w.label[v]) {
        case NodeLabel::unexplored:
          ok = ok && std::isinf(w.cost[v]) && w.parent[v] == -1 && w.iteration_added[v] == -1;
          break;
        case NodeLabel::closed:
          ok = ok && w.cost[v] <= iter * delta + 1e-12;
          [[fallthrough]];
        case NodeLabel::open:
          ok = ok && std::isfinite(w.cost[v]);
          if (v != b.init_index) {
            ok = ok && w.parent[v] >= 0 && w.label[w.parent[v]] != NodeLabel::unexplored;
            ok = ok && w.cost[v] >= w.cost[w.parent[v]];
          }
          break;
      }
    }
  };
  PlanResult res = gmt_plan(b.samples, b.graph, obs, goal, b.init_index, b.params, hook);
  CHECK(calls > 0);
  CHECK(ok);
  CHECK(res.status == PlanStatus::success);
  long long closed = 0;
  for (NodeLabel l : res.tree.label) closed += l == NodeLabel::closed;
  long long swept = 0;
  for (std::size_t k = 0; k + 1 < res.stats.group_sizes.size(); ++k) swept += res.stats.group_sizes[k];
  CHECK(swept == closed);
  CHECK(static_cast<long long>(res.stats.group_sizes.size()) - 1 == calls);
  CHECK(same_as_oracle(b, obs, goal, res));
}

// build_instance (problem.cpp:336-363) on rectangles_2d at n = 2000 gives
// the C1 known answer of BASELINE.md §2.
static void c1_known_answer() {
  ProblemFile p;
  p.dimension = 2;
  p.obstacles.dim = 2;
  p.obstacles.boxes = {Aabb{{0.20, 0.00}, {0.40, 0.60}}, Aabb{{0.45, 0.40}, {0.65, 1.00}},
                       Aabb{{0.70, 0.00}, {0.90, 0.60}}};
  p.init = State{{0.05, 0.30}, std::nullopt};
  p.goal = goal_box({0.92, 0.25}, {0.99, 0.40});
  p.n = 2000;
  ProblemInstance inst = build_instance(p);
  CHECK(inst.init_index == 2000);
  CHECK(inst.graph.edge_count() == 143610);
  GmtParams params;
  params.radius = inst.radius;
  PlanResult res = gmt_plan(inst.samples, inst.graph, p.obstacles, p.goal, inst.init_index, params);
  CHECK(res.status == PlanStatus::success);
  CHECK(res.iterations == 21);
  CHECK(res.total_collision_checks == 1967);
  CHECK(std::fabs(res.cost - 1.6900951384243177) == 0.0);
  // sample_free on the device equals the oracle bit for bit
  detail::FlatScene fs(p.obstacles, p.goal);
  gmt_sample_source src{GMT_SAMPLE_HALTON, 0, 1, 0};
  std::vector<double> coords(4000);
  std::vector<int32_t> gidx(2001);
  int32_t gc = 0;
  CHECK(oracle_sample_free(2000, &fs.s, &src, coords.data(), nullptr, gidx.data(), &gc) == 0);
  bool same = true;
  for (int i = 0; i < 2000; ++i)
    for (int k = 0; k < 2; ++k) same = same && coords[2 * i + k] == inst.samples.states[i].coords[k];
  CHECK(same);
}

// build_instance with a cache file (problem.cpp:353-362): miss -> build +
// save, hit -> the same graph; load_graph_cache rejects a different key.
static void graph_cache_roundtrip() {
  ProblemFile p;
  p.dimension = 2;
  p.obstacles.dim = 2;
  p.obstacles.boxes = {Aabb{{0.20, 0.00}, {0.40, 0.60}}, Aabb{{0.45, 0.40}, {0.65, 1.00}}};
  p.init = State{{0.05, 0.30}, std::nullopt};
  p.goal = goal_box({0.92, 0.25}, {0.99, 0.40});
  p.n = 600;
  const std::string file = "/tmp/gmt_b200_shim_cache.gmtg";
  std::remove(file.c_str());
  ProblemInstance a = build_instance(p, 1, file);
  ProblemInstance b = build_instance(p, 1, file);
  CHECK(a.graph.edge_count() == b.graph.edge_count());
  bool same = a.graph.n == b.graph.n;
  for (int u = 0; same && u < a.graph.n; ++u) {
    same = a.graph.out[u].size() == b.graph.out[u].size();
    for (std::size_t j = 0; same && j < a.graph.out[u].size(); ++j)
      same = a.graph.out[u][j].other == b.graph.out[u][j].other && a.graph.out[u][j].cost == b.graph.out[u][j].cost;
  }
  CHECK(same);
  const std::uint64_t key = problem_key(p);
  CHECK(load_graph_cache(file, key, a.samples.states, p.steering, a.radius).has_value());
  CHECK(!load_graph_cache(file, key + 1, a.samples.states, p.steering, a.radius).has_value());
  std::remove(file.c_str());
}

// load_problem / parse_problem through the shim (problem.cpp:102-231): a
// scene parsed, planned through build_instance + gmt_plan; the reference's
// path-named errors.
static void scene_files() {
  const std::string text = R"({"schema": "gmt-problem/1", "dimension": 2,
    "steering": {"model": "euclidean"},
    "obstacles": [{"lo": [0.2, 0.0], "hi": [0.4, 0.6]}, {"lo": [0.55, 0.4], "hi": [0.75, 1.0]}],
    "init": {"coords": [0.05, 0.3]}, "goal": {"lo": [0.92, 0.25], "hi": [0.99, 0.4]},
    "n": 600, "lambda": 1.0, "notes": "two bars"})";
  const ProblemFile p = parse_problem(text);
  CHECK(p.dimension == 2 && p.obstacles.boxes.size() == 2 && p.n == 600);
  CHECK(p.obstacles.boxes[1].lo[0] == 0.55 && p.goal.box.hi[0] == 0.99);
  CHECK(!p.radius_override && p.sampling.kind == SampleSource::Kind::halton && p.sampling.start_index == 1);
  CHECK(p.notes == "two bars");
  const char* tmp = "/tmp/gmt_shim_scene.json";
  if (FILE* f = std::fopen(tmp, "w")) {
    std::fputs(text.c_str(), f);
    std::fclose(f);
  }
  const ProblemFile q = load_problem(tmp);
  CHECK(q.obstacles.boxes[0].hi[1] == 0.6 && q.init.coords[0] == 0.05);
  const ProblemInstance inst = build_instance(q);
  GmtParams params;
  params.lambda = q.lambda;
  params.radius = inst.radius;
  const PlanResult r = gmt_plan(inst.samples, inst.graph, q.obstacles, q.goal, inst.init_index, params);
  CHECK(r.status == PlanStatus::success);
  if (r.status != PlanStatus::success)
    std::printf("scene_files: status %d, %zu samples, init %d, radius %.17g, iterations %lld\n",
                static_cast<int>(r.status), inst.samples.states.size(), inst.init_index, inst.radius,
                static_cast<long long>(r.iterations));
  auto msg = [&](const std::string& t) {
    try {
      parse_problem(t);
    } catch (const InvalidInputError& e) {
      return std::string(e.what());
    }
    return std::string("no error");
  };
  CHECK(msg(R"({"schema": "gmt-problem/1", "dimension": 2, "steering": {"model": "euclidean"},
    "obstacles": [{"lo": [0.2], "hi": [0.4, 0.6]}], "init": {"coords": [0.05, 0.3]},
    "goal": {"lo": [0.9, 0.2], "hi": [0.99, 0.4]}, "n": 10})") ==
        "obstacles[0].lo: expected 2 coordinates, got 1");
  CHECK(msg(R"({"schema": "gmt-problem/1", "dimensions": 2})") == "dimensions: unknown field");
  CHECK(msg("{\"schema\": ").rfind("invalid JSON: ", 0) == 0);
  CHECK(throws<InvalidInputError>([&] { load_problem("/nonexistent/scene.json"); }));
}

int main() {
  scene_files();
  graph_cache_roundtrip();
  open_field();
  init_in_goal();
  infeasible_and_sealed();
  parameter_validation();
  wavefront_invariants();
  c1_known_answer();
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
