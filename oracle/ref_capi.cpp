// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY (oracle).  Never linked into or
// called by the product library.
//
// A flat C wrapper over the *unmodified* reference library gmtplan, compiled
// from its own sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libgmtref.so.  It lets the Python tests and bench.py's CPU
// baseline call the real reference with the same flat structs the product ABI
// uses (include/gmt_b200.h).  Nothing here re-implements the algorithm: every
// function converts flat arrays to the reference's gmt:: types, calls the
// reference function named in its comment, and converts the result back.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <stdexcept>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "gmt_b200.h"
#include "gmtplan/errors.hpp"
#include "gmtplan/graph.hpp"
#include "gmtplan/parallel.hpp"
#include "gmtplan/planner.hpp"
#include "gmtplan/simulator.hpp"
#include "gmtplan/problem.hpp"
#include "gmtplan/sampling.hpp"
#include "gmtplan/space.hpp"

using namespace gmt;

namespace {

thread_local std::string g_err;

template <typename Fn>
int guard(Fn&& fn) {
  try {
    fn();
    return GMT_OK;
  } catch (const InvalidInputError& e) {
    g_err = e.what();
    return GMT_E_INVALID_INPUT;
  } catch (const InfeasibleSamplingError& e) {
    g_err = e.what();
    return GMT_E_INFEASIBLE_SAMPLING;
  } catch (const GoalBlockedError& e) {
    g_err = e.what();
    return GMT_E_GOAL_BLOCKED;
  } catch (const std::exception& e) {
    g_err = e.what();
    return GMT_E_INTERNAL;
  }
}

ObstacleSet to_obs(const gmt_scene* s) {
  ObstacleSet o;
  o.dim = s->dim;
  for (int b = 0; b < s->num_boxes; ++b) {
    Aabb box;
    box.lo.assign(s->box_lo + (size_t)b * s->dim, s->box_lo + (size_t)(b + 1) * s->dim);
    box.hi.assign(s->box_hi + (size_t)b * s->dim, s->box_hi + (size_t)(b + 1) * s->dim);
    o.boxes.push_back(std::move(box));
  }
  return o;
}

GoalRegion to_goal(const gmt_scene* s) {
  GoalRegion g;
  g.box.lo.assign(s->goal_lo, s->goal_lo + s->dim);
  g.box.hi.assign(s->goal_hi, s->goal_hi + s->dim);
  return g;
}

SampleSource to_src(const gmt_sample_source* s) {
  SampleSource src;
  src.kind = s->kind == GMT_SAMPLE_UNIFORM ? SampleSource::Kind::uniform : SampleSource::Kind::halton;
  src.start_index = s->start_index;
  src.seed = s->seed;
  src.with_heading = s->with_heading != 0;
  return src;
}

SampleSet to_samples(const double* coords, const double* heading, int n, int dim,
                     int goal_count) {
  SampleSet s;
  s.states.resize(n);
  for (int i = 0; i < n; ++i) {
    s.states[i].coords.assign(coords + (size_t)i * dim, coords + (size_t)(i + 1) * dim);
    if (heading) s.states[i].heading = heading[i];
  }
  // Only the emptiness of goal_indices is read by the planners (planner.cpp:39-41).
  for (int k = 0; k < goal_count; ++k) s.goal_indices.push_back(0);
  return s;
}

NeighborGraph to_graph(const gmt_graph_view* v) {
  NeighborGraph g;
  g.n = v->n;
  g.radius = v->radius;
  // A directed graph only changes dijkstra_oracle's mirroring (planner.cpp:278).
  g.model.kind = v->directed ? SteeringModel::Kind::dubins_airplane : SteeringModel::Kind::euclidean;
  g.out.resize(v->n);
  g.in.resize(v->n);
  for (int u = 0; u < v->n; ++u) {
    for (int64_t e = v->out_ptr[u]; e < v->out_ptr[u + 1]; ++e) {
      g.out[u].push_back({v->out_col[e], v->out_cost[e], v->out_path ? v->out_path[e] : -1});
    }
  }
  if (v->directed) {
    for (int x = 0; x < v->n; ++x) {
      for (int64_t e = v->in_ptr[x]; e < v->in_ptr[x + 1]; ++e) {
        g.in[x].push_back({v->in_col[e], v->in_cost[e], v->in_path ? v->in_path[e] : -1});
      }
    }
  } else {
    g.in = g.out;
  }
  if (v->num_paths > 0) {
    g.paths.resize(v->num_paths);
    for (int64_t p = 0; p < v->num_paths; ++p) {
      for (int64_t q = v->path_ptr[p]; q < v->path_ptr[p + 1]; ++q) {
        State st;
        st.coords.assign(v->path_pts + q * v->dim, v->path_pts + (q + 1) * v->dim);
        g.paths[p].push_back(std::move(st));
      }
    }
  }
  return g;
}

void write_out(const PlanResult& r, gmt_plan_out* out) {
  out->status = static_cast<int32_t>(r.status);
  out->goal_node = r.path_indices.empty() ? -1 : r.path_indices.back();
  out->cost = r.cost;
  out->iterations = r.iterations;
  out->total_collision_checks = r.total_collision_checks;
  out->path_len = static_cast<int32_t>(r.path_indices.size());
  out->num_stats = static_cast<int32_t>(r.stats.group_sizes.size());
  out->tree_size = static_cast<int32_t>(r.tree.cost.size());
  if (out->path) std::copy(r.path_indices.begin(), r.path_indices.end(), out->path);
  for (int32_t v = 0; v < out->tree_size; ++v) {
    if (out->label) out->label[v] = static_cast<uint8_t>(r.tree.label[v]);
    if (out->tree_cost) out->tree_cost[v] = r.tree.cost[v];
    if (out->parent) out->parent[v] = r.tree.parent[v];
    if (out->iteration_added) out->iteration_added[v] = r.tree.iteration_added[v];
  }
  int32_t ns = std::min(out->num_stats, out->stats_cap);
  for (int32_t k = 0; k < ns; ++k) {
    if (out->group_sizes) out->group_sizes[k] = r.stats.group_sizes[k];
    if (out->nodes_added) out->nodes_added[k] = r.stats.nodes_added[k];
    if (out->collision_checks) out->collision_checks[k] = r.stats.collision_checks[k];
  }
}

void write_summary(const PlanResult& r, gmt_plan_summary* s) {
  s->status = static_cast<int32_t>(r.status);
  s->goal_node = r.path_indices.empty() ? -1 : r.path_indices.back();
  s->cost = r.cost;
  s->iterations = r.iterations;
  s->total_collision_checks = r.total_collision_checks;
  s->path_len = static_cast<int32_t>(r.path_indices.size());
  s->num_stats = static_cast<int32_t>(r.stats.group_sizes.size());
}

ProblemFile to_problem(const gmt_problem* p) {
  ProblemFile f;
  f.dimension = p->scene.dim;
  f.obstacles = to_obs(&p->scene);
  f.goal = to_goal(&p->scene);
  f.init.coords.assign(p->init, p->init + p->scene.dim);
  if (p->init_has_heading) f.init.heading = p->init_heading;
  f.n = p->n;
  f.lambda = p->lambda;
  f.eta = p->eta;
  if (p->radius_override > 0.0) f.radius_override = p->radius_override;
  f.sampling = to_src(&p->sampling);
  if (p->steering == 1) {  // GMT_STEER_DUBINS_AIRPLANE
    f.steering.kind = SteeringModel::Kind::dubins_airplane;
    f.steering.rho = p->dubins.rho;
    f.steering.discretization_step = p->dubins.discretization_step;
    f.steering.planar_cost_only = p->dubins.planar_cost_only != 0;
  }
  return f;
}

struct RefInstance {
  ProblemFile problem;
  ProblemInstance inst;
};

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// halton / nth_prime / halton_point (sampling.cpp:21-51)
int ref_halton(uint64_t index, uint32_t base, double* out) {
  return guard([&] { *out = halton(index, base); });
}
int ref_nth_prime(int k, uint32_t* out) {
  return guard([&] { *out = nth_prime(k); });
}

// point_free / segment_free (space.cpp:47-90)
int ref_point_free(const gmt_scene* s, const double* p, int32_t* out) {
  return guard([&] {
    std::vector<double> v(p, p + s->dim);
    *out = point_free(v, to_obs(s)) ? 1 : 0;
  });
}
int ref_segment_free(const gmt_scene* s, const double* a, const double* b, int32_t* out) {
  return guard([&] {
    State sa{std::vector<double>(a, a + s->dim), std::nullopt};
    State sb{std::vector<double>(b, b + s->dim), std::nullopt};
    *out = segment_free(sa, sb, to_obs(s)) ? 1 : 0;
  });
}

// segment_free over `count` segments (the corpus form of the tests).
int ref_segment_free_many(const gmt_scene* s, const double* a, const double* b, int64_t count,
                          uint8_t* out) {
  return guard([&] {
    const ObstacleSet obs = to_obs(s);
    const int d = s->dim;
    for (int64_t i = 0; i < count; ++i) {
      State sa{std::vector<double>(a + i * d, a + (i + 1) * d), std::nullopt};
      State sb{std::vector<double>(b + i * d, b + (i + 1) * d), std::nullopt};
      out[i] = segment_free(sa, sb, obs) ? 1 : 0;
    }
  });
}

// sample_free (sampling.cpp:81-142)
int ref_sample_free(int32_t n, const gmt_scene* scene, const gmt_sample_source* src,
                    double* coords, double* heading, int32_t* goal_idx, int32_t* goal_count) {
  return guard([&] {
    SampleSet s = sample_free(n, to_obs(scene), to_goal(scene), to_src(src));
    const int d = scene->dim;
    for (int i = 0; i < n; ++i) {
      std::copy(s.states[i].coords.begin(), s.states[i].coords.end(), coords + (size_t)i * d);
      if (heading) heading[i] = s.states[i].heading ? *s.states[i].heading : 0.0;
    }
    *goal_count = static_cast<int32_t>(s.goal_indices.size());
    std::copy(s.goal_indices.begin(), s.goal_indices.end(), goal_idx);
  });
}

// append_init (sampling.cpp:144-154)
int ref_append_init(int32_t dim, double* coords, double* heading, int32_t* n, const double* init,
                    int32_t init_has_heading, double init_heading, const double* goal_lo,
                    const double* goal_hi, int32_t* goal_idx, int32_t* goal_count,
                    int32_t* index_out) {
  return guard([&] {
    SampleSet s;
    s.states.resize(*n);
    for (int i = 0; i < *n; ++i) {
      s.states[i].coords.assign(coords + (size_t)i * dim, coords + (size_t)(i + 1) * dim);
      if (heading) s.states[i].heading = heading[i];
    }
    s.goal_indices.assign(goal_idx, goal_idx + *goal_count);
    State init_state{std::vector<double>(init, init + dim), std::nullopt};
    if (init_has_heading) init_state.heading = init_heading;
    GoalRegion g;
    g.box.lo.assign(goal_lo, goal_lo + dim);
    g.box.hi.assign(goal_hi, goal_hi + dim);
    int idx = append_init(s, init_state, g);
    if (static_cast<int>(s.states.size()) > *n) {
      std::copy(init, init + dim, coords + (size_t)(*n) * dim);
      if (heading) heading[*n] = init_has_heading ? init_heading : 0.0;
      *n = static_cast<int32_t>(s.states.size());
    }
    *goal_count = static_cast<int32_t>(s.goal_indices.size());
    std::copy(s.goal_indices.begin(), s.goal_indices.end(), goal_idx);
    *index_out = idx;
  });
}

// unit_ball_volume / connection_radius (graph.cpp:14-32)
int ref_unit_ball_volume(int32_t d, double* out) {
  return guard([&] { *out = unit_ball_volume(d); });
}
int ref_connection_radius(int32_t dim, int64_t n, double eta, double mu, double* out) {
  return guard([&] {
    RadiusParams p;
    p.dimension = dim;
    p.n = n;
    p.eta = eta;
    p.mu_free = mu;
    *out = connection_radius(p);
  });
}

// build_neighbor_graph (graph.cpp:117-188), Euclidean model.  Two-call
// pattern like the product ABI: NULL arrays return only the edge count.
int ref_build_neighbor_graph(const double* coords, int32_t n, int32_t dim, double radius,
                             int32_t workers, int64_t* num_edges, int64_t* out_ptr,
                             int32_t* out_col, double* out_cost) {
  return guard([&] {
    std::vector<State> st(n);
    for (int i = 0; i < n; ++i) st[i].coords.assign(coords + (size_t)i * dim, coords + (size_t)(i + 1) * dim);
    NeighborGraph g = build_neighbor_graph(st, SteeringModel{}, radius, workers);
    *num_edges = static_cast<int64_t>(g.edge_count());
    if (!out_ptr) return;
    int64_t e = 0;
    for (int u = 0; u < n; ++u) {
      out_ptr[u] = e;
      for (const auto& ed : g.out[u]) {
        out_col[e] = ed.other;
        out_cost[e] = ed.cost;
        ++e;
      }
    }
    out_ptr[n] = e;
  });
}

// gmt_plan (planner.cpp:94-198)
int ref_gmt_plan(const gmt_scene* scene, const double* coords, int32_t n, int32_t goal_count,
                 const gmt_graph_view* graph, int32_t init_index, double lambda, double radius,
                 int32_t workers, gmt_plan_out* out) {
  return guard([&] {
    SampleSet s = to_samples(coords, nullptr, n, scene->dim, goal_count);
    NeighborGraph g = to_graph(graph);
    GmtParams params;
    params.lambda = lambda;
    params.radius = radius;
    params.workers = workers;
    PlanResult r = gmt_plan(s, g, to_obs(scene), to_goal(scene), init_index, params);
    write_out(r, out);
  });
}

// fmt_plan (planner.cpp:200-262)
int ref_fmt_plan(const gmt_scene* scene, const double* coords, int32_t n, int32_t goal_count,
                 const gmt_graph_view* graph, int32_t init_index, gmt_plan_out* out) {
  return guard([&] {
    SampleSet s = to_samples(coords, nullptr, n, scene->dim, goal_count);
    NeighborGraph g = to_graph(graph);
    PlanResult r = fmt_plan(s, g, to_obs(scene), to_goal(scene), init_index);
    write_out(r, out);
  });
}

// dijkstra_oracle (planner.cpp:264-334)
int ref_dijkstra_oracle(const gmt_scene* scene, const double* coords, int32_t n,
                        int32_t goal_count, const gmt_graph_view* graph, int32_t init_index,
                        gmt_plan_out* out) {
  return guard([&] {
    SampleSet s = to_samples(coords, nullptr, n, scene->dim, goal_count);
    NeighborGraph g = to_graph(graph);
    PlanResult r = dijkstra_oracle(s, g, to_obs(scene), to_goal(scene), init_index);
    write_out(r, out);
  });
}

// ---- ProblemInstance handles: build_instance (problem.cpp:336-363) -------
int ref_instance_build(const gmt_problem* p, int32_t workers, void** out) {
  return guard([&] {
    auto* ri = new RefInstance;
    try {
      ri->problem = to_problem(p);
      ri->inst = build_instance(ri->problem, workers);
    } catch (...) {
      delete ri;
      throw;
    }
    *out = ri;
  });
}

void ref_instance_destroy(void* h) { delete static_cast<RefInstance*>(h); }

int ref_instance_info(void* h, int32_t* n, int32_t* init_index, double* radius,
                      int64_t* num_edges, int32_t* goal_count) {
  return guard([&] {
    auto* ri = static_cast<RefInstance*>(h);
    *n = static_cast<int32_t>(ri->inst.samples.states.size());
    *init_index = ri->inst.init_index;
    *radius = ri->inst.radius;
    *num_edges = static_cast<int64_t>(ri->inst.graph.edge_count());
    *goal_count = static_cast<int32_t>(ri->inst.samples.goal_indices.size());
  });
}

int ref_instance_download(void* h, double* coords, int32_t* goal_idx, int64_t* out_ptr,
                          int32_t* out_col, double* out_cost) {
  return guard([&] {
    auto* ri = static_cast<RefInstance*>(h);
    const auto& st = ri->inst.samples.states;
    const int d = ri->problem.dimension;
    if (coords) {
      for (size_t i = 0; i < st.size(); ++i) std::copy(st[i].coords.begin(), st[i].coords.end(), coords + i * d);
    }
    if (goal_idx) std::copy(ri->inst.samples.goal_indices.begin(), ri->inst.samples.goal_indices.end(), goal_idx);
    if (out_ptr) {
      const auto& g = ri->inst.graph;
      int64_t e = 0;
      for (int u = 0; u < g.n; ++u) {
        out_ptr[u] = e;
        for (const auto& ed : g.out[u]) {
          if (out_col) out_col[e] = ed.other;
          if (out_cost) out_cost[e] = ed.cost;
          ++e;
        }
      }
      out_ptr[g.n] = e;
    }
  });
}

// ---- Dubins steering (steering.cpp:53-112) -----------------------------------
// connect_cost and connect's segment count for state pairs (x, y[, z], heading).
int ref_dubins_costs(const double* x0s, const double* x1s, int64_t count, int32_t dim,
                     const gmt_dubins_params* prm, double* cost, int32_t* segments) {
  return guard([&] {
    SteeringModel m;
    m.kind = SteeringModel::Kind::dubins_airplane;
    m.rho = prm->rho;
    m.discretization_step = prm->discretization_step;
    m.planar_cost_only = prm->planar_cost_only != 0;
    for (int64_t i = 0; i < count; ++i) {
      State a, b;
      a.coords.assign(x0s + i * (dim + 1), x0s + i * (dim + 1) + dim);
      b.coords.assign(x1s + i * (dim + 1), x1s + i * (dim + 1) + dim);
      a.heading = x0s[i * (dim + 1) + dim];
      b.heading = x1s[i * (dim + 1) + dim];
      Connection c = connect(a, b, m);
      cost[i] = c.cost;
      segments[i] = c.path.size() == 1 ? 0 : static_cast<int32_t>(c.path.size()) - 1;
    }
  });
}

// ---- simulator (simulator.cpp:66-227) ---------------------------------------
ScenarioConfig to_scenario(const gmt_scenario* c) {
  ScenarioConfig cfg;
  cfg.base.obstacles = to_obs(&c->scene);
  cfg.base.goal = to_goal(&c->scene);
  cfg.base.init.coords.assign(c->init, c->init + c->scene.dim);
  cfg.base.n = c->n;
  cfg.base.lambda = c->lambda;
  cfg.base.eta = c->eta;
  if (c->radius_override > 0.0) cfg.base.radius_override = c->radius_override;
  cfg.collapse_rate = c->collapse_rate;
  cfg.spawn_box_size = c->spawn_box_size;
  cfg.disturbance_sigma = c->disturbance_sigma;
  cfg.replan_latency = c->replan_latency;
  cfg.control_dt = c->control_dt;
  cfg.robot_speed = c->robot_speed;
  cfg.time_limit = c->time_limit;
  cfg.trials = c->trials;
  cfg.seed = c->seed;
  return cfg;
}

int ref_run_trial(const gmt_scenario* c, uint64_t seed, gmt_trial_outcome* out, double* path,
                  int64_t cap) {
  return guard([&] {
    TrialOutcome o = run_trial(to_scenario(c), seed);
    out->result = static_cast<int32_t>(o.result);
    out->replans = o.replans;
    out->spawned = o.spawned;
    out->noise_outliers = o.noise_outliers;
    out->time = o.time;
    out->path_len = static_cast<int64_t>(o.path_travelled.size());
    const int d = c->scene.dim;
    for (int64_t k = 0; path && k < cap && k < out->path_len; ++k)
      std::copy(o.path_travelled[k].coords.begin(), o.path_travelled[k].coords.end(), path + k * d);
  });
}

int ref_run_campaign(const gmt_scenario* c, const double* lat, int32_t nl, const double* rates,
                     int32_t nr, const double* sig, int32_t ns, int32_t workers, int32_t* successes) {
  return guard([&] {
    auto cells = run_campaign(to_scenario(c), std::vector<double>(lat, lat + nl),
                              std::vector<double>(rates, rates + nr), std::vector<double>(sig, sig + ns),
                              workers);
    for (size_t k = 0; k < cells.size(); ++k) successes[k] = cells[k].successes;
  });
}

// ---- graph cache (GMTG v1, graph.cpp:190-343) and problem_key (problem.cpp:281-303)
int ref_problem_key(const gmt_problem* p, uint64_t* out) {
  return guard([&] { *out = problem_key(to_problem(p)); });
}

// build_instance with a cache file (problem.cpp:354-362): loads on a key /
// shape match, else builds and saves.
int ref_instance_build_cached(const gmt_problem* p, const char* cache_file, void** out) {
  return guard([&] {
    auto* ri = new RefInstance;
    try {
      ri->problem = to_problem(p);
      ri->inst = build_instance(ri->problem, 1, cache_file);
    } catch (...) {
      delete ri;
      throw;
    }
    *out = ri;
  });
}

int ref_save_graph_cache(void* h, const char* file, uint64_t key, int32_t* ok) {
  return guard([&] {
    auto* ri = static_cast<RefInstance*>(h);
    *ok = save_graph_cache(ri->inst.graph, file, key) ? 1 : 0;
  });
}

// load_graph_cache for a Euclidean graph over host states; *hit = 0 on any
// mismatch.  Two-call pattern like ref_build_neighbor_graph.
int ref_load_graph_cache(const char* file, uint64_t key, const double* coords, int32_t n, int32_t dim,
                         double radius, int32_t* hit, int64_t* num_edges, int64_t* out_ptr,
                         int32_t* out_col, double* out_cost) {
  return guard([&] {
    std::vector<State> st(n);
    for (int i = 0; i < n; ++i) st[i].coords.assign(coords + static_cast<size_t>(i) * dim, coords + static_cast<size_t>(i + 1) * dim);
    auto g = load_graph_cache(file, key, st, SteeringModel{}, radius);
    *hit = g ? 1 : 0;
    *num_edges = g ? static_cast<int64_t>(g->edge_count()) : 0;
    if (g && out_ptr) {
      int64_t e = 0;
      for (int u = 0; u < g->n; ++u) {
        out_ptr[u] = e;
        for (const auto& ed : g->out[u]) {
          out_col[e] = ed.other;
          out_cost[e] = ed.cost;
          ++e;
        }
      }
      out_ptr[g->n] = e;
    }
  });
}

// The directed part of an instance's graph: in-rows, path ids and the
// cached edge paths (positions only).  NULL arrays: sizes only.
int ref_instance_download_paths(void* h, int64_t* in_ptr, int32_t* in_col, double* in_cost,
                                int32_t* in_path, int32_t* out_path, int64_t* path_ptr, double* path_pts,
                                int64_t* num_paths, int64_t* num_points) {
  return guard([&] {
    auto* ri = static_cast<RefInstance*>(h);
    const auto& g = ri->inst.graph;
    const int d = ri->problem.dimension;
    *num_paths = static_cast<int64_t>(g.paths.size());
    int64_t pts = 0;
    for (const auto& p : g.paths) pts += static_cast<int64_t>(p.size());
    *num_points = pts;
    if (!in_ptr) return;
    int64_t e = 0;
    for (int x = 0; x < g.n; ++x) {
      in_ptr[x] = e;
      for (const auto& ed : g.in[x]) {
        in_col[e] = ed.other;
        in_cost[e] = ed.cost;
        in_path[e] = ed.path_id;
        ++e;
      }
    }
    in_ptr[g.n] = e;
    e = 0;
    for (int u = 0; u < g.n; ++u)
      for (const auto& ed : g.out[u]) out_path[e++] = ed.path_id;
    int64_t q = 0;
    for (size_t p = 0; p < g.paths.size(); ++p) {
      path_ptr[p] = q;
      for (const auto& st : g.paths[p]) {
        std::copy(st.coords.begin(), st.coords.begin() + d, path_pts + q * d);
        ++q;
      }
    }
    path_ptr[g.paths.size()] = q;
  });
}

int ref_instance_plan(void* h, double lambda, int32_t workers, gmt_plan_out* out) {
  return guard([&] {
    auto* ri = static_cast<RefInstance*>(h);
    GmtParams params;
    params.lambda = lambda;
    params.radius = ri->inst.radius;
    params.workers = workers;
    PlanResult r = gmt_plan(ri->inst.samples, ri->inst.graph, ri->problem.obstacles,
                            ri->problem.goal, ri->inst.init_index, params);
    write_out(r, out);
  });
}

// Single-solve CPU baseline: `reps` timed gmt_plan calls
// on one prebuilt instance, each on the monotonic clock like the reference's
// own `gmtplan plan` timer (tools/gmtplan.cpp:80-90), per-call ms in ms[].
int ref_instance_time_plans(void* h, double lambda, int32_t workers, int32_t reps, double* ms) {
  return guard([&] {
    auto* ri = static_cast<RefInstance*>(h);
    GmtParams params;
    params.lambda = lambda;
    params.radius = ri->inst.radius;
    params.workers = workers;
    for (int32_t k = 0; k < reps; ++k) {
      auto t0 = std::chrono::steady_clock::now();
      PlanResult r = gmt_plan(ri->inst.samples, ri->inst.graph, ri->problem.obstacles,
                              ri->problem.goal, ri->inst.init_index, params);
      ms[k] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      (void)r;
    }
  });
}

// The same on an injected graph (the 12D quadrotor: the device graph with its
// waypoint polylines handed to the unmodified gmt_plan, planner.cpp:54-60).
int ref_time_gmt_plan(const gmt_scene* scene, const double* coords, int32_t n, int32_t goal_count,
                      const gmt_graph_view* graph, int32_t init_index, double lambda, double radius,
                      int32_t workers, int32_t reps, double* ms) {
  return guard([&] {
    SampleSet s = to_samples(coords, nullptr, n, scene->dim, goal_count);
    NeighborGraph g = to_graph(graph);
    ObstacleSet obs = to_obs(scene);
    GoalRegion goal = to_goal(scene);
    GmtParams params;
    params.lambda = lambda;
    params.radius = radius;
    params.workers = workers;
    for (int32_t k = 0; k < reps; ++k) {
      auto t0 = std::chrono::steady_clock::now();
      PlanResult r = gmt_plan(s, g, obs, goal, init_index, params);
      ms[k] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      (void)r;
    }
  });
}

// Batched CPU baseline: one gmt_plan(workers=1) per query under
// parallel_chunks, the pattern of simulator.cpp:212.  Returns wall seconds
// of the whole batch in *seconds.
int ref_plan_many(void** handles, int32_t count, double lambda, int32_t threads,
                  gmt_plan_summary* out, double* seconds) {
  return guard([&] {
    std::vector<PlanResult> results(count);
    auto t0 = std::chrono::steady_clock::now();
    parallel_chunks(threads, static_cast<std::size_t>(count), [&](std::size_t b, std::size_t e) {
      for (std::size_t q = b; q < e; ++q) {
        auto* ri = static_cast<RefInstance*>(handles[q]);
        GmtParams params;
        params.lambda = lambda;
        params.radius = ri->inst.radius;
        params.workers = 1;
        results[q] = gmt_plan(ri->inst.samples, ri->inst.graph, ri->problem.obstacles,
                              ri->problem.goal, ri->inst.init_index, params);
      }
    });
    auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    if (out) {
      for (int32_t q = 0; q < count; ++q) write_summary(results[q], &out[q]);
    }
  });
}

// Parallel build of many instances (setup for the baseline, not timed).
int ref_instance_build_many(const gmt_problem* problems, int32_t count, int32_t threads,
                            void** out) {
  return guard([&] {
    std::vector<std::string> errs(count);
    parallel_chunks(threads, static_cast<std::size_t>(count), [&](std::size_t b, std::size_t e) {
      for (std::size_t q = b; q < e; ++q) {
        auto* ri = new RefInstance;
        try {
          ri->problem = to_problem(&problems[q]);
          ri->inst = build_instance(ri->problem, 1);
          out[q] = ri;
        } catch (const std::exception& ex) {
          delete ri;
          out[q] = nullptr;
          errs[q] = ex.what();
        }
      }
    });
    for (int32_t q = 0; q < count; ++q) {
      if (!out[q]) throw std::runtime_error("query " + std::to_string(q) + ": " + errs[q]);
    }
  });
}

// ---- problem files: parse_problem / problem_key (problem.cpp:102-303) -----
// Parses JSON text and reports the flat fields.  Arrays are caller-owned with
// capacity given by the first call (dim, num_boxes are always written).
int ref_parse_problem(const char* json_text, int32_t* dim, int32_t* num_boxes, double* box_lo,
                      double* box_hi, double* goal_lo, double* goal_hi, double* init,
                      int32_t* n, double* lambda, double* eta, double* radius_override,
                      int32_t* sampling_kind, uint64_t* start_index, uint64_t* seed,
                      uint64_t* key, int32_t* steering_kind) {
  return guard([&] {
    ProblemFile p = parse_problem(json_text);
    *dim = p.dimension;
    *num_boxes = static_cast<int32_t>(p.obstacles.boxes.size());
    if (!box_lo) return;
    for (int b = 0; b < *num_boxes; ++b) {
      std::copy(p.obstacles.boxes[b].lo.begin(), p.obstacles.boxes[b].lo.end(), box_lo + b * p.dimension);
      std::copy(p.obstacles.boxes[b].hi.begin(), p.obstacles.boxes[b].hi.end(), box_hi + b * p.dimension);
    }
    std::copy(p.goal.box.lo.begin(), p.goal.box.lo.end(), goal_lo);
    std::copy(p.goal.box.hi.begin(), p.goal.box.hi.end(), goal_hi);
    std::copy(p.init.coords.begin(), p.init.coords.end(), init);
    *n = p.n;
    *lambda = p.lambda;
    *eta = p.eta;
    *radius_override = p.radius_override ? *p.radius_override : 0.0;
    *sampling_kind = p.sampling.kind == SampleSource::Kind::uniform ? 1 : 0;
    *start_index = p.sampling.start_index;
    *seed = p.sampling.seed;
    *key = problem_key(p);
    *steering_kind = p.steering.kind == SteeringModel::Kind::euclidean ? 0 : 1;
  });
}

}  // extern "C"

// ---- the reference's own seeded problem generator -------------------------
// make_random_problem (tests/support/oracles.cpp:258-327) and its Pcg32
// stream, exposed so the Python tests draw the very problems the reference's
// property tests draw.
#include "support/oracles.hpp"

extern "C" {

void* ref_rng_create(uint64_t seed) { return new Pcg32(seed); }
void ref_rng_destroy(void* h) { delete static_cast<Pcg32*>(h); }
uint32_t ref_rng_next_u32(void* h) { return static_cast<Pcg32*>(h)->next_u32(); }

int ref_random_problem_new(void* rng, int32_t dim, int32_t with_obstacles, int32_t n_min,
                           int32_t n_max, void** out) {
  return guard([&] {
    test::RandomProblemOptions opt;
    opt.dim = dim;
    opt.with_obstacles = with_obstacles != 0;
    opt.n_min = n_min;
    opt.n_max = n_max;
    *out = new test::RandomProblem(test::make_random_problem(*static_cast<Pcg32*>(rng), opt));
  });
}

void ref_random_problem_free(void* h) { delete static_cast<test::RandomProblem*>(h); }

int ref_random_problem_info(void* h, int32_t* num_boxes, int32_t* n_samples, int32_t* init_index,
                            double* radius, int32_t* goal_count, uint64_t* seed) {
  return guard([&] {
    auto* p = static_cast<test::RandomProblem*>(h);
    *num_boxes = static_cast<int32_t>(p->obs.boxes.size());
    *n_samples = static_cast<int32_t>(p->samples.states.size());
    *init_index = p->init_index;
    *radius = p->radius;
    *goal_count = static_cast<int32_t>(p->samples.goal_indices.size());
    *seed = 0;
  });
}

int ref_random_problem_get(void* h, double* box_lo, double* box_hi, double* goal_lo,
                           double* goal_hi, double* init, double* coords, int32_t* goal_idx) {
  return guard([&] {
    auto* p = static_cast<test::RandomProblem*>(h);
    const int d = p->obs.dim;
    for (size_t b = 0; b < p->obs.boxes.size(); ++b) {
      std::copy(p->obs.boxes[b].lo.begin(), p->obs.boxes[b].lo.end(), box_lo + b * d);
      std::copy(p->obs.boxes[b].hi.begin(), p->obs.boxes[b].hi.end(), box_hi + b * d);
    }
    std::copy(p->goal.box.lo.begin(), p->goal.box.lo.end(), goal_lo);
    std::copy(p->goal.box.hi.begin(), p->goal.box.hi.end(), goal_hi);
    std::copy(p->init.coords.begin(), p->init.coords.end(), init);
    for (size_t i = 0; i < p->samples.states.size(); ++i) {
      std::copy(p->samples.states[i].coords.begin(), p->samples.states[i].coords.end(), coords + i * d);
    }
    std::copy(p->samples.goal_indices.begin(), p->samples.goal_indices.end(), goal_idx);
  });
}

}  // extern "C"

extern "C" int ref_struct_sizes(int64_t* out, int32_t count) {
  const int64_t sizes[] = {sizeof(gmt_scene),     sizeof(gmt_sample_source), sizeof(gmt_graph_view),
                           sizeof(gmt_plan_out),  sizeof(gmt_plan_summary),  sizeof(gmt_problem),
                           sizeof(gmt_di_params), sizeof(gmt_batch_host),    sizeof(gmt_quad_params),
                           sizeof(gmt_scenario),  sizeof(gmt_trial_outcome), sizeof(gmt_dubins_params)};
  const int32_t n = static_cast<int32_t>(sizeof(sizes) / sizeof(sizes[0]));
  for (int32_t i = 0; i < count && i < n; ++i) out[i] = sizes[i];
  return n;
}

// ---- double-integrator instances for bench.py's reference arm -------------
// The reference has no double integrator, so a DI instance for
// the UNMODIFIED reference planner is assembled here from (i) the reference's
// own sample_free + append_init (sampling.cpp:81-154), (ii) the oracle's C
// statement of the model (gmt_oracle.c: oracle_di_cost / oracle_di_coord,
// linked in) for edge costs, durations and the cached waypoint polylines the
// reference's motion_free checks (planner.cpp:54-60), and (iii) the shared
// Halton pool of SURVEY.md §8(e): the pool rows are evaluated once, each
// query's rows are the pool rows of its samples re-indexed by rank, plus the
// rows of its non-pool vertices (a substituted goal, the init) evaluated
// directly.  Test/bench infrastructure only.
extern "C" double oracle_di_cost(const double* x0, const double* x1, double vmax, double w, double* tau);
extern "C" double oracle_di_coord(const double* x0, const double* x1, double tau, int k, int i, int M,
                                  double vmax);

namespace {

struct DiPoolRef {
  int K = 0;
  gmt_di_params di{};
  double radius = 0.0;
  double bound = 0.0;
  std::vector<double> pts;                 // K x 6
  std::vector<std::vector<int>> col;       // pool out-rows, targets ascending
  std::vector<std::vector<double>> cost;
  std::vector<std::vector<double>> tau;
};

bool di_may_ref(const double* a, const double* b, double bound) {
  for (int k = 0; k < 3; ++k) {
    const double D = b[k] - a[k];
    if (D > bound || -D > bound) return false;
  }
  return true;
}

// cost(a -> b) <= r with the exact-safe |dp| prefilter; the edge's cost/duration.
bool di_edge(const DiPoolRef& P, const double* a, const double* b, double* c, double* t) {
  if (!di_may_ref(a, b, P.bound)) return false;
  *c = oracle_di_cost(a, b, P.di.vmax, P.di.weight, t);
  return *c <= P.radius;
}

}  // namespace

extern "C" {

void* ref_di_pool_create(uint64_t start_index, int32_t K, const gmt_di_params* di, double radius, int32_t threads) {
  auto* P = new DiPoolRef;
  P->K = K;
  P->di = *di;
  P->radius = radius;
  P->bound = (di->vmax * radius + radius * radius / (2.0 * std::sqrt(3.0 * di->weight))) * (1.0 + 1e-9) + 1e-12;
  P->pts.resize(static_cast<size_t>(K) * 6);
  for (int p = 0; p < K; ++p) {
    const std::vector<double> h = halton_point(start_index + static_cast<uint64_t>(p), 6);  // sampling.cpp:46-51
    std::copy(h.begin(), h.end(), P->pts.begin() + static_cast<size_t>(p) * 6);
  }
  P->col.resize(K);
  P->cost.resize(K);
  P->tau.resize(K);
  parallel_chunks(threads, static_cast<std::size_t>(K), [&](std::size_t b, std::size_t e) {
    for (std::size_t u = b; u < e; ++u) {
      const double* a = P->pts.data() + u * 6;
      for (int v = 0; v < K; ++v) {
        if (v == static_cast<int>(u)) continue;
        double c, t;
        if (di_edge(*P, a, P->pts.data() + static_cast<size_t>(v) * 6, &c, &t)) {
          P->col[u].push_back(v);
          P->cost[u].push_back(c);
          P->tau[u].push_back(t);
        }
      }
    }
  });
  return P;
}

void ref_di_pool_destroy(void* h) { delete static_cast<DiPoolRef*>(h); }

int ref_di_pool_instances(void* pool, const gmt_problem* problems, int32_t count, int32_t threads, void** out) {
  return guard([&] {
    const DiPoolRef& P = *static_cast<const DiPoolRef*>(pool);
    const int M = P.di.segments;
    std::vector<std::string> errs(count);
    parallel_chunks(threads, static_cast<std::size_t>(count), [&](std::size_t b, std::size_t e) {
      for (std::size_t q = b; q < e; ++q) {
        auto* ri = new RefInstance;
        out[q] = nullptr;
        try {
          ri->problem = to_problem(&problems[q]);
          const ProblemFile& pf = ri->problem;
          SampleSet s = sample_free(pf.n, pf.obstacles, pf.goal, pf.sampling);  // the reference's own
          const int init = append_init(s, pf.init, pf.goal);
          const int V = static_cast<int>(s.states.size());
          // samples that are pool points: the free pool points in stream order
          std::vector<int> pid(V, -1), rank(P.K, -1);
          int j = 0;
          for (int p = 0; p < P.K && j < pf.n; ++p) {
            std::vector<double> x(P.pts.begin() + static_cast<size_t>(p) * 6, P.pts.begin() + static_cast<size_t>(p + 1) * 6);
            if (!point_free(x, pf.obstacles)) continue;
            if (s.states[j].coords == x) {
              pid[j] = p;
              rank[p] = j;
            }
            ++j;
          }
          if (j < pf.n - 1) throw std::runtime_error("reference DI pool too small for the query");
          std::vector<int> special;
          for (int v = 0; v < V; ++v)
            if (pid[v] < 0) special.push_back(v);
          NeighborGraph g;
          g.n = V;
          g.radius = P.radius;
          g.model.kind = SteeringModel::Kind::dubins_airplane;  // directed (planner.cpp:278)
          g.out.resize(V);
          g.in.resize(V);
          std::vector<std::vector<double>> otau(V);
          auto X = [&](int v) { return s.states[v].coords.data(); };
          for (int u = 0; u < V; ++u) {
            if (pid[u] >= 0) {
              const int p = pid[u];
              for (size_t k = 0; k < P.col[p].size(); ++k) {
                const int r = rank[P.col[p][k]];
                if (r < 0) continue;
                g.out[u].push_back({r, P.cost[p][k], -1});
                otau[u].push_back(P.tau[p][k]);
              }
              for (int sv : special) {  // the largest indices: appended in order
                double c, t;
                if (sv != u && di_edge(P, X(u), X(sv), &c, &t)) {
                  g.out[u].push_back({sv, c, -1});
                  otau[u].push_back(t);
                }
              }
            } else {
              for (int v = 0; v < V; ++v) {
                double c, t;
                if (v != u && di_edge(P, X(u), X(v), &c, &t)) {
                  g.out[u].push_back({v, c, -1});
                  otau[u].push_back(t);
                }
              }
            }
          }
          // path ids in (source, position) order; in-lists by ascending source
          // (graph.cpp:172-186), sharing the out-edge's path
          int pidx = 0;
          for (int u = 0; u < V; ++u) {
            for (size_t k = 0; k < g.out[u].size(); ++k) {
              auto& ed = g.out[u][k];
              ed.path_id = pidx++;
              std::vector<State> path(M + 1);
              for (int w = 0; w <= M; ++w) {
                path[w].coords.resize(6);
                for (int i = 0; i < 6; ++i)
                  path[w].coords[i] = oracle_di_coord(X(u), X(ed.other), otau[u][k], w, i, M, P.di.vmax);
              }
              g.paths.push_back(std::move(path));
              g.in[ed.other].push_back({u, ed.cost, ed.path_id});
            }
          }
          ri->inst.samples = std::move(s);
          ri->inst.init_index = init;
          ri->inst.radius = P.radius;
          ri->inst.graph = std::move(g);
          out[q] = ri;
        } catch (const std::exception& ex) {
          delete ri;
          errs[q] = ex.what();
        }
      }
    });
    for (int32_t q = 0; q < count; ++q)
      if (!out[q]) throw std::runtime_error("query " + std::to_string(q) + ": " + errs[q]);
  });
}

}  // extern "C"
