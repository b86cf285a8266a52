// sim.cu -- the reference's replanning simulator (simulator.hpp/.cpp) with
// every replan on the B200: campaign trials are
// independent planning queries.  The trial state machine (Poisson obstacle
// collapse, plan tracking, clamped Gaussian disturbance) is host code that
// restates simulator.cpp:68-176 operation for operation with the host's
// libm, so trials replay the reference bit for bit; each replan --
// sample_free (uniform, per-replan seed) -> append_init -> r-disk graph ->
// gmt_plan -- runs through the device path (gmt_instance_build + gmt_plan).
// A campaign (simulator.cpp:178-227) spreads its trials over host worker
// threads, each with its own context / CUDA stream, so the replans of
// different trials overlap on the GPU.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "gmt_b200.h"
#include "internal.cuh"

namespace gmtb {

namespace {

uint64_t mix64(uint64_t x) {  // splitmix64 (rng.hpp:68-73)
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
uint64_t mix64(uint64_t a, uint64_t b) { return mix64(mix64(a) ^ b); }
uint64_t bits_of(double v) {
  uint64_t b;
  std::memcpy(&b, &v, 8);
  return b;
}

// PCG-XSH-RR 32 with the reference's Box-Muller and Knuth Poisson draws
// (rng.hpp:11-60).
struct Rng {
  uint64_t state = 0, inc = 1;
  double spare = 0.0;
  bool has_spare = false;
  explicit Rng(uint64_t seed) {
    state = 0u;
    inc = 1u;  // seq = 0
    next_u32();
    state += seed;
    next_u32();
  }
  uint32_t next_u32() {
    const uint64_t old = state;
    state = old * 6364136223846793005ULL + inc;
    const uint32_t xs = static_cast<uint32_t>(((old >> 18u) ^ old) >> 27u);
    const uint32_t rot = static_cast<uint32_t>(old >> 59u);
    return (xs >> rot) | (xs << ((32u - rot) & 31u));
  }
  double next_double() { return next_u32() * 0x1p-32; }
  double gaussian() {
    if (has_spare) {
      has_spare = false;
      return spare;
    }
    double u1 = next_double();
    const double u2 = next_double();
    while (u1 <= 0.0) u1 = next_double();
    const double mag = std::sqrt(-2.0 * std::log(u1));
    spare = mag * std::sin(2.0 * M_PI * u2);
    has_spare = true;
    return mag * std::cos(2.0 * M_PI * u2);
  }
  int poisson(double mean) {
    const double limit = std::exp(-mean);
    double prod = next_double();
    int k = 0;
    while (prod > limit) {
      ++k;
      prod *= next_double();
    }
    return k;
  }
};

uint64_t draw_seed(Rng& rng) {  // simulator.cpp:17-20
  const uint64_t hi = rng.next_u32();
  return (hi << 32) | rng.next_u32();
}

double euclid(const std::vector<double>& a, const std::vector<double>& b) {  // space.cpp:126-133
  double sq = 0.0;
  for (size_t k = 0; k < a.size(); ++k) {
    const double d = a[k] - b[k];
    sq += d * d;
  }
  return std::sqrt(sq);
}

struct Obstacles {
  int d = 0;
  std::vector<double> lo, hi;  // boxes, row-major
  int count() const { return d ? static_cast<int>(lo.size()) / d : 0; }
};

bool box_contains(const double* lo, const double* hi, const std::vector<double>& p) {  // space.cpp:11-16
  for (size_t k = 0; k < p.size(); ++k)
    if (p[k] < lo[k] || p[k] > hi[k]) return false;
  return true;
}

bool point_free(const std::vector<double>& p, const Obstacles& o) {  // space.cpp:40-54
  for (double x : p)
    if (x < 0.0 || x > 1.0) return false;
  for (int b = 0; b < o.count(); ++b)
    if (box_contains(o.lo.data() + b * o.d, o.hi.data() + b * o.d, p)) return false;
  return true;
}

// plan_from (simulator.cpp:32-64) on the device.  Returns GMT_OK with
// `found` false for the reference's nullopt outcomes.
int plan_from(gmt_ctx* ctx, const gmt_scenario& cfg, const std::vector<double>& pos,
              const Obstacles& obs, uint64_t seed, bool* goal_blocked, bool* found,
              std::vector<std::vector<double>>* path) {
  *found = false;
  gmt_problem p{};
  p.scene = cfg.scene;
  p.scene.num_boxes = obs.count();
  p.scene.box_lo = obs.lo.data();
  p.scene.box_hi = obs.hi.data();
  p.init = pos.data();
  p.n = cfg.n;
  p.lambda = cfg.lambda;
  p.eta = cfg.eta;
  p.radius_override = cfg.radius_override;
  p.sampling.kind = GMT_SAMPLE_UNIFORM;
  p.sampling.start_index = 1;
  p.sampling.seed = seed;
  p.steering = GMT_STEER_EUCLIDEAN;
  gmt_instance* inst = nullptr;
  int rc = gmt_instance_build(ctx, &p, &inst);
  if (rc == GMT_E_GOAL_BLOCKED) {
    if (goal_blocked) *goal_blocked = true;
    return GMT_OK;
  }
  if (rc == GMT_E_INFEASIBLE_SAMPLING) return GMT_OK;
  if (rc) return rc;
  int32_t n = 0, dim = 0, ii = 0, gc = 0;
  double r = 0.0;
  int64_t E = 0;
  rc = gmt_instance_info(inst, &n, &dim, &ii, &r, &E, &gc);
  std::vector<int32_t> path_idx(n);
  gmt_plan_out out{};
  out.path = path_idx.data();
  if (rc == GMT_OK) rc = gmt_plan(ctx, inst, ii, cfg.lambda, r, &out);
  if (rc == GMT_OK && out.status == 0) {
    std::vector<double> coords(static_cast<size_t>(n) * dim);
    rc = gmt_instance_download(ctx, inst, coords.data(), nullptr, nullptr, nullptr, nullptr);
    if (rc == GMT_OK) {
      path->clear();
      for (int k = 0; k < out.path_len; ++k)
        path->emplace_back(coords.begin() + static_cast<size_t>(path_idx[k]) * dim,
                           coords.begin() + static_cast<size_t>(path_idx[k] + 1) * dim);
      *found = true;
    }
  }
  gmt_instance_destroy(inst);
  return rc;
}

int validate_scenario(const gmt_scenario* c) {  // simulator.cpp:67-72
  if (!c) return set_error(GMT_E_INVALID_INPUT, "scenario is null");
  if (!(c->control_dt > 0.0) || !(c->time_limit > 0.0) || !(c->robot_speed >= 0.0) ||
      !(c->replan_latency > 0.0) || !(c->collapse_rate >= 0.0) || !(c->disturbance_sigma >= 0.0) ||
      !(c->spawn_box_size > 0.0))
    return set_error(GMT_E_INVALID_INPUT, "scenario timing/rate parameters must be positive");
  return GMT_OK;
}

// run_trial (simulator.cpp:66-176).
int run_trial(gmt_ctx* ctx, const gmt_scenario& cfg, uint64_t trial_seed, gmt_trial_outcome* out,
              std::vector<double>* travelled) {
  int rc = validate_scenario(&cfg);
  if (rc) return rc;
  const int d = cfg.scene.dim;
  Rng rng(trial_seed);
  Obstacles obstacles;
  obstacles.d = d;
  obstacles.lo.assign(cfg.scene.box_lo, cfg.scene.box_lo + static_cast<size_t>(cfg.scene.num_boxes) * d);
  obstacles.hi.assign(cfg.scene.box_hi, cfg.scene.box_hi + static_cast<size_t>(cfg.scene.num_boxes) * d);
  std::vector<double> pos(cfg.init, cfg.init + d);
  gmt_trial_outcome o{};
  o.result = GMT_TRIAL_TIMED_OUT;
  travelled->assign(pos.begin(), pos.end());
  bool goal_blocked = false;

  std::vector<std::vector<double>> plan;
  bool found = false;
  rc = plan_from(ctx, cfg, pos, obstacles, draw_seed(rng), &goal_blocked, &found, &plan);
  if (rc) return rc;
  if (!found) {
    o.path_len = 1;
    *out = o;
    return GMT_OK;
  }
  size_t waypoint = 1;
  double t = 0.0;
  double next_replan = cfg.replan_latency;
  const double half = 0.5 * cfg.spawn_box_size;
  std::vector<double> lo(d), hi(d);
  for (;;) {
    // (a) collapse events (simulator.cpp:96-113)
    const int events = rng.poisson(cfg.collapse_rate * cfg.control_dt);
    for (int e = 0; e < events; ++e) {
      for (int attempt = 0; attempt < 1000; ++attempt) {
        for (int k = 0; k < d; ++k) {
          const double c = rng.next_double();
          lo[k] = c - half;
          hi[k] = c + half;
        }
        if (box_contains(lo.data(), hi.data(), pos)) continue;
        obstacles.lo.insert(obstacles.lo.end(), lo.begin(), lo.end());
        obstacles.hi.insert(obstacles.hi.end(), hi.begin(), hi.end());
        ++o.spawned;
        break;
      }
    }
    // (b) track the plan, then disturb (simulator.cpp:115-141)
    double advance = cfg.robot_speed * cfg.control_dt;
    while (advance > 0.0 && waypoint < plan.size()) {
      const double seg_len = euclid(pos, plan[waypoint]);
      if (seg_len <= advance) {
        pos = plan[waypoint];
        advance -= seg_len;
        ++waypoint;
      } else {
        const double f = advance / seg_len;
        for (int k = 0; k < d; ++k) pos[k] += f * (plan[waypoint][k] - pos[k]);
        advance = 0.0;
      }
    }
    if (cfg.disturbance_sigma > 0.0) {
      double norm_sq = 0.0;
      for (int k = 0; k < d; ++k) {
        const double g = std::clamp(rng.gaussian(), -6.0, 6.0);
        const double dx = g * cfg.disturbance_sigma;
        pos[k] += dx;
        norm_sq += dx * dx;
      }
      if (std::sqrt(norm_sq) > 3.0 * cfg.disturbance_sigma) ++o.noise_outliers;
    }
    for (int k = 0; k < d; ++k) pos[k] = std::clamp(pos[k], 0.0, 1.0);
    travelled->insert(travelled->end(), pos.begin(), pos.end());
    t += cfg.control_dt;
    // (c) replan completion (simulator.cpp:146-158)
    if (t >= next_replan - 1e-9) {
      if (!goal_blocked) {
        ++o.replans;
        std::vector<std::vector<double>> fresh;
        rc = plan_from(ctx, cfg, pos, obstacles, draw_seed(rng), &goal_blocked, &found, &fresh);
        if (rc) return rc;
        if (found) {
          plan = std::move(fresh);
          waypoint = 1;
        }
      }
      next_replan += cfg.replan_latency;
      if (next_replan <= t) next_replan = t + cfg.replan_latency;
    }
    // (d) end conditions (simulator.cpp:160-172)
    if (!point_free(pos, obstacles)) {
      o.result = GMT_TRIAL_COLLIDED;
      break;
    }
    if (box_contains(cfg.scene.goal_lo, cfg.scene.goal_hi, pos)) {
      o.result = GMT_TRIAL_REACHED_GOAL;
      break;
    }
    if (t >= cfg.time_limit - 1e-9) {
      o.result = GMT_TRIAL_TIMED_OUT;
      break;
    }
  }
  o.time = t;
  o.path_len = static_cast<int64_t>(travelled->size() / d);
  *out = o;
  return GMT_OK;
}

// ---- lockstep campaigns: many trials, replans batched -----------------------
// The trial state machine of run_trial (simulator.cpp:66-176) split at its
// replan points: every trial advances until it needs a plan, the pending
// plan_from requests of all trials go through ONE gmt_plan_problems call
// (batched sampling / graphs / solve), and each trial resumes with its
// result.  Each trial consumes its own generator in exactly the reference's
// order, so outcomes are identical to run_trial's.
struct LockTrial {
  gmt_scenario cfg{};
  Rng rng{0};
  Obstacles obstacles;
  std::vector<double> pos, lo, hi;
  std::vector<std::vector<double>> plan;
  size_t waypoint = 1;
  double t = 0.0, next_replan = 0.0, half = 0.0;
  bool goal_blocked = false;
  gmt_trial_outcome o{};
  int phase = 0;  // 0 initial plan pending, 1 running, 2 replan pending, 3 done
  uint64_t pending_seed = 0;
  explicit LockTrial(const gmt_scenario& c, uint64_t seed) : cfg(c), rng(seed) {
    const int d = cfg.scene.dim;
    obstacles.d = d;
    obstacles.lo.assign(cfg.scene.box_lo, cfg.scene.box_lo + static_cast<size_t>(cfg.scene.num_boxes) * d);
    obstacles.hi.assign(cfg.scene.box_hi, cfg.scene.box_hi + static_cast<size_t>(cfg.scene.num_boxes) * d);
    pos.assign(cfg.init, cfg.init + d);
    lo.resize(d);
    hi.resize(d);
    o.result = GMT_TRIAL_TIMED_OUT;
    next_replan = cfg.replan_latency;
    half = 0.5 * cfg.spawn_box_size;
    pending_seed = draw_seed(rng);  // the initial plan's seed (simulator.cpp:82)
  }
  // After a plan result: the rest of the step, then steps until the next
  // replan request or the end.
  void resume(bool found, std::vector<std::vector<double>>&& fresh) {
    if (phase == 0) {
      if (!found) {
        phase = 3;
        return;
      }
      plan = std::move(fresh);
      waypoint = 1;
      phase = 1;
    } else if (phase == 2) {
      if (found) {
        plan = std::move(fresh);
        waypoint = 1;
      }
      finish_step();
      if (phase == 3) return;
      phase = 1;
    }
    run();
  }
  void finish_step() {  // (c) bookkeeping + (d) end conditions
    next_replan += cfg.replan_latency;
    if (next_replan <= t) next_replan = t + cfg.replan_latency;
    check_end();
  }
  void check_end() {
    o.time = t;
    if (!point_free(pos, obstacles)) {
      o.result = GMT_TRIAL_COLLIDED;
      phase = 3;
    } else if (box_contains(cfg.scene.goal_lo, cfg.scene.goal_hi, pos)) {
      o.result = GMT_TRIAL_REACHED_GOAL;
      phase = 3;
    } else if (t >= cfg.time_limit - 1e-9) {
      o.result = GMT_TRIAL_TIMED_OUT;
      phase = 3;
    }
  }
  void run() {
    const int d = cfg.scene.dim;
    while (phase == 1) {
      const int events = rng.poisson(cfg.collapse_rate * cfg.control_dt);  // (a)
      for (int e = 0; e < events; ++e) {
        for (int attempt = 0; attempt < 1000; ++attempt) {
          for (int k = 0; k < d; ++k) {
            const double c = rng.next_double();
            lo[k] = c - half;
            hi[k] = c + half;
          }
          if (box_contains(lo.data(), hi.data(), pos)) continue;
          obstacles.lo.insert(obstacles.lo.end(), lo.begin(), lo.end());
          obstacles.hi.insert(obstacles.hi.end(), hi.begin(), hi.end());
          ++o.spawned;
          break;
        }
      }
      double advance = cfg.robot_speed * cfg.control_dt;  // (b)
      while (advance > 0.0 && waypoint < plan.size()) {
        const double seg_len = euclid(pos, plan[waypoint]);
        if (seg_len <= advance) {
          pos = plan[waypoint];
          advance -= seg_len;
          ++waypoint;
        } else {
          const double f = advance / seg_len;
          for (int k = 0; k < d; ++k) pos[k] += f * (plan[waypoint][k] - pos[k]);
          advance = 0.0;
        }
      }
      if (cfg.disturbance_sigma > 0.0) {
        double norm_sq = 0.0;
        for (int k = 0; k < d; ++k) {
          const double g = std::clamp(rng.gaussian(), -6.0, 6.0);
          const double dx = g * cfg.disturbance_sigma;
          pos[k] += dx;
          norm_sq += dx * dx;
        }
        if (std::sqrt(norm_sq) > 3.0 * cfg.disturbance_sigma) ++o.noise_outliers;
      }
      for (int k = 0; k < d; ++k) pos[k] = std::clamp(pos[k], 0.0, 1.0);
      t += cfg.control_dt;
      if (t >= next_replan - 1e-9) {  // (c)
        if (!goal_blocked) {
          ++o.replans;
          pending_seed = draw_seed(rng);
          phase = 2;  // wait for the batched plan
          return;
        }
        finish_step();
      } else {
        check_end();
      }
    }
  }
};

int run_lockstep(gmt_ctx* ctx, std::vector<LockTrial>& trials) {
  const int d = trials.empty() ? 0 : trials[0].cfg.scene.dim;
  std::vector<gmt_problem> probs;
  std::vector<int> who;
  std::vector<int32_t> status;
  std::vector<gmt_plan_summary> summ;
  std::vector<double> paths;
  for (;;) {
    probs.clear();
    who.clear();
    for (size_t k = 0; k < trials.size(); ++k) {
      LockTrial& T = trials[k];
      if (T.phase != 0 && T.phase != 2) continue;
      gmt_problem p{};  // plan_from (simulator.cpp:32-64)
      p.scene = T.cfg.scene;
      p.scene.num_boxes = T.obstacles.count();
      p.scene.box_lo = T.obstacles.lo.data();
      p.scene.box_hi = T.obstacles.hi.data();
      p.init = T.pos.data();
      p.n = T.cfg.n;
      p.lambda = T.cfg.lambda;
      p.eta = T.cfg.eta;
      p.radius_override = T.cfg.radius_override;
      p.sampling.kind = GMT_SAMPLE_UNIFORM;
      p.sampling.start_index = 1;
      p.sampling.seed = T.pending_seed;
      p.steering = GMT_STEER_EUCLIDEAN;
      probs.push_back(p);
      who.push_back(static_cast<int>(k));
    }
    if (probs.empty()) return GMT_OK;
    const int m = static_cast<int>(probs.size());
    int cap = 0;
    for (const auto& p : probs) cap = std::max(cap, p.n + 1);
    status.assign(m, 0);
    summ.assign(m, gmt_plan_summary{});
    paths.assign(static_cast<size_t>(m) * cap * d, 0.0);
    const int rc = gmt_plan_problems(ctx, probs.data(), m, status.data(), summ.data(), cap, paths.data());
    if (rc) return rc;
    for (int q = 0; q < m; ++q) {
      LockTrial& T = trials[who[q]];
      bool found = false;
      std::vector<std::vector<double>> fresh;
      if (status[q] == GMT_E_GOAL_BLOCKED) {
        T.goal_blocked = true;
      } else if (status[q] == GMT_OK && summ[q].status == 0) {
        found = true;
        for (int k = 0; k < summ[q].path_len; ++k) {
          const double* s = paths.data() + (static_cast<size_t>(q) * cap + k) * d;
          fresh.emplace_back(s, s + d);
        }
      } else if (status[q] != GMT_OK && status[q] != GMT_E_INFEASIBLE_SAMPLING) {
        return set_error(status[q], "replan failed");
      }
      T.resume(found, std::move(fresh));
    }
  }
}

}  // namespace

}  // namespace gmtb

using namespace gmtb;

extern "C" int gmt_run_trial(gmt_ctx* ctx, const gmt_scenario* cfg, uint64_t trial_seed,
                             gmt_trial_outcome* out, double* path, int64_t path_cap) {
  gmtb::AllocScope alloc_scope_(ctx);
  int rc = validate_scenario(cfg);
  if (rc) return rc;
  rc = validate_scene(&cfg->scene);
  if (rc) return rc;
  std::vector<double> travelled;
  rc = run_trial(ctx, *cfg, trial_seed, out, &travelled);
  if (rc) return rc;
  if (path) {
    const int d = cfg->scene.dim;
    const int64_t k = std::min<int64_t>(path_cap, out->path_len);
    std::memcpy(path, travelled.data(), sizeof(double) * static_cast<size_t>(k) * d);
  }
  return GMT_OK;
}

extern "C" int gmt_run_campaign(int device, const gmt_scenario* cfg, const double* latencies,
                                int32_t num_latencies, const double* rates, int32_t num_rates,
                                const double* sigmas, int32_t num_sigmas, int32_t workers,
                                int32_t* successes) {
  // run_campaign (simulator.cpp:178-227): cells in (latency, rate, sigma)
  // order, trial seeds from the cell parameters and the trial counter.
  if (num_latencies < 1 || num_rates < 1 || num_sigmas < 1 || !cfg || cfg->trials < 1)
    return set_error(GMT_E_INVALID_INPUT, "campaign needs at least one cell and one trial");
  int rc = validate_scene(&cfg->scene);
  if (rc) return rc;
  struct Cell {
    double latency, rate, sigma;
  };
  std::vector<Cell> cells;
  for (int a = 0; a < num_latencies; ++a)
    for (int b = 0; b < num_rates; ++b)
      for (int c = 0; c < num_sigmas; ++c) cells.push_back({latencies[a], rates[b], sigmas[c]});
  struct Task {
    size_t cell;
    uint64_t seed;
  };
  std::vector<Task> tasks;
  for (size_t c = 0; c < cells.size(); ++c) {
    uint64_t key = mix64(cfg->seed, bits_of(cells[c].latency));
    key = mix64(key, bits_of(cells[c].rate));
    key = mix64(key, bits_of(cells[c].sigma));
    for (int t = 0; t < cfg->trials; ++t) tasks.push_back({c, mix64(key, static_cast<uint64_t>(t))});
  }
  for (const Cell& cell : cells) {  // run_trial's parameter check, per cell (simulator.cpp:67-72)
    gmt_scenario c = *cfg;
    c.replan_latency = cell.latency;
    c.collapse_rate = cell.rate;
    c.disturbance_sigma = cell.sigma;
    rc = validate_scenario(&c);
    if (rc) return rc;
  }
  std::vector<uint8_t> success(tasks.size(), 0);
  const int W = std::max(1, std::min<int>(workers, static_cast<int>(tasks.size())));
  std::atomic<int> failed{GMT_OK};
  std::vector<std::string> errors(W);
  // Worker w runs tasks w, w + W, ... in lockstep (batched replans).
  auto work = [&](int w) {
    gmt_ctx* ctx = nullptr;
    int r = gmt_ctx_create(device, &ctx);
    if (r) {
      errors[w] = gmt_last_error();
      failed = r;
      return;
    }
    {
      gmtb::AllocScope scope(ctx);
      std::vector<LockTrial> trials;
      std::vector<size_t> ids;
      for (size_t k = static_cast<size_t>(w); k < tasks.size(); k += static_cast<size_t>(W)) {
        gmt_scenario c = *cfg;
        c.replan_latency = cells[tasks[k].cell].latency;
        c.collapse_rate = cells[tasks[k].cell].rate;
        c.disturbance_sigma = cells[tasks[k].cell].sigma;
        trials.emplace_back(c, tasks[k].seed);
        ids.push_back(k);
      }
      r = run_lockstep(ctx, trials);
      if (r) {
        errors[w] = gmt_last_error();
        failed = r;
      } else {
        for (size_t j = 0; j < trials.size(); ++j)
          success[ids[j]] = trials[j].o.result == GMT_TRIAL_REACHED_GOAL ? 1 : 0;
      }
    }
    gmt_ctx_destroy(ctx);
  };
  std::vector<std::thread> pool;
  for (int w = 0; w < W; ++w) pool.emplace_back(work, w);
  for (auto& th : pool) th.join();
  if (failed != GMT_OK) {
    for (const auto& e : errors)
      if (!e.empty()) return set_error(failed, e);
    return set_error(failed, "campaign worker failed");
  }
  for (size_t c = 0; c < cells.size(); ++c) successes[c] = 0;
  for (size_t k = 0; k < tasks.size(); ++k) successes[tasks[k].cell] += success[k];
  return GMT_OK;
}
