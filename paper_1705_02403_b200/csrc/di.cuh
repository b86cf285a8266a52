// di.cuh -- 6D double-integrator steering (NEW: the
// reference has no double integrator, so this model is defined
// here).
//
// State x = [p_0, p_1, p_2, s_0, s_1, s_2] in [0,1]^6: positions p and
// normalised velocities s, v_k = vmax (2 s_k - 1).  Dynamics p'' = u, cost
// J = tau + w * integral |u|^2 dt (the paper's "mixed time/quadratic control
// effort").  For a fixed duration tau the minimum-effort
// cost is, with D = p1 - p0 per axis,
//   c(tau) = tau + a/tau + b/tau^2 + c0/tau^3,
//   a = 4w sum(v0^2 + v0 v1 + v1^2), b = -12w sum D (v0 + v1), c0 = 12w sum D^2
// and c'(tau) = 0  <=>  g(tau) = tau^4 - a tau^2 - 2 b tau - 3 c0 = 0.
//
// tau* (deterministic, +-*/ only, so host and device agree bit for bit):
// every positive root lies below T = 1 + max(a, 2|b|, 3c0) (Cauchy); g is
// sampled on the geometric grid T q^j (q = 3/4, j = 96 .. 0, ascending tau);
// every sign change g <= 0 -> g > 0 (a local minimum of c) is refined by 64
// bisection steps; tau* is the refined root with the smallest c (ties to the
// smaller tau).  The optimal state trajectory is the cubic
//   p(t) = p0 + v0 t + c2 t^2 + c3 t^3,  v(t) = v0 + 2 c2 t + 3 c3 t^2,
//   c2 = 3D/tau^2 - (2 v0 + v1)/tau,  c3 = (v0 + v1)/tau^2 - 2D/tau^3,
// discretised at t = tau k / M (k = 1..M-1) between the exact endpoint
// states; the lazy check tests the polyline (the reference's
// polyline_free, space.cpp:92-99), so velocities leaving [-vmax, vmax]
// (normalised coordinates outside [0,1]) block the edge.
#pragma once

#include <cmath>
#include <cstdint>

#if defined(__CUDACC__)
#define GMT_HD __host__ __device__ __forceinline__
#else
#define GMT_HD inline
#endif

namespace gmtb {

struct DiParams {
  double vmax;     // velocity bound of the normalised velocity coordinates
  double weight;   // control-effort weight w
  int32_t segments;  // M: polyline segments per trajectory
  int32_t reserved;
};

constexpr int kDiDim = 6;
constexpr int kDiGrid = 96;
constexpr int kDiBisect = 64;

// Correctly rounded arithmetic without contraction on both sides.
#if defined(__CUDA_ARCH__)
GMT_HD double di_add(double a, double b) { return __dadd_rn(a, b); }
GMT_HD double di_sub(double a, double b) { return __dsub_rn(a, b); }
GMT_HD double di_mul(double a, double b) { return __dmul_rn(a, b); }
GMT_HD double di_div(double a, double b) { return __ddiv_rn(a, b); }
#else
GMT_HD double di_add(double a, double b) {
  volatile double r = a + b;
  return r;
}
GMT_HD double di_sub(double a, double b) {
  volatile double r = a - b;
  return r;
}
GMT_HD double di_mul(double a, double b) {
  volatile double r = a * b;
  return r;
}
GMT_HD double di_div(double a, double b) {
  volatile double r = a / b;
  return r;
}
#endif

GMT_HD double di_vel(double s, const DiParams& P) {  // v = vmax (2s - 1)
  return di_mul(P.vmax, di_sub(di_mul(2.0, s), 1.0));
}

struct DiCoef {
  double a, b, c0;
};

GMT_HD DiCoef di_coef(const double* x0, const double* x1, const DiParams& P) {
  double sa = 0.0, sb = 0.0, sc = 0.0;
  for (int k = 0; k < 3; ++k) {
    const double D = di_sub(x1[k], x0[k]);
    const double v0 = di_vel(x0[3 + k], P), v1 = di_vel(x1[3 + k], P);
    sa = di_add(sa, di_add(di_add(di_mul(v0, v0), di_mul(v0, v1)), di_mul(v1, v1)));
    sb = di_add(sb, di_mul(D, di_add(v0, v1)));
    sc = di_add(sc, di_mul(D, D));
  }
  DiCoef c;
  c.a = di_mul(di_mul(4.0, P.weight), sa);
  c.b = di_mul(di_mul(-12.0, P.weight), sb);
  c.c0 = di_mul(di_mul(12.0, P.weight), sc);
  return c;
}

// g(tau) = ((tau^2 - a) tau - 2b) tau - 3 c0
GMT_HD double di_g(const DiCoef& c, double t) {
  return di_sub(di_mul(di_sub(di_mul(di_sub(di_mul(t, t), c.a), t), di_mul(2.0, c.b)), t),
                di_mul(3.0, c.c0));
}

// c(tau) = tau + ((c0/tau + b)/tau + a)/tau
GMT_HD double di_c(const DiCoef& c, double t) {
  return di_add(t, di_div(di_add(di_div(di_add(di_div(c.c0, t), c.b), t), c.a), t));
}

// The duration search shared by the kinodynamic models: the geometric grid
// tau_j = T q^j (j = 0..kDiGrid, each point the rounded product of the
// previous one) walked from large to small tau; every bracket
// [tau_{j+1}, tau_j] with g(tau_{j+1}) <= 0 < g(tau_j) is refined by
// kDiBisect bisection steps; the refined root with the smallest c wins (ties
// to the smaller tau, i.e. the later bracket).  Returns c(tau*) and tau*.
//
// cap < inf (graph construction, where only c <= cap matters): brackets with
// tau_{j+1} > cap are skipped -- their roots exceed cap, so c = tau + effort
// > cap there and they can never be the minimum of a pair that is kept; a
// kept pair's (c, tau) is therefore bit-identical to the uncapped search.
// When no bracket lies below cap: if g(T) > 0 >= g(tau_min) the uncapped
// search has a bracket, all above cap, and the pair is rejected (+inf);
// otherwise the uncapped search runs.
template <class GF, class CF>
GMT_HD double kino_min_scan(double T, const GF& g, const CF& cfun, double cap, double* tau_out) {
  double best_c = 0.0, best_t = 0.0;
  bool have = false;
  double t_hi = T;
  int j = 1;
  if (cap < INFINITY) {
    while (j <= kDiGrid) {
      const double t_lo = di_mul(t_hi, 0.75);
      if (t_lo <= cap) break;
      t_hi = t_lo;
      ++j;
    }
  }
  double g_hi = g(t_hi);
  const double g_top = t_hi == T ? g_hi : (cap < INFINITY ? g(T) : g_hi);
  for (; j <= kDiGrid; ++j) {
    const double t_lo = di_mul(t_hi, 0.75);
    const double g_lo = g(t_lo);
    if (g_lo <= 0.0 && g_hi > 0.0) {
      double lo = t_lo, hi = t_hi;
      for (int it = 0; it < kDiBisect; ++it) {
        const double mid = di_mul(0.5, di_add(lo, hi));
        if (g(mid) > 0.0) {
          hi = mid;
        } else {
          lo = mid;
        }
      }
      const double ct = cfun(hi);
      if (!have || ct <= best_c) {
        best_c = ct;
        best_t = hi;
        have = true;
      }
    }
    t_hi = t_lo;
    g_hi = g_lo;
  }
  if (!have && cap < INFINITY) {
    if (g_top > 0.0 && g_hi <= 0.0) {  // every bracket of the full search lies above cap
      *tau_out = 0.0;
      return INFINITY;
    }
    return kino_min_scan(T, g, cfun, INFINITY, tau_out);
  }
  if (!have) {  // g > 0 on the whole grid: be total
    best_t = t_hi;
    best_c = cfun(best_t);
  }
  *tau_out = best_t;
  return best_c;
}

// Minimum cost and its duration; cost 0 / tau 0 for identical states at rest.
// cap: see kino_min_scan (INFINITY = the exact minimum for every pair).
GMT_HD double di_cost_tau(const double* x0, const double* x1, const DiParams& P, double* tau_out,
                          double cap = INFINITY) {
  const DiCoef c = di_coef(x0, x1, P);
  if (c.a == 0.0 && c.b == 0.0 && c.c0 == 0.0) {
    *tau_out = 0.0;
    return 0.0;
  }
  double T = c.a;
  const double b2 = di_mul(2.0, c.b < 0.0 ? -c.b : c.b);
  const double c3 = di_mul(3.0, c.c0);
  if (b2 > T) T = b2;
  if (c3 > T) T = c3;
  T = di_add(1.0, T);
  return kino_min_scan(
      T, [&](double t) { return di_g(c, t); }, [&](double t) { return di_c(c, t); }, cap, tau_out);
}

// Exact-safe rejection test for graph construction: true only if
// cost(x0 -> x1) > r is certain, so skipping the duration search of such a
// pair never changes a graph (kept pairs still run di_cost_tau unchanged).
// c(tau) - r = P(tau) / tau^3 with the quartic
//   P(tau) = tau^3 (tau - r) + Q(tau),  Q(tau) = a tau^2 + b tau + c0,
// and c(tau) > tau > r for tau > r, so the pair is rejected when P > 0 on
// (0, r].  On each of kDiRejectParts sub-intervals [l, h] the two parts are
// bounded from below separately: tau^3 (tau - r) falls on (0, 3r/4] and
// rises after it; Q's minimum is at an end point or its vertex.  The bound
// must clear a margin far above the rounding of its own evaluation and of the
// search's c(tau) (|P| terms are O(10), errors O(1e-14)): a pair whose true
// minimum is within that margin of r is left to the search.
constexpr int kDiRejectParts = 12;
GMT_HD double di_reject_margin(const DiCoef& c, double r) {
  const double scale = r * r * r * r + c.a * r * r + (c.b < 0.0 ? -c.b : c.b) * r + c.c0 + 1.0;
  return 1e-9 * scale;
}
GMT_HD double di_reject_vertex(const DiCoef& c) {
  return c.a > 0.0 ? -c.b / (2.0 * c.a) : -1.0;  // vertex of Q (a > 0: convex)
}

// The kDiRejectParts-part test.
GMT_HD bool di_cost_exceeds_parts(const DiCoef& c, double r) {
  const double margin = di_reject_margin(c, r);
  const double tm = 0.75 * r;                 // argmin of tau^3 (tau - r)
  const double tv = di_reject_vertex(c);
  double h = r;
  for (int i = 0; i < kDiRejectParts; ++i) {
    const double l = i + 1 == kDiRejectParts ? 0.0 : r * static_cast<double>(kDiRejectParts - 1 - i) / kDiRejectParts;
    // lower bound of tau^3 (tau - r) on [l, h]
    const double t = h <= tm ? h : (l >= tm ? l : tm);
    const double g = t * t * t * (t - r);
    // lower bound of Q on [l, h]
    const double ql = (c.a * l + c.b) * l + c.c0, qh = (c.a * h + c.b) * h + c.c0;
    double q = ql < qh ? ql : qh;
    if (tv > l && tv < h) {
      const double qv = (c.a * tv + c.b) * tv + c.c0;
      q = qv < q ? qv : q;
    }
    if (!(g + q > margin)) return false;
    h = l;
  }
  return true;
}

// The whole interval (0, r] at once: its lower bound is below every part's
// (a >= 0 always: sa = (v0 + v1/2)^2 + 3 v1^2 / 4), so when it clears twice
// the margin -- far above the rounding of either evaluation -- every part
// clears the margin and di_cost_exceeds_parts is true as well
// (tests/cpp/test_di_reject.cpp checks that implication).
GMT_HD bool di_cost_exceeds_whole(const DiCoef& c, double r) {
  const double margin = di_reject_margin(c, r);
  const double tm = 0.75 * r;
  const double tv = di_reject_vertex(c);
  const double g = tm * tm * tm * (tm - r);
  const double q0 = c.c0, qr = (c.a * r + c.b) * r + c.c0;
  double q = q0 < qr ? q0 : qr;
  if (tv > 0.0 && tv < r) {
    const double qv = (c.a * tv + c.b) * tv + c.c0;
    q = qv < q ? qv : q;
  }
  return g + q > 2.0 * margin;
}

// Most rejected pairs are decided by the whole-interval bound; the rest
// take the parts.  Same outcome as di_cost_exceeds_parts alone.
GMT_HD bool di_cost_exceeds(const DiCoef& c, double r) {
  return di_cost_exceeds_whole(c, r) || di_cost_exceeds_parts(c, r);
}

// State at time t on the optimal trajectory x0 -> x1 of duration tau
// (normalised coordinates).  Callers pass the exact endpoints for t = 0, tau.
GMT_HD void di_state_at(const double* x0, const double* x1, double tau, double t,
                        const DiParams& P, double* out) {
  for (int k = 0; k < 3; ++k) {
    const double D = di_sub(x1[k], x0[k]);
    const double v0 = di_vel(x0[3 + k], P), v1 = di_vel(x1[3 + k], P);
    const double tt = di_mul(tau, tau);
    const double c2 = di_sub(di_div(di_mul(3.0, D), tt), di_div(di_add(di_mul(2.0, v0), v1), tau));
    const double c3 = di_sub(di_div(di_add(v0, v1), tt), di_div(di_mul(2.0, D), di_mul(tt, tau)));
    // p(t) = p0 + t (v0 + t (c2 + t c3)),  v(t) = v0 + t (2 c2 + t 3 c3)
    const double p = di_add(x0[k], di_mul(t, di_add(v0, di_mul(t, di_add(c2, di_mul(t, c3))))));
    const double v = di_add(v0, di_mul(t, di_add(di_mul(2.0, c2), di_mul(t, di_mul(3.0, c3)))));
    out[k] = p;
    // s = (v / vmax + 1) / 2
    out[3 + k] = di_mul(0.5, di_add(di_div(v, P.vmax), 1.0));
  }
}

// Coordinate i (0..5) of waypoint k (0..M) of the edge trajectory; k = 0 / M
// return the endpoint coordinates exactly.  The same operations as
// di_state_at, one coordinate at a time (lane-parallel on the device).
GMT_HD double di_coord(const double* x0, const double* x1, double tau, int k, int i,
                       const DiParams& P) {
  const int M = P.segments;
  if (k <= 0 || tau == 0.0) return x0[i];
  if (k >= M) return x1[i];
  const double t = di_div(di_mul(tau, static_cast<double>(k)), static_cast<double>(M));
  const int a = i < 3 ? i : i - 3;
  const double D = di_sub(x1[a], x0[a]);
  const double v0 = di_vel(x0[3 + a], P), v1 = di_vel(x1[3 + a], P);
  const double tt = di_mul(tau, tau);
  const double c2 = di_sub(di_div(di_mul(3.0, D), tt), di_div(di_add(di_mul(2.0, v0), v1), tau));
  const double c3 = di_sub(di_div(di_add(v0, v1), tt), di_div(di_mul(2.0, D), di_mul(tt, tau)));
  if (i < 3) return di_add(x0[a], di_mul(t, di_add(v0, di_mul(t, di_add(c2, di_mul(t, c3))))));
  const double v = di_add(v0, di_mul(t, di_add(di_mul(2.0, c2), di_mul(t, di_mul(3.0, c3)))));
  return di_mul(0.5, di_add(di_div(v, P.vmax), 1.0));
}

GMT_HD void di_waypoint(const double* x0, const double* x1, double tau, int k, const DiParams& P,
                        double* out) {
  for (int i = 0; i < kDiDim; ++i) out[i] = di_coord(x0, x1, tau, k, i, P);
}

// Number of states of an edge's polyline: a single state for the
// degenerate zero-duration edge (the reference's convention for degenerate
// steering, steering.cpp:78-81), else M + 1.
GMT_HD int di_path_len(double tau, const DiParams& P) { return tau == 0.0 ? 1 : P.segments + 1; }

}  // namespace gmtb
