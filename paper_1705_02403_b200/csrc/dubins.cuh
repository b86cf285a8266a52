// dubins.cuh -- Dubins-airplane steering on the device (SURVEY.md §8(f) row
// 1): the planar Dubins shortest path over the six words LSL, RSR, RSL, LSR,
// RLR, LRL (earliest word wins ties), the helical cost sqrt(Lp^2 + dz^2) (or
// Lp alone), and the discretised path of ceil(Lp / step) segments -- the
// algorithm of dubins.cpp:84-167 and steering.cpp:11-101 restated for one
// thread per pose pair.
//
// Parity: the word parameters and sampled poses go through
// sin, cos, atan2 and acos, and the neighbour prune through hypot.  The
// reference gets them from glibc 2.39, which is not correctly rounded (0.06-
// 0.15 % of its sin / cos / atan2 / acos results differ from the correctly
// rounded value), so CUDA's libm cannot reproduce them; libm_port.cuh
// restates glibc's own routines operation for operation (tools/libm_port.py,
// pinned bitwise against the host libm by tests/test_libm_port.py), which
// makes every Dubins cost, path point and graph edge bit-identical.
#pragma once

#include <cmath>
#include <cstdint>

#include "di.cuh"  // GMT_HD
#include "libm_port.cuh"

namespace gmtb {

struct DubinsParams {
  double rho;
  double step;  // discretisation step (steering.hpp:22: rho / 10 when 0)
  int32_t planar_cost_only;
  int32_t dim;  // position coordinates: 2 or 3
};

constexpr double kDubinsTwoPi = 2.0 * 3.14159265358979323846;

GMT_HD double dub_mod2pi(double x) {  // dubins.cpp:49-54
  double r = fmod(x, kDubinsTwoPi);
  if (r < 0.0) r += kDubinsTwoPi;
  if (r >= kDubinsTwoPi) r = 0.0;
  return r;
}

GMT_HD double dub_snap2pi(double x) {  // dubins.cpp:28-32
  double m = dub_mod2pi(x);
  if (kDubinsTwoPi - m < 1e-9) m = 0.0;
  return m;
}

struct DubinsPath {
  double x0, y0, h0;  // start pose
  double t, p, q;     // normalised segment lengths
  int word;           // 0..5 = LSL, RSR, RSL, LSR, RLR, LRL
  double rho;
  GMT_HD double length() const { return (t + p + q) * rho; }
};

// dubins_shortest_path (dubins.cpp:84-167); word = -1 when none is feasible.
GMT_HD DubinsPath dubins_shortest(double ax, double ay, double ah, double bx, double by, double bh,
                                  double rho) {
  const double dx = bx - ax, dy = by - ay;
  const double d = sqrt(dx * dx + dy * dy) / rho;
  const double theta = d > 0.0 ? lmport::lm_atan2(dy, dx) : 0.0;
  const double alpha = dub_mod2pi(ah - theta);
  const double beta = dub_mod2pi(bh - theta);
  const double sa = lmport::lm_sin(alpha), ca = lmport::lm_cos(alpha), sb = lmport::lm_sin(beta), cb = lmport::lm_cos(beta);
  const double cab = ca * cb + sa * sb;
  double wt[6], wp[6], wq[6];
  bool ok[6] = {false, false, false, false, false, false};
  {  // LSL
    const double tmp = 2.0 + d * d - 2.0 * (cab - d * (sa - sb));
    if (tmp >= -1e-9) {
      const double th = lmport::lm_atan2(cb - ca, d + sa - sb);
      wt[0] = dub_snap2pi(-alpha + th);
      wp[0] = sqrt(tmp > 0.0 ? tmp : 0.0);
      wq[0] = dub_snap2pi(beta - th);
      ok[0] = true;
    }
  }
  {  // RSR
    const double tmp = 2.0 + d * d - 2.0 * (cab - d * (sb - sa));
    if (tmp >= -1e-9) {
      const double th = lmport::lm_atan2(ca - cb, d - sa + sb);
      wt[1] = dub_snap2pi(alpha - th);
      wp[1] = sqrt(tmp > 0.0 ? tmp : 0.0);
      wq[1] = dub_snap2pi(-beta + th);
      ok[1] = true;
    }
  }
  {  // RSL
    const double tmp = d * d - 2.0 + 2.0 * (cab - d * (sa + sb));
    if (tmp >= -1e-9) {
      const double p = sqrt(tmp > 0.0 ? tmp : 0.0);
      const double th = lmport::lm_atan2(ca + cb, d - sa - sb) - lmport::lm_atan2(2.0, p);
      wt[2] = dub_snap2pi(alpha - th);
      wp[2] = p;
      wq[2] = dub_snap2pi(beta - th);
      ok[2] = true;
    }
  }
  {  // LSR
    const double tmp = -2.0 + d * d + 2.0 * (cab + d * (sa + sb));
    if (tmp >= -1e-9) {
      const double p = sqrt(tmp > 0.0 ? tmp : 0.0);
      const double th = lmport::lm_atan2(-ca - cb, d + sa + sb) - lmport::lm_atan2(-2.0, p);
      wt[3] = dub_snap2pi(-alpha + th);
      wp[3] = p;
      wq[3] = dub_snap2pi(-beta + th);
      ok[3] = true;
    }
  }
  {  // RLR
    const double tmp = 0.125 * (6.0 - d * d + 2.0 * (cab + d * (sa - sb)));
    if (fabs(tmp) <= 1.0) {
      const double p = kDubinsTwoPi - lmport::lm_acos(tmp);
      const double th = lmport::lm_atan2(ca - cb, d - sa + sb);
      const double t = dub_snap2pi(alpha - th + 0.5 * p);
      wt[4] = t;
      wp[4] = p;
      wq[4] = dub_snap2pi(alpha - beta - t + p);
      ok[4] = true;
    }
  }
  {  // LRL
    const double tmp = 0.125 * (6.0 - d * d + 2.0 * (cab - d * (sa - sb)));
    if (fabs(tmp) <= 1.0) {
      const double p = kDubinsTwoPi - lmport::lm_acos(tmp);
      const double th = lmport::lm_atan2(-ca + cb, d + sa - sb);
      const double t = dub_snap2pi(-alpha + th + 0.5 * p);
      wt[5] = t;
      wp[5] = p;
      wq[5] = dub_snap2pi(beta - alpha - t + p);
      ok[5] = true;
    }
  }
  DubinsPath path;
  path.x0 = ax;
  path.y0 = ay;
  path.h0 = ah;
  path.rho = rho;
  path.word = -1;
  path.t = path.p = path.q = 0.0;
  double best = INFINITY;
  for (int w = 0; w < 6; ++w) {
    const double len = ok[w] ? wt[w] + wp[w] + wq[w] : INFINITY;
    if (len < best) {
      best = len;
      path.word = w;
      path.t = wt[w];
      path.p = wp[w];
      path.q = wq[w];
    }
  }
  return path;
}

// Segment types of the six words (dubins.cpp:36-46): 0 = L, 1 = S, 2 = R.
GMT_HD int dubins_seg(int word, int k) {
  constexpr int8_t segs[6][3] = {{0, 1, 0}, {2, 1, 2}, {2, 1, 0}, {0, 1, 2}, {2, 0, 2}, {0, 2, 0}};
  return segs[word][k];
}

// DubinsPlanarPath::sample (dubins.cpp:56-82): pose after arc length s.
GMT_HD void dubins_sample(const DubinsPath& P, double s, double* x, double* y, double* h) {
  double rem = s / P.rho;
  const double total = P.t + P.p + P.q;
  rem = rem < 0.0 ? 0.0 : (rem > total ? total : rem);
  double px = 0.0, py = 0.0, ph = P.h0;
  const double prm[3] = {P.t, P.p, P.q};
  for (int k = 0; k < 3; ++k) {
    const double v = rem < prm[k] ? rem : prm[k];
    rem -= v;
    const double phi = ph;
    switch (dubins_seg(P.word, k)) {
      case 0:
        px += lmport::lm_sin(phi + v) - lmport::lm_sin(phi);
        py += -lmport::lm_cos(phi + v) + lmport::lm_cos(phi);
        ph = phi + v;
        break;
      case 2:
        px += -lmport::lm_sin(phi - v) + lmport::lm_sin(phi);
        py += lmport::lm_cos(phi - v) - lmport::lm_cos(phi);
        ph = phi - v;
        break;
      default:
        px += v * lmport::lm_cos(phi);
        py += v * lmport::lm_sin(phi);
        break;
    }
    if (rem <= 0.0) break;
  }
  *x = P.x0 + px * P.rho;
  *y = P.y0 + py * P.rho;
  *h = dub_mod2pi(ph);
}

GMT_HD double dub_circular_diff(double ta, double tb) {  // steering.cpp:36-39
  const double d = dub_mod2pi(ta - tb);
  const double e = kDubinsTwoPi - d;
  return d < e ? d : e;
}

// connect() cost and path size (steering.cpp:53-101).  a, b: positions
// (dim 2 or 3), ha, hb: headings.  Returns the cost; *segments = 0 for the
// degenerate pair (path = {a}), else the segment count; *path = the planar
// path (for waypoints).  *feasible = false when no word exists (the
// reference throws; such pairs cannot occur for distinct poses).
GMT_HD double dubins_connect(const double* a, double ha, const double* b, double hb,
                             const DubinsParams& M, int* segments, DubinsPath* path, double* dz_out) {
  const double dz = M.dim == 3 ? b[2] - a[2] : 0.0;
  *dz_out = dz;
  if (fabs(a[0] - b[0]) < 1e-12 && fabs(a[1] - b[1]) < 1e-12 && fabs(dz) < 1e-12 &&
      dub_circular_diff(ha, hb) < 1e-12) {
    *segments = 0;
    path->word = -1;
    return 0.0;
  }
  *path = dubins_shortest(a[0], a[1], ha, b[0], b[1], hb, M.rho);
  const double lp = path->length();
  const double cost = M.planar_cost_only ? lp : sqrt(lp * lp + dz * dz);
  int segs = static_cast<int>(ceil(lp / M.step));
  *segments = segs < 1 ? 1 : segs;
  return cost;
}

// Waypoint i (0..segments) of the connect() path: the endpoints exactly,
// interior poses sampled at s = lp * i / segments; z interpolated linearly.
GMT_HD void dubins_waypoint(const double* a, const double* b, const DubinsPath& P, double dz,
                            int segments, int i, const DubinsParams& M, double* out) {
  if (i <= 0) {
    for (int k = 0; k < M.dim; ++k) out[k] = a[k];
    return;
  }
  if (i >= segments) {
    for (int k = 0; k < M.dim; ++k) out[k] = b[k];
    return;
  }
  const double lp = P.length();
  const double s = lp * static_cast<double>(i) / static_cast<double>(segments);
  double x, y, h;
  dubins_sample(P, s, &x, &y, &h);
  out[0] = x;
  out[1] = y;
  if (M.dim == 3) out[2] = a[2] + dz * (lp > 0.0 ? s / lp : 0.0);
}

}  // namespace gmtb
