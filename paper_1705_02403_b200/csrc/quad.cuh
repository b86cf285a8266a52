// quad.cuh -- 12D linearised quadrotor steering (NEW:
// the reference has no quadrotor).
//
// Normalised state x in [0,1]^12:
//   0-2  position p (workspace units)      3-5  velocity   v = vmax (2s - 1)
//   6-8  roll phi, pitch theta, yaw psi:    phi, theta = amax (2s - 1), psi = ymax (2s - 1)
//   9-11 body rates p, q, r = wmax (2s - 1)
// Hover linearisation: x'' = g theta, y'' = -g phi, z'' = u_z, phi'' = tau_phi,
// theta'' = tau_theta, psi'' = tau_psi; cost J = tau + integral of
// w (tau_phi^2 + tau_theta^2 + u_z^2 + tau_psi^2).  The system splits into
// four integrator chains in unit-gain coordinates:
//   chain 0 (order 4): [p_x, v_x,  g theta,  g q],  input  g tau_theta, weight w/g^2
//   chain 1 (order 4): [p_y, v_y, -g phi,   -g p],  input -g tau_phi,   weight w/g^2
//   chain 2 (order 2): [p_z, v_z],                  input u_z,          weight w
//   chain 3 (order 2): [psi, r],                    input tau_psi,      weight w
// For an order-m chain the Gramian is G(tau) = S H S with S = diag(tau^(m-i+1/2))
// and H_ij = 1/((m-i)!(m-j)!(2m-i-j+1)); H^-1 is integral (12,-6,4 for m = 2;
// the 4x4 below for m = 4), so the minimum effort w d^T G^-1 d is a Laurent
// polynomial and the total cost is
//   c(tau) = tau + sum_{k=1..7} C_k tau^-k,
// minimised exactly like the double integrator (di.cuh): the stationarity
// polynomial tau^8 - sum k C_k tau^(7-k) is scanned on the grid T (3/4)^j and
// every -/+ sign change refined by 64 bisection steps (+-*/ only, so host and
// device agree bit for bit).  The optimal input is w(s) = B^T e^(A^T(tau-s))
// G^-1 d, whose state trajectory has the closed form used by quad_coord.
#pragma once

#include <cstdint>

#include "di.cuh"

namespace gmtb {

struct QuadParams {
  double g;     // gravity in workspace units / s^2
  double vmax;  // velocity bound
  double amax;  // roll / pitch bound (rad)
  double ymax;  // yaw bound (rad)
  double wmax;  // body-rate bound (rad/s)
  double weight;  // control-effort weight w
  int32_t segments;
  int32_t reserved;
};

constexpr int kQuadDim = 12;
constexpr int kQuadK = 7;  // highest inverse power of tau in c(tau)

// Integral inverse of the normalised Gramian for chain orders 2 and 4.
GMT_HD double quad_hinv(int m, int i, int j) {
  constexpr double h2[2][2] = {{12.0, -6.0}, {-6.0, 4.0}};
  constexpr double h4[4][4] = {{100800.0, -50400.0, 10080.0, -840.0},
                               {-50400.0, 25920.0, -5400.0, 480.0},
                               {10080.0, -5400.0, 1200.0, -120.0},
                               {-840.0, 480.0, -120.0, 16.0}};
  return m == 2 ? h2[i][j] : h4[i][j];
}

GMT_HD double quad_fact(int k) {
  double f = 1.0;
  for (int i = 2; i <= k; ++i) f = di_mul(f, static_cast<double>(i));
  return f;
}

GMT_HD int quad_chain_order(int c) { return c < 2 ? 4 : 2; }

GMT_HD double quad_chain_weight(int c, const QuadParams& P) {
  return c < 2 ? di_div(P.weight, di_mul(P.g, P.g)) : P.weight;
}

// Normalised coordinate index of component i of chain c.
GMT_HD int quad_coord_index(int c, int i) {
  constexpr int map[4][4] = {{0, 3, 7, 10}, {1, 4, 6, 9}, {2, 5, -1, -1}, {8, 11, -1, -1}};
  return map[c][i];
}

// Physical value of normalised coordinate `idx` with value s.
GMT_HD double quad_phys(int idx, double s, const QuadParams& P) {
  if (idx < 3) return s;
  double range = P.vmax;
  if (idx == 6 || idx == 7) range = P.amax;
  if (idx == 8) range = P.ymax;
  if (idx >= 9) range = P.wmax;
  return di_mul(range, di_sub(di_mul(2.0, s), 1.0));
}

GMT_HD double quad_norm(int idx, double v, const QuadParams& P) {
  if (idx < 3) return v;
  double range = P.vmax;
  if (idx == 6 || idx == 7) range = P.amax;
  if (idx == 8) range = P.ymax;
  if (idx >= 9) range = P.wmax;
  return di_mul(0.5, di_add(di_div(v, range), 1.0));
}

// Unit-gain chain state of x (z[0..m-1]).
GMT_HD void quad_chain_state(const double* x, int c, const QuadParams& P, double* z) {
  const int m = quad_chain_order(c);
  for (int i = 0; i < m; ++i) {
    const int idx = quad_coord_index(c, i);
    double v = quad_phys(idx, x[idx], P);
    if (c == 0 && i >= 2) v = di_mul(P.g, v);
    if (c == 1 && i >= 2) v = -di_mul(P.g, v);
    z[i] = v;
  }
}

// Inverse of quad_chain_state for one component.
GMT_HD double quad_chain_to_norm(int c, int i, double z, const QuadParams& P) {
  double v = z;
  if (c == 0 && i >= 2) v = di_div(z, P.g);
  if (c == 1 && i >= 2) v = -di_div(z, P.g);
  return quad_norm(quad_coord_index(c, i), v, P);
}

// delta[i][p]: d_i(tau) = sum_p delta[i][p] tau^p, d = z1 - e^(A tau) z0.
GMT_HD void quad_delta(const double* z0, const double* z1, int m, double delta[4][4]) {
  for (int i = 0; i < m; ++i) {
    delta[i][0] = di_sub(z1[i], z0[i]);
    for (int p = 1; p < m - i; ++p) delta[i][p] = -di_div(z0[i + p], quad_fact(p));
  }
}

// C[1..7] of c(tau) = tau + sum C_k tau^-k (C[0] unused).
GMT_HD void quad_coef(const double* x0, const double* x1, const QuadParams& P, double* C) {
  for (int k = 0; k <= kQuadK; ++k) C[k] = 0.0;
  for (int c = 0; c < 4; ++c) {
    const int m = quad_chain_order(c);
    const double wc = quad_chain_weight(c, P);
    double z0[4], z1[4], delta[4][4];
    quad_chain_state(x0, c, P, z0);
    quad_chain_state(x1, c, P, z1);
    quad_delta(z0, z1, m, delta);
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) {
        const double h = di_mul(wc, quad_hinv(m, i, j));
        for (int p = 0; p < m - i; ++p)
          for (int q = 0; q < m - j; ++q) {
            const int k = 2 * m - i - j - 1 - p - q;
            C[k] = di_add(C[k], di_mul(di_mul(h, delta[i][p]), delta[j][q]));
          }
      }
  }
}

// Stationarity polynomial tau^8 - sum_k k C_k tau^(7-k) (Horner).
GMT_HD double quad_g(const double* C, double t) {
  double r = 1.0;
  r = di_mul(r, t);  // tau^7 coefficient is 0
  for (int k = 1; k <= kQuadK; ++k) r = di_sub(di_mul(r, t), di_mul(static_cast<double>(k), C[k]));
  return r;
}

// c(tau) = tau + (((C7/tau + C6)/tau + ...)/tau + C1)/tau
GMT_HD double quad_c(const double* C, double t) {
  double r = di_div(C[kQuadK], t);
  for (int k = kQuadK - 1; k >= 1; --k) r = di_div(di_add(r, C[k]), t);
  return di_add(t, r);
}

GMT_HD double quad_cost_tau(const double* x0, const double* x1, const QuadParams& P, double* tau_out,
                            double cap = INFINITY) {
  double C[kQuadK + 1];
  quad_coef(x0, x1, P, C);
  bool zero = true;
  for (int k = 1; k <= kQuadK; ++k) zero = zero && C[k] == 0.0;
  if (zero) {
    *tau_out = 0.0;
    return 0.0;
  }
  double T = 0.0;
  for (int k = 1; k <= kQuadK; ++k) {
    double a = di_mul(static_cast<double>(k), C[k]);
    a = a < 0.0 ? -a : a;
    if (a > T) T = a;
  }
  T = di_add(1.0, T);
  return kino_min_scan(
      T, [&](double t) { return quad_g(C, t); }, [&](double t) { return quad_c(C, t); }, cap, tau_out);
}

GMT_HD double quad_pow(double t, int e) {
  double r = 1.0;
  for (int i = 0; i < e; ++i) r = di_mul(r, t);
  return r;
}

// Coordinate idx (0..11) of waypoint k (0..M) of the optimal trajectory.
// Chain and component of normalised coordinate idx.
GMT_HD void quad_locate(int idx, int* c, int* i) {
  *c = 0;
  *i = 0;
  for (int cc = 0; cc < 4; ++cc)
    for (int ii = 0; ii < quad_chain_order(cc); ++ii)
      if (quad_coord_index(cc, ii) == idx) *c = cc, *i = ii;
}

// Per-edge, per-chain part of the trajectory: the chain's start state z0 and
// lambda = G^-1 d, G^-1_jl = H^-1_jl / tau^(2m - j - l - 1).
GMT_HD void quad_chain_lambda(const double* x0, const double* x1, double tau, int c, const QuadParams& P,
                              double* z0, double* lam) {
  const int m = quad_chain_order(c);
  double z1[4], delta[4][4], d[4];
  quad_chain_state(x0, c, P, z0);
  quad_chain_state(x1, c, P, z1);
  quad_delta(z0, z1, m, delta);
  for (int j = 0; j < m; ++j) {
    double v = 0.0;
    for (int p = m - j - 1; p >= 0; --p) v = di_add(di_mul(v, tau), delta[j][p]);
    d[j] = v;
  }
  for (int j = 0; j < m; ++j) {
    double v = 0.0;
    for (int l = 0; l < m; ++l)
      v = di_add(v, di_div(di_mul(quad_hinv(m, j, l), d[l]), quad_pow(tau, 2 * m - j - l - 1)));
    lam[j] = v;
  }
}

// Component i of chain c at waypoint k (0 < k < M) from quad_chain_lambda's
// z0 / lambda:  z_i(t) = (e^(A t) z0)_i + sum_j lam_j I(a = m-1-i, b = m-1-j),
// I(a,b) = sum_{r=0..b} (tau-t)^(b-r)/(b-r)! t^(a+r+1) / ((a+r+1) a! r!).
GMT_HD double quad_chain_coord(const double* z0, const double* lam, double tau, int k, int c, int i,
                               const QuadParams& P) {
  const int m = quad_chain_order(c);
  const double t = di_div(di_mul(tau, static_cast<double>(k)), static_cast<double>(P.segments));
  double zi = 0.0;
  for (int q = m - 1; q >= i; --q) zi = di_add(zi, di_div(di_mul(z0[q], quad_pow(t, q - i)), quad_fact(q - i)));
  const int a = m - 1 - i;
  const double u = di_sub(tau, t);
  for (int j = 0; j < m; ++j) {
    const int b = m - 1 - j;
    double I = 0.0;
    for (int r = 0; r <= b; ++r) {
      const double num = di_mul(di_div(quad_pow(u, b - r), quad_fact(b - r)), quad_pow(t, a + r + 1));
      const double den = di_mul(di_mul(static_cast<double>(a + r + 1), quad_fact(a)), quad_fact(r));
      I = di_add(I, di_div(num, den));
    }
    zi = di_add(zi, di_mul(lam[j], I));
  }
  return quad_chain_to_norm(c, i, zi, P);
}

// Coordinate idx (0..11) of waypoint k (0..M) of the optimal trajectory.
GMT_HD double quad_coord(const double* x0, const double* x1, double tau, int k, int idx,
                         const QuadParams& P) {
  const int M = P.segments;
  if (k <= 0 || tau == 0.0) return x0[idx];
  if (k >= M) return x1[idx];
  int c, i;
  quad_locate(idx, &c, &i);
  double z0[4], lam[4];
  quad_chain_lambda(x0, x1, tau, c, P, z0, lam);
  return quad_chain_coord(z0, lam, tau, k, c, i, P);
}

// Necessary condition for cost(x0 -> x1) <= r: for every chain component,
// w d_i^2 / G_ii(tau) <= r with tau <= r (d^T G^-1 d >= d_i^2 / G_ii), and
// |d_i(tau)| >= |delta_i0| - sum_p |delta_ip| r^p.  Widened by 1e-9 relative.
GMT_HD bool quad_may_connect(const double* x0, const double* x1, const QuadParams& P, double r) {
  for (int c = 0; c < 4; ++c) {
    const int m = quad_chain_order(c);
    const double wc = quad_chain_weight(c, P);
    double z0[4], z1[4], delta[4][4];
    quad_chain_state(x0, c, P, z0);
    quad_chain_state(x1, c, P, z1);
    quad_delta(z0, z1, m, delta);
    for (int i = 0; i < m; ++i) {
      double drift = 0.0, rp = 1.0;
      for (int p = 1; p < m - i; ++p) {
        rp = rp * r;
        drift = drift + (delta[i][p] < 0.0 ? -delta[i][p] : delta[i][p]) * rp;
      }
      const double gap = (delta[i][0] < 0.0 ? -delta[i][0] : delta[i][0]) - drift;
      if (gap <= 0.0) continue;
      // G_ii = tau^e / hdiag with e = 2(m-1-i)+1, hdiag = (m-1-i)!^2 e; the
      // effort is >= wc gap^2 hdiag / tau^e and must stay <= r, tau <= r.
      const int e = 2 * (m - 1 - i) + 1;
      const double hdiag = quad_fact(m - 1 - i) * quad_fact(m - 1 - i) * e;
      double re1 = 1.0;
      for (int q = 0; q < e + 1; ++q) re1 = re1 * r;
      if (wc * gap * gap * hdiag > re1 * (1.0 + 1e-9) + 1e-300) return false;
    }
  }
  return true;
}

}  // namespace gmtb
