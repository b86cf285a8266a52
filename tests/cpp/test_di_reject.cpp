// Host check of the double integrator's exact-safe rejection bound
// (di_cost_exceeds, csrc/di.cuh): over random state pairs and radii, every
// rejected pair's exact minimum cost (di_cost_tau, the same header's search)
// exceeds r, and the whole-interval shortcut never decides a pair the
// 12-part bound would keep (so di_cost_exceeds == di_cost_exceeds_parts).
// Prints the rejection rates.  Exit code 1 on a violation.
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "di.cuh"

using namespace gmtb;

static uint64_t s = 0x9E3779B97F4A7C15ull;
static double u01() {
  s ^= s << 13;
  s ^= s >> 7;
  s ^= s << 17;
  return static_cast<double>(s >> 11) * (1.0 / 9007199254740992.0);
}

int main(int argc, char** argv) {
  const long pairs = argc > 1 ? std::atol(argv[1]) : 200000;
  DiParams P{0.5, 1.0, 8, 0};
  const double radii[] = {0.4, 1.0, 1.6, 2.4, 3.5};
  long bad = 0;
  for (double r : radii) {
    long rejected = 0, kept = 0, near = 0, whole = 0;
    for (long i = 0; i < pairs; ++i) {
      double x0[6], x1[6];
      const double spread = (i % 3 == 0) ? 0.15 : 1.0;  // a third of the pairs close together
      for (int k = 0; k < 6; ++k) {
        x0[k] = u01();
        x1[k] = k < 3 ? x0[k] + spread * (u01() - 0.5) : u01();
        if (x1[k] < 0.0) x1[k] = 0.0;
        if (x1[k] > 1.0) x1[k] = 1.0;
      }
      double t;
      const double c = di_cost_tau(x0, x1, P, &t);
      const DiCoef cf = di_coef(x0, x1, P);
      const bool rej = di_cost_exceeds(cf, r);
      const bool w = di_cost_exceeds_whole(cf, r);
      if (w) ++whole;
      if (rej != di_cost_exceeds_parts(cf, r) || (w && !rej)) {
        ++bad;
        std::printf("VIOLATION (shortcut) r=%g\n", r);
      }
      if (rej) ++rejected;
      if (c <= r) ++kept;
      if (c > r && c < r * 1.05) ++near;
      if (rej && !(c > r)) {
        ++bad;
        std::printf("VIOLATION r=%g c=%.17g\n", r, c);
      }
    }
    std::printf("r=%.2f pairs=%ld kept=%ld rejected=%ld (%.1f%% of the non-kept; %ld by the whole interval) near=%ld\n",
                r, pairs, kept, rejected, 100.0 * rejected / (pairs - kept > 0 ? pairs - kept : 1), whole, near);
  }
  return bad ? 1 : 0;
}
